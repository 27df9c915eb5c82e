#!/bin/bash
# round 2 pass zl (final code of the round: packed loops unrolled by 4): default bench line, ncu launch list of the same command, one ncu --set full of
# k_ls_adadelta (7cpa) + SASS source view, and the inter / intra micro captures
set -u
OUT=gpurun_out/r02zl; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > $OUT/bench_default.json 2> $OUT/bench_default.err
tail -c 400 $OUT/bench_default.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_7cpa.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-parts > $OUT/ncu_launches.log 2>&1
python scripts/ncu_summary.py launches $OUT/launches_7cpa.csv > $OUT/launch_share_7cpa.txt 2>&1; cat $OUT/launch_share_7cpa.txt | head -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ls_adadelta -s 3 -c 1 -o /tmp/ls7 python bench.py --steps 1 --warmup 0 --no-cpu --no-parts > $OUT/ncu_ls7.log 2>&1
python scripts/ncu_summary.py full /tmp/ls7.ncu-rep > $OUT/full_ls_7cpa.txt 2>&1
ncu -i /tmp/ls7.ncu-rep --page source --csv --print-source sass > $OUT/sass_ls_7cpa.csv 2>&1
gzip -f $OUT/sass_ls_7cpa.csv
python scripts/sass_blocks.py $OUT/sass_ls_7cpa.csv.gz 25 > $OUT/sass_blocks_ls_7cpa.txt 2>&1
cat $OUT/full_ls_7cpa.txt
timeout 600 ncu --set full --clock-control none -k regex:k_bench_part -s 0 -c 1 -o /tmp/mi python bench.py --micro --steps 1 --micro-iters 5 > $OUT/ncu_mi.log 2>&1
python scripts/ncu_summary.py full /tmp/mi.ncu-rep > $OUT/full_micro_inter_7cpa.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_bench_part -s 3 -c 1 -o /tmp/mp python bench.py --micro --steps 1 --micro-iters 5 > $OUT/ncu_mp.log 2>&1
python scripts/ncu_summary.py full /tmp/mp.ncu-rep > $OUT/full_micro_intra_7cpa.txt 2>&1
head -20 $OUT/full_micro_inter_7cpa.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $OUT/ref.json 2> $OUT/ref.err; tail -c 300 $OUT/ref.json
