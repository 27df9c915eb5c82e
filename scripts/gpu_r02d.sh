#!/bin/bash
# round 2 pass d: pair-loop microbenchmark (scalar vs packed f32x2) + one ncu --set full of k_ls_adadelta 7cpa
set -u
OUT=gpurun_out/r02d; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubp scripts/ubench_pairs.cu && timeout 120 /tmp/ubp > $OUT/ubench_pairs.txt 2>&1; cat $OUT/ubench_pairs.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ls_adadelta -s 3 -c 1 -o /tmp/ls7 python bench.py --steps 1 --warmup 0 --no-cpu > $OUT/ncu_ls7.log 2>&1
python scripts/ncu_summary.py full /tmp/ls7.ncu-rep > $OUT/full_ls_7cpa.txt 2>&1
ncu -i /tmp/ls7.ncu-rep --page raw --csv > $OUT/raw_ls_7cpa.csv 2>&1
ncu -i /tmp/ls7.ncu-rep --page source --csv --print-source sass > $OUT/sass_ls_7cpa.csv 2>&1
cp /tmp/ls7.ncu-rep $OUT/ 2>/dev/null
ls -la $OUT; head -30 $OUT/full_ls_7cpa.txt
