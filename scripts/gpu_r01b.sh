#!/bin/bash
# GPU pass 2: tests (screen, speculative SW), 1stp depth sweep, ADADELTA occupancy variant, HTS sample.
set -u
OUT=gpurun_out/r01b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.log
for D in 1 2 3 0; do
  timeout 600 python bench.py --config 1stp --steps 3 --warmup 3 --no-cpu --sw-depth $D > $OUT/bench_1stp_d$D.json 2>$OUT/bench_1stp_d$D.err; echo "1stp depth $D rc=$?"; python -c "import json;d=json.loads(open('$OUT/bench_1stp_d$D.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['avg_launch_ms'])"
done
for V in default ada3; do
  if [ $V = default ]; then L=""; else L=build/variants/libdock_$V.so; fi
  DOCK_LIB=$L timeout 600 python bench.py --config 7cpa --steps 2 --warmup 3 --no-cpu > $OUT/bench_7cpa_$V.json 2>$OUT/bench_7cpa_$V.err; echo "7cpa $V rc=$?"; python -c "import json;d=json.loads(open('$OUT/bench_7cpa_$V.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'])"
done
timeout 900 python bench.py --config hts --n-ligs 64 --steps 2 --warmup 3 > $OUT/bench_hts.json 2>$OUT/bench_hts.err; echo "hts rc=$?"; tail -c 1500 $OUT/bench_hts.json; tail -5 $OUT/bench_hts.err
