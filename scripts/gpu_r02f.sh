#!/bin/bash
# round 2 pass f: A/B folded D5 slot constants (default) vs unfolded (DK_FOLD=0) on 7cpa / 3ce3,
# the new statistics / multi-rank / verbatim GPU tests, then the full default bench line.
set -u
OUT=gpurun_out/r02f; mkdir -p $OUT
for rep in 1 2; do
for C in 7cpa 3ce3; do
  timeout 300 python bench.py --config $C --steps 3 --warmup 2 --no-cpu --no-parts > $OUT/ab_fold_${C}_$rep.json 2>&1
  DOCK_LIB=build/variants/libdock_nofold.so timeout 300 python bench.py --config $C --steps 3 --warmup 2 --no-cpu --no-parts > $OUT/ab_nofold_${C}_$rep.json 2>&1
  python - <<PY
import json
for t in ("fold", "nofold"):
    d = json.loads(open("$OUT/ab_%s_${C}_$rep.json" % t).read().strip().splitlines()[-1])
    print("$C rep $rep", t, "%.4g" % d["value"])
PY
done; done
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -m gpu -q -x -rf -s -k "statistics or planted or multirank or two_ranks or screen_two or spec_style" > $OUT/pytest_new.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_new.log
grep -E "CFG0|passed|failed|FAILED" $OUT/pytest_new.log | tail -12
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; tail -c 1500 $OUT/bench_default.json
