#!/bin/bash
# One GPU-box pass: build, gpu tests, smoke, bench lines, ncu launch list + one full capture.
# Usage (via gpurun): bash scripts/gpu_round.sh <tag> [configs...]
set -u
TAG=${1:-r01}; shift || true
CFGS=${@:-"1stp 3ce3 7cpa hts"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
for C in $CFGS; do
  timeout 900 python bench.py --config $C > $OUT/bench_$C.json 2> $OUT/bench_$C.err; echo "bench $C rc=$?"; tail -c 600 $OUT/bench_$C.json
done
if [ "${PROFILE:-1}" = "1" ]; then
  SKIP=1 bash scripts/gpu_profile.sh 1stp k_run_sw $TAG
  bash scripts/gpu_profile.sh 7cpa k_ls_adadelta $TAG
  ls -la gpurun_out/
fi
