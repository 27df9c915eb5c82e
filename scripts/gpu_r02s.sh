#!/bin/bash
# round 2 pass s: lean D5 slots (DK_LEAN) -- the -m gpu suite, then an A/B against the
# DK_LEAN=0 build (build/ab/libdock_nolean.so) on 7cpa and 3ce3
set -u
OUT=gpurun_out/r02s; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
bash scripts/gpu_ab.sh $OUT/ab "7cpa 3ce3" "nolean" 2
