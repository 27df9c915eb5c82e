#!/bin/bash
# round 2 pass zn: the packed hybrid tail pair loop unrolled by 2 (hpu2)
# against the default (1)
set -u
OUT=gpurun_out/r02zn; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa" "hpu2" 3
