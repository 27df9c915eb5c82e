#!/bin/bash
# round 2 pass zo: packed loops unrolled by 8 (pu8)
# against the default (4)
set -u
OUT=gpurun_out/r02zo; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa" "pu8" 3
