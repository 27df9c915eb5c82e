#!/bin/bash
# round 2 pass zj: packed loops unrolled by 2 (default) vs 1 (pu1)
set -u
OUT=gpurun_out/r02zj; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa" "pu1" 3
