#!/bin/bash
# round 2 pass zk: packed loops unrolled by 2 (default) vs 4 (pu4)
set -u
OUT=gpurun_out/r02zk; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa" "pu4" 3
