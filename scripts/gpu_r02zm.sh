#!/bin/bash
# round 2 pass zm: torsion walk unrolled by 4 for every shape (walk4) and the scalar tile loop
# unrolled by 8 (tu8) against the defaults
set -u
OUT=gpurun_out/r02zm; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa 3ce3" "walk4 tu8" 2
