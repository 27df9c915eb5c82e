#!/bin/bash
# A/B timing of build/ab/libdock_<tag>.so variants against the default library on one box.
#   bash scripts/gpu_ab.sh OUTDIR "7cpa 3ce3" "tagA tagB ..." [reps]
set -u
OUT=$1; CONFIGS=$2; TAGS=$3; REPS=${4:-2}
mkdir -p $OUT
for rep in $(seq 1 $REPS); do
for C in $CONFIGS; do
  for T in default $TAGS; do
    if [ "$T" = default ]; then L=""; else L="build/ab/libdock_$T.so"; fi
    DOCK_LIB=$L timeout 300 python bench.py --config $C --steps 3 --warmup 2 --no-cpu --no-parts > $OUT/ab_${T}_${C}_$rep.json 2> $OUT/ab_${T}_${C}_$rep.err
    python -c "import json;d=json.loads(open('$OUT/ab_${T}_${C}_$rep.json').read().strip().splitlines()[-1]);print('$C rep $rep $T', '%.4g'%d['value'])" 2>&1 | tail -1
  done
done; done
