#!/bin/bash
OUT=gpurun_out/abun; mkdir -p $OUT
for C in 3ce3 7cpa; do for V in default u8 u2; do
  if [ $V = default ]; then L=""; else L=build/variants/libdock_$V.so; fi
  DOCK_LIB=$L timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu > $OUT/b_${C}_$V.json 2>&1
  python -c "import json;d=json.loads(open('$OUT/b_${C}_$V.json').read().strip().splitlines()[-1]);print('$C $V', '%.4g'%d['value'])"
done; done
