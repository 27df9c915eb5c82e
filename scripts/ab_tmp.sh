#!/bin/bash
set -u
OUT=gpurun_out/ab9; mkdir -p $OUT
bash scripts/gpu_tests.sh ab9t
timeout 600 python bench.py --config hts --n-ligs 256 --steps 2 --warmup 2 --no-cpu > $OUT/hts.json 2>$OUT/hts.err
python -c "import json;d=json.loads(open('$OUT/hts.json').read().strip().splitlines()[-1]);print('hts', '%.4g'%d['value'], '%.1f ms'%d['ms_per_step'], d['score_evals_per_s'])"
