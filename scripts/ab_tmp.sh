#!/bin/bash
set -u
OUT=gpurun_out/ab3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -k "max_size or large or deep" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" $OUT/pytest.log | head -20
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], d.get('score_evals_per_s'))" 2>/dev/null || tail -3 ${1%.json}.err; }
for S in 2 4 8; do
  timeout 600 python bench.py --config hts --n-ligs 256 --steps 2 --warmup 2 --no-cpu --slots $S > $OUT/hts_s$S.json 2>$OUT/hts_s$S.err; j $OUT/hts_s$S.json
done
