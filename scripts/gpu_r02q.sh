#!/bin/bash
# round 2 pass q: the driver's exact commands (timed): our arm and the reference arm
set -u
OUT=gpurun_out/r02q; mkdir -p $OUT
s=$(date +%s); timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "ours rc=$? $(( $(date +%s) - s )) s"
s=$(date +%s); timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$? $(( $(date +%s) - s )) s"
python - <<PY
import json
d = json.loads(open("$OUT/bench.json").read().strip().splitlines()[-1])
print("value %.4g ms %.1f frac %.4f e2e %.4g" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"]))
print(json.dumps(d.get("also")))
print(d["step_ms"], d["clocks"])
r = json.loads(open("$OUT/ref.json").read().strip().splitlines()[-1])
print("ref value %.4g" % r["value"], r["cpu_baseline"].get("cores"))
PY
