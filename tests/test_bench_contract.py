"""bench.py contract on CPU: the reference arm (the oracle on host cores) prints one JSON
line with the fields the driver reads, for the single-ligand and the HTS metric."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "gpu_launches"}


@pytest.mark.parametrize("args,unit", [(["--config", "tiny"], "evals/s"),
                                       (["--config", "tiny", "--scoring", "ad4"], "evals/s")])
def test_reference_arm_line(args, unit):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", *args], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert KEYS <= set(line), KEYS - set(line)
    assert line["impl"] == "reference" and line["unit"] == unit and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["gpu_launches"] == 0 and line["higher_is_better"] is True
    if "ad4" in args:
        assert "AD4" in line["config"]["workload"]
