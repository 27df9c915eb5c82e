"""Multi-GPU paths on the one GPU of the test box.

* bench.py under torchrun with 2 ranks (BENCH_DIST_TEST=1: gloo collectives over CPU
  tensors, both ranks on GPU 0 -- their kernels never wait on each other): the R runs are
  split over the ranks with global run ids, and the gathered per-run results must equal the
  1-rank run's exactly (result_digest of every run's best energy and genotype).
* dock_screen's multi-device dispatcher with devices = [0, 0] (two receptor uploads, worker
  slots on both entries): every ligand's result equals the single-device screen's.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dock():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2203_02096_b200._build import build
    build()
    import paper_2203_02096_b200 as d
    return d


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(args, nproc):
    env = dict(os.environ, BENCH_DIST_TEST="1")
    cmd = [sys.executable, "bench.py", *args]
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", "bench.py", *args]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("config,extra", [("1stp", ["--runs", "5", "--max-evals", "40000"]),
                                          ("3ce3", ["--runs", "3", "--max-evals", "30000"])])
def test_two_ranks_split_runs_equal_one_rank(dock, config, extra):
    args = ["--config", config, "--steps", "1", "--warmup", "1", "--no-cpu", "--no-parts", *extra]
    one = _bench(args, 1)
    two = _bench(["--gpus", "2", *args], 2)
    assert two["n_gpus"] == 2 and two["scaling"] == "strong"
    assert two["config"]["global_runs"] == one["config"]["global_runs"]
    assert two["result_digest"] == one["result_digest"]


def test_screen_two_device_entries_equal_one(dock):
    from gen import hts_ligands
    from gen.synth import TYPE_NAMES, make_grid
    ligs = hts_ligands(6, seed=13)
    grid = make_grid(24, 0.5, list(TYPE_NAMES), seed=77)
    kw = dict(ls_method=0, ls_rate=0.25, ls_max_iters=20)
    a = dock.screen(grid, ligs, 24, 2, 3000, 99, devices=[0], slots_per_device=2, **kw)
    b = dock.screen(grid, ligs, 24, 2, 3000, 99, devices=[0, 0], slots_per_device=2, **kw)
    for k in ("best_E", "best_run", "best_genes", "evals", "status"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert (b["status"] == 0).all()
