"""Host logic of the multi-GPU ligand scheduler, on CPU: the LPT rank
partition and the final result gather over a world_size-2 gloo group."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from gen import CONFIGS, TYPE_TABLE, hts_ligands


def _sched():
    from paper_2203_02096_b200._build import build
    build()
    from paper_2203_02096_b200 import sched
    return sched


def test_lpt_partition_covers_each_ligand_once():
    sched = _sched()
    rng = np.random.default_rng(0)
    costs = rng.uniform(100, 10000, size=257)
    for world in (1, 2, 3, 8):
        parts = sched.lpt_partition(costs, world)
        allidx = np.concatenate(parts)
        assert sorted(allidx.tolist()) == list(range(257))
        loads = np.array([costs[p].sum() for p in parts])
        # LPT bound: no rank exceeds the mean load by more than the largest single job
        assert loads.max() - loads.mean() <= costs.max() + 1e-9
        assert [p.tolist() for p in sched.lpt_partition(costs, world)] == [p.tolist() for p in parts]


def test_lpt_partition_ties_and_degenerate():
    sched = _sched()
    parts = sched.lpt_partition([5.0, 5.0, 5.0, 5.0], 2)
    assert [p.tolist() for p in parts] == [[0, 2], [1, 3]]
    parts = sched.lpt_partition([1.0], 4)
    assert [len(p) for p in parts] == [1, 0, 0, 0]
    assert [len(p) for p in sched.lpt_partition([], 2)] == [0, 0]


def test_cost_model_uses_topology_pairs():
    sched = _sched()
    import paper_2203_02096_b200 as dock
    ligs = hts_ligands(6)
    names = list(TYPE_TABLE)
    tp = np.array([TYPE_TABLE[t][:4] for t in names], np.float32)
    roles = np.array([TYPE_TABLE[t][4] for t in names], np.int32)
    for lig in ligs:
        _, _, pairs = dock.topology(lig.types, lig.charges, lig.xyz, lig.bonds, lig.rotatable, tp, roles)
        c = sched.ligand_cost(len(lig.types), pairs.shape[0])
        assert c == 40.0 * pairs.shape[0] + 133.0 * len(lig.types)


def _worker(rank, world, port, n_total, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_02096_b200 import sched
    costs = np.arange(n_total, dtype=np.float64) % 7 + 1.0
    mine = sched.lpt_partition(costs, world)[rank]
    G = 38
    rec = {"best_E": -(mine.astype(np.float32) + 0.25), "best_run": (mine % 5).astype(np.int32),
           "evals": (mine * 1000 + 7).astype(np.int64), "status": np.zeros(len(mine), np.int32),
           "best_genes": np.tile(mine[:, None].astype(np.float32), (1, G)) * 0.5}
    res = sched.gather_records(mine, rec, n_total)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, res))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_gather_records_world2_gloo():
    _sched()
    n_total = 23
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=100) for _ in range(2))
    for p in ps:
        p.join(timeout=30)
        assert p.exitcode == 0
    idx = np.arange(n_total)
    for r in (0, 1):
        res = out[r]
        np.testing.assert_array_equal(res["best_E"], -(idx.astype(np.float32) + 0.25))
        np.testing.assert_array_equal(res["best_run"], idx % 5)
        np.testing.assert_array_equal(res["evals"], idx * 1000 + 7)
        np.testing.assert_array_equal(res["status"], np.zeros(n_total))
        np.testing.assert_array_equal(res["best_genes"][:, 3], idx.astype(np.float32) * 0.5)
