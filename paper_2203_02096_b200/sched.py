"""Rank-level ligand sharding for one-process-per-GPU screens.

Above dock_screen (which balances ligands over the slots and devices of ONE process),
a torchrun job with one rank per GPU splits the library with a deterministic
longest-processing-time-first partition. The partition uses the §8(e) cost model
cost = 40 P + 133 N, and the C++ scheduler uses the same model. Each rank docks its share
with global ligand ids, so the Philox key (D2) and every result are independent of the
rank count. The only collective is one gather of fixed-size result records at the end
(NS: "NCCL appears only for a final gather of best poses"). This module is host
plumbing: it does no docking arithmetic.
"""
from __future__ import annotations

import heapq

import numpy as np

RECORD_FIELDS = ("best_E", "best_run", "evals", "status")


def ligand_cost(n_atoms, n_pairs):
    """§8(e) cost model per ligand (runs x max_evals is common to a screen)."""
    return 40.0 * np.asarray(n_pairs, np.float64) + 133.0 * np.asarray(n_atoms, np.float64)


def lpt_partition(costs, world):
    """Greedy LPT: ligands by decreasing cost (ties: lower index first), each to the
    currently least-loaded rank (ties: lower rank). Returns `world` sorted index arrays."""
    costs = np.asarray(costs, np.float64)
    order = sorted(range(costs.shape[0]), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    parts = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        parts[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [np.array(sorted(p), dtype=np.int64) for p in parts]


def gather_records(local_idx, records, n_total, group=None, device="cpu"):
    """All-gather per-ligand result records into global order.

    local_idx: global indices of this rank's ligands; records: dict with best_E [n],
    best_run [n], evals [n], status [n], best_genes [n, 38] for those ligands. Every rank
    returns the full arrays (index-ordered). Uses one all_gather of a padded float64
    record tensor. This works with gloo (CPU tensors) and nccl (device="cuda:k")."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n_local = int(len(local_idx))
    G = records["best_genes"].shape[1] if n_local else 38
    width = 1 + len(RECORD_FIELDS) + G
    counts = torch.tensor([n_local], dtype=torch.int64, device=device)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts, group=group)
    cap = int(max(int(c.item()) for c in all_counts))
    buf = np.zeros((max(cap, 1), width), np.float64)
    buf[:, 0] = -1
    if n_local:
        buf[:n_local, 0] = np.asarray(local_idx, np.float64)
        for k, f in enumerate(RECORD_FIELDS):
            buf[:n_local, 1 + k] = np.asarray(records[f], np.float64)
        buf[:n_local, 1 + len(RECORD_FIELDS):] = records["best_genes"]
    t = torch.from_numpy(buf).to(device)
    outs = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    full = np.concatenate([o.cpu().numpy() for o in outs])
    full = full[full[:, 0] >= 0]
    res = {"best_E": np.full(n_total, np.nan, np.float32), "best_run": np.full(n_total, -1, np.int32),
           "evals": np.zeros(n_total, np.int64), "status": np.full(n_total, -1, np.int32),
           "best_genes": np.zeros((n_total, G), np.float32)}
    idx = full[:, 0].astype(np.int64)
    if np.unique(idx).shape[0] != idx.shape[0]:
        raise RuntimeError("gather_records: a ligand was docked by two ranks")
    res["best_E"][idx] = full[:, 1]
    res["best_run"][idx] = full[:, 2]
    res["evals"][idx] = full[:, 3]
    res["status"][idx] = full[:, 4]
    res["best_genes"][idx] = full[:, 5:]
    return res
