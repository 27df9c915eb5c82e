#!/usr/bin/env python
"""bench.py — score evaluations/s of the B200 LGA docking hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1stp] [--impl ours|reference]

A step = one complete docking job of the config (all hot-path rows: init, GA generations
with offspring scoring, local search with scoring(+gradient), sum_evals/termination,
best-of-run) on synthetic inputs already resident in HBM.  Under torchrun every rank
docks its own `runs` independent runs (global run indices rank*runs.., weak scaling); the
only collective is the final NCCL all-gather of the best poses (NS).  Timing: CUDA
events on the launching stream, barrier + synchronize around the timed region, L2
flushed (256 MiB write) between steps, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "score evals/sec"
UNIT = "evals/s"


# ---------------------------------------------------------------------------
# Algorithmic work model: FP32 flops per energy evaluation, FMA = 2.
# ---------------------------------------------------------------------------
F_ORIENT = 30          # n, q, R(q) from (phi, theta, alpha)
F_TORSION = 110        # Rodrigues matrix + composite with the parent transform
F_ATOM_POSE = 18       # one 3x4 transform per atom
F_ATOM_INTER = 77      # trilinear: corner combine (3 maps), value and gradient
F_PAIR_E = 33          # D5 energy of one pair
F_PAIR_EG = 55         # D5 energy + dE/drho2 + force on both atoms (unique pair)
F_ATOM_BACK = 18       # (r - t) x g, sums
F_TORSION_BACK = 20    # per-torsion projection (plus 6 per moved atom)
F_GENE_ADADELTA = 12


def flops_per_eval(N, T, P, moved_total, grad):
    f = F_ORIENT + T * F_TORSION + N * (F_ATOM_POSE + F_ATOM_INTER)
    if grad:
        f += P * F_PAIR_EG + N * F_ATOM_BACK + T * F_TORSION_BACK + 6 * moved_total + (6 + T) * F_GENE_ADADELTA
    else:
        f += P * F_PAIR_E
    return f


def fp32_peak_tflops(sm_mhz):
    """148 SMs x 128 FP32 lanes x 2 flop/FMA x clock (B200_PROFILING.md: 148 SMs)."""
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def workload_desc(cfg):
    ls = "Solis-Wets" if cfg.ls_method == 1 else "ADADELTA"
    return (f"{cfg.name}-shaped ({cfg.note.split(':')[0]}): {cfg.n_atoms} atoms, {cfg.n_tors} torsions, "
            f"{cfg.grid_n}^3 grid, pop {cfg.pop}, {cfg.runs} runs/GPU, {cfg.max_evals} evals/run, {ls} "
            f"ls_rate {cfg.ls_rate}, {cfg.ls_iters} iters")


# ---------------------------------------------------------------------------
# CPU oracle baseline (rank 0, N = 1): bounded sample of the same workload.
# ---------------------------------------------------------------------------
def oracle_sample(cfg, lig, grid, budget, threads, seed=42):
    import oracle
    P = oracle.Problem(grid, lig)
    pp = oracle.params(ls_method=cfg.ls_method, ls_rate=cfg.ls_rate, ls_max_iters=cfg.ls_iters)
    out = [None] * threads

    def work(i):
        out[i] = oracle.dock_run(P, pp, cfg.pop, budget, seed, run=i)["evals"]
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    return sum(out), dt


def cpu_budget(cfg):
    # ~2-4 s of one core per run (oracle rates: 1stp 1.6e5, 3ce3 3e4, 7cpa 1e4 evals/s/core)
    return {"tiny": 2000, "1stp": 400_000, "3ce3": 90_000, "7cpa": 30_000}.get(cfg.name, 50_000)


def run_reference(args, cfg, lig, grid):
    """--impl reference: the oracle (as it stands) on the host cores, rank 0 only."""
    rank, _, world = env_rank()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    budget = cpu_budget(cfg)
    for _ in range(args.warmup):
        oracle_sample(cfg, lig, grid, budget, threads)
    tot_e, tot_t, per = 0, 0.0, []
    for s in range(args.steps):
        e, t = oracle_sample(cfg, lig, grid, budget, threads, seed=42 + s)
        tot_e += e; tot_t += t; per.append(t)
    v = tot_e / tot_t
    sample = f"{threads} independent runs of the {cfg.name} workload, each capped at {budget} evals, per step"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gen/synth.py, seeded)",
            "config": {"workload": workload_desc(cfg), "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_ours(args, cfg, lig, grid):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2203_02096_b200 as dock

    rank, local, world = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    d = dock.Docker.from_inputs(grid, lig, ls_method=cfg.ls_method, ls_rate=cfg.ls_rate,
                                ls_max_iters=cfg.ls_iters, profile=1, device=local)
    runs = cfg.runs
    run_base = rank * runs
    stream = torch.cuda.Stream(device=dev)
    bE = torch.empty(runs, dtype=torch.float32, device=dev)
    bG = torch.empty(runs, d.G, dtype=torch.float32, device=dev)
    ev = torch.empty(runs, dtype=torch.int64, device=dev)
    gens = torch.empty(runs, dtype=torch.int32, device=dev)
    gather_E = torch.empty(world * runs, dtype=torch.float32, device=dev)
    gather_G = torch.empty(world * runs, d.G, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    moved_total = int(np.asarray(d.torsions()[1]).sum())
    f_e = flops_per_eval(d.N, d.T, d.P, moved_total, grad=False)
    f_eg = flops_per_eval(d.N, d.T, d.P, moved_total, grad=True)

    def step(seed):
        with torch.cuda.stream(stream):
            d.run_device(cfg.pop, runs, cfg.max_evals, seed, bE, bG, ev, gens, run_base=run_base,
                         stream=stream.cuda_stream)
            if world > 1:   # NS: NCCL only for the final gather of best poses
                dist.all_gather_into_tensor(gather_E, bE)
                dist.all_gather_into_tensor(gather_G, bG)

    for w in range(args.warmup):
        step(42)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    times, evals, ls_ms, ls_n, ga_ms, ga_n = [], 0, 0.0, 0, 0.0, 0
    launches0 = d.launches
    for s in range(args.steps):
        flush.zero_()                               # L2 flush between timed steps
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(42)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        times.append(e0.elapsed_time(e1))
        evals += int(ev.sum().item())
        ms, n = d.kernel_stats()
        ga_ms += ms[0]; ga_n += int(n[0]); ls_ms += ms[1]; ls_n += int(n[1])
    launches = d.launches - launches0
    clk = clocks.stop()
    t_local = sum(times)
    t_max = t_local
    tot_evals = evals
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        te = torch.tensor([evals], dtype=torch.int64, device=dev)
        dist.all_reduce(te)
        tot_evals = int(te.item())
    value = tot_evals / (t_max / 1e3)
    ms_per_step = t_max / args.steps

    # ---- roofline of the dominant kernel (local search) from live CUDA events ----
    evals_step = evals // args.steps
    per_gen_ga = cfg.pop - 1
    gens_np = gens.cpu().numpy()
    ga_evals_step = int(gens_np.sum()) * per_gen_ga + runs * cfg.pop
    ls_evals_step = evals_step - ga_evals_step
    grad = cfg.ls_method == 0
    ls_flops = ls_evals_step * args.steps * (f_eg if grad else f_e)
    ga_flops = ga_evals_step * args.steps * f_e
    peaks = measured_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    peak = fp32_peak_tflops(sm_mhz)
    ls_tflops = ls_flops / (ls_ms / 1e3) / 1e12 if ls_ms > 0 else 0.0
    ga_tflops = ga_flops / (ga_ms / 1e3) / 1e12 if ga_ms > 0 else 0.0
    roofline = {"kernel": "k_ls_sw" if not grad else "k_ls_adadelta", "bound": "alu", "achieved": ls_tflops,
                "peak": peak, "unit": "TFLOP/s", "frac": ls_tflops / peak,
                "traffic": None,
                "flops_per_eval": f_eg if grad else f_e, "evals_per_launch": ls_evals_step * args.steps / max(ls_n, 1),
                "avg_launch_ms": ls_ms / max(ls_n, 1), "share_of_step": ls_ms / t_local if t_local else None,
                "peak_source": f"derived: 148 SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                "ga_kernel": {"achieved": ga_tflops, "avg_launch_ms": ga_ms / max(ga_n, 1),
                              "share_of_step": ga_ms / t_local if t_local else None}}

    # ---- end to end through the public API with host buffers ----
    e2e_steps = max(1, min(args.steps, 3))
    tp, roles = grid.type_params()
    e2e_t, e2e_evals = 0.0, 0
    h2d = d2h = 0
    for s in range(e2e_steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dd = dock.Docker(grid.maps, grid.n, grid.spacing, grid.origin, tp, roles, lig.types, lig.charges,
                         lig.xyz, lig.bonds, lig.rotatable, ls_method=cfg.ls_method, ls_rate=cfg.ls_rate,
                         ls_max_iters=cfg.ls_iters, device=local)
        r = dd.run(cfg.pop, runs, cfg.max_evals, 42, run_base=run_base, xyz=True)
        h2d = dd.upload_bytes
        dd.close()
        t1 = time.perf_counter()
        e2e_t = max(e2e_t, 0) + (t1 - t0)
        e2e_evals += int(r["evals"].sum())
        d2h = r["best_E"].nbytes + r["best_genes"].nbytes + r["best_xyz"].nbytes + r["evals"].nbytes + \
            r["generations"].nbytes + 16 * runs * int(np.ceil(r["generations"].max() / 16 + 1))
    if world > 1:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())
        te = torch.tensor([e2e_evals], dtype=torch.int64, device=dev)
        dist.all_reduce(te)
        e2e_evals = int(te.item())
    e2e_value = e2e_evals / e2e_t

    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (gen/synth.py, seeded ligand + pseudo-receptor maps)",
                "config": {"workload": workload_desc(cfg), "runs_per_gpu": runs, "global_runs": runs * world,
                           "l2": "flushed between steps (256 MiB write); grid pinned by an L2 access window",
                           "parallelism": f"dp{world} (independent runs per GPU)"},
                "ligands_per_hour": 3600.0 * world / (ms_per_step / 1e3),
                "gpu_launches": launches,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "note": "dock_init (host grid+ligand upload) + dock_run_ex (host outputs) + dock_free, wall clock"},
                "roofline": roofline,
                "clocks": clk}
        if world == 1 and not args.no_cpu:
            threads = os.cpu_count() or 1
            budget = cpu_budget(cfg)
            ce, ct = oracle_sample(cfg, lig, grid, budget, threads)
            line["cpu_baseline"] = {"value": ce / ct, "unit": UNIT, "cores": threads, "kind": "oracle",
                                    "sample": f"{threads} runs x {budget} evals of the same workload, one per thread"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    d.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="1stp", choices=["tiny", "1stp", "3ce3", "7cpa"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    from gen import config_inputs
    cfg, lig, grid = config_inputs(args.config)
    if args.impl == "reference":
        run_reference(args, cfg, lig, grid)
    else:
        run_ours(args, cfg, lig, grid)


if __name__ == "__main__":
    main()
