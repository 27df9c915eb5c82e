#!/usr/bin/env python
"""bench.py — score evaluations/s of the B200 LGA docking hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 7cpa] [--impl ours|reference]

The default config is BASELINE.json configs[3] (7cpa-shaped), the largest single-GPU config.

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
# Algorithmic work model: SURVEY.md §8(d) "Op-count model" (FP32 flops, FMA = 2), used
# verbatim for roofline.achieved:
#   per pair   21 (energy) / 40 (energy + gradient)
#   per atom   60 / 100 interpolation + 18 pose (+ 15 back-projection with the gradient)
#   per torsion 55 / 92;  per gene 12 (ADADELTA update, gradient path only)
# C3 (N 70, T 15, P 2,000): 48.3 k / 91.1 k flop per evaluation, as §8(d)'s table.
# ---------------------------------------------------------------------------
F_PAIR = (21, 40)
F_ATOM_INTER = (60, 100)
F_ATOM_POSE = 18
F_ATOM_BACK = 15
F_TORSION = (55, 92)
F_GENE_ADADELTA = 12
# NEXT-2 D5-AD4 pair: + r, smoothing, the sigmoidal dielectric and two cutoffs;
# not in §8(d), scaled from D5's pair by the AD4 pair's extra XU + FMA work (5 vs 2 XU ops)
F_PAIR_AD4 = (33, 62)

SCORING = 0            # --scoring: 0 = D5, 1 = D5-AD4 (dock_params.scoring)


def flops_per_eval(N, T, P, grad):
    """§8(d) op-count model of one evaluation (energy only, or energy + gradient + ADADELTA)."""
    g = 1 if grad else 0
    f = P * (F_PAIR_AD4 if SCORING else F_PAIR)[g] + N * (F_ATOM_INTER[g] + F_ATOM_POSE) + T * F_TORSION[g]
    if grad:
        f += N * F_ATOM_BACK + (6 + T) * F_GENE_ADADELTA
    return f


def fp32_peak_tflops(sm_mhz):
    """148 SMs x 128 FP32 lanes x 2 flop/FMA x clock (B200_PROFILING.md: 148 SMs)."""
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    captures (profiles/ncu_traffic.json); absent -> null."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return {}


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


def dist_setup(local, world):
    """One process per GPU, NCCL.  Returns (device, collective device).  BENCH_DIST_TEST=1 is
    a test-only mode: gloo over CPU tensors and GPU local % device_count, so the multi-rank
    path (sharding, barriers, max-over-ranks, gathers) runs on a 1-GPU box."""
    import torch
    import torch.distributed as dist
    test = os.environ.get("BENCH_DIST_TEST") == "1"
    idx = local % max(1, torch.cuda.device_count()) if test else local
    torch.cuda.set_device(idx)
    dev = torch.device("cuda", idx)
    if world > 1:
        if test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    return dev, (torch.device("cpu") if test else dev)


def all_gather_cat(t, cdev):
    """Concatenate `t` from every rank (rank order) on the collective device."""
    import torch
    import torch.distributed as dist
    x = t.to(cdev)
    parts = [torch.empty_like(x) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, x)
    return torch.cat(parts)


def reduce_scalar(v, dtype, op, cdev):
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=dtype, device=cdev)
    dist.all_reduce(t, op=op)
    return t.item()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def workload_desc(cfg):
    ls = "Solis-Wets" if cfg.ls_method == 1 else "ADADELTA"
    return (f"{cfg.name}-shaped ({cfg.note.split(':')[0]}): {cfg.n_atoms} atoms, {cfg.n_tors} torsions, "
            f"{cfg.grid_n}^3 grid, pop {cfg.pop}, {cfg.runs} runs/GPU, {cfg.max_evals} evals/run, {ls} "
            f"ls_rate {cfg.ls_rate}, {cfg.ls_iters} iters" + (", AD4.1-calibrated scoring (NEXT-2)" if SCORING else ""))


# ---------------------------------------------------------------------------
# CPU oracle baseline (rank 0, N = 1): bounded sample of the same workload.
# ---------------------------------------------------------------------------
def oracle_sample(cfg, lig, grid, budget, threads, seed=42):
    import oracle
    P = oracle.Problem(grid, lig, sf={} if SCORING else None)
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


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(cfg, lig, grid, repeats=3):
    """The oracle as it stands on the host (SURVEY.md §8(d) "CPU oracle baseline"): per core
    (one run on one thread) and per box (one run per hardware thread, `repeats` times: median
    and spread), on a bounded sample of the same workload."""
    threads = os.cpu_count() or 1
    budget = cpu_budget(cfg)
    e1, t1 = oracle_sample(cfg, lig, grid, budget, 1)
    box = []
    for r in range(repeats):
        e, t = oracle_sample(cfg, lig, grid, budget, threads, seed=42 + r)
        box.append(e / t)
    med = statistics.median(box)
    return {"value": med, "unit": UNIT, "cores": threads, "kind": "oracle",
            "per_core": e1 / t1, "box_runs": box, "box_spread": (max(box) - min(box)) / med,
            "cpu_model": cpu_model(),
            "sample": f"{threads} runs x {budget} evals of the same workload, one per hardware thread, median of "
                      f"{repeats}; per_core: one run of {budget} evals on one thread",
            "note": "double-precision C oracle, gcc -O2, no fast-math: a reported baseline, not the target"}


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
def other_configs(gpu, steps=3):
    """The other BASELINE.json configs in the same run (C1-C3 at 1 GPU, and
    the HTS sample), each device-timed like the headline: one warm-up job, then `steps` jobs
    with CUDA events around dock_run_device (HTS: wall clock around dock_screen)."""
    import torch
    import paper_2203_02096_b200 as dock
    from gen import config_inputs, hts_ligands
    out = {}
    dev = torch.device("cuda", gpu)
    for name in ("1stp", "3ce3"):
        c, lg, gr = config_inputs(name)
        d = dock.Docker.from_inputs(gr, lg, ls_method=c.ls_method, ls_rate=c.ls_rate, ls_max_iters=c.ls_iters,
                                    device=gpu)
        st = torch.cuda.Stream(device=dev)
        bE = torch.empty(c.runs, dtype=torch.float32, device=dev)
        bG = torch.empty(c.runs, d.G, dtype=torch.float32, device=dev)
        ev = torch.empty(c.runs, dtype=torch.int64, device=dev)
        gens = torch.empty(c.runs, dtype=torch.int32, device=dev)
        ms, evals = [], 0
        for s in range(steps + 1):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            d.run_device(c.pop, c.runs, c.max_evals, 42, bE, bG, ev, gens, stream=st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            if s > 0:
                ms.append(e0.elapsed_time(e1)); evals += int(ev.sum().item())
        out[f"configs[{1 if name == '1stp' else 2}] {name}"] = {
            "value": evals / (sum(ms) / 1e3), "unit": UNIT, "ms_per_step": statistics.median(ms),
            "engine": d.engine, "workload": workload_desc(c), "steps": steps}
        d.close()
    c, _, gr = config_inputs("hts")
    ligs = hts_ligands(256)
    kw = dict(ls_method=c.ls_method, ls_rate=c.ls_rate, ls_max_iters=c.ls_iters)
    dock.screen(gr, ligs[:8], c.pop, c.runs, c.max_evals // 10, 7, devices=[gpu], **kw)
    t = []
    for s in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dock.screen(gr, ligs, c.pop, c.runs, c.max_evals, 42, devices=[gpu], **kw)
        t.append(time.perf_counter() - t0)
    out["configs[4] hts"] = {"value": 3600.0 * len(ligs) * len(t) / sum(t), "unit": "ligands/h",
                             "workload": f"256-ligand sample of configs[4] (N ~ U{{10..70}}), pop {c.pop}, "
                                         f"{c.runs} runs x {c.max_evals} evals, dock_screen wall clock", "steps": 2}
    return out


def run_ours(args, cfg, lig, grid):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2203_02096_b200 as dock

    rank, local, world = env_rank()
    dev, cdev = dist_setup(local, world)
    gpu = dev.index
    def make(prof):
        return dock.Docker.from_inputs(grid, lig, ls_method=cfg.ls_method, ls_rate=cfg.ls_rate,
                                       ls_max_iters=cfg.ls_iters, profile=prof, device=gpu, sw_depth=args.sw_depth,
                                       scoring=SCORING, sw_split=args.sw_split, run_branches=args.run_branches)
    d = make(1)          # profiled context (CUDA events around the LS launches)
    # the config's R runs are split contiguously over the ranks, rank k docks
    # global runs [kR/G, (k+1)R/G) (strong scaling; the Philox counter carries the global run
    # index, so the results equal the 1-GPU run's).  --weak: every rank docks R runs of its own.
    total_runs = cfg.runs * world if args.weak else cfg.runs
    run_base = rank * cfg.runs if args.weak else rank * total_runs // world
    runs = cfg.runs if args.weak else (rank + 1) * total_runs // world - run_base
    rmax = -(-total_runs // world)                  # gather rows per rank (padded)
    if runs < 1:
        raise SystemExit(f"rank {rank}: no runs ({total_runs} runs over {world} ranks); use fewer GPUs or --runs")
    stream = torch.cuda.Stream(device=dev)
    bE = torch.empty(runs, dtype=torch.float32, device=dev)
    bG = torch.empty(runs, d.G, dtype=torch.float32, device=dev)
    ev = torch.empty(runs, dtype=torch.int64, device=dev)
    gens = torch.empty(runs, dtype=torch.int32, device=dev)
    gathered = {}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    f_e = flops_per_eval(d.N, d.T, d.P, grad=False)
    f_eg = flops_per_eval(d.N, d.T, d.P, grad=True)

    def step(seed, ctx=None, gather=True):
        # gather=False: this rank's extra (unprofiled-context warm-up / profiled) steps, which
        # other ranks may not run (engines can differ per rank), so no collective in them
        with torch.cuda.stream(stream):
            (ctx or d).run_device(cfg.pop, runs, cfg.max_evals, seed, bE, bG, ev, gens, run_base=run_base,
                                  stream=stream.cuda_stream)
            if world > 1 and gather:   # NS: NCCL only for the final gather of best poses (rows padded to rmax)
                pE = torch.full((rmax,), float("nan"), dtype=torch.float32, device=dev)
                pG = torch.zeros(rmax, d.G, dtype=torch.float32, device=dev)
                pE[:runs] = bE; pG[:runs] = bG
                gathered["E"] = all_gather_cat(pE, cdev)
                gathered["G"] = all_gather_cat(pG, cdev)

    for w in range(args.warmup):
        step(42)
    torch.cuda.synchronize()
    # Run branches (Solis-Wets): timing events inside the branched generation
    # graph perturb it (1stp 455 vs 302 ms per step), so the timed region runs an
    # unprofiled context and the LS launch times come from one extra profiled step after it.
    branches = d.run_branches
    engine = d.engine
    dt = d
    if branches > 1:
        dt = make(0)
        for w in range(args.warmup):
            step(42, dt, gather=False)
        torch.cuda.synchronize()
    clocks = ClockSampler(gpu)
    clocks.start()
    times, evals, ls_ms, ls_n = [], 0, 0.0, 0
    launches0 = dt.launches
    for s in range(args.steps):
        flush.zero_()                               # L2 flush between timed steps
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(42, dt)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        times.append(e0.elapsed_time(e1))
        evals += int(ev.sum().item())
        if branches == 1:
            ms, n = d.kernel_stats()
            ls_ms += ms[1]; ls_n += int(n[1])
    launches = dt.launches - launches0
    prof_steps, t_share = args.steps, sum(times)
    if branches > 1:
        # the profiled step: the events time run 0's LS launches; the other runs' identical
        # launches run concurrently with them
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(42, gather=False)
        e1.record(stream)
        torch.cuda.synchronize()
        ms, n = d.kernel_stats()
        ls_ms, ls_n, prof_steps, t_share = ms[1], int(n[1]), 1, e0.elapsed_time(e1)
    clk = clocks.stop()
    t_local = sum(times)
    t_max = t_local
    tot_evals = evals
    if world > 1:
        t_max = float(reduce_scalar(t_local, torch.float64, dist.ReduceOp.MAX, cdev))
        tot_evals = int(reduce_scalar(evals, torch.int64, dist.ReduceOp.SUM, cdev))
    value = tot_evals / (t_max / 1e3)
    ms_per_step = t_max / args.steps

    # ---- roofline of the dominant kernel (local search) from live CUDA events ----
    evals_step = evals // args.steps
    per_gen_ga = cfg.pop - 1
    gens_np = gens.cpu().numpy()
    ga_evals_step = int(gens_np.sum()) * per_gen_ga + runs * cfg.pop
    ls_evals_step = evals_step - ga_evals_step
    grad = cfg.ls_method == 0
    ls_flops = ls_evals_step * prof_steps * (f_eg if grad else f_e)
    peaks = measured_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    peak = fp32_peak_tflops(sm_mhz)
    ls_tflops = ls_flops / (ls_ms / 1e3) / 1e12 if ls_ms > 0 else 0.0
    tr = ncu_traffic().get(cfg.name) or {}
    if grad:
        kname = "k_ls_adadelta"
    elif engine == "clusters":
        kname = "k_run_sw (persistent cluster engine; timed unit: one LS phase of run 0, GA barrier -> LS barrier)"
    else:
        kname = "k_ls_sw_tree / k_ls_sw (Solis-Wets LS, depth auto)"
    roofline = {"kernel": kname, "engine": engine,
                "bound": "alu", "achieved": ls_tflops,
                "peak": peak, "unit": "TFLOP/s", "frac": ls_tflops / peak,
                "traffic": tr.get("dram_bytes_per_launch"),
                "traffic_source": tr.get("source"),
                "flops_per_eval": f_eg if grad else f_e,
                "evals_per_launch": ls_evals_step * prof_steps / max(ls_n * branches, 1),
                "run_branches": branches,
                "avg_launch_ms": ls_ms / max(ls_n, 1), "share_of_step": ls_ms / t_share if t_share else None,
                "peak_source": f"derived: 148 SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                "note": ("Solis-Wets chains are a dependent sequence of energy evaluations and only "
                         f"{runs * int(cfg.ls_rate * cfg.pop + 0.9999)} chains run per generation: the kernel is "
                         "latency-bound (DESIGN.md §7), so this ALU fraction is low by construction"
                         + (f"; {branches} concurrent runs ({engine}): achieved = all runs' LS flops / run 0's "
                            "LS time (the runs execute concurrently), share_of_step = run 0's LS time / step"
                            if branches > 1 else ""))
                if not grad else "issue-bound pair tiles (ncu: profiles/)"}

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
                         ls_max_iters=cfg.ls_iters, device=gpu, scoring=SCORING)
        r = dd.run(cfg.pop, runs, cfg.max_evals, 42, run_base=run_base, xyz=True)
        h2d = dd.upload_bytes
        dd.close()
        t1 = time.perf_counter()
        e2e_t = max(e2e_t, 0) + (t1 - t0)
        e2e_evals += int(r["evals"].sum())
        d2h = r["best_E"].nbytes + r["best_genes"].nbytes + r["best_xyz"].nbytes + r["evals"].nbytes + \
            r["generations"].nbytes + 16 * runs * int(np.ceil(r["generations"].max() / 16 + 1))
    if world > 1:
        e2e_t = float(reduce_scalar(e2e_t, torch.float64, dist.ReduceOp.MAX, cdev))
        e2e_evals = int(reduce_scalar(e2e_evals, torch.int64, dist.ReduceOp.SUM, cdev))
    e2e_value = e2e_evals / e2e_t

    # digest of every run's best energy and genotype (all ranks' runs, global run order): equal
    # at any rank count (the R split) -- tests/test_gpu_multirank.py compares 1 and 2 ranks
    import hashlib
    if world > 1:
        gE = gathered["E"].cpu().numpy().reshape(world, rmax)
        gG = gathered["G"].cpu().numpy().reshape(world, rmax, d.G)
        cnt = [(k + 1) * total_runs // world - k * total_runs // world for k in range(world)] if not args.weak \
            else [runs] * world
        allE = np.concatenate([gE[k, :cnt[k]] for k in range(world)])
        allG = np.concatenate([gG[k, :cnt[k]] for k in range(world)])
    else:
        allE, allG = bE.cpu().numpy(), bG.cpu().numpy()
    result_digest = hashlib.sha256(allE.astype(np.float32).tobytes() + allG.astype(np.float32).tobytes()).hexdigest()[:16]

    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (gen/synth.py, seeded ligand + pseudo-receptor maps)",
                "config": {"workload": workload_desc(cfg), "runs_per_gpu": runs if args.weak else rmax,
                           "global_runs": total_runs,
                           "l2": "flushed between steps (256 MiB write); grid pinned by an L2 access window",
                           "parallelism": (f"dp{world} (every rank its own {cfg.runs} runs, global run ids)" if args.weak
                                           else f"dp{world} (rank k docks runs [kR/G, (k+1)R/G) of R = {total_runs})")},
                "ligands_per_hour": 3600.0 * (world if args.weak else 1) / (ms_per_step / 1e3),
                "result_digest": result_digest,
                "gpu_launches": launches,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "note": "dock_init (host grid+ligand upload) + dock_run_ex (host outputs) + dock_free, wall clock"},
                "roofline": roofline,
                "clocks": clk,
                "step_ms": {"median": statistics.median(times), "min": min(times), "max": max(times),
                            "spread": (max(times) - min(times)) / statistics.median(times),
                            "note": "this rank's timed steps (the paper reports means of 10 replicas, P:153)"}}
        if world == 1 and not args.no_parts:
            line["roofline_parts"] = parts_roofline(d, cfg, grid, dev)
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(cfg, lig, grid)
        if world == 1 and not args.no_also and args.config == "7cpa":
            line["also"] = other_configs(gpu)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if dt is not d:
        dt.close()
    d.close()


# ---------------------------------------------------------------------------
# configs[4] HTS: ligands/hour through dock_screen, ranks sharded by LPT (sched.py)
# ---------------------------------------------------------------------------
def hts_oracle_sample(cfg, grid, ligs, threads, budget):
    """One run of `budget` evals for each of `threads` ligands, one per thread."""
    import oracle
    pp = oracle.params(ls_method=cfg.ls_method, ls_rate=cfg.ls_rate, ls_max_iters=cfg.ls_iters)
    out = [0] * threads

    def work(i):
        P = oracle.Problem(grid, ligs[i % len(ligs)], sf={} if SCORING else None)
        out[i] = oracle.dock_run(P, pp, cfg.pop, budget, 42, ligand_id=i, run=0)["evals"]
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return sum(out), time.perf_counter() - t0


def run_hts(args, cfg, grid):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2203_02096_b200 as dock
    from paper_2203_02096_b200 import sched
    from gen import hts_ligands

    rank, local, world = env_rank()
    if args.impl == "reference":
        if rank != 0:
            return
    else:
        dev, cdev = dist_setup(local, world)
        local = dev.index
    ligs = hts_ligands(args.n_ligs)
    per_lig_evals = cfg.runs * cfg.max_evals
    sample_desc = (f"configs[4] sample: {args.n_ligs} of the 10k synthetic ligands (N ~ U{{10..70}}, "
                   f"T = clip(N/5 + U{{-1,0,1}}, 0, 15), 8 types), 64^3 receptor, pop {cfg.pop}, {cfg.runs} runs x "
                   f"{cfg.max_evals} evals, ADADELTA ls_rate {cfg.ls_rate}, {cfg.ls_iters} iters"
                   + (", AD4.1-calibrated scoring (NEXT-2)" if SCORING else ""))
    if args.impl == "reference":
        threads = os.cpu_count() or 1
        budget = 20_000
        for _ in range(args.warmup):
            hts_oracle_sample(cfg, grid, ligs, threads, 2_000)
        te, tt = 0, 0.0
        for s in range(args.steps):
            e, t = hts_oracle_sample(cfg, grid, ligs, threads, budget)
            te += e; tt += t
        lph = 3600.0 * (te / tt) / per_lig_evals
        sample = f"{threads} threads, one run of {budget} evals of one ligand each, extrapolated at {per_lig_evals} evals/ligand"
        print(json.dumps({"impl": "reference", "metric": "ligands/hour", "value": lph, "unit": "ligands/h",
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": 1e3 * tt / args.steps, "higher_is_better": True, "scaling": "strong",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic (gen/synth.py, seeded)",
                          "config": {"workload": sample_desc, "sample": sample},
                          "cpu_baseline": {"value": lph, "unit": "ligands/h", "cores": threads, "kind": "oracle",
                                           "sample": sample},
                          "e2e": {"value": lph, "unit": "ligands/h", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                          "gpu_launches": 0}), flush=True)
        return
    tp, roles = grid.type_params()
    n_pairs = [dock.topology(l.types, l.charges, l.xyz, l.bonds, l.rotatable, tp, roles)[2].shape[0] for l in ligs]
    costs = sched.ligand_cost([len(l.types) for l in ligs], n_pairs)
    mine = sched.lpt_partition(costs, world)[rank]
    my_ligs = [ligs[i] for i in mine]
    kw = dict(ls_method=cfg.ls_method, ls_rate=cfg.ls_rate, ls_max_iters=cfg.ls_iters, scoring=SCORING,
              run_branches=args.run_branches)
    for _ in range(args.warmup):   # warm-up on a slice: context, kernels, graphs
        dock.screen(grid, my_ligs[:8], cfg.pop, cfg.runs, cfg.max_evals // 10, 7, ligand_ids=mine[:8],
                    devices=[local], slots_per_device=args.slots, **kw)
    dev = torch.device("cuda", local)
    clocks = ClockSampler(local)
    clocks.start()
    times, launches, evals, prep_ms = [], 0, 0, 0.0
    out = None
    for s in range(args.steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        out = dock.screen(grid, my_ligs, cfg.pop, cfg.runs, cfg.max_evals, 42, ligand_ids=mine,
                          devices=[local], slots_per_device=args.slots, **kw)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        launches += out["stats"]["launches"]
        evals += int(out["evals"].sum())
        prep_ms += out["stats"]["prep_ms"]
    clk = clocks.stop()
    t_local = sum(times)
    t_max = t_local
    tot_evals = evals
    if world > 1:
        t_max = float(reduce_scalar(t_local, torch.float64, dist.ReduceOp.MAX, cdev))
        tot_evals = int(reduce_scalar(evals, torch.int64, dist.ReduceOp.SUM, cdev))
        res = sched.gather_records(mine, out, len(ligs), device=cdev)   # NCCL: final gather only
    else:
        res = out
    lph = 3600.0 * len(ligs) * args.steps / t_max
    line = None
    if rank == 0:
        assert np.all(res["status"] == 0), "a ligand failed"
        h2d = int(np.prod(grid.maps.shape)) * 4 + sum(len(l.types) * 40 + len(l.bonds) * 9 for l in my_ligs)
        line = {"metric": "ligands/hour", "value": lph, "unit": "ligands/h", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (gen/synth.py hts_ligands, seeded)",
                "config": {"workload": sample_desc, "parallelism": f"dp{world} (LPT ligand shards per rank)",
                           "slots_per_gpu": args.slots,
                           "l2": "receptor 32 MiB pinned by an L2 access window; ligands stream through",
                           "timing": "wall clock around the synchronous dock_screen call (host prep + all device "
                                     "work + result copies), max over ranks"},
                "score_evals_per_s": tot_evals / t_max,
                "prep_ms_per_step": prep_ms / args.steps,
                "gpu_launches": launches,
                "e2e": {"value": lph, "unit": "ligands/h", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": len(my_ligs) * 4 * (cfg.runs * (2 + 2 + 38)),
                        "note": "dock_screen is host-to-host: its timed region already includes every copy"},
                "roofline": None,
                "best_E_median": float(np.median(res["best_E"])),
                "clocks": clk}
        if world == 1 and not args.no_cpu:
            threads = os.cpu_count() or 1
            ce, ct = hts_oracle_sample(cfg, grid, ligs, threads, 20_000)
            line["cpu_baseline"] = {"value": 3600.0 * (ce / ct) / per_lig_evals, "unit": "ligands/h", "cores": threads,
                                    "kind": "oracle", "sample": f"{threads} ligands x one run of 20000 evals, "
                                    f"extrapolated at {per_lig_evals} evals/ligand"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# The two isolated parts of an evaluation (SURVEY.md §8(d) "isolating the two kernels for
# ncu"): k_bench_part inter (pose + trilinear E+G) and intra (pose + pair tiles E+forces) on
# the config's population, each against its own roofline: the interpolation against the
# measured L2 gather ceiling (k_l2_gather: random 16-byte __ldg over a resident buffer the
# size of the grid), the pair tiles against the FP32 peak.
# ---------------------------------------------------------------------------
def parts_roofline(d, cfg, grid, dev, reps=3, iters=5):
    import numpy as np
    import torch
    import paper_2203_02096_b200 as dock
    from gen import random_genotypes
    n = cfg.runs * cfg.pop
    X = torch.from_numpy(random_genotypes(grid, d.T, n, seed=5, frac_out=0.0, shrink=0.2)).to(dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    st = torch.cuda.Stream(device=dev)
    res = {}
    for part, name in ((0, "inter"), (1, "intra")):
        with torch.cuda.stream(st):
            d.bench_part(part, X, out, iters, stream=st.cuda_stream)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                d.bench_part(part, X, out, iters, stream=st.cuda_stream)
            e1.record(st)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / reps / 1e3
    grid_mib = max(16, int(np.ceil(grid.maps.nbytes * 4 / 3 / 2 ** 20)))   # the packed float4 grid
    l2_gbs, _ = dock.bench_l2_gather(dev.index, grid_mib, 8, 64)
    peaks = measured_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    lookups = n * iters * d.N
    alg = 96 * lookups / res["inter"] / 1e9
    pairs = n * iters * d.P
    fl = pairs * (F_PAIR_AD4 if SCORING else F_PAIR)[1] / res["intra"] / 1e12
    pk = fp32_peak_tflops(sm_mhz)
    return {"inter": {"kernel": "k_bench_part<kInter> (pose + trilinear E+G; 8 float4 corner __ldg per atom)",
                      "ms": 1e3 * res["inter"], "atom_lookups_per_s": lookups / res["inter"],
                      "algorithmic_GBps_96B": alg, "moved_GBps_128B": 128 * lookups / res["inter"] / 1e9,
                      "l2_gather_ceiling_GBps": l2_gbs, "l2_gather_buffer_MiB": grid_mib,
                      "frac_of_l2_gather": 128 * lookups / res["inter"] / 1e9 / l2_gbs,
                      "hbm_peak_GBps": peaks.get("hbm_gbs"),
                      "note": "fraction = moved bytes (128 B: 8 float4 corners) / the measured random-gather ceiling"},
            "intra": {"kernel": "k_bench_part<kIntra> (pose + pair tiles E+forces)", "ms": 1e3 * res["intra"],
                      "pairs_per_s": pairs / res["intra"], "tflops_8d_model": fl, "fp32_peak_tflops": pk,
                      "frac": fl / pk, "flop_per_pair": (F_PAIR_AD4 if SCORING else F_PAIR)[1]}}


def run_micro(args, cfg, lig, grid):
    import torch
    import paper_2203_02096_b200 as dock
    dev = torch.device("cuda", 0)
    d = dock.Docker.from_inputs(grid, lig, ls_method=0, scoring=SCORING)
    line = {"metric": "microbench", "config": {"workload": workload_desc(cfg), "genotypes": cfg.runs * cfg.pop,
                                               "iters": args.micro_iters}}
    line.update(parts_roofline(d, cfg, grid, dev, reps=args.steps, iters=args.micro_iters))
    print(json.dumps(line), flush=True)
    d.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="7cpa", choices=["tiny", "1stp", "3ce3", "7cpa", "hts", "ps", "pm", "pl"])
    ap.add_argument("--runs", type=int, default=0, help="override runs per GPU (NEXT-1 sweeps)")
    ap.add_argument("--max-evals", type=int, default=0, help="override evals per run (NEXT-1 sweeps)")
    ap.add_argument("--micro", action="store_true", help="isolated inter/intra microbenchmarks (roofline evidence)")
    ap.add_argument("--micro-iters", type=int, default=20)
    ap.add_argument("--sw-depth", type=int, default=0, help="Solis-Wets speculation depth (0 = auto)")
    ap.add_argument("--sw-split", type=int, default=0, help="Solis-Wets warps per evaluation (0 = auto)")
    ap.add_argument("--run-branches", type=int, default=0, help="dock_params.run_branches (0 = auto, 1 lockstep, 2 branches, 3 clusters)")
    ap.add_argument("--n-ligs", type=int, default=256, help="hts: ligands per step (sample of configs[4])")
    ap.add_argument("--slots", type=int, default=4, help="hts: ligands in flight per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-parts", action="store_true", help="skip the inter / intra / L2-gather roofline parts")
    ap.add_argument("--no-also", action="store_true", help="skip the other configs (1stp, 3ce3, HTS sample) of the 7cpa line")
    ap.add_argument("--weak", action="store_true", help="N > 1: every rank docks the config's runs (default: split them)")
    ap.add_argument("--scoring", default="d5", choices=["d5", "ad4"],
                    help="intramolecular scoring: D5 (default) or the NEXT-2 AD4.1-calibrated variant")
    args = ap.parse_args()
    global SCORING
    SCORING = 1 if args.scoring == "ad4" else 0
    from gen import config_inputs
    cfg, lig, grid = config_inputs(args.config)
    if args.runs > 0:
        cfg.runs = args.runs
    if args.max_evals > 0:
        cfg.max_evals = args.max_evals
    if args.micro:
        run_micro(args, cfg, lig, grid)
    elif args.config == "hts":
        run_hts(args, cfg, grid)
    elif args.impl == "reference":
        run_reference(args, cfg, lig, grid)
    else:
        run_ours(args, cfg, lig, grid)


if __name__ == "__main__":
    main()
