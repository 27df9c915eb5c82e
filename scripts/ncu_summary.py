"""Summarise ncu evidence for profiles/: per-kernel launch shares from a
`--metrics gpu__time_duration.sum` launch list, and the key counters of a
`--set full` capture (read with `ncu -i <rep> --page raw --csv`).

  python scripts/ncu_summary.py launches <launches.csv>
  python scripts/ncu_summary.py full <report.ncu-rep>
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"), ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "SM instr throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "thread FFMA"),
    ("derived__smsp__sass_thread_inst_executed_op_ffma_pred_on_x2", "thread FFMA x2 (flops)"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "thread FADD"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "thread FMUL"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__t_sectors.sum", "L2 sectors"),
    ("lts__t_sectors.sum.pct_of_peak_sustained_elapsed", "L2 sector throughput % of peak"),
    ("lts__t_bytes.sum.per_second", "L2 bytes/s"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("dram__bytes_read.sum", "DRAM read bytes"),
    ("dram__bytes_write.sum", "DRAM write bytes"),
    ("dram__bytes_read.sum.per_second", "DRAM read B/s"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected"),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio", "stall branch_resolving"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = None
    for r in rows[1:]:
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        unit = r[iu]
        k = r[ik].split("(")[0].replace("void ", "").split("<")[0]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"| kernel | launches | total ({unit}) | mean ({unit}) | share |\n|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {t:.0f} | {t / n:.0f} | {100 * t / tot:.1f}% |")


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")]
        print(f"kernel: {name}")
        for key, label in KEYS:
            if key in h:
                i = h.index(key)
                print(f"  {label:28s} {v[i]} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
