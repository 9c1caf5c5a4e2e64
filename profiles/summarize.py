"""Turn ncu outputs (brought back from the GPU box into gpurun_out/) into the
committed summaries under profiles/.

    python profiles/summarize.py launches <launches.csv> <steps> <out.txt>
    python profiles/summarize.py full <report.ncu-rep> <out_prefix> [config]

`launches` aggregates an `ncu --metrics gpu__time_duration.sum
--clock-control none --csv` launch list per kernel (ms per step, share,
launches per step).  `full` extracts the headline sections, the stall
reasons and the raw metrics the DESIGN.md roofline cites from an
`ncu --set full` capture (one kernel)."""

import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, steps, out):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg, tot = collections.OrderedDict(), 0.0
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        name = r[ki].split("(")[0][:80]
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    lines = [f"# {path}: {steps} render steps, gpu__time_duration.sum per kernel "
             "(ncu --clock-control none; cold-cache, serialised launches)",
             f"{'ms/step':>10s} {'share':>6s} {'launch/step':>11s}  kernel"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v / 1e6 / steps:10.3f} {100 * v / tot:5.1f}% {n / steps:11.1f}  {k}")
    lines.append(f"total kernel time per step: {tot / 1e6 / steps:.3f} ms")
    open(out, "w").write("\n".join(lines) + "\n")


def _ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def full(rep, prefix, config=""):
    want = ["Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread",
            "Achieved Occupancy", "Theoretical Occupancy", "Executed Ipc Active",
            "Issue Slots Busy", "Eligible Warps Per Scheduler", "No Eligible",
            "L1/TEX Hit Rate", "L2 Hit Rate", "L1/TEX Cache Throughput", "L2 Cache Throughput",
            "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
            "Warp Cycles Per Issued Instruction", "Executed Instructions",
            "Avg. Active Threads Per Warp"]
    rows = list(csv.reader(io.StringIO(_ncu(rep, "--page", "details", "--csv"))))
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    seen, lines = set(), [f"# ncu --set full --clock-control none: {rep} {config}"]
    for r in rows[1:]:
        if len(r) <= vi or r[mi] not in want:
            continue
        k = r[ki].split("(")[0][-40:]
        if (k, r[mi]) in seen:
            continue
        seen.add((k, r[mi]))
        lines.append(f"{k:42s} {r[mi]:38s} {r[vi]:>16s} {r[ui]}")
    raw = list(csv.reader(io.StringIO(_ncu(rep, "--page", "raw", "--csv"))))
    rh, rv = raw[0], raw[2]
    d = {rh[i]: rv[i] for i in range(len(rh))}
    stalls = sorted(((float(d[k].replace(",", "") or 0), k) for k in rh
                     if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
                     and d[k] not in ("", "n/a")), reverse=True)
    tot = sum(v for v, _ in stalls) or 1.0
    lines.append("# warp stall samples (share of all samples)")
    lines += [f"  {100 * v / tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}"
              for v, k in stalls[:10]]
    keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "sm__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
            "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
            "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
            "smsp__inst_executed_op_ldgsts.sum", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    unit_row = raw[1]
    sel = {k: f"{d[k]} {unit_row[rh.index(k)]}".strip() for k in keys if k in d}
    json.dump({"report": rep, "config": config, "kernel": d.get("Kernel Name", ""),
               "metrics": sel}, open(prefix + "_raw.json", "w"), indent=1)
    open(prefix + "_summary.txt", "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], float(sys.argv[3]), sys.argv[4])
    else:
        full(sys.argv[2], sys.argv[3], " ".join(sys.argv[4:]))
