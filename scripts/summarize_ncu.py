"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python scripts/summarize_ncu.py <tag> [launches.csv] [report.ncu-rep ...]

Writes profiles/<tag>/: launches.csv (copy), launches_summary.txt (per-kernel
device time and share of the step), <report>_summary.txt (key metrics of each
captured kernel) and stall/opcode breakdown of the fused GEMM.
"""

import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
]


def ncu_csv(args):
    r = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def summarize_report(rep, out):
    rows = ncu_csv(["-i", rep, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        lines.append(f"== {d.get('Kernel Name', '?')[:100]}")
        for k in KEYS:
            if k in hdr:
                lines.append(f"  {k} = {d[k]} {units[hdr.index(k)]}")
        stalls = []
        for k, u, v in zip(hdr, units, r):
            if k.startswith("smsp__average_warps_issue_stalled_") and \
                    k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):
                                                 -len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        lines.append("  top stall reasons (warps per issue): " + ", ".join(
            f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:6]))
    # opcode breakdown of sampled stalls (source page)
    src = ncu_csv(["-i", rep, "--page", "source", "--print-source", "sass"])
    if len(src) > 2:
        h = src[1]
        agg = defaultdict(float)
        tot = 0.0
        for r in src[2:]:
            if len(r) != len(h):
                continue
            d = dict(zip(h, r))
            try:
                s = float(d.get("Warp Stall Sampling (All Samples)") or 0)
            except ValueError:
                continue
            toks = d["Source"].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            agg[op.split(".")[0]] += s
            tot += s
        if tot:
            lines.append("  stall samples by opcode: " + ", ".join(
                f"{k}={100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    return rows


def summarize_launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0]
            per[name].append(float(d["Metric Value"]))
    # two steps share the launch list: the north star's FP64 cascade (casc::) and
    # the NEXT-3 INT8 cascade (i8::); shares are within each step
    def step_of(k):
        base = k.replace("void ", "")
        if "i8::" in base or base.startswith("i8_"):
            return "int8"
        if "casc::" in base or base.startswith("casc_") or base.startswith("split_"):
            return "fp64"
        return None
    steps = defaultdict(float)
    for k, v in per.items():
        if step_of(k):
            steps[step_of(k)] += sum(v) / len(v)
    lines = ["kernel | launches | mean ms | step | share of its step (our kernels)"]
    for k, v in sorted(per.items(), key=lambda x: -sum(x[1])):
        mean = sum(v) / len(v) / 1e6
        st = step_of(k)
        share = (sum(v) / len(v)) / steps[st] if st else None
        lines.append(f"{k} | {len(v)} | {mean:.3f} | {st or ''} | "
                     f"{'' if share is None else f'{100 * share:.2f}%'}")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


def main():
    tag = sys.argv[1]
    outdir = os.path.join(ROOT, "profiles", tag)
    os.makedirs(outdir, exist_ok=True)
    for a in sys.argv[2:]:
        base = os.path.basename(a)
        if a.endswith(".csv"):
            shutil.copy(a, os.path.join(outdir, base))
            summarize_launches(a, os.path.join(outdir, base.replace(".csv", "_summary.txt")))
        elif a.endswith(".ncu-rep"):
            summarize_report(a, os.path.join(outdir, base.replace(".ncu-rep", "_summary.txt")))


if __name__ == "__main__":
    main()
