#!/usr/bin/env python
"""Turn gpurun_out/ ncu artefacts into the small, committed summaries under profiles/.

  python tools/summarize_profiles.py --tag r01_C2 [--launches gpurun_out/launches.csv]
                                     [--rep gpurun_out/prof.ncu-rep]

Writes profiles/<tag>_launches.md (per-kernel share of the step, from the
`ncu --metrics gpu__time_duration.sum --clock-control none` launch list) and
profiles/<tag>_<kernel>.json (the key counters of one `ncu --set full` capture).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio")


def launches(path, tag):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[r[ki][:90]][0] += 1
        agg[r[ki][:90]][1] += v
        tot += v
    out = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
           "Cold-cache, serialised per-launch times: read the SHARE column, not the absolutes.", "",
           "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {c} | {v / 1e6:.3f} | {100 * v / tot:.1f}% |")
    out.append(f"| **all** | {sum(c for c, _ in agg.values())} | {tot / 1e6:.3f} | 100% |")
    dst = os.path.join(ROOT, "profiles", f"{tag}_launches.md")
    open(dst, "w").write("\n".join(out) + "\n")
    print("wrote", dst)


def full(path, tag):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        rec = {"kernel": name, "source": os.path.basename(path)}
        for k in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                try:
                    rec[k] = [float(d[k].replace(",", "")), u.get(k, "")]
                except ValueError:
                    rec[k] = [d[k], u.get(k, "")]
        short = name.split("(")[0].replace("void ", "").replace("kj::", "").replace(" ", "")
        short = "".join(ch if ch.isalnum() else "_" for ch in short).strip("_")
        dst = os.path.join(ROOT, "profiles", f"{tag}_{short}.json")
        json.dump(rec, open(dst, "w"), indent=1)
        print("wrote", dst)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches.csv"))
    ap.add_argument("--rep", default=os.path.join(ROOT, "gpurun_out", "prof.ncu-rep"))
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.launches and os.path.exists(a.launches):
        launches(a.launches, a.tag)
    if a.rep and os.path.exists(a.rep):
        full(a.rep, a.tag)


if __name__ == "__main__":
    main()
