#!/usr/bin/env python3
"""Summarise an ncu capture + launch list into profiles/ (tracked, per round).

    python scripts/summarize_profile.py <tag> <round> [--traffic-key concat]

Reads gpurun_out/prof_<tag>.ncu-rep (ncu --set full of one launch) and
gpurun_out/launches_<tag>.csv (gpu__time_duration of every launch of one solve)
and writes profiles/<round>_<tag>.md and .json.
"""
import csv
import json
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    # why warps wait (cycles per issued instruction)
    "smsp__average_warp_latency_per_inst_issued.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for n, u, v in zip(h, units, vals):
        d[n] = (v, u)
    return d


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    out = []
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        m = re.search(r"(k_\w+|cub::\w+)", d["Kernel Name"])
        out.append((m.group(1) if m else d["Kernel Name"][:40], float(d["Metric Value"].replace(",", "")) / 1e6))
    return out


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    rep = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    lpath = os.path.join(OUT, f"launches_{tag}.csv")
    os.makedirs(PROF, exist_ok=True)
    res = {"tag": tag, "round": rnd}
    lines = [f"# ncu summary `{tag}` (round {rnd})", ""]
    if os.path.exists(lpath):
        L = launches(lpath)
        tot = sum(ms for _, ms in L)
        by = Counter()
        cnt = Counter()
        for n, ms in L:
            by[n] += ms
            cnt[n] += 1
        res["launch_list"] = {"launches": len(L), "total_ms": tot,
                              "by_kernel": {k: {"launches": cnt[k], "ms": v, "share": v / tot} for k, v in by.items()}}
        lines += ["## Launch list (ncu gpu__time_duration, cold-cache, serialised: compare shares)", "",
                  f"{len(L)} launches, {tot:.2f} ms total", "", "| kernel | launches | ms | share |", "|---|---|---|---|"]
        for k, v in by.most_common():
            lines.append(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / tot:.1f}% |")
        lines.append("")
    if os.path.exists(rep):
        d = raw_metrics(rep)
        sel = {m: d[m][0] for m in METRICS if m in d}
        res["top_launch_metrics"] = sel
        kname = d.get("Kernel Name", ("?",))[0] if "Kernel Name" in d else "?"
        res["kernel"] = kname
        lines += ["## Longest launch, `ncu --set full`", "", f"kernel: `{kname}`", "", "| metric | value |", "|---|---|"]
        for m in METRICS:
            if m in d:
                lines.append(f"| {m} | {d[m][0]} {d[m][1]} |")
        try:
            b = float(sel.get("dram__bytes_read.sum", "0").replace(",", "")) + \
                float(sel.get("dram__bytes_write.sum", "0").replace(",", ""))
            res["dram_bytes_per_launch_MB"] = b
        except ValueError:
            pass
        lines.append("")
    json.dump(res, open(os.path.join(PROF, f"{rnd}_{tag}.json"), "w"), indent=1)
    open(os.path.join(PROF, f"{rnd}_{tag}.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
