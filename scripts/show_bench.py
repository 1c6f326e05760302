#!/usr/bin/env python3
"""Print the key fields of bench.py JSON lines (log files given as arguments)."""
import json
import sys


def show(d, ind=""):
    print(ind, "value %.4g" % d["value"], "ms/step %.3f" % d["ms_per_step"])
    r = d.get("roofline") or {}
    print(ind, "roof", {k: r.get(k) for k in ["kernel", "bound", "achieved", "peak", "frac", "frac_issue",
                                              "frac_of_copy_bw", "frac_timed_region", "share_of_step",
                                              "candidates_per_s", "avg_launch_ms", "traffic"]})
    e = d.get("e2e") or {}
    print(ind, "e2e", {k: e.get(k) for k in ["value", "time_to_minimal_re_ms", "solve_ms_median"]})
    print(ind, "cfg", {k: d["config"].get(k) for k in ["workload", "cstar", "time_to_minimal_re_ms",
                                                        "candidates_per_step"]})
    print(ind, "complete", d.get("complete_levels"))


for path in sys.argv[1:]:
    print("==", path)
    lines = [l for l in open(path) if l.startswith("{")]
    if not lines:
        print(open(path).read()[-1500:])
        continue
    d = json.loads(lines[-1])
    show(d)
    if d.get("secondary"):
        show(d["secondary"], "   SEC")
    print(" clocks", d.get("clocks"), "launches", d.get("gpu_launches"))
    print(" cpu", d.get("cpu_baseline"))
