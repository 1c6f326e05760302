#!/usr/bin/env python3
"""A/B of a level's launch order (concat first vs REI_UNION_FIRST), interleaved per rep.

    python scripts/ab_launch_order.py [workload] [repeats]

Prints, per variant, the solve-time distribution (ms) and candidates/s over all
reps (total candidates / total time), with Python GC off.  The early exit at c*
depends on which kernel meets the precise CS first, so the spread matters as
much as the median.
"""
import gc
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2305_18575_b200 import Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "table1-row1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
spec, max_cost, _ = bench.WORKLOADS[name]
gc.disable()
res = {"concat_first": [], "union_first": []}
for i in range(reps + 1):
    for var in res:
        os.environ["REI_UNION_FIRST"] = "1" if var == "union_first" else "0"
        s = Solver.from_spec(spec, device=0)
        t0 = time.perf_counter()
        r = s.solve(max_cost)
        t1 = time.perf_counter()
        s.close()
        if i:
            res[var].append((1e3 * (t1 - t0), r.candidates, r.cost))
for var, xs in res.items():
    ms = sorted(x[0] for x in xs)
    tot = sum(x[1] for x in xs) / (sum(x[0] for x in xs) / 1e3)
    print(f"{name} {var}: median {statistics.median(ms):.2f} ms  min {ms[0]:.2f}  "
          f"p90 {ms[int(0.9 * (len(ms) - 1))]:.2f}  max {ms[-1]:.2f}  "
          f"{tot / 1e9:.1f} G cand/s  cost {set(x[2] for x in xs)}", flush=True)
