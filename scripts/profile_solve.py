#!/usr/bin/env python3
"""One rei_solve of a bench workload (for ncu capture; not a timing source).

    ncu ... python scripts/profile_solve.py [workload] [--complete]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2305_18575_b200 import Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "table1-row1"
spec, max_cost, _ = bench.WORKLOADS[name]
s = Solver.from_spec(spec, device=0, complete_final_level="--complete" in sys.argv)
s.reset_kernel_stats()  # per-kernel CUDA events on (include/rei.h rei_kernel_stats)
r = s.solve(max_cost)
print(r.status, r.cost, r.regex, r.candidates, f"{r.seconds * 1000:.2f} ms")
for l in r.levels:
    print(f"  level {l.cost:3d} unique {l.unique:10d} cand {l.cand:14d} eval {l.evaluated:14d} {l.ms:8.3f} ms")
print(s.kernel_stats())
