#!/usr/bin/env python3
"""Host-side phase timings of rei_init / rei_solve (REI_TRACE=1), repeated contexts.

    REI_TRACE=1 python scripts/trace_e2e.py [workload] [repeats]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2305_18575_b200 import Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "table1-row1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec, max_cost, _ = bench.WORKLOADS[name]
for i in range(reps):
    t0 = time.perf_counter()
    s = Solver.from_spec(spec, device=0)
    t1 = time.perf_counter()
    r = s.solve(max_cost)
    t2 = time.perf_counter()
    s.close()
    t3 = time.perf_counter()
    print(f"rep {i}: init {1e3 * (t1 - t0):.2f} ms solve {1e3 * (t2 - t1):.2f} ms "
          f"(device {r.seconds * 1e3:.2f}) close {1e3 * (t3 - t2):.2f} ms  {r.status} {r.cost}", flush=True)
