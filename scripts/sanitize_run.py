#!/usr/bin/env python3
"""Small solves that exercise every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), SURVEY 4b.6:

    compute-sanitizer --tool memcheck --error-exitcode 1 python scripts/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import specgen  # noqa: E402
from paper_2305_18575_b200 import Solver, solve_batch, solve_group, solve_packed  # noqa: E402

CASES = [
    (specgen.C1_TOY, 12, {}),                                       # bitmap, fast kernels
    (specgen.E1, 12, {"complete_final_level": True}),
    (specgen.gen_type2("01", 7, 6, 6, 0), 14, {}),                  # 64-bit-key hash set
    (specgen.gen_planted("01", "1(0+11)*0?", 8, 8, 6, 12, 0), 9, {}),   # indexed hash, W32=4
    (specgen.Spec("01", ("0" * 20, "1"), ("0" * 19, "11")), 10, {}),    # generic kernels
    (specgen.TABLE1_ROW1, 30, {"error": (20, 100)}),                # allowed error
    (specgen.TABLE1_ROW1, 15, {}),                                  # level sort (levels >= 2^14)
    (specgen.C1_TOY.with_costs((1, 3, 3, 1, 3)), 40, {"max_entries": 160}),  # OnTheFly
]


def main():
    for sp, mc, kw in CASES:
        r = Solver.from_spec(sp, device=0, **kw).solve(mc)
        print(sp.name or sp.alphabet, r.status, r.cost, r.regex)
    g = solve_group([Solver.from_spec(specgen.C1_TOY, device=0) for _ in range(2)], 12)
    print("group", g.status, g.cost)
    rs = solve_batch([Solver.from_spec(specgen.gen_type1("01", 4, 5, 5, s), device=0) for s in range(4)], 20, 4)
    print("batch", [r.cost for r in rs])
    specs = specgen.suite_f4(12)
    rp, _ = solve_packed([Solver.from_spec(sp, device=0, small_cache=True) for sp in specs], 60)
    print("packed", [r.cost for r in rp])


if __name__ == "__main__":
    main()
