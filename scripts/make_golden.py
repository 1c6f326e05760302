#!/usr/bin/env python3
"""Write oracle golden files under tests/golden/ (calls only oracle/).

Every value written here comes from ``oracle/`` on specs from ``specgen``;
nothing comes from the CUDA path.  Usage:

    python scripts/make_golden.py table1_row1 [--max-cost 28]
    python scripts/make_golden.py table1_row8
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import specgen  # noqa: E402

SPECS = {
    "table1_row1": (specgen.TABLE1_ROW1, 28),
    "table1_row8": (specgen.TABLE1_ROW8, 208),
    "c1_toy": (specgen.C1_TOY, 20),
    "e1": (specgen.E1, 20),
    "intro": (specgen.INTRO, 20),
    # BASELINE configs[1]: Type 1, binary, le = 6, p = n = 10, seed 0
    "c2_t1_s0": (specgen.gen_type1("01", 6, 10, 10, 0), 40),
    # BASELINE configs[2]: binary, |IC| = 115 (two-u64 CS), planted target, unit and the
    # non-uniform cost function (20,20,20,5,30) (the paper's AlphaRegex-style costs)
    "c3_planted_s1": (specgen.gen_planted("01", "(0+1)*1(0+1)(0+1)(0+1)", 10, 10, 6, 10, 1), 40),
    "c3_planted_s1_nu": (specgen.gen_planted("01", "(0+1)*1(0+1)(0+1)(0+1)", 10, 10, 6, 10, 1,
                                             costs=(20, 20, 20, 5, 30)), 800),
    # BASELINE configs[3]: 4 symbols, planted target (DESIGN.md input recipe), |IC| = 148
    "c4_planted_s0": (specgen.gen_planted("abcd", "(a+b+c)*d(a+c)(b+d)", 10, 10, 4, 8, 0), 40),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name", choices=sorted(SPECS))
    ap.add_argument("--max-cost", type=int, default=None)
    ap.add_argument("--stop-at-first", action="store_true",
                    help="stop at the first precise candidate (do not finish level c*)")
    args = ap.parse_args()
    spec, mc = SPECS[args.name]
    mc = args.max_cost or mc
    t0 = time.time()
    o = oracle.Oracle.from_spec(spec)
    r = o.solve(mc, complete_final_level=not args.stop_at_first)
    out = {
        "spec": {"alphabet": spec.alphabet, "P": list(spec.P), "N": list(spec.N),
                 "costs": list(spec.costs), "name": spec.name},
        "generator": "scripts/make_golden.py (oracle/ only)",
        "oracle_host": platform.processor() or platform.machine(),
        "wall_seconds": time.time() - t0,
        "n_ic": o.n,
        "status": r.status,
        "cstar": r.cost,
        "regex": r.regex,
        "candidates_through_found": r.candidates,
        "complete_final_level": not args.stop_at_first,
        "levels": [
            {"cost": l.cost, "unique": l.unique, "cand_q": l.cand_q, "cand_s": l.cand_s,
             "cand_c": l.cand_c, "cand_u": l.cand_u, "complete": l.complete}
            for l in r.levels
        ],
    }
    path = os.path.join(ROOT, "tests", "golden", f"{args.name}_oracle.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, r.status, r.cost, r.regex, f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
