#!/usr/bin/env python3
"""Scan seeded planted instances on the GPU to pick BASELINE configs[2]/[3]
workloads with a large search (not a timing source; the bench re-times them).

configs[2]: binary, |IC| in [65, 128] (two-u64 CS);  configs[3]: 4 symbols,
|IC| in [129, 512].  One JSON line per instance: n, c*, candidates, unique, ms.
    python scripts/scan_wide.py c3|c4 [out.jsonl]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import specgen  # noqa: E402
from paper_2305_18575_b200 import Solver  # noqa: E402

C3_TARGETS = ["(0+1)*0(0+1)(0+1)", "(0+1)*11(0+1)*", "1(0+11)*0?", "0(10+1)*(01)?",
              "(00+11)*(01+10)", "(0+10)*1(1+01)*", "((0+1)(0+1))*1", "(01+10)*(0+11)?"]
C3B_TARGETS = ["(0+1)*1(0+1)(0+1)(0+1)", "(0+1)*0(0+1)(0+1)(0+1)(0+1)", "((0+1)(0+1)(0+1))*",
               "(0(0+1)1+1(0+1)0)*", "(0+1)*(00+11)(0+1)*(01+10)", "1(0+1)*0(0+1)*1", "(01*0+1)*0?"]
C4_TARGETS = ["(ab+c)*d(a+b)?", "(a+b)*c(a+d)*", "(a+bc)*(d+ca)", "(ab+cd)*(a+d)?",
              "a(b+c)*d(a+b)*", "(a+b+c)*d(a+c)(b+d)"]
COSTS = [(1, 1, 1, 1, 1), (20, 20, 20, 5, 30)]


def run(sp, max_cost, budget=120 << 30):
    t = time.perf_counter()
    s = Solver.from_spec(sp, device=0, mem_budget_bytes=budget)
    n = s.n_ic
    r = s.solve(max_cost)
    dt = time.perf_counter() - t
    out = {"name": sp.name, "costs": list(sp.costs), "n": n, "W32": r.cs_words, "status": r.status,
           "cstar": r.cost, "cand": r.candidates, "unique": r.unique, "ms": dt * 1e3,
           "regex": r.regex, "levels": [(l.cost, l.unique, l.cand) for l in r.levels if l.complete]}
    s.close()
    return out


def main():
    which = sys.argv[1]
    path = sys.argv[2] if len(sys.argv) > 2 else None
    f = open(path, "a") if path else None
    if which == "c3":
        alpha, targets, lens, nlo, nhi = "01", C3_TARGETS, [(4, 8), (5, 9), (6, 10), (7, 11)], 65, 128
    elif which == "c3b":
        alpha, targets, lens, nlo, nhi = "01", C3B_TARGETS, [(6, 10), (7, 11), (8, 12)], 65, 128
    else:
        alpha, targets, lens, nlo, nhi = "abcd", C4_TARGETS, [(4, 8), (5, 9), (6, 10), (6, 12)], 129, 512
    for tgt in targets:
        for lo, hi in lens:
            for costs in COSTS:
                for seed in range(3):
                    try:
                        sp = specgen.gen_planted(alpha, tgt, 10, 10, lo, hi, seed, costs=costs,
                                                 max_attempts=200000)
                    except Exception as e:  # noqa: BLE001
                        print(json.dumps({"target": tgt, "lo": lo, "hi": hi, "seed": seed, "err": str(e)}))
                        continue
                    try:
                        s = Solver.from_spec(sp, device=0)
                        n = s.n_ic
                        s.close()
                    except Exception as e:  # noqa: BLE001
                        print(json.dumps({"name": sp.name, "err": str(e)}))
                        continue
                    if not (nlo <= n <= nhi):
                        continue
                    mc = 40 if costs[0] == 1 else 800
                    try:
                        out = run(sp, mc)
                    except Exception as e:  # noqa: BLE001
                        out = {"name": sp.name, "n": n, "err": str(e)}
                    out.update({"target": tgt, "lo": lo, "hi": hi, "seed": seed})
                    line = json.dumps(out)
                    print(line, flush=True)
                    if f:
                        f.write(line + "\n")
                        f.flush()


if __name__ == "__main__":
    main()
