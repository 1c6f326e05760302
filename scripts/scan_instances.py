#!/usr/bin/env python3
"""Scan seeded synthetic instances on the GPU (n, c*, candidates, time) to pick
bench / test workloads for BASELINE configs[1..3].  Not a timing source."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import specgen  # noqa: E402
from paper_2305_18575_b200 import Solver  # noqa: E402


def run(sp, max_cost=60, budget=100 << 30):
    try:
        s = Solver.from_spec(sp, device=0, mem_budget_bytes=budget)
    except Exception as e:  # noqa: BLE001
        return f"init error {e}"
    t = time.perf_counter()
    r = s.solve(max_cost)
    dt = time.perf_counter() - t
    out = (f"n={r.n_ic:3d} W={r.cs_words} {r.status:13s} c*={r.cost:3d} cand={r.candidates:.3e} "
           f"uniq={r.unique:.3e} {dt * 1000:9.1f} ms {r.candidates / max(dt, 1e-9) / 1e9:7.1f} Gc/s {r.regex}")
    s.close()
    return out


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c2"
    if which == "c2":
        for seed in range(12):
            sp = specgen.gen_type1("01", 6, 10, 10, seed)
            print("T1 le6 p10 s", seed, run(sp, 40), flush=True)
        for seed in range(6):
            sp = specgen.gen_type2("01", 6, 10, 10, seed)
            print("T2 le6 p10 s", seed, run(sp, 40), flush=True)
    elif which == "c3":
        for tgt, lo, hi in [("1(0+11)*0?", 6, 12), ("(0+1)*11(0+1)*", 6, 12), ("(01+1)*0", 6, 12),
                            ("0(10+1)*(01)?", 8, 14), ("(0+1)*0(0+1)(0+1)", 6, 12)]:
            for seed in range(3):
                try:
                    sp = specgen.gen_planted("01", tgt, 10, 10, lo, hi, seed)
                except Exception as e:  # noqa: BLE001
                    print(tgt, seed, e)
                    continue
                print(tgt, seed, run(sp, 30), flush=True)
    elif which == "c4":
        for tgt, lo, hi in [("(ab+c)*d(a+b)?", 6, 14), ("(a+b)*c(a+d)*", 6, 14), ("a(b+c)*d", 8, 16),
                            ("(ab)*(cd)*", 8, 16), ("(a+bc)*(d+ca)", 6, 14)]:
            for seed in range(2):
                try:
                    sp = specgen.gen_planted("abcd", tgt, 10, 10, lo, hi, seed)
                except Exception as e:  # noqa: BLE001
                    print(tgt, seed, e)
                    continue
                print(tgt, seed, run(sp, 30), flush=True)
    elif which == "row8":
        print("table1-row8", run(specgen.TABLE1_ROW8, 400), flush=True)


if __name__ == "__main__":
    main()
