#!/usr/bin/env python3
"""Solve a few large planted configs[2]/[3] candidates once each (selection only; the
bench re-times the chosen ones).  python scripts/try_big.py [out.jsonl]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import specgen  # noqa: E402
from scan_wide import run  # noqa: E402

NU = (20, 20, 20, 5, 30)
CANDS = [
    ("01", "(0+1)*0(0+1)(0+1)(0+1)(0+1)", 6, 10, 0, NU, 800),
    ("01", "(0+1)*0(0+1)(0+1)(0+1)(0+1)", 6, 10, 2, NU, 800),
    ("01", "(0+1)*0(0+1)(0+1)(0+1)(0+1)", 6, 10, 1, (1, 1, 1, 1, 1), 40),
    ("01", "(0+1)*1(0+1)(0+1)(0+1)(0+1)", 6, 10, 0, (1, 1, 1, 1, 1), 40),
    ("abcd", "(a+b+c)*d(a+c)(b+d)", 6, 10, 1, NU, 800),
]
out = open(sys.argv[1], "a") if len(sys.argv) > 1 else None
for alpha, tgt, lo, hi, seed, costs, mc in CANDS:
    try:
        sp = specgen.gen_planted(alpha, tgt, 10, 10, lo, hi, seed, costs=costs, max_attempts=200000)
        r = run(sp, mc, budget=150 << 30)
    except Exception as e:  # noqa: BLE001
        r = {"target": tgt, "seed": seed, "costs": list(costs), "err": str(e)}
    r.pop("levels", None)
    line = json.dumps(r)
    print(line, flush=True)
    if out:
        out.write(line + "\n")
        out.flush()
