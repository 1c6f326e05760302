#!/usr/bin/env python3
"""A/B of environment variants over FRESH contexts (experiments only; not a bench number).

Every repetition creates a new context (rei_init), solves and destroys it -- the e2e
path bench.py times -- and records the device time of the solve and of its deepest
levels.  Variants run in separate processes, interleaved.

    AB_ENVS="tag:K=V,K2=V2;tag2:K=V" python scripts/ab_fresh.py [workload] [reps] [rounds]
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import bench
from paper_2305_18575_b200 import Solver
spec, mc, _ = bench.WORKLOADS[%r]
out = []
for i in range(%d + 1):
    s = Solver.from_spec(spec, device=0)
    r = s.solve(mc)
    s.close()
    if i:
        out.append({"ms": r.seconds * 1000, "lv": {l.cost: round(l.ms, 3) for l in r.levels[-4:]}})
print(json.dumps(out))
"""


def main():
    workload = sys.argv[1] if len(sys.argv) > 1 else "table1-row1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    envs = [("base", {})]
    for item in [x for x in os.environ.get("AB_ENVS", "").split(";") if x]:
        tag, kvs = item.split(":", 1)
        envs.append((tag, dict(kv.split("=", 1) for kv in kvs.split(",") if kv)))
    res = {t: [] for t, _ in envs}
    for _ in range(rounds):
        for tag, extra in envs:
            env = dict(os.environ, **extra)
            p = subprocess.run([sys.executable, "-c", CHILD % (ROOT, workload, reps)], env=env,
                               capture_output=True, text=True, timeout=900)
            if p.returncode:
                print(tag, "FAILED", p.stderr[-600:], flush=True)
                continue
            res[tag] += json.loads(p.stdout.strip().splitlines()[-1])
    for tag, runs in res.items():
        if not runs:
            continue
        ms = sorted(r["ms"] for r in runs)
        print(f"{tag:14s} median {statistics.median(ms):7.2f} ms  min {ms[0]:7.2f}  max {ms[-1]:7.2f}  "
              f"all {[round(x, 1) for x in ms]}")
        levels = sorted({c for r in runs for c in r["lv"]})
        for c in levels:
            v = sorted(r["lv"][str(c)] if str(c) in r["lv"] else r["lv"].get(c) for r in runs
                       if str(c) in r["lv"] or c in r["lv"])
            print(f"{'':14s}   level {c}: {[round(x, 1) for x in v]}")


if __name__ == "__main__":
    main()
