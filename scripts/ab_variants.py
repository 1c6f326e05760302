#!/usr/bin/env python3
"""A/B timing of compile-time kernel variants on one GPU (experiments only).

    python scripts/ab_variants.py build name:DEF1,DEF2 ...   # here (nvcc, no GPU)
    python scripts/ab_variants.py run [workload] [reps]      # under gpurun

`run` times every librei_b200*.so found in the package (the default build is
"base") with REI_LIB, in fresh processes, interleaved, and prints the median
solve time and per-kernel-class device ms.  Not a bench.py number.
"""
import glob
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2305_18575_b200")
sys.path.insert(0, ROOT)

CHILD = r"""
import json, sys, time
sys.path.insert(0, %r)
import bench
from paper_2305_18575_b200 import Solver
spec, mc, _ = bench.WORKLOADS[%r]
s = Solver.from_spec(spec, device=0, complete_final_level=%r)
s.solve(mc)
out = []
for _ in range(%d):
    s.reset_kernel_stats()
    r = s.solve(mc)
    out.append({"ms": r.seconds * 1000, "k": s.kernel_stats(), "cand": r.candidates})
print(json.dumps(out))
"""


def main():
    if sys.argv[1] == "build":
        from paper_2305_18575_b200 import build
        for arg in sys.argv[2:]:
            name, defs = arg.split(":")
            print(build.build_variant(name, [d for d in defs.split(",") if d]))
        return
    workload = sys.argv[2] if len(sys.argv) > 2 else "table1-row1"
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    libs = {"base": os.path.join(PKG, "librei_b200.so")}
    for f in sorted(glob.glob(os.path.join(PKG, "librei_b200_*.so"))):
        libs[os.path.basename(f)[len("librei_b200_"):-3]] = f
    modes = [m for m in os.environ.get("AB_CONC", "").split(",") if m]  # REI_CONCURRENT modes
    # AB_ENVS="tag:K=V,K2=V2;tag2:K=V": extra environment variants of every library
    envs = [("", {})]
    for item in [x for x in os.environ.get("AB_ENVS", "").split(";") if x]:
        tag, kvs = item.split(":", 1)
        envs.append((tag, dict(kv.split("=", 1) for kv in kvs.split(","))))
    runs_of = {}
    for name, path in libs.items():
        for m in modes or [None]:
            for tag, extra in envs:
                key = (name if m is None else f"{name}/c{m}") + (f"/{tag}" if tag else "")
                runs_of[key] = (path, m, extra)
    res = {k: [] for k in runs_of}
    for rnd in range(2):
        for name, (path, m, extra) in runs_of.items():
            env = dict(os.environ, REI_LIB=path, **extra)
            if m is not None:
                env["REI_CONCURRENT"] = m
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, workload, os.environ.get("AB_COMPLETE") == "1", reps)], env=env,
                                 capture_output=True, text=True, timeout=600)
            if out.returncode != 0:
                print(name, "FAILED", out.stderr[-400:])
                continue
            res[name] += json.loads(out.stdout.strip().splitlines()[-1])
    for name, runs in res.items():
        if not runs:
            continue
        ms = statistics.median(r["ms"] for r in runs)
        kc = {k: statistics.median(r["k"][k][1] for r in runs) for k in ("concat", "union", "unary")}
        print(f"{name:16s} solve {ms:8.2f} ms  concat {kc['concat']:7.2f}  union {kc['union']:7.2f}  "
              f"unary {kc['unary']:6.2f}  ({len(runs)} runs)")


if __name__ == "__main__":
    main()
