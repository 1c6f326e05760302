#!/usr/bin/env python3
"""The f4 suite (specgen.suite_f4): many small specifications on one GPU.

    python scripts/suite_run.py [count] [chunk] [max_cost] [--modes packed,single,batch]

For each mode, every spec is solved once (contexts created per chunk with the
small-cache flag, rei_init outside the timed solve); prints specs/s, candidates/s and
per-spec time percentiles, and checks that the modes agree on status and c*.
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import specgen  # noqa: E402


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(q * len(xs)))] if xs else None


def run(mode, specs, chunk, max_cost):
    from paper_2305_18575_b200 import Solver, solve_batch, solve_packed
    res, per = [], []
    total = 0.0
    for i in range(0, len(specs), chunk):
        part = specs[i:i + chunk]
        solvers = [Solver.from_spec(sp, device=0, small_cache=True) for sp in part]
        t0 = time.perf_counter()
        if mode == "packed":
            rs, done = solve_packed(solvers, max_cost)
        elif mode == "batch":
            rs = solve_batch(solvers, max_cost, threads=8)
            done = [r.seconds for r in rs]
        else:  # one spec after another: each spec's own solve time
            rs, done = [], []
            for s in solvers:
                t1 = time.perf_counter()
                rs.append(s.solve(max_cost))
                done.append(time.perf_counter() - t1)
        total += time.perf_counter() - t0
        res += rs
        per += done
        for s in solvers:
            s.close()
    return res, per, total


def summary(mode, res, per, total):
    cand = sum(r.candidates for r in res)
    return {"specs": len(res), "seconds": total, "specs_per_s": len(res) / total,
            "cand_per_s": cand / total, "candidates": cand,
            "found": sum(r.status == "found" for r in res),
            "not_found": sum(r.status == "not_found" for r in res),
            "oom": sum(r.status == "out_of_memory" for r in res),
            # packed: completion time of each spec from its chunk's start; single: own solve time
            "time_s_p50": pct(per, 0.5), "time_s_p90": pct(per, 0.9), "time_s_max": max(per),
            "frac_under_10ms": sum(t < 0.01 for t in per) / len(per),
            "frac_under_100ms": sum(t < 0.1 for t in per) / len(per),
            "frac_under_1s": sum(t < 1.0 for t in per) / len(per)}


def main():
    """Whole suite in each mode; then the small specs (found with < 1e8 candidates in
    the first mode) again, packed vs one after another: the latency-bound workload f4
    is about (most of the paper's suite finishes in under a second)."""
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    count = int(args[0]) if args else 1024
    chunk = int(args[1]) if len(args) > 1 else 128
    max_cost = int(args[2]) if len(args) > 2 else 40
    modes = "single,packed"
    for a in sys.argv[1:]:
        if a.startswith("--modes="):
            modes = a.split("=", 1)[1]
    specs = specgen.suite_f4(count)
    out = {"config": {"count": count, "chunk": chunk, "max_cost": max_cost, "generator": "specgen.suite_f4"}}
    base = None
    for mode in modes.split(","):
        res, per, total = run(mode, specs, chunk, max_cost)
        key = [(r.status, r.cost) for r in res]
        if base is None:
            base = (key, res)
        out[mode] = summary(mode, res, per, total)
        out[mode]["agree_with_first_mode"] = sum(a == b for a, b in zip(key, base[0]))
        print(json.dumps({mode: out[mode]}), flush=True)
    small = [sp for sp, r in zip(specs, base[1]) if r.status == "found" and r.candidates < 1e8]
    out["small"] = {"specs": len(small), "rule": "found with < 1e8 candidates in the first mode"}
    for mode in modes.split(","):
        res, per, total = run(mode, small, chunk, max_cost)
        out["small"][mode] = summary(mode, res, per, total)
    print(json.dumps({"small": out["small"]}), flush=True)
    return out


if __name__ == "__main__":
    main()
