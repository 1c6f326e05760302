#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum of every launch) into profiles/.

    python scripts/summarize_launches.py gpurun_out/launches_bench.csv profiles/r01_bench_launches.md "<command>"

The launches are cold-cache and serialised by ncu: compare kernel SHARES with the
bench's own CUDA-event numbers, not absolute times.
"""
import collections
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_top_kernel import parse_launches  # noqa: E402


def short(name):
    base = re.sub(r"^void\s+", "", name.replace("<unnamed>", "anon").replace("(anonymous namespace)", "anon"))
    base = base.split("(")[0].split("<")[0].strip()
    return base.split("::")[-1] or base


def main():
    src, dst = sys.argv[1], sys.argv[2]
    cmd = sys.argv[3] if len(sys.argv) > 3 else ""
    launches = parse_launches(src)
    tot = sum(ms for _, ms in launches)
    by = collections.defaultdict(lambda: [0, 0.0])
    for n, ms in launches:
        k = short(n)
        by[k][0] += 1
        by[k][1] += ms
    lines = [f"# ncu launch list: `{cmd}`", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` (every launch cold-cache and "
             "serialised: compare shares, not absolute times).", "",
             f"{len(launches)} launches, {tot:.2f} ms total", "",
             "| kernel | launches | ms | share |", "|---|---|---|---|"]
    for k, (n, ms) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:16]))


if __name__ == "__main__":
    main()
