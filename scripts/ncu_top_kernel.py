#!/usr/bin/env python3
"""Launch list + full ncu capture of the longest launch of a kernel (run under gpurun).

    python scripts/ncu_top_kernel.py <tag> [kernel_regex] [-- solve args]

1. ncu --metrics gpu__time_duration.sum over one scripts/profile_solve.py run
   -> gpurun_out/launches_<tag>.csv (every launch, cold-cache, serialised);
2. picks the longest launch whose name matches kernel_regex (default k_concat);
3. ncu --set full --import-source on on exactly that launch
   -> gpurun_out/prof_<tag>.ncu-rep.
"""
import csv
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def parse_launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    out = []
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
        out.append((d["Kernel Name"], v * scale))
    return out


def main():
    tag = sys.argv[1]
    regex = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "--" else "k_concat"
    extra = sys.argv[sys.argv.index("--") + 1:] if "--" in sys.argv else []
    os.makedirs(OUT, exist_ok=True)
    cmd = [sys.executable, os.path.join(ROOT, "scripts", "profile_solve.py"), *extra]
    lpath = os.path.join(OUT, f"launches_{tag}.csv")
    subprocess.run(["ncu", "--metrics", "gpu__time_duration.sum", "--clock-control", "none", "--csv",
                    "--log-file", lpath, *cmd], check=True, stdout=subprocess.DEVNULL)
    launches = parse_launches(lpath)
    matching = [(i, ms) for i, (name, ms) in enumerate(launches) if re.search(regex, name)]
    idx_in_match = max(range(len(matching)), key=lambda k: matching[k][1])
    total = sum(ms for _, ms in launches)
    print(f"{len(launches)} launches, {total:.2f} ms total; longest {regex}: #{idx_in_match} "
          f"{matching[idx_in_match][1]:.3f} ms")
    subprocess.run(["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on",
                    "-k", f"regex:{regex}", "-s", str(idx_in_match), "-c", "1", "-f",
                    "-o", os.path.join(OUT, f"prof_{tag}"), *cmd], check=True, stdout=subprocess.DEVNULL)


if __name__ == "__main__":
    main()
