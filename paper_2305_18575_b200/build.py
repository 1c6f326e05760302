"""Build librei_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_2305_18575_b200.build        # or build() from Python
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "librei_b200.so")
SOURCES = ["precompute.cu", "levels.cu", "exchange.cu", "devmem.cu", "rei_api.cu"]
HEADERS = ["rei_common.cuh", "rei_host.h"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--shared",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-ldl"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "rei.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    import fcntl
    # one builder at a time (test workers / ranks may call build() together)
    with open(LIB + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and not _stale():
            return LIB
        return _build_locked(verbose)


def _build_locked(verbose: bool) -> str:
    # one nvcc per translation unit, in parallel, then one link
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    comp = [f for f in FLAGS if f not in ("--shared", "-ldl")]

    def compile_one(f):
        obj = os.path.join(objdir, f.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *comp, "-c", "-o", obj, os.path.join(CSRC, f)]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        outs = list(ex.map(compile_one, SOURCES))
    report = ""
    for obj, r in outs:
        report += r.stderr
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building librei_b200.so")
    cmd = [NVCC, *ARCH, "--shared", "-Xcompiler", "-fPIC", "-o", LIB + ".tmp", *[o for o, _ in outs], "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking librei_b200.so")
    with open(os.path.join(PKG, "ptxas_report.txt"), "w") as f:
        f.write(report)
    if verbose:
        sys.stderr.write(report)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_variant(name: str, defines) -> str:
    """Build librei_b200_<name>.so with extra -D flags (A/B experiments only)."""
    out = os.path.join(PKG, f"librei_b200_{name}.so")
    cmd = [NVCC, *ARCH, *[f for f in FLAGS if f != "-v" and f != "-Xptxas"], *[f"-D{d}" for d in defines],
           "-o", out, *[os.path.join(CSRC, f) for f in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed building variant {name}")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
