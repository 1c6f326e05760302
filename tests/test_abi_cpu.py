"""C-ABI library checks that need no GPU: it builds, loads, exports every symbol
declared in include/rei.h, and its pure host logic (partition) is right."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rei.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rei_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2305_18575_b200 import build
    build.build()
    from paper_2305_18575_b200 import rei
    return rei.load_library()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("rei_init", "rei_solve", "rei_level_stats", "rei_destroy", "rei_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_init_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2305_18575_b200 import ReiError, Solver
    with pytest.raises(ReiError):
        Solver("01", ["1"], ["0"])


def test_partition_covers_space_exactly(lib):
    from paper_2305_18575_b200 import partition
    for total in (0, 1, 7, 100, 2 ** 40 + 3):
        for G in (1, 2, 3, 8):
            spans = [partition(total, G, g) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_sass_is_sm100a():
    from paper_2305_18575_b200 import build
    path = build.build()
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_nccl_is_resolved_at_run_time(lib):
    # the library has no link-time NCCL dependency; NCCL is dlopen'ed (torch's copy)
    # only for multi-GPU contexts -- ncclGetUniqueId works without a GPU
    import subprocess
    from paper_2305_18575_b200 import build, nccl_unique_id
    deps = subprocess.run(["ldd", build.LIB], capture_output=True, text=True).stdout
    assert "nccl" not in deps
    a, b = nccl_unique_id(), nccl_unique_id()
    assert len(a) == 128 and a != b


def test_binding_flags_match_header():
    # the ctypes binding's option flags are the header's REI_FLAG_* values
    import re
    from paper_2305_18575_b200 import rei
    hdr = open(os.path.join(ROOT, "include", "rei.h")).read()
    flags = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define REI_FLAG_(\w+) (\d+)u", hdr)}
    assert flags["EXCHANGE_SELF"] == rei.FLAG_EXCHANGE_SELF
    for name in ("COMPLETE_FINAL_LEVEL", "NO_ONTHEFLY", "SHARDED_CACHE", "SMALL_CACHE"):
        assert flags[name] == getattr(rei, "FLAG_" + name), name
    assert len(set(flags.values())) == len(flags)  # distinct bits


def test_sass_has_device_loop_and_wide_concat():
    # the cooperative level loop and the wide concatenation kernels are in the library
    import subprocess
    lib_path = os.path.join(ROOT, "paper_2305_18575_b200", "librei_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    syms = subprocess.run(["cuobjdump", "-symbols", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "k_level_loop" in syms and "k_concat_wide" in syms
