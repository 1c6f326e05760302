"""CPU oracle for the Paresy REI search -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product path (``paper_2305_18575_b200``) never imports it, and the two
share no code: the oracle is ``oracle/rei_oracle.cpp`` (plain sequential
Algorithm 1 / Algorithm 2 of PAPER.md) behind a ctypes wrapper.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie it to the paper:
worked example E1, the introduction example
(P:142-161), the Section 5 allowed-error table, brute-force
enumeration of syntactic regexes matched with Python ``re``, closed forms
(overfit bound P:1540-1545), and semiring laws.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rei_oracle.cpp")
_LIB = os.path.join(_HERE, "librei_oracle.so")
_lib = None

WORDS = 8  # the oracle's CS width in u64 words (|IC| <= 512)


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (plain -O2; the oracle is never tuned)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        c = ctypes
        lib.orc_create.restype = c.c_void_p
        lib.orc_create.argtypes = [c.c_char_p, c.POINTER(c.c_char_p), c.c_int,
                                   c.POINTER(c.c_char_p), c.c_int, c.POINTER(c.c_int),
                                   c.c_char_p, c.c_int]
        lib.orc_destroy.argtypes = [c.c_void_p]
        lib.orc_n.argtypes = [c.c_void_p]
        lib.orc_ic_word.argtypes = [c.c_void_p, c.c_int, c.c_char_p, c.c_int]
        lib.orc_gt_row.argtypes = [c.c_void_p, c.c_int, c.POINTER(c.c_int), c.c_int]
        lib.orc_masks.argtypes = [c.c_void_p, c.POINTER(c.c_uint64), c.POINTER(c.c_uint64)]
        lib.orc_op.argtypes = [c.c_void_p, c.c_int, c.POINTER(c.c_uint64),
                               c.POINTER(c.c_uint64), c.POINTER(c.c_uint64)]
        lib.orc_solve.argtypes = [c.c_void_p, c.c_int, c.c_long, c.c_long, c.c_int, c.c_ulonglong, c.c_int]
        lib.orc_otf_level.argtypes = [c.c_void_p]
        lib.orc_result.argtypes = [c.c_void_p, c.POINTER(c.c_longlong), c.POINTER(c.c_double)]
        lib.orc_regex.argtypes = [c.c_void_p, c.c_char_p, c.c_int]
        lib.orc_num_stats.argtypes = [c.c_void_p]
        lib.orc_stat.argtypes = [c.c_void_p, c.c_int, c.POINTER(c.c_ulonglong)]
        lib.orc_level_size.restype = c.c_long
        lib.orc_level_size.argtypes = [c.c_void_p, c.c_int]
        lib.orc_level_cs.restype = c.c_long
        lib.orc_level_cs.argtypes = [c.c_void_p, c.c_int, c.POINTER(c.c_uint64), c.c_long]
        lib.orc_entry_regex.argtypes = [c.c_void_p, c.c_int, c.c_long, c.c_char_p, c.c_int]
        _lib = lib
    return _lib


STATUS = {0: "found", 2: "not_found", 3: "out_of_memory"}


@dataclasses.dataclass
class LevelStat:
    cost: int
    cand_q: int
    cand_s: int
    cand_c: int
    cand_u: int
    unique: int
    complete: bool

    @property
    def cand(self) -> int:
        return self.cand_q + self.cand_s + self.cand_c + self.cand_u


@dataclasses.dataclass
class Result:
    status: str
    regex: str
    cost: int
    candidates: int          # through the found candidate, sequential order
    cand_complete: int       # through the last complete level
    last_complete_cost: int
    entries: int
    seconds: float
    levels: List[LevelStat]


def _cs_from_int(x: int) -> "ctypes.Array":
    arr = (ctypes.c_uint64 * WORDS)()
    for k in range(WORDS):
        arr[k] = (x >> (64 * k)) & ((1 << 64) - 1)
    return arr


def _cs_to_int(arr) -> int:
    return sum(int(arr[k]) << (64 * k) for k in range(WORDS))


class Oracle:
    """One specification (P, N) with its IC, guide table and masks."""

    def __init__(self, alphabet: str, P: Sequence[str], N: Sequence[str],
                 costs: Sequence[int] = (1, 1, 1, 1, 1)):
        lib = _load()
        self._lib = lib
        enc = lambda xs: (ctypes.c_char_p * max(1, len(xs)))(*[x.encode() for x in xs])
        c5 = (ctypes.c_int * 5)(*[int(c) for c in costs])
        err = ctypes.create_string_buffer(256)
        h = lib.orc_create(alphabet.encode(), enc(P), len(P), enc(N), len(N), c5, err, 256)
        if not h:
            raise ValueError(err.value.decode())
        self._h = ctypes.c_void_p(h)
        self.alphabet, self.P, self.N, self.costs = alphabet, list(P), list(N), tuple(costs)

    @classmethod
    def from_spec(cls, spec) -> "Oracle":
        return cls(spec.alphabet, spec.P, spec.N, spec.costs)

    def __del__(self):
        if getattr(self, "_h", None) is not None:
            self._lib.orc_destroy(self._h)
            self._h = None

    # ---- staged precompute views -------------------------------------
    @property
    def n(self) -> int:
        return self._lib.orc_n(self._h)

    def ic(self) -> List[str]:
        buf = ctypes.create_string_buffer(4096)
        out = []
        for k in range(self.n):
            self._lib.orc_ic_word(self._h, k, buf, 4096)
            out.append(buf.value.decode())
        return out

    def gt_row(self, w: int) -> List[Tuple[int, int]]:
        cap = 4096
        arr = (ctypes.c_int * (2 * cap))()
        m = self._lib.orc_gt_row(self._h, w, arr, cap)
        return [(arr[2 * k], arr[2 * k + 1]) for k in range(m)]

    def masks(self) -> Tuple[int, int]:
        p = (ctypes.c_uint64 * WORDS)()
        q = (ctypes.c_uint64 * WORDS)()
        self._lib.orc_masks(self._h, p, q)
        return _cs_to_int(p), _cs_to_int(q)

    # ---- CS operations (integers as bitvectors, bit i = IC word i) -----
    def _op(self, op: int, a: int, b: int = 0) -> int:
        out = (ctypes.c_uint64 * WORDS)()
        self._lib.orc_op(self._h, op, _cs_from_int(a), _cs_from_int(b), out)
        return _cs_to_int(out)

    def union(self, a: int, b: int) -> int:
        return self._op(0, a, b)

    def concat(self, a: int, b: int) -> int:
        return self._op(1, a, b)

    def star(self, a: int) -> int:
        return self._op(2, a)

    def question(self, a: int) -> int:
        return self._op(3, a)

    def satisfies(self, a: int) -> bool:
        return bool(self._op(4, a))

    # ---- search --------------------------------------------------------
    def solve(self, max_cost: int = 500, error: Optional[Tuple[int, int]] = None,
              complete_final_level: bool = False, max_entries: int = 0,
              onthefly: bool = False) -> Result:
        """max_entries caps the language cache (0 = unlimited); with onthefly the
        level that overflows and later ones are only checked."""
        num, den = error if error else (0, 1)
        self._lib.orc_solve(self._h, int(max_cost), int(num), int(den),
                            1 if complete_final_level else 0, int(max_entries), 1 if onthefly else 0)
        out6 = (ctypes.c_longlong * 6)()
        secs = ctypes.c_double()
        self._lib.orc_result(self._h, out6, ctypes.byref(secs))
        buf = ctypes.create_string_buffer(1 << 16)
        self._lib.orc_regex(self._h, buf, 1 << 16)
        levels = []
        st = (ctypes.c_ulonglong * 7)()
        for k in range(self._lib.orc_num_stats(self._h)):
            self._lib.orc_stat(self._h, k, st)
            levels.append(LevelStat(int(st[0]), int(st[1]), int(st[2]), int(st[3]),
                                    int(st[4]), int(st[5]), bool(st[6])))
        return Result(STATUS.get(int(out6[1]), str(out6[1])), buf.value.decode(),
                      int(out6[0]), int(out6[2]), int(out6[3]), int(out6[4]), int(out6[5]),
                      secs.value, levels)

    @property
    def otf_level(self) -> int:
        """First cost level checked on the fly (not cached) by the last solve; 0 = none."""
        return self._lib.orc_otf_level(self._h)

    def level_cs(self, cost: int) -> List[int]:
        m = self._lib.orc_level_size(self._h, cost)
        if m == 0:
            return []
        arr = (ctypes.c_uint64 * (m * WORDS))()
        self._lib.orc_level_cs(self._h, cost, arr, m)
        return [sum(int(arr[i * WORDS + k]) << (64 * k) for k in range(WORDS)) for i in range(m)]

    def entry_regex(self, cost: int, i: int) -> str:
        buf = ctypes.create_string_buffer(1 << 16)
        self._lib.orc_entry_regex(self._h, cost, i, buf, 1 << 16)
        return buf.value.decode()


def solve_spec(spec, max_cost: int = 500, **kw) -> Result:
    return Oracle.from_spec(spec).solve(max_cost, **kw)
