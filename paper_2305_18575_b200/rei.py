"""ctypes binding of librei_b200.so (include/rei.h) -- argument marshalling only.

Every step of the search runs in the CUDA library; this module converts Python
strings / ints to the C ABI and back.  There is no CPU fallback: if the shared
library is missing or no CUDA device is usable, construction raises.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Dict, List, Optional, Sequence, Tuple

_PKG = os.path.dirname(os.path.abspath(__file__))
# REI_LIB selects an alternative build (A/B experiments, scripts/ab_variants.py)
LIB_PATH = os.environ.get("REI_LIB") or os.path.join(_PKG, "librei_b200.so")

REI_OK, REI_EINVAL, REI_NOT_FOUND, REI_OUT_OF_MEMORY, REI_ECUDA, REI_ENCCL = range(6)
STATUS_NAMES = {0: "found", 1: "invalid", 2: "not_found", 3: "out_of_memory", 4: "cuda_error",
                5: "nccl_error"}
FLAG_COMPLETE_FINAL_LEVEL = 1
FLAG_NO_ONTHEFLY = 2
FLAG_SHARDED_CACHE = 4
FLAG_SMALL_CACHE = 8
FLAG_EXCHANGE_SELF = 16
KERNEL_CLASSES = ("precompute", "unary", "concat", "union", "transpose", "other")


class ReiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Costs(ctypes.Structure):
    _fields_ = [("sym", ctypes.c_uint32), ("opt", ctypes.c_uint32), ("star", ctypes.c_uint32),
                ("cat", ctypes.c_uint32), ("alt", ctypes.c_uint32)]


# rei_allgather_fn: int (*)(void* user, const void* send, void* recv, size_t bytes)
_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_size_t)


class _Options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("mem_budget_bytes", ctypes.c_uint64), ("err_num", ctypes.c_uint32),
                ("err_den", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("world_size", ctypes.c_int), ("rank", ctypes.c_int),
                ("nccl_unique_id", ctypes.c_void_p), ("max_entries", ctypes.c_uint64),
                ("allgather", _ALLGATHER), ("allgather_user", ctypes.c_void_p)]


def torch_allgather(group=None):
    """Host all-gather over torch.distributed for REI_FLAG_SHARDED_CACHE: bytes -> the
    ranks' bytes in rank order.  Runs on a gloo group (CPU tensors); with another
    default backend a gloo group is created (collective: every rank calls this)."""
    import torch
    import torch.distributed as dist
    if group is None and dist.get_backend() != "gloo":
        group = dist.new_group(backend="gloo")
    world = dist.get_world_size(group)

    def gather(data: bytes):
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        return [bytes(o.numpy().tobytes()) for o in out]
    return gather


def c_allgather(fn):
    """Wrap a Python all-gather (bytes -> list of bytes, rank order) as the C callback."""
    def cb(user, send, recv, n):
        try:
            parts = fn(ctypes.string_at(send, n))
            buf = b"".join(parts)
            if any(len(x) != n for x in parts):
                return 1
            ctypes.memmove(recv, buf, len(buf))
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1
    return _ALLGATHER(cb)


class _Result(ctypes.Structure):
    _fields_ = [("regex", ctypes.c_char_p), ("cost", ctypes.c_uint32),
                ("last_complete_cost", ctypes.c_uint32), ("candidates", ctypes.c_uint64),
                ("cand_complete", ctypes.c_uint64), ("unique", ctypes.c_uint64),
                ("seconds", ctypes.c_double), ("n_ic", ctypes.c_uint32),
                ("cs_words", ctypes.c_uint32)]


class _LevelStat(ctypes.Structure):
    _fields_ = [("cost", ctypes.c_uint32), ("complete", ctypes.c_uint32),
                ("cand_q", ctypes.c_uint64), ("cand_s", ctypes.c_uint64),
                ("cand_c", ctypes.c_uint64), ("cand_u", ctypes.c_uint64),
                ("unique", ctypes.c_uint64), ("evaluated", ctypes.c_uint64),
                ("eval_c", ctypes.c_uint64), ("eval_u", ctypes.c_uint64), ("ms", ctypes.c_double)]


_lib = None


def load_library():
    """Load librei_b200.so; raises if it was not built (no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2305_18575_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    c = ctypes
    vp = c.c_void_p
    lib.rei_init.restype = c.c_int
    lib.rei_init.argtypes = [c.POINTER(vp), c.c_char_p, c.POINTER(c.c_char_p), c.c_size_t,
                             c.POINTER(c.c_char_p), c.c_size_t, _Costs, c.POINTER(_Options)]
    lib.rei_solve.restype = c.c_int
    lib.rei_solve.argtypes = [vp, c.c_uint32, c.POINTER(_Result)]
    lib.rei_level_stats.restype = c.c_int
    lib.rei_level_stats.argtypes = [vp, c.POINTER(_LevelStat), c.c_size_t, c.POINTER(c.c_size_t)]
    lib.rei_kernel_stats.restype = c.c_int
    lib.rei_kernel_stats.argtypes = [vp, c.c_int, c.POINTER(c.c_uint64), c.POINTER(c.c_double)]
    lib.rei_reset_kernel_stats.argtypes = [vp]
    lib.rei_launch_count.restype = c.c_uint64
    lib.rei_launch_count.argtypes = [vp]
    lib.rei_dedup_mode.restype = c.c_int
    lib.rei_dedup_mode.argtypes = [vp]
    lib.rei_transfer_bytes.restype = c.c_int
    lib.rei_transfer_bytes.argtypes = [vp, c.POINTER(c.c_uint64), c.POINTER(c.c_uint64)]
    lib.rei_last_error.restype = c.c_char_p
    lib.rei_last_error.argtypes = [vp]
    lib.rei_last_init_error.restype = c.c_char_p
    lib.rei_destroy.argtypes = [vp]
    lib.rei_release_cached_memory.argtypes = []
    lib.rei_release_cached_memory.restype = None
    lib.rei_ic.restype = c.c_int
    lib.rei_ic.argtypes = [vp, c.c_uint32, c.c_char_p, c.c_size_t, c.POINTER(c.c_uint32)]
    lib.rei_splits.restype = c.c_int
    lib.rei_splits.argtypes = [vp, c.c_uint32, c.POINTER(c.c_uint32), c.c_size_t, c.POINTER(c.c_uint32)]
    lib.rei_masks.restype = c.c_int
    lib.rei_masks.argtypes = [vp, c.POINTER(c.c_uint32), c.POINTER(c.c_uint32)]
    lib.rei_level_cs.restype = c.c_int
    lib.rei_level_cs.argtypes = [vp, c.c_uint32, c.POINTER(c.c_uint32), c.c_size_t, c.POINTER(c.c_size_t)]
    lib.rei_entry_regex.restype = c.c_int
    lib.rei_entry_regex.argtypes = [vp, c.c_uint32, c.c_uint64, c.c_char_p, c.c_size_t]
    lib.rei_cs_ops.restype = c.c_int
    lib.rei_cs_ops.argtypes = [vp, c.c_int, c.POINTER(c.c_uint32), c.POINTER(c.c_uint32),
                               c.POINTER(c.c_uint32), c.c_size_t]
    lib.rei_partition.argtypes = [c.c_uint64, c.c_int, c.c_int, c.POINTER(c.c_uint64), c.POINTER(c.c_uint64)]
    lib.rei_cs_owner.restype = c.c_int
    lib.rei_cs_owner.argtypes = [c.POINTER(c.c_uint32), c.c_uint32, c.c_int]
    lib.rei_exchange_offsets.restype = None
    lib.rei_exchange_offsets.argtypes = [c.c_int, c.POINTER(c.c_uint64), c.c_int, c.POINTER(c.c_uint64),
                                         c.POINTER(c.c_uint64)]
    lib.rei_nccl_unique_id.restype = c.c_int
    lib.rei_nccl_unique_id.argtypes = [c.c_void_p, c.c_size_t]
    lib.rei_solve_batch.restype = c.c_int
    lib.rei_solve_batch.argtypes = [c.POINTER(c.c_void_p), c.c_size_t, c.c_uint32, c.c_int,
                                    c.POINTER(_Result), c.POINTER(c.c_int)]
    lib.rei_solve_packed.restype = c.c_int
    lib.rei_solve_packed.argtypes = [c.POINTER(c.c_void_p), c.c_size_t, c.c_uint32, c.POINTER(_Result),
                                     c.POINTER(c.c_int), c.POINTER(c.c_double)]
    lib.rei_solve_group.restype = c.c_int
    lib.rei_solve_group.argtypes = [c.POINTER(c.c_void_p), c.c_int, c.c_uint32, c.POINTER(_Result)]
    _lib = lib
    return lib


@dataclasses.dataclass
class LevelStat:
    cost: int
    complete: int  # 1 cached, 2 checked on the fly (not cached), 0 stopped inside
    cand_q: int
    cand_s: int
    cand_c: int
    cand_u: int
    unique: int
    evaluated: int
    eval_c: int
    eval_u: int
    ms: float

    @property
    def cand(self) -> int:
        return self.cand_q + self.cand_s + self.cand_c + self.cand_u


@dataclasses.dataclass
class Result:
    status: str
    regex: str
    cost: int
    last_complete_cost: int
    candidates: int
    cand_complete: int
    unique: int
    seconds: float
    n_ic: int
    cs_words: int
    levels: List[LevelStat]


def release_cached_memory() -> None:
    """Return the device / pinned blocks that destroyed contexts left in the
    library's caches to the driver (rei_release_cached_memory)."""
    load_library().rei_release_cached_memory()


def _strs(xs: Sequence[str]):
    arr = (ctypes.c_char_p * max(1, len(xs)))()
    for i, x in enumerate(xs):
        arr[i] = x.encode("latin-1")
    return arr


class Solver:
    """One specification on one GPU (a librei_b200 context)."""

    def __init__(self, alphabet: str, P: Sequence[str], N: Sequence[str],
                 costs: Sequence[int] = (1, 1, 1, 1, 1), device: int = -1, stream=None,
                 mem_budget_bytes: int = 0, error: Optional[Tuple[int, int]] = None,
                 complete_final_level: bool = False, world_size: int = 1, rank: int = 0,
                 nccl_id: Optional[bytes] = None, max_entries: int = 0, onthefly: bool = True,
                 sharded_cache: bool = False, allgather=None, small_cache: bool = False,
                 exchange_self: bool = False):
        """world_size > 1 (one process per rank, rei_solve collective): the level
        exchange runs over NCCL with `nccl_id` (rank 0's nccl_unique_id()), or, with
        `allgather` and no nccl_id, through that host all-gather (bytes -> list of
        bytes in rank order, e.g. torch_allgather() over gloo).
        sharded_cache: capacity mode (include/rei.h REI_FLAG_SHARDED_CACHE); `allgather`
        defaults to torch_allgather() there."""
        lib = load_library()
        self._lib = lib
        self._h = ctypes.c_void_p()
        opts = _Options()
        self._nccl_id = None
        self._allgather = None
        if world_size > 1 and sharded_cache:
            self._allgather = c_allgather(allgather or torch_allgather())
            opts.allgather = self._allgather
        elif world_size > 1 and allgather is not None and nccl_id is None:
            # host-staged level exchange through the caller's all-gather (e.g. gloo)
            self._allgather = c_allgather(allgather)
            opts.allgather = self._allgather
        elif world_size > 1 or exchange_self:
            if nccl_id is None or len(nccl_id) < 128:
                raise ValueError("world_size > 1 needs the 128-byte nccl_id from rank 0 "
                                 "(or an allgather callable for the host-staged exchange)")
            _use_torch_nccl()
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            opts.nccl_unique_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        opts.device = device
        if stream is not None:
            opts.stream = int(getattr(stream, "cuda_stream", stream))
        opts.mem_budget_bytes = int(mem_budget_bytes)
        if error:
            opts.err_num, opts.err_den = int(error[0]), int(error[1])
        else:
            opts.err_num, opts.err_den = 0, 1
        opts.flags = (FLAG_COMPLETE_FINAL_LEVEL if complete_final_level else 0) | \
            (0 if onthefly else FLAG_NO_ONTHEFLY) | (FLAG_SHARDED_CACHE if sharded_cache else 0) | \
            (FLAG_SMALL_CACHE if small_cache else 0) | (FLAG_EXCHANGE_SELF if exchange_self else 0)
        opts.max_entries = int(max_entries)
        opts.world_size, opts.rank = int(world_size), int(rank)
        costs_c = _Costs(*[int(c) for c in costs])
        self._keep = (_strs(P), _strs(N))
        st = lib.rei_init(ctypes.byref(self._h), alphabet.encode("latin-1"), self._keep[0], len(P),
                          self._keep[1], len(N), costs_c, ctypes.byref(opts))
        if st != REI_OK:
            raise ReiError(st, lib.rei_last_init_error().decode())
        self.alphabet, self.P, self.N, self.costs = alphabet, list(P), list(N), tuple(costs)

    @classmethod
    def from_spec(cls, spec, **kw) -> "Solver":
        return cls(spec.alphabet, spec.P, spec.N, spec.costs, **kw)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.rei_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _err(self) -> str:
        return self._lib.rei_last_error(self._h).decode()

    # ---- search ---------------------------------------------------------
    def solve(self, max_cost: int = 500) -> Result:
        r = _Result()
        st = self._lib.rei_solve(self._h, int(max_cost), ctypes.byref(r))
        if st not in (REI_OK, REI_NOT_FOUND, REI_OUT_OF_MEMORY):
            raise ReiError(st, self._err())
        return Result(STATUS_NAMES[st], (r.regex or b"").decode("latin-1"), r.cost,
                      r.last_complete_cost, r.candidates, r.cand_complete, r.unique, r.seconds,
                      r.n_ic, r.cs_words, self.level_stats())

    def level_stats(self) -> List[LevelStat]:
        n = ctypes.c_size_t()
        self._lib.rei_level_stats(self._h, None, 0, ctypes.byref(n))
        buf = (_LevelStat * max(1, n.value))()
        self._lib.rei_level_stats(self._h, buf, n.value, ctypes.byref(n))
        return [LevelStat(b.cost, int(b.complete), b.cand_q, b.cand_s, b.cand_c, b.cand_u,
                          b.unique, b.evaluated, b.eval_c, b.eval_u, b.ms) for b in buf[:n.value]]

    def kernel_stats(self) -> Dict[str, Tuple[int, float]]:
        out = {}
        for k, name in enumerate(KERNEL_CLASSES):
            n = ctypes.c_uint64()
            ms = ctypes.c_double()
            self._lib.rei_kernel_stats(self._h, k, ctypes.byref(n), ctypes.byref(ms))
            out[name] = (n.value, ms.value)
        return out

    def reset_kernel_stats(self):
        self._lib.rei_reset_kernel_stats(self._h)

    def launch_count(self) -> int:
        return int(self._lib.rei_launch_count(self._h))

    DEDUP_MODES = ("bitmap", "hash64", "indexed", "inline")

    def dedup_mode(self) -> str:
        """The dedup set rei_init chose (include/rei.h rei_dedup_mode)."""
        return self.DEDUP_MODES[self._lib.rei_dedup_mode(self._h)]

    def transfer_bytes(self) -> Tuple[int, int]:
        h, d = ctypes.c_uint64(), ctypes.c_uint64()
        self._lib.rei_transfer_bytes(self._h, ctypes.byref(h), ctypes.byref(d))
        return h.value, d.value

    # ---- introspection ----------------------------------------------------
    @property
    def n_ic(self) -> int:
        n = ctypes.c_uint32()
        self._lib.rei_ic(self._h, 0, None, 0, ctypes.byref(n))
        return n.value

    @property
    def cs_words(self) -> int:
        w = 1
        while 32 * w < self.n_ic:
            w *= 2
        return w

    def ic(self) -> List[str]:
        out = []
        buf = ctypes.create_string_buffer(4096)
        for k in range(self.n_ic):
            if self._lib.rei_ic(self._h, k, buf, 4096, None) != REI_OK:
                raise ReiError(REI_EINVAL, "rei_ic")
            out.append(buf.value.decode("latin-1"))
        return out

    def splits(self, w: int) -> List[Tuple[int, int]]:
        cap = 4096
        arr = (ctypes.c_uint32 * (2 * cap))()
        cnt = ctypes.c_uint32()
        st = self._lib.rei_splits(self._h, w, arr, cap, ctypes.byref(cnt))
        if st != REI_OK:
            raise ReiError(st, self._err())
        return [(arr[2 * k], arr[2 * k + 1]) for k in range(cnt.value)]

    def masks(self) -> Tuple[int, int]:
        W = self.cs_words
        p = (ctypes.c_uint32 * W)()
        q = (ctypes.c_uint32 * W)()
        self._lib.rei_masks(self._h, p, q)
        return _words_to_int(p, W), _words_to_int(q, W)

    def level_cs_array(self, cost: int):
        """The CSs of level `cost` as a numpy uint32 array of shape (m, cs_words)."""
        import numpy as np
        W = self.cs_words
        cnt = ctypes.c_size_t()
        self._lib.rei_level_cs(self._h, cost, None, 0, ctypes.byref(cnt))
        m = cnt.value
        arr = np.zeros(max(1, m) * W, dtype=np.uint32)
        if m:
            st = self._lib.rei_level_cs(self._h, cost, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                        m, ctypes.byref(cnt))
            if st != REI_OK:
                raise ReiError(st, self._err())
        return arr[:m * W].reshape(m, W)

    def level_cs(self, cost: int) -> List[int]:
        W = self.cs_words
        arr = self.level_cs_array(cost)
        m = arr.shape[0]
        if m == 0:
            return []
        arr = arr.reshape(-1)
        if W == 1:
            return [int(x) for x in arr]
        arr = arr.reshape(m, W).astype(object)
        return [sum(int(row[q]) << (32 * q) for q in range(W)) for row in arr]

    def entry_regex(self, cost: int, i: int) -> str:
        buf = ctypes.create_string_buffer(1 << 16)
        st = self._lib.rei_entry_regex(self._h, cost, i, buf, 1 << 16)
        if st != REI_OK:
            raise ReiError(st, self._err())
        return buf.value.decode("latin-1")

    def cs_ops(self, op: int, a: Sequence[int], b: Optional[Sequence[int]] = None) -> List[int]:
        """op 0 union, 1 concat, 2 star, 3 question, 4 precise -- on the device."""
        W = self.cs_words
        m = len(a)
        A = (ctypes.c_uint32 * (m * W))()
        B = (ctypes.c_uint32 * (m * W))()
        O = (ctypes.c_uint32 * (m * W))()
        for i, x in enumerate(a):
            for q in range(W):
                A[i * W + q] = (x >> (32 * q)) & 0xFFFFFFFF
        if b is not None:
            for i, x in enumerate(b):
                for q in range(W):
                    B[i * W + q] = (x >> (32 * q)) & 0xFFFFFFFF
        st = self._lib.rei_cs_ops(self._h, op, A, B if b is not None else None, O, m)
        if st != REI_OK:
            raise ReiError(st, self._err())
        return [sum(int(O[i * W + q]) << (32 * q) for q in range(W)) for i in range(m)]


def _words_to_int(arr, W) -> int:
    return sum(int(arr[q]) << (32 * q) for q in range(W))


def partition(total: int, G: int, g: int) -> Tuple[int, int]:
    """rei_partition: rank g's contiguous share of a flattened space (host logic)."""
    lib = load_library()
    b, e = ctypes.c_uint64(), ctypes.c_uint64()
    lib.rei_partition(total, G, g, ctypes.byref(b), ctypes.byref(e))
    return b.value, e.value


def cs_owner(cs: int, cs_words: int, world: int) -> int:
    """rei_cs_owner: the hash owner of a CS among `world` ranks (host logic)."""
    lib = load_library()
    arr = (ctypes.c_uint32 * cs_words)(*[(cs >> (32 * q)) & 0xFFFFFFFF for q in range(cs_words)])
    return lib.rei_cs_owner(arr, cs_words, world)


def exchange_offsets(world: int, counts: Sequence[int], rank: int) -> Tuple[List[int], List[int]]:
    """rei_exchange_offsets: (send offsets by owner, receive offsets by source) of the
    level all-to-all for `rank`, from the world x world count matrix (row = source)."""
    lib = load_library()
    c = (ctypes.c_uint64 * (world * world))(*counts)
    so = (ctypes.c_uint64 * world)()
    ro = (ctypes.c_uint64 * world)()
    lib.rei_exchange_offsets(world, c, rank, so, ro)
    return list(so), list(ro)


def _use_torch_nccl():
    """Point the library's dlopen at the NCCL build torch loaded (one NCCL per process)."""
    import torch  # noqa: F401
    if "REI_NCCL_LIB" in os.environ:
        return
    try:
        import nvidia.nccl
        cand = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["REI_NCCL_LIB"] = cand
    except Exception:  # noqa: BLE001 -- fall back to the soname lookup in the library
        pass


def nccl_unique_id() -> bytes:
    """rank 0's ncclUniqueId (128 bytes) for Solver(..., world_size, rank, nccl_id)."""
    _use_torch_nccl()
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.rei_nccl_unique_id(buf, 128)
    if st != REI_OK:
        raise ReiError(st, "ncclGetUniqueId failed")
    return buf.raw


def solve_group(solvers: Sequence["Solver"], max_cost: int = 500) -> Result:
    """Run G single-GPU contexts as ranks 0..G-1 of one sharded search (virtual ranks)."""
    lib = load_library()
    arr = (ctypes.c_void_p * len(solvers))(*[s._h.value for s in solvers])
    r = _Result()
    st = lib.rei_solve_group(arr, len(solvers), int(max_cost), ctypes.byref(r))
    if st not in (REI_OK, REI_NOT_FOUND, REI_OUT_OF_MEMORY):
        raise ReiError(st, solvers[0]._err())
    s0 = solvers[0]
    return Result(STATUS_NAMES[st], (r.regex or b"").decode("latin-1"), r.cost, r.last_complete_cost,
                  r.candidates, r.cand_complete, r.unique, r.seconds, r.n_ic, r.cs_words,
                  s0.level_stats())


def solve_batch(solvers: Sequence["Solver"], max_cost: int = 500, threads: int = 8) -> List[Result]:
    """Independent searches, `threads` host threads, one stream per context (f4)."""
    lib = load_library()
    n = len(solvers)
    arr = (ctypes.c_void_p * max(1, n))(*[s._h.value for s in solvers])
    res = (_Result * max(1, n))()
    sts = (ctypes.c_int * max(1, n))()
    lib.rei_solve_batch(arr, n, int(max_cost), int(threads), res, sts)
    out = []
    for i, s in enumerate(solvers):
        r, st = res[i], sts[i]
        if st not in (REI_OK, REI_NOT_FOUND, REI_OUT_OF_MEMORY):
            raise ReiError(st, s._err())
        out.append(Result(STATUS_NAMES[st], (r.regex or b"").decode("latin-1"), r.cost,
                          r.last_complete_cost, r.candidates, r.cand_complete, r.unique, r.seconds,
                          r.n_ic, r.cs_words, s.level_stats()))
    return out


def solve_packed(solvers: Sequence["Solver"], max_cost: int = 500) -> Tuple[List[Result], List[float]]:
    """Packed launches over many small specifications on one device (f4, include/rei.h
    rei_solve_packed): results, and each spec's host seconds from the call to its result."""
    lib = load_library()
    n = len(solvers)
    arr = (ctypes.c_void_p * max(1, n))(*[s._h.value for s in solvers])
    res = (_Result * max(1, n))()
    sts = (ctypes.c_int * max(1, n))()
    done = (ctypes.c_double * max(1, n))()
    st = lib.rei_solve_packed(arr, n, int(max_cost), res, sts, done)
    if st != REI_OK:
        raise ReiError(st, solvers[0]._err() if solvers else "")
    out = []
    for i, s in enumerate(solvers):
        r, sti = res[i], sts[i]
        if sti not in (REI_OK, REI_NOT_FOUND, REI_OUT_OF_MEMORY):
            raise ReiError(sti, s._err())
        out.append(Result(STATUS_NAMES[sti], (r.regex or b"").decode("latin-1"), r.cost,
                          r.last_complete_cost, r.candidates, r.cand_complete, r.unique, r.seconds,
                          r.n_ic, r.cs_words, s.level_stats()))
    return out, [done[i] for i in range(n)]


def solve(spec, max_cost: int = 500, **kw) -> Result:
    with Solver.from_spec(spec, **kw) as s:
        return s.solve(max_cost)
