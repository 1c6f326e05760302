"""World-size-2 host-side checks of the multi-GPU path on CPU (gloo, 127.0.0.1).

* every rank's share of a level's work lists (rei_partition, the C ABI's pure host
  function) is disjoint and the shares cover the list exactly;
* the level exchange protocol driven by the library's host functions (rei_cs_owner,
  rei_exchange_offsets): bucket by hash owner, all-to-all, owner dedup, all-gather
  of the owners' lists -- every rank derives the same level, the union of the
  staged lists (the device side of the same exchange runs in
  tests/test_gpu_multiproc.py);
* bench.py's cross-rank reduction: time = max over ranks, work = sum;
* the sharded cache's host transport (REI_FLAG_SHARDED_CACHE): the C all-gather
  callback the binding builds on torch.distributed returns every rank's bytes in
  rank order (IPC-handle exchange and the per-level barrier go through it), and
  hash ownership splits a level into disjoint shards that cover it.
"""
import os
import random
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_18575_b200 import build, partition
        build.build()
        # 1) partitions
        for total in (0, 1, 5, 1000, 10 ** 12 + 7):
            b, e = partition(total, world, rank)
            spans = [None] * world
            dist.all_gather_object(spans, (b, e))
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
                assert e0 == b1 and b0 <= e0
        # 2) the level exchange protocol with the library's host functions: a rank's
        #    staged CSs are bucketed by rei_cs_owner, sent to their owners at the
        #    rei_exchange_offsets positions (all-to-all over gloo), deduplicated by the
        #    owner, and the owners' lists all-gathered in owner order -- every rank gets
        #    the same level, the union of the staged lists without duplicates
        from paper_2305_18575_b200 import cs_owner, exchange_offsets
        for words in (1, 2, 4, 16):
            rng = random.Random(100 + rank + words)
            pool = [rng.getrandbits(32 * words) for _ in range(60)]
            pool_all = [None] * world
            dist.all_gather_object(pool_all, pool)
            common = pool_all[0][:20]  # CSs several ranks find (cross-rank duplicates)
            mine = list(dict.fromkeys(common + pool[20:]))
            owners = [cs_owner(x, words, world) for x in mine]
            assert all(0 <= o < world for o in owners)
            buckets = [[x for x, o in zip(mine, owners) if o == d] for d in range(world)]
            row = [len(b) for b in buckets]
            rows = [None] * world
            dist.all_gather_object(rows, row)
            counts = [c for r in rows for c in r]
            send_off, recv_off = exchange_offsets(world, counts, rank)
            flat = [x for b in buckets for x in b]
            assert all(flat[send_off[d]:send_off[d] + row[d]] == buckets[d] for d in range(world))
            sent = [None] * world
            dist.all_gather_object(sent, flat)  # gloo stands in for the all-to-all
            recv = []
            for src in range(world):
                so, _ = exchange_offsets(world, counts, src)
                chunk = sent[src][so[rank]:so[rank] + counts[src * world + rank]]
                assert len(recv) == recv_off[src]
                recv += chunk
            assert all(cs_owner(x, words, world) == rank for x in recv)
            uniq = list(dict.fromkeys(recv))
            lists = [None] * world
            dist.all_gather_object(lists, uniq)
            level = [x for l in lists for x in l]
            views = [None] * world
            dist.all_gather_object(views, level)
            assert all(v == views[0] for v in views)
            staged = [None] * world
            dist.all_gather_object(staged, mine)
            assert sorted(level) == sorted(set().union(*map(set, staged)))
        # 3) bench.py reduction
        import bench
        t, c = bench.reduce_over_ranks(10.0 + rank, 1000 * (rank + 1), torch.device("cpu"), world)
        assert t == 10.0 + world - 1 and c == sum(1000 * (r + 1) for r in range(world))
        # 4) sharded-cache transport: the C callback over torch.distributed (gloo)
        import ctypes
        from paper_2305_18575_b200.rei import c_allgather, torch_allgather
        cb = c_allgather(torch_allgather())
        for n in (1, 7, 400):  # 1 byte = the per-level barrier; 400 = IPC handle records
            send = ctypes.create_string_buffer(bytes([(rank * 31 + i) % 256 for i in range(n)]), n)
            recv = ctypes.create_string_buffer(n * world)
            assert cb(None, ctypes.cast(send, ctypes.c_void_p), ctypes.cast(recv, ctypes.c_void_p), n) == 0
            want = b"".join(bytes([(r * 31 + i) % 256 for i in range(n)]) for r in range(world))
            assert recv.raw == want
        keys = list(range(0, 5000, 7))
        mine = [k for k in keys if ((k * 0x9E3779B97F4A7C15 & (2 ** 64 - 1)) >> 40) % world == rank]
        shards = [None] * world
        dist.all_gather_object(shards, mine)
        assert sorted(x for sh in shards for x in sh) == keys
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, "ok") for r in range(world)], res
