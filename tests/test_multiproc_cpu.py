"""World-size-2 host-side checks of the multi-GPU path on CPU (gloo, 127.0.0.1).

* every rank's share of a level's work lists (rei_partition, the C ABI's pure host
  function) is disjoint and the shares cover the list exactly;
* the level exchange protocol: ranks all-gather their new-CS lists in rank order
  and keep first occurrences -- every rank derives the same canonical list, equal
  to the union of the lists;
* bench.py's cross-rank reduction: time = max over ranks, work = sum.
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
        # 2) canonical merge of per-rank lists (first occurrence, rank order)
        rng = random.Random(100 + rank)
        mine = [rng.randrange(50) for _ in range(40)]
        mine = list(dict.fromkeys(mine))  # a rank's own list has no duplicates
        lists = [None] * world
        dist.all_gather_object(lists, mine)
        merged = list(dict.fromkeys(x for l in lists for x in l))
        views = [None] * world
        dist.all_gather_object(views, merged)
        assert all(v == views[0] for v in views)
        assert set(merged) == set().union(*map(set, lists))
        # 3) bench.py reduction
        import bench
        t, c = bench.reduce_over_ranks(10.0 + rank, 1000 * (rank + 1), torch.device("cpu"), world)
        assert t == 10.0 + world - 1 and c == sum(1000 * (r + 1) for r in range(world))
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
