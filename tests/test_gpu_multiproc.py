"""World size 2, one process per rank, both on GPU 0 (``-m gpu``): the library's own
level exchange (owner bucketing, all-to-all, owner dedup, all-gather of the uniques,
re-pointing of tentative indexed-hash slots) through the host-staged transport --
rei_options.allgather over torch.distributed gloo (NCCL cannot put two ranks on one
GPU).  Checked against the oracle (same c*, same CS set at every complete level) and
across ranks (byte-identical caches, same regex)."""
import os
import socket

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_18575_b200 import build
    build.build()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spec(name):
    import specgen
    return {
        "c1": (specgen.C1_TOY, 12),
        "row1": (specgen.TABLE1_ROW1, 17),
        "t1": (specgen.gen_type1("01", 4, 5, 5, 3), 20),
        "w4": (specgen.gen_planted("01", "(0+1)*0(0+1)(0+1)", 10, 10, 4, 8, 1), 11),
        "w16": (specgen.gen_planted("abcd", "(a+b)*c(a+d)*", 10, 10, 6, 14, 1), 8),
    }[name]


def _worker(rank, world, port, name, redundant, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["REI_REDUNDANT_CAND"] = redundant
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_18575_b200 import Solver
        from paper_2305_18575_b200.rei import torch_allgather
        sp, K = _spec(name)
        s = Solver.from_spec(sp, device=0, world_size=world, rank=rank, allgather=torch_allgather(),
                             complete_final_level=True)
        r = s.solve(K)
        last = r.cost if r.status == "found" else K
        levels = {c: s.level_cs(c) for c in range(1, last + 1)}
        q.put((rank, "ok", r.status, r.cost, r.regex, levels, s.transfer_bytes()))
        s.close()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), None, None, None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("redundant", ["0", "3000"], ids=["exchange-all", "redundant-small"])
@pytest.mark.parametrize("name", ["c1", "row1", "t1", "w4", "w16"])
def test_two_processes_host_exchange(name, redundant):
    import torch.multiprocessing as mp
    import oracle
    from regex_tools import precise
    if redundant != "0" and name.startswith("w"):
        pytest.skip("no redundant levels above 64 bits")
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, redundant, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    assert [x[1] for x in res] == ["ok", "ok"], res
    sp, K = _spec(name)
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K, complete_final_level=True)
    (_, _, st0, c0, rx0, lv0, tb0), (_, _, st1, c1, rx1, lv1, _) = res
    assert st0 == st1 == ro.status
    if ro.status == "found":
        assert c0 == c1 == ro.cost
        assert rx0 == rx1 and precise(rx0, sp.P, sp.N)
    assert lv0 == lv1                      # byte-identical caches on both ranks
    for c, cs in lv0.items():
        assert sorted(cs) == sorted(o.level_cs(c)), c
    assert tb0[0] > 0 and tb0[1] > 0      # the host-staged transport moved the levels
