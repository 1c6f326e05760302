"""Sharded cache (include/rei.h REI_FLAG_SHARDED_CACHE) on one GPU
(``-m gpu``).

G contexts act as ranks 0..G-1: rank o owns the CSs whose hash is o mod G (dedup
slot, cache entry, back-pointer); every rank enumerates its share of each level and
inserts candidates into the owners' buffers through peer mappings.  Virtual ranks
share one process (rei_solve_group); the cross-process case maps the owners'
buffers with CUDA IPC and meets through a gloo all-gather.  Checked against the
oracle: the same c*, the same set of CSs at every level (the owners' shards
concatenated), the same candidate counts through the last complete level, and
regexes rebuilt across shards that denote their CSs.  Capacity: G ranks hold a
cache that one context with the same per-context cap cannot."""
import os

import pytest

import oracle
import specgen
from regex_tools import cost as re_cost, language_on, parse, precise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_18575_b200 import build
    build.build()


def group(sp, G, **kw):
    from paper_2305_18575_b200 import Solver
    return [Solver.from_spec(sp, device=0, sharded_cache=True, mem_budget_bytes=kw.pop("budget", 1 << 28), **kw)
            for _ in range(G)]


def planted(alpha, tgt, p, n, lo, hi, s):
    return specgen.gen_planted(alpha, tgt, p, n, lo, hi, s)


CASES = [(specgen.C1_TOY, 12), (specgen.E1, 12), (specgen.TABLE1_ROW1, 15),
         (specgen.gen_type1("01", 4, 5, 5, 3), 20), (specgen.gen_type2("01", 7, 6, 6, 0), 16),
         (specgen.C1_TOY.with_costs((2, 1, 3, 1, 1)), 20),
         (planted("01", "1(0+11)*0?", 8, 8, 6, 12, 0), 10),     # |IC| > 64: indexed dedup, W = 4
         (planted("01", "0(10)*1?", 8, 8, 6, 14, 0), 9)]        # W = 8


def check_against_oracle(sp, K, members, rg, ro, o):
    assert rg.status == ro.status
    last = ro.cost if ro.status == "found" else K
    for c in range(1, last + 1):
        lists = [m.level_cs(c) for m in members]
        for other in lists[1:]:
            assert other == lists[0], c            # every rank sees the same shards
        got = lists[0]
        assert len(set(got)) == len(got), c       # each CS has exactly one owner
        assert sorted(got) == sorted(o.level_cs(c)), c
    if ro.status == "found":
        assert rg.cost == ro.cost
        assert precise(rg.regex, sp.P, sp.N)
        assert re_cost(parse(rg.regex), sp.costs) == ro.cost
    want = {l.cost: l for l in ro.levels}
    for l in rg.levels:  # candidates per constructor (A9) and new CSs, level by level
        w = want.get(l.cost)
        if w is None:
            continue
        assert (l.cand_q, l.cand_s, l.cand_c, l.cand_u, l.unique) == \
            (w.cand_q, w.cand_s, w.cand_c, w.cand_u, w.unique), l.cost


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("sp,K", CASES, ids=[f"{i}-{c[0].name or 'rand'}" for i, c in enumerate(CASES)])
def test_sharded_cache_matches_oracle(sp, K, G):
    from paper_2305_18575_b200 import solve_group
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K, complete_final_level=True)
    members = group(sp, G, complete_final_level=True)
    rg = solve_group(members, K)
    check_against_oracle(sp, K, members, rg, ro, o)


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_cache_early_exit(G):
    from paper_2305_18575_b200 import solve_group
    sp = specgen.INTRO
    ro = oracle.Oracle.from_spec(sp).solve(20)
    rg = solve_group(group(sp, G), 20)
    assert rg.status == "found" and rg.cost == ro.cost
    assert precise(rg.regex, sp.P, sp.N)
    assert rg.cand_complete == ro.cand_complete
    assert rg.cand_complete <= rg.candidates


def test_sharded_cache_reconstruction_across_shards():
    # every entry's regex, rebuilt through back-pointers that live on other
    # ranks, denotes its stored CS and has the level's cost
    from paper_2305_18575_b200 import solve_group
    sp = specgen.C1_TOY
    members = group(sp, 3, complete_final_level=True)
    solve_group(members, 8)
    g = members[1]
    ic = g.ic()
    idx = {w: i for i, w in enumerate(ic)}
    for c in range(1, 9):
        for i, cs in enumerate(g.level_cs(c)):
            rx = g.entry_regex(c, i)
            assert sum(1 << idx[w] for w in language_on(rx, ic)) == cs
            assert re_cost(parse(rx), sp.costs) == c


def test_sharded_cache_capacity():
    # a cap that one context cannot search under holds when G = 4 ranks share the cache
    from paper_2305_18575_b200 import Solver, solve_group
    sp, K = specgen.gen_type1("01", 4, 5, 5, 3), 20
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K, complete_final_level=True)
    total = sum(l.unique for l in ro.levels if l.complete)
    cap = total // 2
    single = Solver.from_spec(sp, device=0, max_entries=cap, onthefly=False, complete_final_level=True)
    assert single.solve(K).status == "out_of_memory"
    members = group(sp, 4, max_entries=cap, onthefly=False, complete_final_level=True)
    rg = solve_group(members, K)
    check_against_oracle(sp, K, members, rg, ro, o)


def test_sharded_cache_onthefly():
    # an owner's shard fills: the level is re-checked without caching
    from paper_2305_18575_b200 import solve_group
    sp, K = specgen.TABLE1_ROW1, 40
    o = oracle.Oracle.from_spec(sp)
    members = group(sp, 2, max_entries=30000)
    rg = solve_group(members, K)
    stats = rg.levels
    assert any(l.complete == 2 for l in stats) or rg.status == "out_of_memory"
    cached = [l.cost for l in stats if l.complete == 1]
    ro = o.solve(max(cached), complete_final_level=True)
    for c in cached:
        assert sorted(members[0].level_cs(c)) == sorted(o.level_cs(c)), c
    if rg.status == "found":
        assert precise(rg.regex, sp.P, sp.N)
        assert re_cost(parse(rg.regex), sp.costs) == rg.cost
        assert rg.cost == 28  # c* of Table 1 row 1 (golden / paper)
    assert ro.status in ("found", "not_found")


def test_sharded_cache_repeated_solves():
    from paper_2305_18575_b200 import solve_group
    sp = specgen.E1
    members = group(sp, 2)
    a = solve_group(members, 20)
    b = solve_group(members, 20)
    assert (a.status, a.cost, a.cand_complete) == (b.status, b.cost, b.cand_complete)


def _ipc_worker(rank, world, init_file, K, out_dir):
    import json
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank, world_size=world)
    from paper_2305_18575_b200 import Solver
    sp = specgen.gen_type1("01", 4, 5, 5, 3)
    s = Solver.from_spec(sp, device=0, world_size=world, rank=rank, sharded_cache=True,
                         mem_budget_bytes=1 << 27, complete_final_level=True)
    r = s.solve(K)
    levels = {c: sorted(s.level_cs(c)) for c in range(1, (r.cost if r.status == "found" else K) + 1)}
    stats = [(l.cost, l.cand_q, l.cand_s, l.cand_c, l.cand_u, l.unique) for l in r.levels]
    json.dump({"status": r.status, "cost": r.cost, "regex": r.regex, "stats": stats,
               "levels": levels}, open(os.path.join(out_dir, f"r{rank}.json"), "w"))
    dist.barrier()
    s.close()
    dist.destroy_process_group()


def test_sharded_cache_two_processes(tmp_path):
    # one process per rank: buffers mapped with CUDA IPC, barriers over gloo
    import json
    import torch.multiprocessing as mp
    K = 20
    mp.start_processes(_ipc_worker, args=(2, str(tmp_path / "init"), K, str(tmp_path)), nprocs=2,
                       start_method="spawn")
    sp = specgen.gen_type1("01", 4, 5, 5, 3)
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K, complete_final_level=True)
    res = [json.load(open(tmp_path / f"r{r}.json")) for r in range(2)]
    for r in res:
        assert r["status"] == ro.status
        want = {l.cost: (l.cost, l.cand_q, l.cand_s, l.cand_c, l.cand_u, l.unique) for l in ro.levels}
        for st in r["stats"]:
            if st[0] in want:
                assert tuple(st) == want[st[0]]
        if ro.status == "found":
            assert r["cost"] == ro.cost and precise(r["regex"], sp.P, sp.N)
        for c, cs in r["levels"].items():
            assert cs == sorted(o.level_cs(int(c))), c
