"""The device-resident level loop (k_level_loop) against the host level
loop and the oracle (``-m gpu``).

The small levels of a search run inside one cooperative kernel that plans each level
on the device exactly as the host's plan_level does (Alg. 1 lines 5-8),
so every level's CS set, its per-constructor candidate counts (reading A9) and the
back-pointer ranks must be identical to the host loop's; the loop hands over to the
host at a level that is too big (REI_DEVICE_LOOP_CAND), would overflow the cache,
must be sorted (bitmap mode), or holds the first precise candidate.
"""
import random

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


def solve(sp, K, monkeypatch, env=None, **kw):
    from paper_2305_18575_b200 import Solver
    for k in ("REI_NO_DEVICE_LOOP", "REI_DEVICE_LOOP_CAND", "REI_LOOP_RESUME"):
        monkeypatch.delenv(k, raising=False)
    for k, v in (env or {}).items():
        monkeypatch.setenv(k, v)
    g = Solver.from_spec(sp, device=0, **kw)
    return g, g.solve(K)


def levels_of(g, r):
    return {l.cost: (l.unique, l.cand_q, l.cand_s, l.cand_c, l.cand_u, l.complete) for l in r.levels}


CASES = [
    (specgen.C1_TOY, 12, {}),                                   # found inside the loop
    (specgen.E1, 12, {"complete_final_level": True}),
    (specgen.TABLE1_ROW1, 16, {}),                              # loop stops for the level sort
    (specgen.TABLE1_ROW1, 30, {"error": (25, 100)}),            # allowed error (f1)
    (specgen.C1_TOY.with_costs((2, 1, 3, 1, 1)), 20, {}),        # cost gaps
    (specgen.gen_type1("01", 4, 5, 5, 3, costs=(1, 2, 2, 1, 3)), 30, {}),
    (specgen.gen_type2("01", 7, 6, 6, 0), 16, {}),              # two-word CSs, 64-bit-key set
    (specgen.gen_type1("abc", 3, 5, 5, 1), 16, {}),
    (specgen.Spec("01x", ("01", "1"), ("0",)), 10, {}),         # zero seed (A2)
]


@pytest.mark.parametrize("sp,K,kw", CASES, ids=[f"{c[0].name or c[0].alphabet}-{i}" for i, c in enumerate(CASES)])
@pytest.mark.parametrize("cand", [None, "3000", "3000-resume"])
def test_device_loop_equals_host_loop(sp, K, kw, cand, monkeypatch):
    env = {"REI_DEVICE_LOOP_CAND": cand.split("-")[0]} if cand else {}
    if cand and cand.endswith("resume"):  # the loop resumes after every big host level
        env["REI_LOOP_RESUME"] = "1"
    gd, rd = solve(sp, K, monkeypatch, env, **kw)
    gh, rh = solve(sp, K, monkeypatch, {"REI_NO_DEVICE_LOOP": "1"}, **kw)
    assert (rd.status, rd.cost) == (rh.status, rh.cost)
    ld, lh = levels_of(gd, rd), levels_of(gh, rh)
    last = rd.cost if rd.status == "found" else K
    for c in lh:
        if c < last or kw.get("complete_final_level"):
            assert ld[c] == lh[c], c
            assert sorted(gd.level_cs(c)) == sorted(gh.level_cs(c)), c
    assert rd.cand_complete == rh.cand_complete
    if rd.status == "found" and rd.regex not in ("empty", "eps") and "error" not in kw:
        assert precise(rd.regex, sp.P, sp.N), rd.regex
        assert re_cost(parse(rd.regex), sp.costs) == rd.cost


@pytest.mark.parametrize("sp,K", [(specgen.TABLE1_ROW1, 14), (specgen.gen_type2("01", 7, 6, 6, 1), 14)],
                         ids=["n25", "w2"])
def test_device_loop_back_pointers(sp, K, monkeypatch):
    # every entry of the loop's levels reconstructs to a regex that denotes
    # exactly its CS on IC and costs exactly its level
    g, r = solve(sp, K, monkeypatch)
    ic = g.ic()
    idx = {w: i for i, w in enumerate(ic)}
    rng = random.Random(11)
    for l in r.levels:
        if not l.unique or l.cost > 13:
            continue
        arr = g.level_cs(l.cost)
        for i in rng.sample(range(len(arr)), min(25, len(arr))):
            rx = g.entry_regex(l.cost, i)
            assert sum(1 << idx[w] for w in language_on(rx, ic)) == arr[i], (l.cost, i, rx)
            assert re_cost(parse(rx), sp.costs) == l.cost


@pytest.mark.parametrize("sp,K", [(specgen.C1_TOY, 12), (specgen.gen_type1("01", 4, 5, 5, 2), 20),
                                  (specgen.gen_type2("01", 7, 6, 6, 3), 16)], ids=["toy", "t1", "w2"])
def test_device_loop_vs_oracle(sp, K, monkeypatch):
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K, complete_final_level=True)
    g, rg = solve(sp, K, monkeypatch, complete_final_level=True)
    assert (rg.status, rg.cost) == (ro.status, ro.cost)
    last = ro.cost if ro.status == "found" else K
    for c in range(1, last + 1):
        assert sorted(g.level_cs(c)) == sorted(o.level_cs(c)), c
    want = {l.cost: (l.unique, l.cand_q, l.cand_s, l.cand_c, l.cand_u) for l in ro.levels}
    for l in rg.levels:
        assert (l.unique, l.cand_q, l.cand_s, l.cand_c, l.cand_u) == want[l.cost], l.cost


def test_device_loop_capacity_handover(monkeypatch):
    # a cache cap stops the loop before a level that might not fit; the host loop then
    # grows / goes OnTheFly exactly as without the device loop (f2)
    sp = specgen.C1_TOY.with_costs((1, 3, 3, 1, 3))
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(40, max_entries=120, onthefly=True)
    g, rg = solve(sp, 40, monkeypatch, max_entries=120, onthefly=True)
    assert (rg.status, rg.last_complete_cost) == (ro.status, ro.last_complete_cost)
    if ro.status == "found":
        assert rg.cost == ro.cost and precise(rg.regex, sp.P, sp.N)


# Lagged levels (rei_api.cu solve_lagged): with unary costs > 1 a level is launched
# before the previous level's count is back.  The result must not depend on it.
LAG_CASES = [
    (specgen.TABLE1_ROW1.with_costs((10, 10, 10, 1, 10)), 150, {}),     # Table 1 row 8 costs
    (specgen.C1_TOY.with_costs((2, 3, 3, 1, 2)), 30, {}),
    (specgen.gen_type1("01", 4, 5, 5, 3, costs=(1, 2, 2, 1, 3)), 30, {}),
    (specgen.gen_type2("01", 7, 6, 6, 0, costs=(2, 3, 3, 1, 2)), 30, {}),   # two-word CSs
    (specgen.gen_type2("01", 7, 6, 6, 1, costs=(2, 3, 3, 1, 2)), 30, {"small_cache": True}),  # growth
]


@pytest.mark.parametrize("sp,K,kw", LAG_CASES, ids=[f"lag-{i}" for i in range(len(LAG_CASES))])
def test_lagged_levels_equal_synchronous(sp, K, kw, monkeypatch):
    gl, rl = solve(sp, K, monkeypatch, {"REI_NO_DEVICE_LOOP": "1"}, **kw)
    gs, rs = solve(sp, K, monkeypatch, {"REI_NO_DEVICE_LOOP": "1", "REI_NO_LAG": "1"}, **kw)
    assert (rl.status, rl.cost) == (rs.status, rs.cost)
    ll, ls = levels_of(gl, rl), levels_of(gs, rs)
    last = rl.cost if rl.status == "found" else K
    for c in ls:
        if c < last:
            assert ll[c] == ls[c], c
            assert sorted(gl.level_cs(c)) == sorted(gs.level_cs(c)), c
    assert rl.cand_complete == rs.cand_complete
    if rl.status == "found":
        assert precise(rl.regex, sp.P, sp.N), rl.regex
        assert re_cost(parse(rl.regex), sp.costs) == rl.cost


def test_lagged_levels_vs_oracle(monkeypatch):
    sp = specgen.gen_type1("01", 4, 5, 5, 3, costs=(1, 2, 2, 1, 3))
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(30)
    g, rg = solve(sp, 30, monkeypatch, {"REI_NO_DEVICE_LOOP": "1"})
    assert (rg.status, rg.cost) == (ro.status, ro.cost)
    want = {l.cost: (l.unique, l.cand_q, l.cand_s, l.cand_c, l.cand_u) for l in ro.levels if l.complete}
    for l in rg.levels:
        if l.complete == 1 and l.cost in want:
            assert (l.unique, l.cand_q, l.cand_s, l.cand_c, l.cand_u) == want[l.cost], l.cost
