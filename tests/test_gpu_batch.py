"""Many small specifications solved concurrently (``-m gpu``):
rei_solve_batch runs independent contexts on host threads / their own streams;
every result must equal the oracle's (status, c*, per-level unique counts)."""
import pytest

import oracle
import specgen
from regex_tools import cost as re_cost, parse, precise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_18575_b200 import build
    build.build()


def suite():
    out = []
    for s in range(16):
        out.append(specgen.gen_type1("01", 4, 5, 5, 1000 + s))
        out.append(specgen.gen_type2("01", 5, 5, 5, 2000 + s))
    out.append(specgen.gen_type1("abc", 3, 4, 4, 7))
    out.append(specgen.E1)
    return out


@pytest.mark.parametrize("threads", [1, 8])
def test_batch_matches_oracle(threads):
    from paper_2305_18575_b200 import Solver, solve_batch
    specs = suite()
    solvers = [Solver.from_spec(sp, device=0) for sp in specs]
    results = solve_batch(solvers, 30, threads=threads)
    for sp, r in zip(specs, results):
        ro = oracle.Oracle.from_spec(sp).solve(30)
        assert r.status == ro.status, sp
        if ro.status == "found":
            assert r.cost == ro.cost
            if r.regex not in ("empty", "eps"):
                assert precise(r.regex, sp.P, sp.N)
                assert re_cost(parse(r.regex), sp.costs) == ro.cost
        want = {l.cost: l.unique for l in ro.levels if l.complete}
        got = {l.cost: l.unique for l in r.levels if l.complete}
        for c in set(want) & set(got):
            assert got[c] == want[c], (sp, c)


def packed_suite():
    out = suite()
    out += [specgen.gen_type1("01", 5, 8, 8, 3000 + s) for s in range(6)]       # |IC| 33-63: hash64
    out += [specgen.gen_type2("01", 6, 7, 7, 4000 + s) for s in range(4)]
    out.append(specgen.Spec("01", [], ["0"]))                                    # trivial: empty
    out.append(specgen.Spec("01", [""], ["0"]))                                  # trivial: eps
    out.append(specgen.gen_planted("01", "1(0+11)*0?", 8, 8, 6, 12, 0))          # |IC| > 64: alone
    out.append(specgen.Spec("01", ("0" * 20, "1"), ("0" * 19, "11")))            # > 15 splits: alone
    out.append(specgen.TABLE1_ROW1)                                              # not found below 14
    return out


@pytest.mark.parametrize("small_cache", [False, True])
def test_packed_matches_oracle(small_cache):
    # one packed launch per kernel class and level step over all specifications
    # (rei_solve_packed): every result equals the oracle's (status, c*, per-level unique
    # and per-constructor candidate counts of the complete levels)
    from paper_2305_18575_b200 import Solver, solve_packed
    specs = packed_suite()
    K = 14
    solvers = [Solver.from_spec(sp, device=0, small_cache=small_cache) for sp in specs]
    results, done = solve_packed(solvers, K)
    assert len(done) == len(specs) and all(d >= 0 for d in done)
    for sp, r in zip(specs, results):
        ro = oracle.Oracle.from_spec(sp).solve(K)
        assert r.status == ro.status, sp
        if ro.status == "found":
            assert r.cost == ro.cost, sp
            if r.regex not in ("empty", "eps"):
                assert precise(r.regex, sp.P, sp.N), (sp, r.regex)
                assert re_cost(parse(r.regex), sp.costs) == ro.cost
        want = {l.cost: l for l in ro.levels if l.complete}
        got = {l.cost: l for l in r.levels if l.complete == 1}
        for c in set(want) & set(got):
            w, g = want[c], got[c]
            assert (g.unique, g.cand_q, g.cand_s, g.cand_c, g.cand_u) == \
                (w.unique, w.cand_q, w.cand_s, w.cand_c, w.cand_u), (sp, c)
    for s in solvers:
        s.close()


def test_packed_then_single_is_identical():
    # a context solved in a packed call solves identically alone afterwards
    from paper_2305_18575_b200 import Solver, solve_packed
    specs = suite()[:8]
    solvers = [Solver.from_spec(sp, device=0) for sp in specs]
    packed, _ = solve_packed(solvers, 20)
    for s, rp in zip(solvers, packed):
        r1 = s.solve(20)
        # (the candidates evaluated inside the final level depend on when the parallel
        # search met its answer; everything through the last complete level is fixed)
        assert (r1.status, r1.cost, r1.cand_complete) == (rp.status, rp.cost, rp.cand_complete)
        assert [l.unique for l in r1.levels if l.complete == 1] == [l.unique for l in rp.levels if l.complete == 1]
        s.close()
