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
