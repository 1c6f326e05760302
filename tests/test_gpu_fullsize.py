"""Full-size BASELINE configs, launched as bench.py launches them (``-m gpu``).

The oracle cannot finish these, so parity is checked by
properties that hold at any size and by the oracle on what it can compute:
* the returned regex is precise under Python's ``re`` and costs exactly c*;
* the oracle's per-level unique and candidate counts for the levels it finishes;
* sampled cache entries of the deepest levels: the regex reconstructed from each
  entry's back-pointer denotes exactly the stored CS on IC (checked
  with ``re``) and costs exactly its level;
* no cached CS of a level below c* is precise (the search would have stopped).
C5 (Table 1 row 1) is compared against the oracle's golden file in
test_gpu_parity.py.
"""
import json
import os
import random

import pytest

import bench
import oracle
import specgen
from regex_tools import cost as re_cost, language_on, parse, precise

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_18575_b200 import build
    build.build()


def check_full(name, oracle_levels):
    from paper_2305_18575_b200 import Solver
    spec, max_cost, _ = bench.WORKLOADS[name]
    g = Solver.from_spec(spec, device=0)
    r = g.solve(max_cost)
    assert r.status == "found"
    assert precise(r.regex, spec.P, spec.N), r.regex
    assert re_cost(parse(r.regex), spec.costs) == r.cost
    # oracle on the levels it can finish in seconds
    ro = oracle.Oracle.from_spec(spec).solve(oracle_levels)
    got = {l.cost: (l.unique, l.cand) for l in r.levels}
    for l in ro.levels:
        if l.complete and l.cost in got:
            assert got[l.cost] == (l.unique, l.cand), l.cost
    # sampled reconstruction audit of the deepest complete levels
    ic = g.ic()
    idx = {w: i for i, w in enumerate(ic)}
    pm, nm = g.masks()
    rng = random.Random(5)
    deep = [l.cost for l in r.levels if l.complete and l.unique][-3:]
    for c in deep:
        cs = g.level_cs(c)
        for i in rng.sample(range(len(cs)), min(40, len(cs))):
            rx = g.entry_regex(c, i)
            assert sum(1 << idx[w] for w in language_on(rx, ic)) == cs[i], (c, i, rx)
            assert re_cost(parse(rx), spec.costs) == c
        # P12 / minimality: nothing cached below c* is precise
        assert not any((x & pm) == pm and not (x & nm) for x in cs)
    return r


def test_c2_type1_seed0_full():
    # BASELINE configs[1]: |IC| = 58, two-word CSs, 64-bit-key hash set, c* = 23
    r = check_full("c2-t1-s0", 14)
    assert r.cost == 23 and r.cs_words == 2


def test_table1_row8_full():
    # Table 1 row 8: the row-1 spec with costs (10,10,10,1,10); c* = 208
    r = check_full("table1-row8", 130)
    assert r.cost == 208
    path = os.path.join(GOLDEN, "table1_row8_oracle.json")
    if os.path.exists(path):
        gold = json.load(open(path))
        assert gold["cstar"] == r.cost
        want = {l["cost"]: l["unique"] for l in gold["levels"]}
        for l in r.levels:
            if l.complete:
                assert l.unique == want[l.cost], l.cost


@pytest.mark.parametrize("alpha,tgt,lo,hi,seed", [
    ("01", "(0+1)*0(0+1)(0+1)", 6, 12, 0),       # configs[2]: W32 = 8
    ("abcd", "(ab+c)*d(a+b)?", 6, 14, 1),        # configs[3]: W32 = 16
])
def test_planted_wide_full(alpha, tgt, lo, hi, seed):
    from paper_2305_18575_b200 import Solver
    sp = specgen.gen_planted(alpha, tgt, 10, 10, lo, hi, seed)
    g = Solver.from_spec(sp, device=0)
    r = g.solve(30)
    assert r.status == "found"
    assert precise(r.regex, sp.P, sp.N)
    assert re_cost(parse(r.regex), sp.costs) == r.cost
    assert r.cost <= re_cost(parse(tgt), sp.costs)  # the planted target bounds c*
