"""The NCCL data plane of the multi-GPU level exchange on one GPU
(``-m gpu``): REI_FLAG_EXCHANGE_SELF makes a one-rank NCCL world that still runs
every exchange step -- small levels computed redundantly and canonically sorted,
staged levels bucketed by hash owner, grouped ncclSend/ncclRecv (to itself), owner
dedup, the ncclBroadcast all-gather of the unique lists, the control-line
ncclAllGather.  NCCL cannot place two ranks on one GPU, so this is how the NCCL
calls run on the one-GPU boxes; the result must equal the oracle's exactly (level
sets, per-constructor counts, c*)."""
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


CASES = [
    (specgen.C1_TOY, 12),
    (specgen.TABLE1_ROW1, 16),                                       # one-word, level sort
    (specgen.gen_type2("01", 7, 6, 6, 0), 16),                       # two-word, 64-bit keys
    (specgen.gen_planted("01", "1(0+11)*0?", 8, 8, 6, 12, 0), 10),   # W32 = 4, inline keys
    (specgen.gen_planted("abcd", "(ab+c)*d(a+b)?", 6, 6, 6, 14, 0), 11),  # W32 = 8
]


@pytest.mark.parametrize("redundant", ["0", "2000"], ids=["exchange-all", "redundant-small"])
@pytest.mark.parametrize("sp,K", CASES, ids=[c[0].name or f"{c[0].alphabet}-{i}" for i, c in enumerate(CASES)])
def test_exchange_self_over_nccl(sp, K, redundant, monkeypatch):
    from paper_2305_18575_b200 import Solver, nccl_unique_id
    monkeypatch.setenv("REI_REDUNDANT_CAND", redundant)
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K, complete_final_level=True)
    g = Solver.from_spec(sp, device=0, complete_final_level=True, exchange_self=True, nccl_id=nccl_unique_id())
    rg = g.solve(K)
    assert (rg.status, rg.cost) == (ro.status, ro.cost)
    last = ro.cost if ro.status == "found" else K
    for c in range(1, last + 1):
        assert sorted(g.level_cs(c)) == sorted(o.level_cs(c)), c
    want = {l.cost: (l.unique, l.cand_q, l.cand_s, l.cand_c, l.cand_u) for l in ro.levels}
    for l in rg.levels:
        assert (l.unique, l.cand_q, l.cand_s, l.cand_c, l.cand_u) == want[l.cost], l.cost
    if ro.status == "found" and rg.regex not in ("empty", "eps"):
        assert precise(rg.regex, sp.P, sp.N), rg.regex
        assert re_cost(parse(rg.regex), sp.costs) == ro.cost
    g.close()


def test_exchange_self_needs_nccl_id():
    from paper_2305_18575_b200 import Solver
    with pytest.raises(ValueError):
        Solver.from_spec(specgen.C1_TOY, device=0, exchange_self=True)
