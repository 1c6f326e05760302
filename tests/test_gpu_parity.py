"""GPU <-> oracle parity (``-m gpu``): the CUDA path through the C ABI against the
plain CPU oracle on the same seeded inputs.  Integer work: every comparison is
bit-exact (IC, guide-table splits, masks, CS operations, the set of CSs of every
completed cost level, c*), and the returned regex must be precise under Python's
``re`` with cost exactly c* (SURVEY 8(c) P11)."""
import json
import os
import random

import pytest

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


def gpu_solver(spec, **kw):
    from paper_2305_18575_b200 import Solver
    return Solver.from_spec(spec, **kw)


# ----------------------------------------------------------------- instances

def planted(alpha, tgt, p, n, lo, hi, s, costs=(1, 1, 1, 1, 1)):
    return specgen.gen_planted(alpha, tgt, p, n, lo, hi, s, costs=costs)


SMALL = [
    (specgen.E1, 12),
    (specgen.C1_TOY, 12),
    (specgen.INTRO, 12),
    (specgen.C1_TOY.with_costs((2, 1, 3, 1, 1)), 20),
    (specgen.TABLE1_ROW1, 14),                      # not found below 28: NOT_FOUND path
    (specgen.Spec("abc", ("abc", "c", "ac"), ("a", "bc", "")), 14),
    (specgen.Spec("01", ("0", "00"), ("1", "")), 10),
    (specgen.Spec("0", ("00", "0000"), ("", "0", "000")), 12),   # unary alphabet
    (specgen.Spec("012", ("01", "1"), ("2", "")), 10),            # '2' never in P: still in IC
    (specgen.Spec("01x", ("01", "1"), ("0",)), 10),               # 'x' not in IC: zero seed (A2)
]
RANDOM_W1 = [(specgen.gen_type1("01", 4, 5, 5, s), 20) for s in range(6)] + \
            [(specgen.gen_type2("01", 5, 5, 5, s), 20) for s in range(6)] + \
            [(specgen.gen_type1("01", 4, 5, 5, s, costs=(1, 2, 2, 1, 3)), 30) for s in range(3)] + \
            [(specgen.gen_type1("abc", 3, 5, 5, s), 16) for s in range(3)]
W2 = [(specgen.gen_type1("01", 5, 5, 5, s), 16) for s in (0, 5)] + \
     [(specgen.gen_type2("01", 7, 6, 6, s), 16) for s in (0, 1, 3)]
W4 = [(planted("01", "1(0+11)*0?", 8, 8, 6, 12, 0), 10),
      (planted("01", "(0+1)*11(0+1)*", 8, 8, 6, 12, 0), 14),
      (planted("01", "(01+1)*0", 8, 8, 6, 12, 1), 9)]
W8 = [(planted("abcd", "(ab+c)*d(a+b)?", 6, 6, 6, 14, 0), 13),
      (planted("01", "0(10)*1?", 8, 8, 6, 14, 0), 9),
      (planted("01", "(01+1)*0", 8, 8, 6, 12, 0), 9)]
W16 = [(planted("abcd", "(a+b)*c(a+d)*", 6, 6, 6, 14, 1), 12),
       (planted("abcd", "a(b+c)*d", 6, 6, 8, 16, 0), 9),
       (planted("abcd", "(ab)*(cd)*", 6, 6, 8, 16, 1), 9)]


def ids(cases):
    return [sp.name or f"{sp.alphabet}-{len(sp.P)}-{len(sp.N)}" for sp, _ in cases]


# ------------------------------------------------------------ precompute

@pytest.mark.parametrize("sp,K", SMALL + W2[:2] + W4[:1] + W8[:1] + W16[:1],
                         ids=ids(SMALL + W2[:2] + W4[:1] + W8[:1] + W16[:1]))
def test_precompute_parity(sp, K):
    o = oracle.Oracle.from_spec(sp)
    g = gpu_solver(sp)
    ic = o.ic()
    assert g.ic() == ic
    for w in range(len(ic)):
        want = [(l, r) for (l, r) in o.gt_row(w) if ic[l] and ic[r]]   # proper splits
        assert g.splits(w) == want
    assert g.masks() == o.masks()


@pytest.mark.parametrize("sp", [specgen.TABLE1_ROW1, W2[0][0], W4[0][0], W8[0][0], W16[0][0]],
                         ids=["n25", "w2", "w4", "w8", "w16"])
def test_cs_ops_parity(sp):
    o = oracle.Oracle.from_spec(sp)
    g = gpu_solver(sp)
    n = o.n
    rng = random.Random(99)
    a = [rng.getrandbits(n) & rng.getrandbits(n) for _ in range(200)]
    b = [rng.getrandbits(n) | rng.getrandbits(n) for _ in range(200)]
    a[:4] = [0, 1, (1 << n) - 1, 2]
    assert g.cs_ops(0, a, b) == [o.union(x, y) for x, y in zip(a, b)]
    assert g.cs_ops(1, a, b) == [o.concat(x, y) for x, y in zip(a, b)]
    assert g.cs_ops(2, a) == [o.star(x) for x in a]
    assert g.cs_ops(3, a) == [o.question(x) for x in a]
    assert g.cs_ops(4, a) == [int(o.satisfies(x)) for x in a]


# ------------------------------------------------------------ search parity

def compare_search(sp, K, error=None):
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K, error=error, complete_final_level=True)
    g = gpu_solver(sp, error=error, complete_final_level=True)
    rg = g.solve(K)
    assert rg.status == ro.status
    last = ro.cost if ro.status == "found" else K
    # every level, including c* (complete_final_level): identical sets of CSs
    for c in range(1, last + 1):
        want = o.level_cs(c)
        got = g.level_cs(c)
        assert len(got) == len(want), (c, len(got), len(want))
        assert sorted(got) == sorted(want), c
    go = {l.cost: l for l in rg.levels}
    for l in ro.levels:
        if l.cost in go:
            gl = go[l.cost]
            assert (gl.cand_q, gl.cand_s, gl.cand_c, gl.cand_u) == (l.cand_q, l.cand_s, l.cand_c, l.cand_u)
            assert gl.unique == l.unique
    if ro.status == "found":
        assert rg.cost == ro.cost
        if rg.regex not in ("empty", "eps"):
            if error is None:
                assert precise(rg.regex, sp.P, sp.N), rg.regex
            assert re_cost(parse(rg.regex), sp.costs) == ro.cost
    return o, g, ro, rg


# The small levels of a search run in the device level loop (k_level_loop) by
# default; "host" runs every level through the host loop and the level kernels
# (REI_NO_DEVICE_LOOP), so both paths are held to the oracle.
@pytest.fixture(params=["device_loop", "host_loop"])
def loop_mode(request, monkeypatch):
    if request.param == "host_loop":
        monkeypatch.setenv("REI_NO_DEVICE_LOOP", "1")
    return request.param


@pytest.mark.parametrize("sp,K", SMALL, ids=ids(SMALL))
def test_search_parity_small(sp, K, loop_mode):
    compare_search(sp, K)


@pytest.mark.parametrize("sp,K", RANDOM_W1, ids=ids(RANDOM_W1))
def test_search_parity_random_w1(sp, K, loop_mode):
    compare_search(sp, K)


@pytest.mark.parametrize("sp,K", W2, ids=ids(W2))
def test_search_parity_w2(sp, K, loop_mode):
    compare_search(sp, K)


@pytest.mark.parametrize("sp,K", W4 + W8 + W16, ids=ids(W4 + W8 + W16))
def test_search_parity_wide(sp, K):
    compare_search(sp, K)


@pytest.mark.parametrize("sp,K", W4 + W8, ids=ids(W4 + W8))
def test_indexed_keys_parity(sp, K, monkeypatch):
    # the fingerprint + arena-index hash set (REI_INDEXED_KEYS; the default for |IC| in
    # 65..127 / 129..254 keeps the whole CS in the slot) reaches the same level sets
    monkeypatch.setenv("REI_INDEXED_KEYS", "1")
    compare_search(sp, K)


@pytest.mark.parametrize("sp", [W4[1][0], W8[0][0]], ids=["w4", "w8"])
def test_inline_keys_growth(sp):
    # a small first cache forces growths of the inline-key table (rehash of every entry)
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(12)
    rg = gpu_solver(sp, mem_budget_bytes=48 << 20).solve(12)
    assert rg.status in (ro.status, "out_of_memory")
    if rg.status == ro.status:
        assert rg.cost == ro.cost
    want = {l.cost: l.unique for l in ro.levels}
    got = {l.cost: l.unique for l in rg.levels if l.complete == 1}
    assert got and all(got[c] == want[c] for c in got)


def test_ic_over_512_is_einval_and_device_stays_usable():
    # |IC| > 512 (a binary string of length 57 has ~1.6k infixes) is rejected at rei_init
    # without touching out-of-bounds shared memory; the CUDA context stays usable
    from paper_2305_18575_b200 import ReiError
    rng = random.Random(3)
    long_word = "".join(rng.choice("01") for _ in range(57))
    with pytest.raises(ReiError):
        gpu_solver(specgen.Spec("01", (long_word,), ("0",)))
    sp, K = SMALL[1]
    ro = oracle.Oracle.from_spec(sp).solve(K)
    rg = gpu_solver(sp).solve(K)
    assert (rg.status, rg.cost) == (ro.status, ro.cost)


@pytest.mark.parametrize("sp,K", RANDOM_W1[:4] + RANDOM_W1[12:14] + W2[:1], ids=ids(RANDOM_W1[:4] + RANDOM_W1[12:14] + W2[:1]))
def test_small_cache_parity(sp, K):
    # REI_FLAG_SMALL_CACHE: the cache starts at 2^16 entries and grows; |IC| in 21..32
    # runs on the two-word 64-bit-key hash set instead of the 2^|IC|-bit bitmap
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K, complete_final_level=True)
    g = gpu_solver(sp, complete_final_level=True, small_cache=True)
    rg = g.solve(K)
    assert (rg.status, rg.cost) == (ro.status, ro.cost)
    last = ro.cost if ro.status == "found" else K
    for c in range(1, last + 1):
        assert sorted(g.level_cs(c)) == sorted(o.level_cs(c)), c


@pytest.mark.parametrize("var", ["REI_GENERIC_CONCAT", "REI_GENERIC_UNARY"])
@pytest.mark.parametrize("sp,K", RANDOM_W1[:3] + W2[:2] + W4[:1] + W8[:1],
                         ids=ids(RANDOM_W1[:3] + W2[:2] + W4[:1] + W8[:1]))
def test_generic_kernels_parity(sp, K, var, monkeypatch):
    # the generic (any split count) concat / unary kernels, used when a word has > 15
    # proper splits, exercised on one- and two-word CSs too; on wide CSs the generic
    # unary kernel is the per-thread star (the default is the sliced k_unary_wide)
    monkeypatch.setenv(var, "1")
    compare_search(sp, K)


@pytest.mark.parametrize("order", ["0", "1"])
@pytest.mark.parametrize("conc", ["0", "2", "3", "5"])
@pytest.mark.parametrize("sp,K", RANDOM_W1[:2] + W2[:1], ids=ids(RANDOM_W1[:2] + W2[:1]))
def test_launch_order_and_streams_parity(sp, K, order, conc, monkeypatch):
    # a level's kernels are independent (REI_UNION_FIRST = launch order, REI_CONCURRENT =
    # stream layout): every combination reaches the oracle's level sets, both in the
    # complete-final-level mode and with the early exit
    monkeypatch.setenv("REI_UNION_FIRST", order)
    monkeypatch.setenv("REI_CONCURRENT", conc)
    compare_search(sp, K)
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K)
    rg = gpu_solver(sp).solve(K)
    assert (rg.status, rg.cost) == (ro.status, ro.cost)
    if ro.status == "found" and rg.regex not in ("empty", "eps"):
        assert precise(rg.regex, sp.P, sp.N)


@pytest.mark.parametrize("waves", ["4", "64"])
@pytest.mark.parametrize("sp,K", RANDOM_W1[:2] + W2[:1], ids=ids(RANDOM_W1[:2] + W2[:1]))
def test_concat_waves_parity(sp, K, waves, monkeypatch):
    # concat grids of several waves of CTAs (REI_CONCAT_WAVES) cover the same work items
    monkeypatch.setenv("REI_CONCAT_WAVES", waves)
    compare_search(sp, K)


@pytest.mark.parametrize("sp", [specgen.Spec("01", ("0" * 20, "1"), ("0" * 19, "11")),
                                specgen.Spec("01", ("0" * 40, "1"), ("0" * 39, "11"))],
                         ids=["w1-len20", "w2-len40"])
def test_long_words_use_generic_kernel(sp):
    # words with more than 15 proper splits take the generic concat kernel
    compare_search(sp, 12)


@pytest.mark.parametrize("pct", [50, 45, 40, 35, 25, 20, 15])
def test_allowed_error_parity(pct, loop_mode):
    # Section 5 table rows, REI with allowed error.
    compare_search(specgen.TABLE1_ROW1, 30, error=(pct, 100))


@pytest.mark.parametrize("sp,K", SMALL[:3] + RANDOM_W1[:4] + W2[:2] + W4[:1],
                         ids=ids(SMALL[:3] + RANDOM_W1[:4] + W2[:2] + W4[:1]))
def test_early_exit_mode(sp, K, loop_mode):
    # default mode stops inside level c*: same c*, same complete levels, precise regex
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(K)
    g = gpu_solver(sp)
    rg = g.solve(K)
    assert rg.status == ro.status
    if ro.status == "found":
        assert rg.cost == ro.cost
        assert precise(rg.regex, sp.P, sp.N)
        assert re_cost(parse(rg.regex), sp.costs) == ro.cost
        assert rg.cand_complete == ro.cand_complete
        assert ro.cand_complete <= rg.candidates
    for c in range(1, (ro.cost if ro.status == "found" else K + 1)):
        assert sorted(g.level_cs(c)) == sorted(o.level_cs(c))


def test_reconstruction_audit():
    # every cache entry's reconstructed regex denotes its stored CS.
    sp = specgen.C1_TOY
    g = gpu_solver(sp, complete_final_level=True)
    g.solve(7)
    ic = g.ic()
    idx = {w: i for i, w in enumerate(ic)}
    for c in range(1, 8):
        for i, cs in enumerate(g.level_cs(c)):
            rx = g.entry_regex(c, i)
            assert sum(1 << idx[w] for w in language_on(rx, ic)) == cs
            assert re_cost(parse(rx), sp.costs) == c


def test_trivial_and_invalid():
    from paper_2305_18575_b200 import ReiError, Solver
    r = Solver("01", [], ["0"]).solve(10)
    assert r.status == "found" and r.regex == "empty" and r.cost == 1
    r = Solver("01", [""], ["0"], costs=(3, 1, 1, 1, 1)).solve(10)
    assert r.status == "found" and r.regex == "eps" and r.cost == 3
    with pytest.raises(ReiError):
        Solver("01", ["0"], ["0"])
    with pytest.raises(ReiError):
        Solver("01", ["2"], [])
    with pytest.raises(ReiError):
        Solver("01", ["0"], [], costs=(0, 1, 1, 1, 1))
    r = Solver.from_spec(specgen.TABLE1_ROW1).solve(5)
    assert r.status == "not_found" and r.last_complete_cost == 5


def test_repeated_solve_is_identical():
    g = gpu_solver(specgen.TABLE1_ROW1, complete_final_level=True)
    a = g.solve(16)
    b = g.solve(16)
    assert [l.unique for l in a.levels] == [l.unique for l in b.levels]
    for c in range(1, 17):
        assert sorted(g.level_cs(c)) == sorted(g.level_cs(c))


def test_small_budget_growth_and_oom():
    # the arena starts small and grows by retrying a level; a budget
    # too small for the search reports out_of_memory with the last complete level
    sp = W2[0][0]
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(16)
    g = gpu_solver(sp, mem_budget_bytes=64 << 20)
    rg = g.solve(16)
    assert rg.status == ro.status and rg.cost == ro.cost
    tiny = gpu_solver(sp, mem_budget_bytes=40 << 10)
    rt = tiny.solve(16)
    assert rt.status == "out_of_memory"
    assert 1 <= rt.last_complete_cost < ro.cost


# ------------------------------------------------ full size (BASELINE configs)

def test_table1_row1_full_vs_golden():
    # BASELINE config 5 / Table 1 row 1: c* = 28;
    # per-level unique and candidate counts of levels 1..27 against the oracle's
    # golden file (scripts/make_golden.py, oracle only); launched like bench.py.
    path = os.path.join(GOLDEN, "table1_row1_oracle.json")
    if not os.path.exists(path):
        pytest.skip("golden not generated")
    gold = json.load(open(path))
    sp = specgen.TABLE1_ROW1
    g = gpu_solver(sp)
    r = g.solve(40)
    assert r.status == "found" and r.cost == 28
    assert precise(r.regex, sp.P, sp.N) and re_cost(parse(r.regex), sp.costs) == 28
    want = {l["cost"]: l for l in gold["levels"]}
    for l in r.levels:
        if l.cost < 28:
            w = want[l.cost]
            assert l.unique == w["unique"], l.cost
            assert (l.cand_q, l.cand_s, l.cand_c, l.cand_u) == (w["cand_q"], w["cand_s"], w["cand_c"], w["cand_u"])
    # full final level too
    g2 = gpu_solver(sp, complete_final_level=True)
    r2 = g2.solve(40)
    assert {l.cost: l.unique for l in r2.levels} == {c: w["unique"] for c, w in want.items()}


@pytest.mark.parametrize("cap", [40, 80, 120, 160, 200, 300])
@pytest.mark.parametrize("otf", [True, False])
def test_onthefly_parity(cap, otf, loop_mode):
    # f2: the same cache cap on both sides -> same outcome, same last
    # checked level, same cached level sets below the first OnTheFly level
    sp = specgen.C1_TOY.with_costs((1, 3, 3, 1, 3))
    o = oracle.Oracle.from_spec(sp)
    ro = o.solve(40, max_entries=cap, onthefly=otf)
    first_otf = o.otf_level or 10 ** 9
    g = gpu_solver(sp, max_entries=cap, onthefly=otf)
    rg = g.solve(40)
    assert rg.status == ro.status
    assert rg.last_complete_cost == ro.last_complete_cost
    if ro.status == "found":
        assert rg.cost == ro.cost
        assert precise(rg.regex, sp.P, sp.N)
    for c in range(1, min(first_otf, ro.last_complete_cost + 1)):
        assert sorted(g.level_cs(c)) == sorted(o.level_cs(c)), c


@pytest.mark.parametrize("bits", [None, "25"])
def test_level_sort_mode_parity(monkeypatch, bits):
    # finished bitmap-mode levels (>= 2^14 entries) are reordered by bitmap position
    # (default: top 12 bits; "25": the whole key); level sets, counts and every
    # back-pointer must be unaffected
    if bits:
        monkeypatch.setenv("REI_LEVEL_SORT_BITS", bits)
    sp = specgen.TABLE1_ROW1
    o, g, ro, rg = compare_search(sp, 16)
    assert max(l.unique for l in rg.levels) >= 1 << 14  # some level was sorted
    ic = g.ic()
    idx = {w: i for i, w in enumerate(ic)}
    rnd = random.Random(7)
    for c in (14, 15, 16):  # entries built from sorted operand levels
        cs_list = g.level_cs(c)
        for i in rnd.sample(range(len(cs_list)), 60):
            rx = g.entry_regex(c, i)
            assert sum(1 << idx[w] for w in language_on(rx, ic)) == cs_list[i], (c, i, rx)
            assert re_cost(parse(rx), sp.costs) == c


def test_cached_allocator_reuse_and_release():
    # contexts created after others were destroyed reuse their cached device / pinned
    # blocks (devmem.cu); results must not depend on the blocks' previous contents, and
    # rei_release_cached_memory may run at any time
    from paper_2305_18575_b200 import release_cached_memory
    cases = [(specgen.C1_TOY, 12), (W2[0][0], 16), (specgen.C1_TOY, 12), (W2[0][0], 16)]
    want = {}
    for i, (sp, K) in enumerate(cases):
        g = gpu_solver(sp, complete_final_level=True)
        r = g.solve(K)
        key = sp.name or id(sp)
        sets = [sorted(g.level_cs(c)) for c in range(1, r.cost + 1)]
        if key in want:
            assert (r.cost, sets) == want[key]
        else:
            ro = oracle.Oracle.from_spec(sp).solve(K, complete_final_level=True)
            assert r.cost == ro.cost
            want[key] = (r.cost, sets)
        g.close()
        if i == 1:
            release_cached_memory()


# |IC| = 64 exactly: the all-ones CS (the language of (0+1)*, cost 4 under unit costs)
# equals the empty-slot sentinel of the 64-bit-key hash set and takes its flag path
N64 = [(specgen.gen_type1("01", 7, 5, 5, 3), 11), (specgen.gen_type1("01", 7, 4, 4, 15), 11)]


@pytest.mark.parametrize("sp,K", N64, ids=["t1-le7-s3", "t1-le7-s15"])
def test_ic_64_all_ones_sentinel(sp, K, loop_mode):
    o, g, ro, rg = compare_search(sp, K)
    assert o.n == 64
    ones = (1 << 64) - 1
    assert ones in g.level_cs(4) and ones in o.level_cs(4)
    # nowhere else: the flag makes it a single cached language
    assert sum(l.count(ones) for l in (g.level_cs(c) for c in range(1, K + 1))) == 1
