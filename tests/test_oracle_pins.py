"""Pins of the CPU oracle to the paper and to mathematics (``-m "not gpu"``).

Each test names the passage it pins (P:n = PAPER.md line n).  None of them
re-derives an expected value from the oracle itself: expected values are the
paper's printed ones, results of an independent matcher (Python ``re``) or of
brute-force enumeration of syntactic regexes, closed forms, or laws.
"""
import json
import os
import random

import pytest

import oracle
import specgen
from regex_tools import (brute_force_levels, cost, enumerate_trees, infixes, language_on,
                         parse, precise, to_python_re)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def bits_of(o, words):
    idx = {w: i for i, w in enumerate(o.ic())}
    return sum(1 << idx[w] for w in words)


def sym(o, a):
    return bits_of(o, [a]) if a in o.ic() else 0


# ------------------------------------------------------------- P1: E1

def test_e1_infix_closure_is_papers_listing():
    # P:661-676 lists IC(P u N) for example_standard_1 (15 words).
    paper = {"11011", "1101", "110", "11", "1011", "101", "10", "1", "011", "01",
             "0011", "001", "00", "0", ""}
    o = oracle.Oracle.from_spec(specgen.E1)
    assert set(o.ic()) == paper and o.n == 15


def test_e1_guide_table_figure_indices():
    # word "110" sits at index 10; split "11"."0" is entry (6, 1).
    o = oracle.Oracle.from_spec(specgen.E1)
    ic = o.ic()
    assert ic[10] == "110" and ic[6] == "11" and ic[1] == "0"
    assert (6, 1) in o.gt_row(10)
    # every gt row lists exactly the |w|+1 splits of w
    for w, word in enumerate(ic):
        row = o.gt_row(w)
        assert sorted(ic[l] + "|" + ic[r] for l, r in row) == \
            sorted(word[:k] + "|" + word[k:] for k in range(len(word) + 1))


def test_e1_cs_of_example_regex():
    # L((0?1)*1) cap IC = {11011, 1011, 011, 11, 1}; built with the
    # oracle's IPS ops from the symbol CSs.
    o = oracle.Oracle.from_spec(specgen.E1)
    s0, s1 = sym(o, "0"), sym(o, "1")
    cs = o.concat(o.star(o.concat(o.question(s0), s1)), s1)
    assert cs == bits_of(o, ["11011", "1011", "011", "11", "1"])
    assert o.satisfies(cs)


def test_e1_minimal_cost_is_7():
    # (0?1)*1 is minimal under (1,1,1,1,1); its cost is 7.
    assert cost(parse("(0?1)*1"), (1, 1, 1, 1, 1)) == 7
    r = oracle.solve_spec(specgen.E1, 30)
    assert r.status == "found" and r.cost == 7
    assert precise(r.regex, specgen.E1.P, specgen.E1.N)
    assert cost(parse(r.regex), (1, 1, 1, 1, 1)) == 7


def test_spec_worked_ops_on_e1():
    # P10: CS{1}.CS{10} = {110}; CS(0)* = {eps,0,00}; CS{1}? = {eps,1}.
    o = oracle.Oracle.from_spec(specgen.E1)
    ten = bits_of(o, ["10"])
    assert o.concat(sym(o, "1"), ten) == bits_of(o, ["110"])
    assert o.star(sym(o, "0")) == bits_of(o, ["", "0", "00"])
    assert o.question(sym(o, "1")) == bits_of(o, ["", "1"])


# ---------------------------------------------------------- P3: intro

def test_intro_example():
    # the intro spec "should, ideally, lead to" 10(0+1)*, cost 8.
    sp = specgen.INTRO
    r = oracle.solve_spec(sp, 30)
    assert r.status == "found"
    assert cost(parse("10(0+1)*"), sp.costs) == 8 == r.cost
    assert precise(r.regex, sp.P, sp.N)
    words = infixes(sp.P + sp.N)
    assert language_on(r.regex, words) == language_on("10(0+1)*", words)


# ------------------------------------------- P5: Table 1 row 1 / Section 5

def test_table1_row1_paper_regex_is_precise_with_cost_28():
    # P:1779-1782 spec, P:1798 regex and cost: pins our reading of the spec.
    sp = specgen.TABLE1_ROW1
    rx = "10?+0?(00+10*10?(0+1))1?"
    assert precise(rx, sp.P, sp.N)
    assert cost(parse(rx), (1, 1, 1, 1, 1)) == 28


def test_table1_row1_no_precise_language_below_17():
    # Part of P:1798's minimality claim (c* = 28) that is cheap on CPU.
    r = oracle.solve_spec(specgen.TABLE1_ROW1, 16)
    assert r.status == "not_found"


@pytest.mark.parametrize("pct,paper_cost,paper_regex", [
    (50, 1, "empty"), (45, 1, "1"), (40, 4, "10?"), (35, 7, "1+(0+1)0"),
    (30, 8, "(0+11)*1"), (25, 8, "(0+11)*1"), (20, 12, "(0+11)*(1+00)"),
    (15, 14, "(0+1)0+(0+11)*1"),
])
def test_allowed_error_table(pct, paper_cost, paper_regex):
    # Section 5 table: with Q->S->C->U order the oracle returns the
    # paper's regex text, not just its cost; cost and text are the paper's.
    sp = specgen.TABLE1_ROW1
    r = oracle.solve_spec(sp, 40, error=(pct, 100))
    assert r.status == "found"
    assert r.cost == paper_cost
    assert r.regex == paper_regex
    if paper_regex != "empty":
        assert cost(parse(paper_regex), (1, 1, 1, 1, 1)) == paper_cost


def test_allowed_error_table_paper_counts_bracket():
    # Reading A9: the paper's |REs| lies between our cumulative count before and
    # after the level that holds the solution.
    sp = specgen.TABLE1_ROW1
    paper = {50: 1, 45: 3, 40: 50, 35: 1124, 25: 2073, 20: 116912, 15: 794598}
    for pct, reps in paper.items():
        r = oracle.solve_spec(sp, 40, error=(pct, 100), complete_final_level=True)
        before = r.cand_complete if r.levels and not r.levels[-1].complete else None
        # cumulative counts through the level before c* and through c*
        cum, prev = 1 + len(sp.alphabet), None
        for l in r.levels:
            if l.cost == r.cost:
                prev = cum
                cum += l.cand
                break
            cum += l.cand
        if r.cost <= 1:
            assert reps <= 1 + len(sp.alphabet)
            continue
        assert prev <= reps <= cum, (pct, prev, reps, cum)
        del before


# ------------------------------------------------ P2: brute force

BRUTE_CASES = [
    (specgen.E1, (1, 1, 1, 1, 1), 7),
    (specgen.C1_TOY, (1, 1, 1, 1, 1), 6),
    (specgen.C1_TOY, (2, 1, 3, 1, 1), 8),
    (specgen.Spec("01", ("0", "00"), ("1", "")), (1, 1, 1, 1, 1), 7),
    (specgen.Spec("ab", ("ab", "ba", "aa"), ("b", "bb", "")), (1, 1, 1, 1, 1), 7),
    (specgen.Spec("abc", ("abc", "c", "ac"), ("a", "bc", "")), (1, 2, 1, 1, 2), 7),
    # reading A2: symbol c occurs in no example, so its seed is the empty language
    # (the brute force matches `c` against IC and finds nothing); it changes the counts
    (specgen.Spec("abc", ("ab", "ba", "aa"), ("b", "bb", "")), (1, 1, 1, 1, 1), 6),
    (specgen.Spec("abc", ("a", "aa", "ab"), ("b", "", "ba")), (1, 1, 1, 1, 1), 6),
]


@pytest.mark.parametrize("sp,costs,K", BRUTE_CASES)
def test_brute_force_level_histogram(sp, costs, K):
    # The method reaches exactly the plain definition: the number
    # of IC-languages whose cheapest syntactic regex costs c equals the oracle's
    # unique count at level c; the least precise cost equals c*.
    hist, cstar, words = brute_force_levels(sp.alphabet, sp.P, sp.N, costs, K)
    o = oracle.Oracle(sp.alphabet, sp.P, sp.N, costs)
    assert sorted(o.ic(), key=lambda s: (len(s), s)) == words or set(o.ic()) == set(words)
    r = o.solve(K, complete_final_level=True)
    got = {l.cost: l.unique for l in r.levels if l.unique}
    want = {c: h for c, h in hist.items() if c <= (r.cost if r.status == "found" else K)}
    got = {c: u for c, u in got.items() if c <= (r.cost if r.status == "found" else K)}
    assert got == want
    if cstar is not None:
        assert r.status == "found" and r.cost == cstar
    else:
        assert r.status == "not_found"


def test_enumerator_counts():
    # binary alphabet, unit costs: 2 / 4 / 16 trees at cost 1/2/3.
    t = enumerate_trees("01", (1, 1, 1, 1, 1), 3)
    assert [len(t[c]) for c in (1, 2, 3)] == [2, 4, 16]


# ------------------------------------- language-restriction homomorphism

def _random_tree(rng, alphabet, depth):
    if depth == 0 or rng.random() < 0.25:
        return ("sym", rng.choice(alphabet))
    k = rng.choice("?*.+.+")
    if k in "?*":
        return (k, _random_tree(rng, alphabet, depth - 1))
    return (k, _random_tree(rng, alphabet, depth - 1), _random_tree(rng, alphabet, depth - 1))


@pytest.mark.parametrize("sp", [specgen.E1, specgen.C1_TOY, specgen.TABLE1_ROW1,
                                specgen.Spec("abc", ("abcab", "cc", "bca"), ("a", "cab", ""))])
def test_ops_agree_with_re_matcher(sp):
    # IC is infix-closed, so CS(r.s) = CS(r).CS(s), CS(r*) = CS(r)*, etc.
    # (P:616-648).  The right-hand sides come from Python re.
    o = oracle.Oracle.from_spec(sp)
    ic = o.ic()
    idx = {w: i for i, w in enumerate(ic)}
    import re as _re

    def cs_re(tree):
        pat = _re.compile(to_python_re(tree))
        return sum(1 << idx[w] for w in ic if pat.fullmatch(w))

    rng = random.Random(1234)
    for _ in range(300):
        a = _random_tree(rng, sp.alphabet, 3)
        b = _random_tree(rng, sp.alphabet, 3)
        A, B = cs_re(a), cs_re(b)
        assert o.union(A, B) == cs_re(("+", a, b))
        assert o.concat(A, B) == cs_re((".", a, b))
        assert o.star(A) == cs_re(("*", a))
        assert o.question(A) == cs_re(("?", a))


def test_semiring_laws_on_random_cs():
    # (B, v, ^, 0, 1) lifted to IPS: laws on random CSs.
    o = oracle.Oracle.from_spec(specgen.TABLE1_ROW1)
    n = o.n
    one = 1  # eps is word 0 (shortlex)
    rng = random.Random(7)
    for _ in range(500):
        a, b, c = (rng.getrandbits(n) for _ in range(3))
        assert o.concat(a, one) == a == o.concat(one, a)
        assert o.concat(a, 0) == 0 == o.concat(0, a)
        assert o.concat(o.concat(a, b), c) == o.concat(a, o.concat(b, c))
        assert o.concat(a, o.union(b, c)) == o.union(o.concat(a, b), o.concat(a, c))
        assert o.concat(o.union(a, b), c) == o.union(o.concat(a, c), o.concat(b, c))
        s = o.star(a)
        assert s == o.union(one, o.concat(a, s))        # r* = 1 + r r*
        assert o.star(s) == s
        assert o.question(a) == o.union(one, a)


# --------------------------------------------------- P7 / P12 invariants

def overfit_cost(P, costs):
    c1, c2, c3, c4, c5 = costs
    ws = [w for w in P if w]
    total = sum(len(w) * c1 + (len(w) - 1) * c4 for w in ws) + (len(ws) - 1) * c5
    return total + (c2 if "" in P else 0)


@pytest.mark.parametrize("seed", range(12))
def test_random_specs_invariants(seed):
    # search ends no later than the overfit union's cost; the found
    # regex is precise under re and has cost c* (P:474-477); level
    # candidate counts follow reading A9 from level sizes; total uniques <= 2^n.
    sp = specgen.gen_type1("01", 4, 5, 5, seed) if seed % 2 else specgen.gen_type2("01", 4, 5, 5, seed)
    costs = [(1, 1, 1, 1, 1), (2, 1, 3, 1, 1), (1, 2, 2, 1, 3)][seed % 3]
    o = oracle.Oracle(sp.alphabet, sp.P, sp.N, costs)
    bound = overfit_cost(sp.P, costs)
    r = o.solve(bound, complete_final_level=True)
    assert r.status == "found" and r.cost <= bound
    assert precise(r.regex, sp.P, sp.N)
    assert cost(parse(r.regex), costs) == r.cost
    sizes = {l.cost: l.unique for l in r.levels}
    c1, c2, c3, c4, c5 = costs
    for l in r.levels:
        if l.cost == c1:
            continue
        c = l.cost
        assert l.cand_q == sizes.get(c - c2, 0)
        assert l.cand_s == sizes.get(c - c3, 0)
        assert l.cand_c == sum(sizes.get(L, 0) * sizes.get(c - c4 - L, 0) for L in range(1, c))
        exp_u = 0
        for L in range(1, c):
            R = c - c5 - L
            if L < R:
                exp_u += sizes.get(L, 0) * sizes.get(R, 0)
            elif L == R:
                exp_u += sizes.get(L, 0) * (sizes.get(L, 0) - 1) // 2
        assert l.cand_u == exp_u
    assert sum(sizes.values()) <= 2 ** o.n


def test_reconstruction_audit_e1():
    # every cache entry's reconstructed regex denotes exactly the
    # stored CS (checked with re) and has cost equal to its level.
    sp = specgen.E1
    o = oracle.Oracle.from_spec(sp)
    o.solve(7, complete_final_level=True)
    ic = o.ic()
    for c in range(1, 8):
        for i, cs in enumerate(o.level_cs(c)):
            rx = o.entry_regex(c, i)
            lang = language_on(rx, ic)
            assert sum(1 << ic.index(w) for w in lang) == cs
            assert cost(parse(rx), sp.costs) == c


def test_trivial_cases():
    # Alg. 1 lines 1-2.
    r = oracle.Oracle("01", [], ["0"]).solve(10)
    assert r.status == "found" and r.regex == "empty" and r.cost == 1
    r = oracle.Oracle("01", [""], ["0"], (3, 1, 1, 1, 1)).solve(10)
    assert r.status == "found" and r.regex == "eps" and r.cost == 3


def test_validation_errors():
    with pytest.raises(ValueError):
        oracle.Oracle("01", ["0"], ["0"])
    with pytest.raises(ValueError):
        oracle.Oracle("01", ["2"], [])
    with pytest.raises(ValueError):
        oracle.Oracle("01", ["0"], [], (0, 1, 1, 1, 1))


def test_golden_table1_row1_if_present():
    # Written by scripts/make_golden.py (oracle only): c* = 28.
    path = os.path.join(GOLDEN, "table1_row1_oracle.json")
    if not os.path.exists(path):
        pytest.skip("golden not generated yet")
    g = json.load(open(path))
    assert g["cstar"] == 28 and g["status"] == "found"
    assert precise(g["regex"], specgen.TABLE1_ROW1.P, specgen.TABLE1_ROW1.N)
    assert cost(parse(g["regex"]), (1, 1, 1, 1, 1)) == 28
    # the paper's |REs| is bracketed by our counts before/after level 28
    cum = 1 + 2
    for l in g["levels"]:
        if l["cost"] == 28:
            lo = cum
        cum += l["cand_q"] + l["cand_s"] + l["cand_c"] + l["cand_u"]
    assert lo <= 26774099142 <= cum


# ------------------------------------------------------ f2: OnTheFly mode

@pytest.mark.parametrize("cap", [40, 80, 120, 160, 200, 300, 10 ** 6])
def test_onthefly_keeps_minimality(cap):
    # OnTheFly continues from cached levels "without compromising on
    # minimality and precision"; when it needs an uncached level it stops (OOM).
    sp = specgen.C1_TOY.with_costs((1, 3, 3, 1, 3))
    o = oracle.Oracle.from_spec(sp)
    full = o.solve(40)
    r = o.solve(40, max_entries=cap, onthefly=True)
    if r.status == "found":
        assert r.cost == full.cost
        assert precise(r.regex, sp.P, sp.N)
    else:
        assert r.status == "out_of_memory"
    plain = o.solve(40, max_entries=cap, onthefly=False)
    assert plain.status in ("found", "out_of_memory")
    # OnTheFly checks at least as many levels as the plain cache-limited search
    assert r.last_complete_cost >= plain.last_complete_cost
    if cap >= 10 ** 6:
        assert r.status == plain.status == "found" and o.otf_level == 0
