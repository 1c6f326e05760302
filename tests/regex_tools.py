"""Independent regex utilities for the tests (no CS bitvectors anywhere).

* ``parse``: the paper's concrete syntax (union ``+``, juxtaposition for
  concatenation, postfix ``?`` and ``*``; ``empty``/``eps`` for the trivial
  answers) into a tuple AST.
* ``cost``: the cost homomorphism on that AST.
* ``to_python_re`` / ``matches``: membership by Python's ``re`` engine, a
  matcher that knows nothing about infix closures or guide tables.
* ``enumerate_trees``: brute-force enumeration of every syntactic regex in
  RE+ (symbols closed under ?, *, concatenation, union; reading A4) by exact
  cost, used to pin the oracle's per-level unique counts (pin P2).
"""
from __future__ import annotations

import functools
import re
from typing import Dict, Iterable, List, Sequence, Tuple


def parse(r: str):
    if r == "empty":
        return ("empty",)
    if r == "eps":
        return ("eps",)
    pos = 0

    def peek():
        return r[pos] if pos < len(r) else None

    def union():
        nonlocal pos
        node = concat()
        while peek() == "+":
            pos += 1
            node = ("+", node, concat())
        return node

    def concat():
        node = postfix()
        while peek() is not None and peek() not in "+)":
            node = (".", node, postfix())
        return node

    def postfix():
        nonlocal pos
        node = atom()
        while peek() is not None and peek() in "*?":
            node = (peek(), node)
            pos += 1
        return node

    def atom():
        nonlocal pos
        c = peek()
        if c == "(":
            pos += 1
            node = union()
            if peek() != ")":
                raise ValueError(f"unbalanced: {r!r}")
            pos += 1
            return node
        if c is None or c in "+)*?":
            raise ValueError(f"unexpected {c!r} in {r!r}")
        pos += 1
        return ("sym", c)

    tree = union()
    if pos != len(r):
        raise ValueError(f"trailing input in {r!r}")
    return tree


def cost(tree, costs: Sequence[int]) -> int:
    c1, c2, c3, c4, c5 = costs
    k = tree[0]
    if k in ("sym", "empty", "eps"):
        return c1
    if k == "?":
        return cost(tree[1], costs) + c2
    if k == "*":
        return cost(tree[1], costs) + c3
    if k == ".":
        return cost(tree[1], costs) + cost(tree[2], costs) + c4
    if k == "+":
        return cost(tree[1], costs) + cost(tree[2], costs) + c5
    raise ValueError(k)


def to_python_re(tree) -> str:
    k = tree[0]
    if k == "sym":
        return re.escape(tree[1])
    if k == "eps":
        return "(?:)"
    if k == "empty":
        return "(?!)"
    if k in "?*":
        return "(?:" + to_python_re(tree[1]) + ")" + k
    if k == ".":
        return "(?:" + to_python_re(tree[1]) + to_python_re(tree[2]) + ")"
    if k == "+":
        return "(?:" + to_python_re(tree[1]) + "|" + to_python_re(tree[2]) + ")"
    raise ValueError(k)


@functools.lru_cache(maxsize=1 << 16)
def _compiled(pattern: str):
    return re.compile(pattern)


def matches(regex: str, word: str) -> bool:
    return _compiled(to_python_re(parse(regex))).fullmatch(word) is not None


def language_on(regex: str, words: Sequence[str]) -> frozenset:
    pat = _compiled(to_python_re(parse(regex)))
    return frozenset(w for w in words if pat.fullmatch(w) is not None)


def precise(regex: str, P: Iterable[str], N: Iterable[str]) -> bool:
    pat = _compiled(to_python_re(parse(regex)))
    return all(pat.fullmatch(p) for p in P) and not any(pat.fullmatch(q) for q in N)


def infixes(words: Iterable[str]) -> List[str]:
    """All infixes of the given words (plain set comprehension, unordered)."""
    out = set()
    for w in words:
        for i in range(len(w) + 1):
            for j in range(i, len(w) + 1):
                out.add(w[i:j])
    return sorted(out, key=lambda s: (len(s), s))


def enumerate_trees(alphabet: str, costs: Sequence[int], max_cost: int) -> Dict[int, List]:
    """Every syntactic regex of RE+ with cost exactly c, for c <= max_cost."""
    c1, c2, c3, c4, c5 = costs
    by_cost: Dict[int, List] = {c: [] for c in range(1, max_cost + 1)}
    for c in range(1, max_cost + 1):
        out = by_cost[c]
        if c == c1:
            out.extend(("sym", a) for a in alphabet)
        if c - c2 >= 1:
            out.extend(("?", t) for t in by_cost[c - c2])
        if c - c3 >= 1:
            out.extend(("*", t) for t in by_cost[c - c3])
        for L in range(1, c - c4):
            R = c - c4 - L
            if R >= 1:
                out.extend((".", a, b) for a in by_cost[L] for b in by_cost[R])
        for L in range(1, c - c5):
            R = c - c5 - L
            if R >= 1:
                out.extend(("+", a, b) for a in by_cost[L] for b in by_cost[R])
    return by_cost


def brute_force_levels(alphabet: str, P: Sequence[str], N: Sequence[str],
                       costs: Sequence[int], max_cost: int):
    """Per-cost histogram of IC-languages by the cost of their cheapest tree.

    Returns (hist, cstar): hist[c] = number of distinct languages L(r) cap IC
    whose cheapest syntactic regex costs exactly c; cstar = the least cost of
    a tree whose language satisfies (P, N) (None if above max_cost).
    """
    words = infixes(list(P) + list(N))
    trees = enumerate_trees(alphabet, costs, max_cost)
    best: Dict[frozenset, int] = {}
    cstar = None
    Pset, Nset = set(P), set(N)
    for c in range(1, max_cost + 1):
        for t in trees[c]:
            pat = _compiled(to_python_re(t))
            lang = frozenset(w for w in words if pat.fullmatch(w) is not None)
            if lang not in best:
                best[lang] = c
            if cstar is None and Pset <= lang and not (Nset & lang):
                cstar = c
    hist: Dict[int, int] = {}
    for lang, c in best.items():
        hist[c] = hist.get(c, 0) + 1
    return hist, cstar, words
