"""Seeded synthetic REI specifications (inputs only; no method arithmetic).

This module is shared by the oracle tests, the CUDA-path tests and bench.py.
It contains NONE of the method's arithmetic (no infix closure, no CS, no
guide table, no search): only random-number generation, the paper's two
benchmark sampling schemes, a planted-target scheme, the named fixed specs
the paper prints, and the spec-file format.

Citations: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n.

* SplitMix64: seed 0 -> first output 0xE220A8397B1DCDAF.
* Type 1: p+n distinct strings drawn uniformly from
  Sigma^{<=le}; the first p go to P (union sampled first, then split).
* Type 2: a uniform length per slot, then a uniform
  string of that length not already used by the same polarity and not used by
  the opposite polarity at that length (P_i cap N_i = empty).
* Planted (not in the paper): P sampled from the
  language of a target regex, N sampled from its complement, so that wide-IC
  instances stay solvable (c* <= cost(target)).
"""
from __future__ import annotations

import dataclasses
import re
from typing import List, Optional, Sequence, Tuple

MASK64 = (1 << 64) - 1


class SplitMix64:
    """SplitMix64. Public-domain recurrence, fixed constants."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def below(self, bound: int) -> int:
        """Uniform integer in [0, bound) by rejection (no modulo bias)."""
        if bound <= 0:
            raise ValueError("bound must be positive")
        limit = (1 << 64) - ((1 << 64) % bound)
        while True:
            x = self.next()
            if x < limit:
                return x % bound

    def uniform(self) -> float:
        return (self.next() >> 11) / float(1 << 53)


@dataclasses.dataclass(frozen=True)
class Spec:
    """A specification (P, N) over an explicit alphabet.

    ``alphabet`` is the ordered symbol string (its order lifts to the shortlex
    order); ``""`` denotes epsilon.  ``costs`` is the cost
    homomorphism (c1..c5) = (sym, ?, *, concat, union).
    """

    alphabet: str
    P: Tuple[str, ...]
    N: Tuple[str, ...]
    costs: Tuple[int, int, int, int, int] = (1, 1, 1, 1, 1)
    name: str = ""

    def with_costs(self, costs: Sequence[int], name: Optional[str] = None) -> "Spec":
        return dataclasses.replace(self, costs=tuple(int(c) for c in costs),
                                   name=self.name if name is None else name)


class InfeasibleParams(ValueError):
    pass


# ---------------------------------------------------------------- sampling


def _count_upto(k: int, le: int) -> int:
    """|Sigma^{<=le}| for |Sigma| = k."""
    return le + 1 if k == 1 else (k ** (le + 1) - 1) // (k - 1)


def _unrank_shortlex(alphabet: str, rank: int) -> str:
    """The rank-th string of Sigma^* in shortlex order (rank 0 = epsilon)."""
    k = len(alphabet)
    length = 0
    block = 1
    while rank >= block:
        rank -= block
        length += 1
        block *= k
    digits = []
    for _ in range(length):
        digits.append(alphabet[rank % k])
        rank //= k
    return "".join(reversed(digits))


def gen_type1(alphabet: str, le: int, p: int, n: int, seed: int,
              costs=(1, 1, 1, 1, 1)) -> Spec:
    """Type 1: p+n distinct strings uniform over Sigma^{<=le}."""
    total = _count_upto(len(alphabet), le)
    if p + n > total:
        raise InfeasibleParams(f"p+n={p + n} > |Sigma^<={le}|={total}")
    rng = SplitMix64(seed)
    chosen: List[int] = []
    used = set()
    while len(chosen) < p + n:
        r = rng.below(total)
        if r not in used:
            used.add(r)
            chosen.append(r)
    words = [_unrank_shortlex(alphabet, r) for r in chosen]
    return Spec(alphabet, tuple(words[:p]), tuple(words[p:]), tuple(costs),
                f"type1-k{len(alphabet)}-le{le}-p{p}-n{n}-s{seed}")


def gen_type2(alphabet: str, le: int, p: int, n: int, seed: int,
              costs=(1, 1, 1, 1, 1), max_attempts: int = 10 ** 6) -> Spec:
    """Type 2: uniform length per slot, per-length disjointness."""
    rng = SplitMix64(seed)
    k = len(alphabet)
    P: List[str] = []
    N: List[str] = []
    Ps, Ns = set(), set()
    attempts = 0
    for pol in [0] * p + [1] * n:
        while True:
            attempts += 1
            if attempts > max_attempts:
                raise InfeasibleParams("Type 2 resample limit exceeded")
            length = rng.below(le + 1)
            idx = rng.below(k ** length) if length else 0
            digits = []
            for _ in range(length):
                digits.append(alphabet[idx % k])
                idx //= k
            w = "".join(reversed(digits))
            mine, other = (Ps, Ns) if pol == 0 else (Ns, Ps)
            if w in mine or w in other:
                continue
            mine.add(w)
            (P if pol == 0 else N).append(w)
            break
    return Spec(alphabet, tuple(P), tuple(N), tuple(costs),
                f"type2-k{k}-le{le}-p{p}-n{n}-s{seed}")


# ------------------------------------------------ planted-target generator


def _regex_to_python(r: str) -> str:
    """Paper regex syntax (union '+', postfix '?', '*') -> Python re syntax."""
    return r.replace("+", "|")


def _parse(r: str):
    """Tiny recursive-descent parser of the paper's regex syntax into tuples."""
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
            assert peek() == ")", r
            pos += 1
            return node
        pos += 1
        return ("sym", c)

    tree = union()
    assert pos == len(r), r
    return tree


def _sample_from(tree, rng: SplitMix64, star_p: float = 0.55, depth: int = 0) -> str:
    kind = tree[0]
    if kind == "sym":
        return tree[1]
    if kind == ".":
        return _sample_from(tree[1], rng, star_p, depth) + _sample_from(tree[2], rng, star_p, depth)
    if kind == "+":
        return _sample_from(tree[1 + rng.below(2)], rng, star_p, depth)
    if kind == "?":
        return _sample_from(tree[1], rng, star_p, depth) if rng.below(2) else ""
    if kind == "*":
        out = []
        while rng.uniform() < star_p and len(out) < 32:
            out.append(_sample_from(tree[1], rng, star_p, depth + 1))
        return "".join(out)
    raise ValueError(kind)


def gen_planted(alphabet: str, target: str, p: int, n: int, lo: int, hi: int,
                seed: int, costs=(1, 1, 1, 1, 1), n_lo: int = 0,
                max_attempts: int = 2 * 10 ** 6) -> Spec:
    """Planted target (DESIGN.md input recipe; not in the paper).

    P: p distinct strings of L(target) with length in [lo, hi] (sampled from
    the regex tree, rejection on length).  N: n distinct strings of length in
    [n_lo, hi] drawn uniformly per length and rejected if in L(target).
    """
    tree = _parse(target)
    pat = re.compile(_regex_to_python(target))
    rng = SplitMix64(seed)
    P: List[str] = []
    seen = set()
    attempts = 0
    while len(P) < p:
        attempts += 1
        if attempts > max_attempts:
            raise InfeasibleParams("planted: not enough positive strings")
        w = _sample_from(tree, rng)
        if lo <= len(w) <= hi and w not in seen:
            seen.add(w)
            P.append(w)
    N: List[str] = []
    k = len(alphabet)
    while len(N) < n:
        attempts += 1
        if attempts > max_attempts:
            raise InfeasibleParams("planted: not enough negative strings")
        length = n_lo + rng.below(hi - n_lo + 1)
        w = "".join(alphabet[rng.below(k)] for _ in range(length))
        if w in seen or pat.fullmatch(w):
            continue
        seen.add(w)
        N.append(w)
    return Spec(alphabet, tuple(P), tuple(N), tuple(costs),
                f"planted-{target}-p{p}-n{n}-L{lo}-{hi}-s{seed}")


# ------------------------------------------------------------ fixed specs

# Example `example_standard_1`.
E1 = Spec("01", ("1", "011", "1011", "11011"), ("", "10", "101", "0011"), name="E1")

# Introduction example.
INTRO = Spec("01", ("10", "101", "100", "1010", "1011", "1000", "1001"),
             ("", "0", "1", "00", "11", "010"), name="intro")

# BASELINE.json configs[0]: the paper-style toy.
C1_TOY = Spec("01", ("10", "100", "101", "1010", "1011"),
              ("", "0", "1", "01", "11", "001"), name="C1-toy")

# Table 1 row 1 (Type 1 no. 50) = the Section 5 spec.
TABLE1_ROW1 = Spec("01",
                   ("00", "1101", "0001", "0111", "001", "1", "10", "1100", "111", "1010"),
                   ("", "0", "0000", "0011", "01", "010", "011", "100", "1000", "1001", "11", "1110"),
                   name="table1-row1")

# Table 1 row 8: same spec, cost function (10,10,10,1,10).
TABLE1_ROW8 = TABLE1_ROW1.with_costs((10, 10, 10, 1, 10), name="table1-row8")


def c2_instances(count: int = 8, seed0: int = 0, le: int = 6, p: int = 10, n: int = 10,
                 max_ic: int = 64, ic_size=None) -> List[Spec]:
    """BASELINE configs[1]: Type 1 binary, le<=6, p=n=10, IC fits one u64.

    ``ic_size`` is a callable returning |IC| (supplied by the caller from
    either side; this module does not compute infix closures itself).
    """
    out = []
    s = seed0
    while len(out) < count:
        sp = gen_type1("01", le, p, n, s)
        s += 1
        if ic_size is not None and ic_size(sp) > max_ic:
            continue
        out.append(sp)
    return out


# The many-small-specifications suite, after the paper's benchmark
# suites (Type 1 with p, n in 8..12; Type 2 with p, n in 7..14; binary;
# 12 cost functions).  Lengths are capped (le = 4, |IC| <= 31) so that
# every spec is a small, latency-bound search; the cost functions rotate through the
# paper's single-expensive-constructor family.
SUITE_COSTS = [(1, 1, 1, 1, 1), (1, 1, 10, 1, 1), (1, 10, 1, 1, 1), (1, 1, 1, 10, 1),
               (10, 1, 1, 1, 1), (1, 1, 1, 1, 10)]


def suite_f4(count: int = 1024, seed0: int = 0) -> List[Spec]:
    """`count` seeded specs: alternately Type 1 (le 4, p, n in 8..12) and Type 2
    (le 4, p, n in 7..14), cost functions from SUITE_COSTS.  Infeasible draws are
    skipped."""
    rng = SplitMix64(seed0 ^ 0x5EED5)
    out: List[Spec] = []
    i = 0
    while len(out) < count:
        costs = SUITE_COSTS[i % len(SUITE_COSTS)]
        le = 4
        try:
            if i % 2 == 0:
                sp = gen_type1("01", le, 8 + rng.below(5), 8 + rng.below(5), seed0 + i, costs=costs)
            else:
                sp = gen_type2("01", le, 7 + rng.below(8), 7 + rng.below(8), seed0 + i, costs=costs)
            out.append(sp)
        except InfeasibleParams:
            pass
        i += 1
    return out


# Planted wide-IC instances (BASELINE configs[2], configs[3]); parameters fixed
# here so every side regenerates byte-identical specs.
C3_PLANTED = [
    ("01", "1(0+11)*0?", 10, 10, 6, 12, s) for s in range(8)
]
C4_PLANTED = [
    ("abcd", "(ab+c)*d(a+b)?", 10, 10, 6, 14, s) for s in range(4)
] + [
    ("abcd", "(a+b)*c(a+d)*", 10, 10, 6, 14, s) for s in range(4)
]


# ------------------------------------------------------------- spec files


def write_spec(spec: Spec) -> str:
    """Spec file format: '+w' / '-w' lines, '#' comments."""
    lines = [f"# {spec.name}", f"# alphabet {spec.alphabet}",
             "# costs " + ",".join(map(str, spec.costs))]
    lines += ["+" + w for w in spec.P]
    lines += ["-" + w for w in spec.N]
    return "\n".join(lines) + "\n"


def read_spec(text: str, alphabet: Optional[str] = None,
              costs=(1, 1, 1, 1, 1), name: str = "") -> Spec:
    P, N = [], []
    for line in text.splitlines():
        if line.startswith("# alphabet ") and alphabet is None:
            alphabet = line[len("# alphabet "):]
            continue
        if line.startswith("# costs "):
            costs = tuple(int(x) for x in line[len("# costs "):].split(","))
            continue
        if not line or line.startswith("#"):
            continue
        if line[0] == "+":
            P.append(line[1:])
        elif line[0] == "-":
            N.append(line[1:])
        else:
            raise ValueError(f"bad spec line {line!r}")
    if alphabet is None:
        alphabet = "".join(sorted(set("".join(P + N))))
    return Spec(alphabet, tuple(P), tuple(N), tuple(costs), name)


def spec_alphabet_from_examples(P: Sequence[str], N: Sequence[str]) -> str:
    """Sigma = symbols of P cup N in sorted order (A2 reading)."""
    return "".join(sorted(set("".join(list(P) + list(N)))))
