"""Input generators (specgen): determinism and the paper's sampling shapes."""
import specgen


def test_splitmix64_seed0():
    # seed 0 -> first output 0xE220A8397B1DCDAF (published recurrence).
    assert specgen.SplitMix64(0).next() == 0xE220A8397B1DCDAF
    assert specgen.SplitMix64(1).next() != specgen.SplitMix64(2).next()


def test_type1_shape_and_determinism():
    a = specgen.gen_type1("01", 6, 10, 10, 3)
    b = specgen.gen_type1("01", 6, 10, 10, 3)
    assert a == b
    assert len(a.P) == 10 and len(a.N) == 10
    assert not set(a.P) & set(a.N)
    assert all(len(w) <= 6 for w in a.P + a.N)


def test_type1_skews_long():
    # Type 1 is dominated by long strings (uniform over Sigma^<=le).
    n7 = tot = 0
    for s in range(200):
        sp = specgen.gen_type1("01", 7, 10, 10, s)
        n7 += sum(len(w) == 7 for w in sp.P + sp.N)
        tot += 20
    assert abs(n7 / tot - 128 / 255) < 0.05


def test_type2_contains_eps_often():
    # short strings like eps are likely in most Type 2 specs.
    hits = sum("" in (sp.P + sp.N) for sp in
               (specgen.gen_type2("01", 10, 10, 10, s) for s in range(300)))
    assert hits / 300 >= 0.8


def test_planted_is_consistent():
    import re
    sp = specgen.gen_planted("abcd", "(ab+c)*d(a+b)?", 8, 8, 4, 10, 0)
    pat = re.compile("(ab|c)*d(a|b)?")
    assert all(pat.fullmatch(w) for w in sp.P)
    assert not any(pat.fullmatch(w) for w in sp.N)


def test_spec_file_roundtrip():
    sp = specgen.TABLE1_ROW1
    back = specgen.read_spec(specgen.write_spec(sp), name=sp.name)
    assert back.P == sp.P and back.N == sp.N and back.alphabet == sp.alphabet
    assert back.costs == sp.costs
