#!/usr/bin/env python3
"""Probe locality of the dedup bitmap under bit permutations of the CS (offline, CPU).

Builds Table 1 row 1 levels 1..19 with the oracle, forms concat groups like the
kernel's (one uniform operand x 32 consecutive cached operands, level-20 candidates,
oracle cache order) and counts the distinct 32-byte sectors / 128-byte lines the 32
probes of a group touch for: identity, bit-reversal, every rotation, and the
variability-sorted permutation.  Motivates bm_pos() in levels.cu.

    python scripts/probe_locality.py
"""
import os
import random
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, specgen
sp = specgen.TABLE1_ROW1
o = oracle.Oracle.from_spec(sp)
t=time.time(); r = o.solve(19); print("solve", r.status, time.time()-t)
n = o.n
lv = {c: o.level_cs(c) for c in range(1, 20)}
print({c: len(v) for c, v in lv.items()})
# concat via the oracle's op (slow per call) -> vectorise with gt rows
gt = [o.gt_row(w) for w in range(n)]
def concat_vec(x, ys):
    out = np.zeros(len(ys), dtype=np.int64)
    ys = np.asarray(ys, dtype=np.int64)
    for w in range(n):
        acc = np.zeros(len(ys), dtype=bool)
        for (u, v) in gt[w]:
            if (x >> u) & 1:
                acc |= ((ys >> v) & 1).astype(bool)
        out |= acc.astype(np.int64) << w
    return out
def brev(v, n):
    r = np.zeros_like(v)
    for i in range(n):
        r |= ((v >> i) & 1) << (n - 1 - i)
    return r
def rot(v, r, n):
    m = (1 << n) - 1
    return ((v >> r) | (v << (n - r))) & m
random.seed(1)
samples = []
for _ in range(3000):
    L = random.randint(1, 17); R = 19 - L
    if not lv.get(L) or not lv.get(R): continue
    x = random.choice(lv[L]); ys = lv[R]
    s0 = random.randrange(0, max(1, len(ys) - 32 + 1)); grp = ys[s0:s0 + 32]
    samples.append(concat_vec(x, grp))
def sectors(perm):
    tot = 0
    for c in samples:
        idx = perm(c)
        tot += len(set((idx >> 8).tolist()))
    return tot / len(samples)
def lines(perm):
    return sum(len(set((perm(c) >> 10).tolist())) for c in samples) / len(samples)
print("groups", len(samples))
print("identity sectors", sectors(lambda c: c), "lines", lines(lambda c: c))
print("reverse  sectors", sectors(lambda c: brev(c, n)), "lines", lines(lambda c: brev(c, n)))
best = []
for r in range(1, n):
    best.append((sectors(lambda c, r=r: rot(c, r, n)), r))
best.sort(); print("rotations best", best[:5], "worst", best[-3:])
# per-bit within-group variability
var = np.zeros(n)
for c in samples:
    for w in range(n):
        b = (c >> w) & 1
        var[w] += min(b.sum(), len(b) - b.sum()) / len(b)
order = np.argsort(-var)
print("bit variability", np.round(var / len(samples), 3))
print("ideal order", order)
pos = np.zeros(n, dtype=np.int64); pos[order] = np.arange(n)
def ideal(c):
    r = np.zeros_like(c)
    for w in range(n):
        r |= ((c >> w) & 1) << pos[w]
    return r
print("ideal sectors", sectors(ideal), "lines", lines(ideal))
