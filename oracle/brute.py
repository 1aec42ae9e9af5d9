"""Pure-Python brute force of Eq. 5 for tiny inputs — TEST INFRASTRUCTURE ONLY.

Triple loop over rows, hashes and sampled slots, in the order PAPER.md:150-159 (§3.1) states:
sample S(v), project with a, add b, divide by w, floor. Python floats are IEEE doubles and each
product of two f32 values is exact in double, so with the same left-to-right order this equals
oracle/fastlsh_oracle.c bit for bit.
"""
from __future__ import annotations

import math


def sample(v, S):
    """S(v) for a multiset S of 0-based indices."""
    return [v[i] for i in S]


def fastlsh_hash(v, S, a, b, w):
    """h(v) = floor((a . S(v) + b) / w) — Eq. 5. Returns (p, code)."""
    sv = sample(v, S)
    p = 0.0
    for aj, xj in zip(a, sv):
        p += float(aj) * float(xj)
    return p, math.floor((p + float(b)) / float(w))


def e2lsh_hash(v, a, b, w):
    """h(v) = floor((a . v + b) / w) — Eq. 1."""
    p = 0.0
    for aj, xj in zip(a, v):
        p += float(aj) * float(xj)
    return p, math.floor((p + float(b)) / float(w))


def hash_all(X, idx, a, b, w):
    """[[code of row r under hash i]] and the projections, for lists/arrays of tiny size."""
    P, C = [], []
    for v in X:
        pr, cr = [], []
        for i in range(len(idx)):
            p, c = fastlsh_hash([float(x) for x in v], [int(t) for t in idx[i]], a[i], b[i], w)
            pr.append(p)
            cr.append(c)
        P.append(pr)
        C.append(cr)
    return P, C
