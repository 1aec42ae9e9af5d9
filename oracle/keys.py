"""Compound bucket keys with exact Python integers — TEST INFRASTRUCTURE ONLY.

PAPER.md:167 (§3.2): "H(v) = (h_1(v), ..., h_k(v)) is the concatenation of k elementary LSH codes"
and L groups H_1..H_L give L tables. A literal bit concatenation of K codes does not fit in 64
bits (reading R9), so a table's key is the multilinear form, exactly mod p = 2^61 - 1:

    key_l(v) = ( r[l][0] + sum_{j<K} r[l][j+1] * u32(code[v][l*K + j]) )  mod  (2^61 - 1)

u32(c) is the two's-complement bit pattern of the int32 code. Table l uses code columns
[l*K, (l+1)*K). Equal code tuples give equal keys; distinct tuples collide with probability
<= 1/p over the draw of r.
"""
from __future__ import annotations

import numpy as np

P61 = (1 << 61) - 1


def u32(c: int) -> int:
    return int(c) & 0xFFFFFFFF


def key(codes_row, r_l, K: int, l: int) -> int:
    acc = int(r_l[0])
    for j in range(K):
        acc += int(r_l[j + 1]) * u32(codes_row[l * K + j])
    return acc % P61


def build_keys(codes, r, L: int, K: int):
    """keys[l][v] for codes int[N][k] (k >= L*K), r uint64[L][K+1]; returns uint64 [L, N]."""
    codes = np.asarray(codes)
    N = codes.shape[0]
    out = np.zeros((L, N), dtype=np.uint64)
    for v in range(N):
        row = [int(c) for c in codes[v]]
        for l in range(L):
            out[l, v] = key(row, r[l], K, l)
    return out
