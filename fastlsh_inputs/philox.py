"""Counter-based Philox4x32-10 generator (numpy, vectorised) — seeded input generation only.

This module holds none of the method's arithmetic (no projection, no floor, no key mixing).
It produces the random draws the method consumes (the sampled multisets S_i, the Gaussian
coefficients a_i, the offsets b_i, and the key multipliers), addressed by a counter so that any
single value can be regenerated independently of the order in which values are produced
(reading R11).

Counter layout (shared, as a written spec, with the library's own C++ generator in
paper_2309_15479_b200/csrc/philox.h — the two are independent implementations of the same spec
and are cross-checked by tests/test_inputs.py):

    key     = (seed & 0xffffffff, seed >> 32)
    counter = (j, i, stream, 0)          -> four uint32 words

Streams: 1 = sampled indices, 2 = Gaussian coefficients, 3 = offsets b, 4 = key multipliers.
"""
from __future__ import annotations

import math

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)

STREAM_IDX = 1
STREAM_A = 2
STREAM_B = 3
STREAM_KEYS = 4


def philox4x32_10(c0, c1, c2, c3, seed: int):
    """Philox4x32 with 10 rounds on uint32 counter arrays; returns four uint32 arrays."""
    c0 = np.asarray(c0, dtype=np.uint64) & MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    c0, c1, c2, c3 = (x.copy() for x in (c0, c1, c2, c3))
    k0 = seed & 0xFFFFFFFF
    k1 = (seed >> 32) & 0xFFFFFFFF
    for rnd in range(10):
        p0 = c0 * M0
        p1 = c2 * M1
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        n0 = hi1 ^ c1 ^ np.uint64(k0)
        n1 = lo1
        n2 = hi0 ^ c3 ^ np.uint64(k1)
        n3 = lo0
        c0, c1, c2, c3 = n0, n1, n2, n3
        if rnd != 9:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
    return (c0.astype(np.uint32), c1.astype(np.uint32), c2.astype(np.uint32), c3.astype(np.uint32))


def _grid(rows: int, cols: int):
    i = np.repeat(np.arange(rows, dtype=np.uint64), cols)
    j = np.tile(np.arange(cols, dtype=np.uint64), rows)
    return i, j


def _u64(lo, hi):
    return (np.asarray(hi, dtype=np.uint64) << np.uint64(32)) | np.asarray(lo, dtype=np.uint64)


def sample_indices(n: int, m: int, k: int, seed: int) -> np.ndarray:
    """S_i for i<k: m i.i.d. uniform draws from [0, n), with replacement (§3.1).

    idx = floor(u64 * n / 2^64) — the high 64 bits of the 128-bit product, exact integer math.
    Returns int32 [k, m] (0-based; the paper's example is 1-based — DESIGN.md reading R2).
    """
    i, j = _grid(k, m)
    r0, r1, _, _ = philox4x32_10(j, i, STREAM_IDX, 0, seed)
    u = _u64(r0, r1)
    # high 64 bits of u * n, computed exactly with a 32-bit split of u
    n64 = np.uint64(n)
    lo = u & MASK32
    hi = u >> np.uint64(32)
    t = lo * n64  # < 2^64 because n < 2^32
    t2 = hi * n64 + (t >> np.uint64(32))
    idx = (t2 >> np.uint64(32)).astype(np.int64)
    return idx.reshape(k, m).astype(np.int32)


def _u53(lo, hi) -> np.ndarray:
    return (_u64(lo, hi) >> np.uint64(11)).astype(np.float64)


def gaussian_coefficients(m: int, k: int, seed: int) -> np.ndarray:
    """a_i ~ N(0,1)^m via Box–Muller (cos branch) in double, rounded to f32.

    u1 = (h53(r0,r1) + 1) / 2^53 in (0,1], u2 = h53(r2,r3) / 2^53 in [0,1).
    Python's math module (the platform libm) is used element by element so that the value is
    the same function of the counter as the library's C++ generator on the same host.
    """
    i, j = _grid(k, m)
    r0, r1, r2, r3 = philox4x32_10(j, i, STREAM_A, 0, seed)
    u1 = (_u53(r0, r1) + 1.0) * 2.0 ** -53
    u2 = _u53(r2, r3) * 2.0 ** -53
    out = np.empty(u1.shape, dtype=np.float32)
    for t in range(u1.shape[0]):
        out[t] = np.float32(math.sqrt(-2.0 * math.log(u1[t])) * math.cos(2.0 * math.pi * u2[t]))
    return out.reshape(k, m)


def uniform_offsets(k: int, w: float, seed: int) -> np.ndarray:
    """b_i ~ U[0, w) rounded to f32 and clamped below w (reading R1)."""
    i = np.arange(k, dtype=np.uint64)
    r0, r1, _, _ = philox4x32_10(0, i, STREAM_B, 0, seed)
    u = _u53(r0, r1) * 2.0 ** -53
    wf = np.float32(w)
    b = (np.float64(wf) * u).astype(np.float32)
    below = np.nextafter(wf, np.float32(0))
    return np.where(b >= wf, below, b).astype(np.float32)


MERSENNE61 = (1 << 61) - 1


def key_multipliers(L: int, K: int, seed: int) -> np.ndarray:
    """r_{l,j} uniform in [0, 2^61-1) for l<L, j<=K (reading R9), uint64 [L, K+1].

    r = (u64 >> 3), with the single value 2^61-1 folded to 0.
    """
    i, j = _grid(L, K + 1)
    r0, r1, _, _ = philox4x32_10(j, i, STREAM_KEYS, 0, seed)
    r = _u64(r0, r1) >> np.uint64(3)
    r = np.where(r == np.uint64(MERSENNE61), np.uint64(0), r)
    return r.astype(np.uint64).reshape(L, K + 1)


def identity_indices(n: int, k: int) -> np.ndarray:
    """The identity plan S = (0..n-1) for every hash: FastLSH with it is E2LSH."""
    return np.tile(np.arange(n, dtype=np.int32), (k, 1))
