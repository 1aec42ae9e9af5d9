"""Seeded input generators shared by the tests, the oracle runs and bench.py.

Holds none of the method's arithmetic: only random draws (Philox, counter-addressed) and
synthetic datasets. Both the CUDA path and the oracle consume what this module produces.
"""
from __future__ import annotations

import numpy as np

from . import configs, data, philox  # noqa: F401


def fastlsh_arrays(n: int, m: int, k: int, w: float, seed: int):
    """(idx int32[k,m], a f32[k,m], b f32[k]) for FastLSH (Eq. 5)."""
    return (philox.sample_indices(n, m, k, seed),
            philox.gaussian_coefficients(m, k, seed),
            philox.uniform_offsets(k, w, seed))


def e2lsh_arrays(n: int, k: int, w: float, seed: int):
    """(identity idx, a f32[k,n], b f32[k]) for E2LSH (Eq. 1): m = n, S = identity.

    The coefficient stream is the FastLSH one addressed by (i, j<n), so identity-FastLSH and
    E2LSH drawn from the same seed are the same function.
    """
    return (philox.identity_indices(n, k),
            philox.gaussian_coefficients(n, k, seed),
            philox.uniform_offsets(k, w, seed))


def tiny_case(N: int, n: int, m: int, k: int, w: float, seed: int, scale: float = 1.0):
    """Small random X (float32, seeded numpy) plus FastLSH arrays, for host-only tests."""
    rng = np.random.default_rng(seed)
    X = (rng.standard_normal((N, n)) * scale).astype(np.float32)
    idx, a, b = fastlsh_arrays(n, m, k, w, seed)
    return X, idx, a, b
