"""Preprocessing transforms of the paper's extensions — TEST INFRASTRUCTURE ONLY.

PAPER.md:481 (§5): "one can use FastLSH for the angular similarity directly after data
normalization" -> normalize(x) = x / ||x||_2 (a zero row stays zero; reading R17).

PAPER.md:830-834 (App. B, maximum inner product search, after [MIPS]): data rows are mapped by
P(v) = (sqrt(kappa^2 - ||v||^2), v) and queries by Q(u) = (0, u), kappa = max_i ||v_i||_2; then
argmax_i P(v_i).Q(u) / (||P(v_i)|| ||Q(u)||) = argmin_i ||P(v_i) - Q(u)|| for ||u|| = 1, so FastLSH
(an l2 LSH) answers MIPS on the transformed vectors. The extra coordinate is prepended, as written.
Computed in float64 from the f32 inputs.
"""
from __future__ import annotations

import numpy as np


def normalize(X):
    X = np.asarray(X, dtype=np.float64)
    nrm = np.sqrt((X * X).sum(axis=1, keepdims=True))
    return np.where(nrm > 0, X / np.where(nrm > 0, nrm, 1.0), 0.0)


def max_norm(X):
    X = np.asarray(X, dtype=np.float64)
    return float(np.sqrt((X * X).sum(axis=1)).max()) if len(X) else 0.0


def mips_data(X, kappa: float):
    """P(v) = (sqrt(kappa^2 - ||v||^2), v); kappa >= max ||v|| (clamped at 0 against rounding)."""
    X = np.asarray(X, dtype=np.float64)
    sq = (X * X).sum(axis=1)
    head = np.sqrt(np.maximum(kappa * kappa - sq, 0.0))
    return np.concatenate([head[:, None], X], axis=1)


def mips_query(U):
    """Q(u) = (0, u)."""
    U = np.asarray(U, dtype=np.float64)
    return np.concatenate([np.zeros((len(U), 1)), U], axis=1)
