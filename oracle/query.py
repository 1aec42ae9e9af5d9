"""LSH query with exact re-ranking — TEST INFRASTRUCTURE ONLY.

PAPER.md:171-172 (§3.2): to answer a query u, compute H_l(u) for every table l, take the points in
the L buckets H_l(u) as candidates, compute their exact distances to u and return the closest
(the paper re-ranks all candidates exactly). DESIGN.md reading R16 fixes the details:
  - candidates = the DISTINCT points v with key_l(v) == key_l(u) for at least one table l;
  - distance = squared Euclidean distance ||x_v - u||^2 (monotone in l2, PAPER.md:65 uses l2);
  - result = the top-k candidates by (distance, id) ascending; fewer than k candidates pad with
    id -1 and distance +inf.

`query` follows that with the canonical tables of oracle/tables.py (binary search of the bucket);
`candidates_brute` recomputes the candidate set directly from the keys (no tables) to pin it.
"""
from __future__ import annotations

import numpy as np


def _bucket(sorted_keys_l, ids_l, key):
    lo = np.searchsorted(sorted_keys_l, np.uint64(key), side="left")
    hi = np.searchsorted(sorted_keys_l, np.uint64(key), side="right")
    return ids_l[lo:hi]


def query(X, Q, sorted_keys, ids, qkeys, topk: int):
    """X f32 [N, n] data, Q f32 [nq, n] queries, tables (sorted_keys u64 [L, N], ids u32 [L, N]),
    qkeys u64 [L, nq]. Returns (ids int64 [nq, topk], dist float64 [nq, topk], ncand int64 [nq])."""
    X = np.asarray(X, dtype=np.float64)
    Q = np.asarray(Q, dtype=np.float64)
    L = sorted_keys.shape[0]
    nq = Q.shape[0]
    out_i = np.full((nq, topk), -1, dtype=np.int64)
    out_d = np.full((nq, topk), np.inf, dtype=np.float64)
    ncand = np.zeros(nq, dtype=np.int64)
    for q in range(nq):
        cand = set()
        for l in range(L):
            cand.update(int(v) for v in _bucket(sorted_keys[l], ids[l], qkeys[l, q]))
        ncand[q] = len(cand)
        if not cand:
            continue
        c = np.array(sorted(cand), dtype=np.int64)
        diff = X[c] - Q[q]
        d = np.einsum("ij,ij->i", diff, diff)
        order = np.lexsort((c, d))[:topk]  # primary distance, secondary id
        out_i[q, :len(order)] = c[order]
        out_d[q, :len(order)] = d[order]
    return out_i, out_d, ncand


def candidates_brute(keys, qkeys, q: int):
    """Distinct points sharing a key with query q in some table, straight from the keys [L, N]."""
    L, N = keys.shape
    hit = np.zeros(N, dtype=bool)
    for l in range(L):
        hit |= keys[l] == qkeys[l, q]
    return set(np.flatnonzero(hit).tolist())
