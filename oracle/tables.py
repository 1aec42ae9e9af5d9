"""Bucket tables from compound keys — TEST INFRASTRUCTURE ONLY.

PAPER.md:167 (§3.2): every point v is stored in bucket H_l(v) of each of the L hash tables; a
query probes bucket H_l(u) of every table. With the 64-bit compound keys of
DESIGN.md reading R9, table l is the multiset of pairs (key_l(v), v). The library stores it in
canonical bulk form (reading R15):

  sorted_keys[l]  the N keys of table l in ascending (unsigned) order,
  ids[l]          the row id v of each entry; entries with equal keys (one bucket) in ascending v,
  bucket_start[l] the first position of every bucket, in ascending key order, then N.

So bucket b of table l holds ids[l][bucket_start[l][b] : bucket_start[l][b+1]], all with key
sorted_keys[l][bucket_start[l][b]].

`build_tables` follows that definition with a library sort; `buckets_brute` is a pure-Python
dictionary grouping (a different formulation) used to pin it.
"""
from __future__ import annotations

import numpy as np


def build_tables(keys):
    """keys uint64 [L, N] -> (sorted_keys uint64 [L, N], ids uint32 [L, N], starts: list of int64 arrays)."""
    keys = np.asarray(keys, dtype=np.uint64)
    L, N = keys.shape
    ids = np.arange(N, dtype=np.int64)
    sk = np.empty_like(keys)
    si = np.empty((L, N), dtype=np.uint32)
    starts = []
    for l in range(L):
        order = np.lexsort((ids, keys[l]))  # primary: key, secondary: row id (stable bucket order)
        sk[l] = keys[l][order]
        si[l] = order.astype(np.uint32)
        if N:
            first = np.ones(N, dtype=bool)
            first[1:] = sk[l][1:] != sk[l][:-1]
            starts.append(np.flatnonzero(first).astype(np.int64))
        else:
            starts.append(np.zeros(0, dtype=np.int64))
    return sk, si, starts


def buckets_brute(keys_l):
    """Pure-Python grouping of one table: {key: [ids in ascending order]} (insertion order = row order)."""
    out: dict[int, list[int]] = {}
    for v, kk in enumerate(keys_l):
        out.setdefault(int(kk), []).append(v)
    return out
