"""The parity rule of north_star / SURVEY.md §8(c), applied to GPU results vs the CPU oracle.

  projections: |p_gpu - p| <= 1e-5 * ||a_i|| * ||S_i(v)||               (north_star tolerance)
  codes:       equal wherever floor((p - tau + b)/w) == floor((p + tau + b)/w);
               inside that band, one of the two values,
               with tau = 1e-5 * scale + 2^-22 * (|p| + |b|)            (reading R5:
               the fp32 +b and /w roundings add at most ~1.5 ulp of |p + b|)
  sentinel:    INT32_MIN where the oracle's quotient is non-finite or outside (-2^31, 2^31).
"""
from __future__ import annotations

import numpy as np

INT32_MIN = -(2 ** 31)


def check_projections(p_gpu, p, scale, tol=1e-5):
    p_gpu = np.asarray(p_gpu, np.float64)
    err = np.abs(p_gpu - p)
    bound = tol * scale
    bad = ~(err <= bound)
    assert not bad.any(), (f"{int(bad.sum())} projections outside 1e-5*scale; worst rel "
                           f"{float(np.max(err / np.maximum(scale, 1e-300)))}")
    rel = err / np.maximum(scale, 1e-300)
    return float(rel.max()) if rel.size else 0.0


def expected_code_band(p, scale, b, w):
    tau = 1e-5 * scale + 2.0 ** -22 * (np.abs(p) + np.abs(b)[None, :])
    lo = np.floor((p - tau + b[None, :]) / w)
    hi = np.floor((p + tau + b[None, :]) / w)
    return lo, hi


def check_codes(codes_gpu, p, scale, code_oracle, b, w):
    """Returns the fraction of (row, hash) pairs whose oracle projection lies in the ambiguity band."""
    codes_gpu = np.asarray(codes_gpu, np.int64)
    b = np.asarray(b, np.float64)
    lo, hi = expected_code_band(p, scale, b, w)
    out_of_range = (code_oracle <= INT32_MIN) | (code_oracle > 2 ** 31 - 1)
    ambig = (lo != hi) & ~out_of_range
    exact = ~ambig & ~out_of_range
    mism = exact & (codes_gpu != code_oracle)
    assert not mism.any(), (f"{int(mism.sum())} code mismatches outside the band, e.g. at "
                            f"{np.argwhere(mism)[:5].tolist()}")
    inb = ambig & ((codes_gpu < lo) | (codes_gpu > hi))
    assert not inb.any(), f"{int(inb.sum())} codes outside their band"
    if out_of_range.any():
        assert (codes_gpu[out_of_range] == INT32_MIN).all()
    return float(ambig.mean()) if ambig.size else 0.0


def stats(codes_gpu, proj_gpu, p, scale, code_oracle, b, w, keys_gpu=None, keys_ref=None):
    """The per-config parity record of BASELINE.md §3 / VERDICT r1 item 1, on one row sample:
    max relative projection error (vs ||a|| ||S(v)||), ambiguous fraction (oracle projection inside
    the band of DESIGN.md R5), code mismatches outside the band (must be 0), codes outside their
    band, sentinel mismatches, and key mismatches given the GPU's codes (must be 0)."""
    codes_gpu = np.asarray(codes_gpu, np.int64)
    b = np.asarray(b, np.float64)
    lo, hi = expected_code_band(p, scale, b, w)
    out_of_range = (code_oracle <= INT32_MIN) | (code_oracle > 2 ** 31 - 1)
    ambig = (lo != hi) & ~out_of_range
    exact = ~ambig & ~out_of_range
    rec = {"rows": int(codes_gpu.shape[0]), "hashes": int(codes_gpu.size),
           "ambiguous_frac": float(ambig.mean()) if ambig.size else 0.0,
           "out_of_band_mismatches": int((exact & (codes_gpu != code_oracle)).sum()),
           "in_band_outside_band": int((ambig & ((codes_gpu < lo) | (codes_gpu > hi))).sum()),
           "in_band_differ_from_oracle": int((ambig & (codes_gpu != code_oracle)).sum()),
           "sentinel_mismatches": int((out_of_range & (codes_gpu != INT32_MIN)).sum())}
    if proj_gpu is not None:
        err = np.abs(np.asarray(proj_gpu, np.float64) - p)
        rel = err / np.maximum(scale, 1e-300)
        rec["max_rel_proj_err"] = float(rel.max()) if rel.size else 0.0
        rec["proj_outside_tol"] = int((err > 1e-5 * scale).sum())
    if keys_gpu is not None:
        rec["key_mismatches_given_codes"] = int((np.asarray(keys_gpu) != np.asarray(keys_ref)).sum())
    return rec


def record(rec: dict):
    """Append one parity record (JSON line) to $FASTLSH_PARITY_LOG when set (the GPU runs collect
    them into profiles/r02_parity.jsonl)."""
    import json
    import os
    path = os.environ.get("FASTLSH_PARITY_LOG")
    if path:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
