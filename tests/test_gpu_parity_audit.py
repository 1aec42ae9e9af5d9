"""Large-sample parity audit (65 s on a B200; FASTLSH_AUDIT=0 skips it): the CUDA path at BASELINE sizes, in the
launch configuration the bench times, against the CPU oracle on 1e8-3e8 (row, hash) pairs per
config — whole row blocks spread over the resident workload, not single sampled rows, so every
lane / warp / CTA position of the kernels is covered. Same rule as test_gpu_parity.py
(parity.stats: north_star tolerance, boundary band of DESIGN.md R5); the records go to
$FASTLSH_PARITY_LOG (committed as profiles/r02_parity_audit.jsonl).

PAPER.md:157 (Eq. 5: h(v) = floor((a . S(v) + b) / w)), PAPER.md:167 (K codes per table key).
"""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, fastlsh_arrays
from oracle import keys as okeys
from parity import record, stats

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(os.environ.get("FASTLSH_AUDIT") == "0", reason="FASTLSH_AUDIT=0")]
THREADS = max(1, min(16, len(os.sched_getaffinity(0))))

# (config, m, resident rows N, blocks, rows per block, rows per block whose keys are recomputed)
AUDIT = [("C1", None, None, 16, 16384, 64), ("C2", 32, None, 8, 16384, 32), ("C2", 128, 262_144, 8, 8192, 32),
         ("C3", None, 25_000_000, 16, 65536, 128), ("C4", None, None, 4, 25000, 64)]


@pytest.mark.parametrize("name,m,N,blocks,rpb,krows", AUDIT)
def test_parity_audit(name, m, N, blocks, rpb, krows):
    c = configs.get(name)
    m = m or c.m
    N = N or c.N
    idx, a, b = fastlsh_arrays(c.n, m, c.k, c.w, c.seed)
    P = fl.Params.from_arrays(c.n, c.w, idx, a, b)
    X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
    K = fl.Keys.create(c.L, c.K, seed=1) if c.L else None
    if K is not None:
        codes, gkeys = fl.hash_keys(P, K, X)
    else:
        codes, gkeys = fl.fastlsh_hash(P, X), None
    torch.cuda.synchronize()
    tot = {"rows": 0, "hashes": 0, "ambiguous": 0, "out_of_band_mismatches": 0, "in_band_outside_band": 0,
           "in_band_differ_from_oracle": 0, "sentinel_mismatches": 0, "proj_outside_tol": 0,
           "key_mismatches_given_codes": 0, "key_rows": 0}
    worst = 0.0
    # blocks spread over the workload: the first, the last (ragged tail included) and evenly between
    starts = sorted({min(max(0, N - rpb), (N - rpb) * i // max(1, blocks - 1)) for i in range(blocks)})
    for s in starts:
        e = min(N, s + rpb)
        Xb = X[s:e]
        pg = fl.fastlsh_project(P, Xb.contiguous()).cpu().numpy()
        cg = codes[s:e].cpu().numpy()
        p, scale, code = oracle.fastlsh(Xb.cpu().numpy(), idx, a, b, c.w, threads=THREADS)
        kg = kr = None
        rec = stats(cg, pg, p, scale, code, b, c.w)
        if K is not None:
            kk = min(krows, e - s)
            kg = gkeys[:, s:s + kk].cpu().numpy().view(np.uint64)
            kr = okeys.build_keys(cg[:kk].astype(np.int64), K.export(), K.L, K.K)
            tot["key_mismatches_given_codes"] += int((kg != kr).sum())
            tot["key_rows"] += kk
        tot["rows"] += rec["rows"]
        tot["hashes"] += rec["hashes"]
        tot["ambiguous"] += int(round(rec["ambiguous_frac"] * rec["hashes"]))
        for f in ("out_of_band_mismatches", "in_band_outside_band", "in_band_differ_from_oracle",
                  "sentinel_mismatches", "proj_outside_tol"):
            tot[f] += rec[f]
        worst = max(worst, rec["max_rel_proj_err"])
        del pg, cg, p, scale, code
    out = {"config": name, "m": m, "test": "audit", "N": N, "blocks": len(starts),
           "kernel": fl.Params.KERNELS.get(P.info()["kernel"], "?"),
           "ambiguous_frac": tot["ambiguous"] / max(1, tot["hashes"]), "max_rel_proj_err": worst}
    out.update({k: v for k, v in tot.items() if k != "ambiguous"})
    record(out)
    assert tot["out_of_band_mismatches"] == 0 and tot["in_band_outside_band"] == 0
    assert tot["sentinel_mismatches"] == 0 and tot["proj_outside_tol"] == 0
    assert tot["key_mismatches_given_codes"] == 0
    assert worst < 1e-6
