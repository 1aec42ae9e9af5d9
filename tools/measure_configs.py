"""Per-config measurement: K1r, K1 (and K1t where it applies) and the dense tcgen05
E2LSH comparator on every BASELINE.json config, with the north-star roofline fraction
t_roof / t_kernel, t_roof = max((4Nn + 4Nk)/BW_HBM, N*k*m/G_s). One JSON object per line.

  python tools/measure_configs.py [--out profiles/r01_configs.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_15479_b200 as fl  # noqa: E402
from fastlsh_inputs import configs, data  # noqa: E402

G_S = 148 * 32 * 1.965e9


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
    except Exception:
        return 6.65e12


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


CASES = [  # name, m override, rows, note
    ("C0", None, None, "full config (10^4 rows, L2-resident)"),
    ("C1", None, None, "full config"),
    ("C2", 32, None, "full config, m sweep"),
    ("C2", 128, None, "m sweep"),
    ("C2", 512, 250_000, "m sweep, 250k-row sample"),
    ("C2", 4096, 20_000, "m = n (i.i.d. sampling), 20k-row sample"),
    ("C3", None, 25_000_000, "one GPU's shard at G = 8 (2e8 / 8 rows)"),
    ("C4", None, None, "one streaming batch (1e5 rows)"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_configs.jsonl"))
    args = ap.parse_args()
    bw = hbm_peak()
    out = open(args.out, "w")
    for name, m_over, rows, note in CASES:
        c = configs.get(name)
        m = m_over or c.m
        N = rows or c.N
        P = fl.Params.create(c.n, m, c.k, c.w, seed=c.seed)
        X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
        codes = torch.empty((N, c.k), dtype=torch.int32, device="cuda")
        gathers = N * c.k * m
        iters = max(3, min(20, int(2e11 / max(gathers, 1))))
        t_hbm = (4.0 * N * c.n + 4.0 * N * c.k) / bw
        t_smem = gathers / G_S
        t_roof = max(t_hbm, t_smem)
        rec = {"config": name, "m": m, "rows": N, "n": c.n, "k": c.k, "note": note,
               "t_roof_ms": t_roof * 1e3, "bound": "smem" if t_smem >= t_hbm else "hbm"}
        info = P.info()
        if info["kernel"] == 5:
            P.row_packing()  # builds the gather packings (reported below) without leaving auto mode
            info = P.info()
        rec["packing"] = {kk: info[kk] for kk in ("parts", "slots", "warps_per_block", "hash_blocks",
                                                  "bank_efficiency")}
        rp = P.row_packing()
        if rp is not None:
            rec["row_packing"] = {kk: rp[kk] for kk in ("parts", "slots", "warps", "hash_blocks", "S", "n1")}
        rec["auto_kernel"] = fl.Params.KERNELS[info["kernel"]]
        ms = timed(lambda: fl.fastlsh_hash(P, X, out=codes), iters)  # the automatic choice (fastlsh_hash)
        rec["auto"] = {"kernel": rec["auto_kernel"], "ms": ms, "hashes_per_s": N * c.k / (ms / 1e3),
                       "roofline_frac": t_roof / (ms / 1e3)}
        for kern, key in (("jit", "K1j"), ("rows", "K1r"), ("smem", "K1"), ("tmem", "K1t")):
            try:
                P.set_kernel(kern)
                ms = timed(lambda: fl.fastlsh_hash(P, X, out=codes), iters)
                rec[key] = {"ms": ms, "hashes_per_s": N * c.k / (ms / 1e3), "roofline_frac": t_roof / (ms / 1e3),
                            "smem_frac": t_smem / (ms / 1e3), "hbm_frac": t_hbm / (ms / 1e3)}
            except fl.FastLSHError as ex:
                rec[key] = {"unavailable": str(ex)}
        P.set_kernel("auto")
        best = min((rec[k]["ms"] for k in ("K1j", "K1r", "K1") if "ms" in rec[k]))
        if c.L:  # the bench's step: hash + keys through fastlsh_hash_keys with the automatic kernel
            Kobj = fl.Keys.create(c.L, c.K, seed=c.seed)
            keys = torch.empty((c.L, N), dtype=torch.int64, device="cuda")
            ms = timed(lambda: fl.hash_keys(P, Kobj, X, codes=codes, keys_out=keys), iters)
            rec["hash_keys_auto"] = {"ms": ms, "hashes_per_s": N * c.k / (ms / 1e3),
                                     "hbm_bytes_per_row": 4 * c.n + 4 * c.k + 8 * c.L}
            del keys
        try:
            Pd = fl.Params.e2lsh(c.n, c.k, c.w, seed=c.seed)
            for prec in (3, 2, 1):
                ms = timed(lambda: fl.e2lsh_hash(Pd, X, out=codes, precision=prec), 3)
                rec["dense_fp16x3" if prec == 2 else f"dense_tf32x{prec}"] = {
                    "ms": ms, "hashes_per_s": N * c.k / (ms / 1e3), "fastlsh_speedup": ms / best}
            del Pd
        except fl.FastLSHError as ex:
            rec["dense"] = {"unavailable": str(ex)}
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
        del X, codes, P
        torch.cuda.empty_cache()
    out.close()


if __name__ == "__main__":
    main()
