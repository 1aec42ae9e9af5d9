"""Short driver for ncu captures of the hot-path kernels (one config, a few launches)."""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_15479_b200 as fl  # noqa: E402
from fastlsh_inputs import configs, data  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--rows", type=int, default=262144)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--keys", action="store_true")
    ap.add_argument("--fused-keys", action="store_true", help="hash_keys (K1r builds keys from its code tile)")
    ap.add_argument("--kernel", default="auto", choices=["auto", "smem", "tmem", "rows"])
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--dense", action="store_true", help="time the tcgen05 dense baseline too")
    ap.add_argument("--dense-e2lsh", action="store_true", help="dense baseline on E2LSH params (m = n)")
    args = ap.parse_args()
    c = configs.get(args.config)
    m = args.m or c.m
    P = fl.Params.create(c.n, m, c.k, c.w, seed=c.seed)
    P.set_kernel(args.kernel)
    K = fl.Keys.create(c.L, c.K, seed=c.seed) if ((args.keys or args.fused_keys) and c.L) else None
    X = data.generate(c.data, c.n, 0, args.rows, seed=c.seed, device="cuda")
    codes = torch.empty((args.rows, c.k), dtype=torch.int32, device="cuda")
    keys = torch.empty((c.L, args.rows), dtype=torch.int64, device="cuda") if K else None
    for _ in range(args.iters):
        if K and args.fused_keys:
            fl.hash_keys(P, K, X, codes=codes, keys_out=keys)
            continue
        fl.fastlsh_hash(P, X, out=codes)
        if K:
            fl.build_keys(K, codes, out=keys)
    torch.cuda.synchronize()
    if args.dense:
        Pd = fl.Params.e2lsh(c.n, c.k, c.w, seed=c.seed) if args.dense_e2lsh else P
        for prec in (3, 1):
            fl.e2lsh_hash(Pd, X, out=codes, precision=prec)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                fl.e2lsh_hash(Pd, X, out=codes, precision=prec)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            kpad = (c.k + 255) // 256 * 256
            flops = 2.0 * args.rows * c.n * kpad * (3 if prec == 3 else 1)
            print(f"dense e2lsh {args.config} prec={prec} rows={args.rows}: {ms:.3f} ms, "
                  f"{args.rows * c.k / ms / 1e6:.3e} hashes/s, {flops / ms / 1e9:.1f} TFLOP/s (tf32 MMA rate)")
    if args.time:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fl.fastlsh_hash(P, X, out=codes)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        gathers = args.rows * c.k * m
        peak = 148 * 32 * 1.965e9
        print(f"{args.config} m={m} rows={args.rows}: {ms:.3f} ms/launch, {gathers / ms / 1e6:.1f} Ggather/s, "
              f"{gathers / (ms / 1e3) / peak:.3f} of smem roofline; info={P.info()}")


if __name__ == "__main__":
    main()
