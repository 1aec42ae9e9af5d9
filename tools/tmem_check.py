"""Quick GPU check of the TMEM kernel K1t vs the shared-memory kernel K1 and the oracle; timings."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2309_15479_b200 as fl  # noqa: E402
from fastlsh_inputs import configs, data, fastlsh_arrays  # noqa: E402
from parity import check_codes, check_projections  # noqa: E402


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    only = sys.argv[1:] or ["C0", "C1", "C3", "C4", "C1full", "C3full", "C4full", "C2"]
    for name in only:
        full = name.endswith("full")
        c = configs.get(name.replace("full", ""))
        N = c.N if full else {"C0": c.N, "C1": 2003, "C3": 4099, "C4": 1001, "C2": 517}[c.name]
        if full and c.name == "C3":
            N = 4_000_000
        idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, c.seed)
        P = fl.Params.from_arrays(c.n, c.w, idx, a, b)
        info = P.info()
        X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
        res = {}
        for kern in ("smem", "tmem"):
            try:
                P.set_kernel(kern)
            except Exception as ex:  # noqa: BLE001
                print(f"{name}: {kern} unavailable: {ex}")
                continue
            codes = fl.fastlsh_hash(P, X)
            proj = fl.fastlsh_project(P, X)
            torch.cuda.synchronize()
            ms = timed(lambda: fl.fastlsh_hash(P, X, out=codes))
            res[kern] = (codes, proj, ms)
        rows = np.arange(N) if N <= 5000 else np.unique(np.r_[np.random.default_rng(0).choice(N, 1500, replace=False), 0, N - 1])
        ri = torch.as_tensor(rows, device="cuda")
        Xh = X[ri].cpu().numpy()
        p, s, code = oracle.fastlsh(Xh, idx, a, b, c.w, threads=8)
        for kern, (codes, proj, ms) in res.items():
            try:
                rel = check_projections(proj[ri].cpu().numpy(), p, s)
                amb = check_codes(codes[ri].cpu().numpy(), p, s, code, b, c.w)
                ok = f"parity ok (max rel {rel:.2e}, amb {amb:.1e})"
            except AssertionError as ex:
                ok = f"PARITY FAIL: {str(ex)[:200]}"
            g = N * c.k * c.m / (ms / 1e3)
            print(f"{name} N={N} {kern}: {ms:.3f} ms  {N * c.k / ms / 1e6:.3e} hashes/s  "
                  f"{g / 9.306e12:.3f} of smem roofline  {ok}  [tmem HB={info['tmem_hash_blocks']} "
                  f"nhw={info['tmem_hashes_per_warp']}]", flush=True)
        if len(res) == 2:
            same = torch.equal(res["smem"][0], res["tmem"][0])
            print(f"   codes identical smem vs tmem: {same}", flush=True)


if __name__ == "__main__":
    main()
