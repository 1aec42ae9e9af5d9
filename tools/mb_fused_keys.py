"""Time K1r with keys built from its code tile (hash_keys) vs codes + the standalone key kernel."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data


def timed(fn, iters=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for name, rows in (("C1", 1_000_000), ("C3", 8_388_608), ("C4", 100_000)):
    c = configs.get(name)
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=c.seed)
    K = fl.Keys.create(c.L, c.K, seed=c.seed)
    X = data.generate(c.data, c.n, 0, rows, seed=c.seed, device="cuda")
    codes = torch.empty((rows, c.k), dtype=torch.int32, device="cuda")
    keys = torch.empty((c.L, rows), dtype=torch.int64, device="cuda")
    t_f = timed(lambda: fl.hash_keys(P, K, X, codes=codes, keys_out=keys))
    try:
        t_fk = timed(lambda: fl.hash_keys(P, K, X, keys_out=keys, with_codes=False))
    except fl.FastLSHError:
        t_fk = float("nan")  # keys-only needs a fused path (one CTA block, or K1 with table size)
    t_h = timed(lambda: fl.fastlsh_hash(P, X, out=codes))
    t_k = timed(lambda: fl.build_keys(K, codes, out=keys))
    print(f"{name} rows={rows}: fused {t_f:.3f} ms, fused keys-only {t_fk:.3f}, hash {t_h:.3f} + keys {t_k:.3f} = {t_h + t_k:.3f} ms")
