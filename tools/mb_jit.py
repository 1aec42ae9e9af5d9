"""Time K1j (params-specialised lane = row kernel) vs K1r on the n = 128 configs: codes,
codes + keys in one launch, keys only; and the same rows through K1r + the key kernel."""
import os, sys, time
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


for name, rows in (("C3", 8_388_608), ("C0", 10_000)):
    c = configs.get(name)
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=c.seed)
    L, Kc = (c.L, c.K) if c.L else (4, 16)
    K = fl.Keys.create(L, Kc, seed=c.seed)
    t0 = time.perf_counter()
    P.prepare(keys=K, codes=True)
    print(f"{name}: prepare {time.perf_counter() - t0:.1f} s, {P.jit_status()}", flush=True)
    X = data.generate(c.data, c.n, 0, rows, seed=c.seed, device="cuda")
    codes = torch.empty((rows, c.k), dtype=torch.int32, device="cuda")
    keys = torch.empty((L, rows), dtype=torch.int64, device="cuda")
    assert P.info()["kernel"] == 4
    t_h = timed(lambda: fl.fastlsh_hash(P, X, out=codes))
    t_f = timed(lambda: fl.hash_keys(P, K, X, codes=codes, keys_out=keys))
    t_fk = timed(lambda: fl.hash_keys(P, K, X, keys_out=keys, with_codes=False))
    P.set_kernel("rows")
    t_rh = timed(lambda: fl.fastlsh_hash(P, X, out=codes))
    t_rk = timed(lambda: fl.build_keys(K, codes, out=keys))
    gath = rows * c.k * c.m
    hbm_codes = rows * (4 * c.n + 4 * c.k)
    hbm_all = hbm_codes + rows * 8 * L
    print(f"{name} rows={rows}: K1j codes {t_h:.3f} ms ({hbm_codes / t_h / 1e6:.0f} GB/s), "
          f"codes+keys {t_f:.3f} ms ({hbm_all / t_f / 1e6:.0f} GB/s), keys-only {t_fk:.3f} ms "
          f"({(rows * (4 * c.n + 8 * L)) / t_fk / 1e6:.0f} GB/s); "
          f"K1r {t_rh:.3f} + K3 {t_rk:.3f} = {t_rh + t_rk:.3f} ms; G_s roofline {gath / 9.306e12 * 1e3:.3f} ms",
          flush=True)
