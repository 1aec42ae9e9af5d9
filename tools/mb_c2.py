"""Time the automatic kernel on C2 (n = 4096, k = 1000, 10^6 rows) for m = 32 and 128 (K1r): the
row-stage geometry A/B of DESIGN.md "K1r" (C2 wavefront budget)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data

c = configs.get("C2")
X = data.generate(c.data, c.n, 0, c.N, seed=c.seed, device="cuda")
out = torch.empty((c.N, c.k), dtype=torch.int32, device="cuda")
for m in (32, 128):
    P = fl.Params.create(c.n, m, c.k, c.w, seed=c.seed)
    fl.fastlsh_hash(P, X, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fl.fastlsh_hash(P, X, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    roof = c.N * c.k * m / (148 * 32 * 1.965e9) * 1e3
    info = P.info()
    print(f"C2 m={m}: {ms:.3f} ms, G_s roofline {roof:.3f} ms, frac {roof / ms:.3f}, kernel {info.get('kernel')}, "
          f"rows {P.row_packing() and {k: v for k, v in P.row_packing().items() if not hasattr(v, 'shape')}}", flush=True)
