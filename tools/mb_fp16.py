"""K4 dense E2LSH comparator: 3xFP16 (precision 2) vs 3xTF32 (3) vs 1xTF32 (1) on C1 (10^6 rows,
n = 960, k = 500), a C3 chunk (8.4M rows, n = 128, k = 256) and C2 (250k rows, n = 4096, k = 1000),
CUDA-event timed; prints the MMA-work rate (3 products at 2, 3; 1 at 1) and the max projection error
vs 3xTF32 relative to ||a|| ||x|| on the first rows."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2309_15479_b200 as fl  # noqa: E402
from fastlsh_inputs import configs, data  # noqa: E402


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


for name, rows in (("C1", 1_000_000), ("C3", 8_388_608), ("C2", 250_000)):
    c = configs.get(name)
    P = fl.Params.e2lsh(c.n, c.k, c.w, seed=c.seed)
    X = data.generate(c.data, c.n, 0, rows, seed=c.seed, device="cuda")
    codes = torch.empty((rows, c.k), dtype=torch.int32, device="cuda")
    flops = 2.0 * rows * c.n * c.k
    res = {}
    for prec in (3, 2, 1):
        ms = timed(lambda: fl.e2lsh_hash(P, X, out=codes, precision=prec))
        res[prec] = ms
    pr3 = fl.e2lsh_project(P, X[:4096], precision=3).double()
    pr2 = fl.e2lsh_project(P, X[:4096], precision=2).double()
    scale = X[:4096].double().norm(dim=1, keepdim=True) * (c.n ** 0.5)
    err = ((pr2 - pr3).abs() / scale).max().item()
    print(f"{name} rows={rows}: 3xTF32 {res[3]:.3f} ms ({3 * flops / res[3] / 1e9:.0f} TF/s MMA work), "
          f"3xFP16 {res[2]:.3f} ms ({3 * flops / res[2] / 1e9:.0f}), 1xTF32 {res[1]:.3f} ms; "
          f"max |p2 - p3| / (sqrt(n) ||x||) = {err:.2e}", flush=True)
    del P, X, codes
