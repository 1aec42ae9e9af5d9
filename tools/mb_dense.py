"""C2's m sweep through the automatic kernel choice (dense path for m >= n/8) at full size, plus the
K4 comparator on C1, CUDA-event timed. Prints one JSON object per case."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2309_15479_b200 as fl  # noqa: E402
from fastlsh_inputs import configs, data  # noqa: E402

G_S = 148 * 32 * 1.965e9


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


bw = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
c = configs.get("C2")
X = data.generate(c.data, c.n, 0, c.N, seed=c.seed, device="cuda")
codes = torch.empty((c.N, c.k), dtype=torch.int32, device="cuda")
for m in [int(a) for a in (sys.argv[1:] or ["128", "512", "4096"])]:
    P = fl.Params.create(c.n, m, c.k, c.w, seed=c.seed)
    kern = fl.Params.KERNELS[P.info()["kernel"]]
    ms = timed(lambda: fl.fastlsh_hash(P, X, out=codes), 3 if m >= 512 else 5)
    t_roof = max((4.0 * c.N * c.n + 4.0 * c.N * c.k) / bw, c.N * c.k * m / G_S) * 1e3
    print(json.dumps({"config": "C2", "m": m, "rows": c.N, "kernel": kern, "ms": ms, "t_roof_ms": t_roof,
                      "roofline_frac": t_roof / ms, "hashes_per_s": c.N * c.k / (ms / 1e3)}), flush=True)
    del P
del X, codes
torch.cuda.empty_cache()
c = configs.get("C1")
X = data.generate(c.data, c.n, 0, c.N, seed=c.seed, device="cuda")
codes = torch.empty((c.N, c.k), dtype=torch.int32, device="cuda")
Pd = fl.Params.e2lsh(c.n, c.k, c.w, seed=c.seed)
for prec in (3, 1):
    ms = timed(lambda: fl.e2lsh_hash(Pd, X, out=codes, precision=prec))
    print(json.dumps({"config": "C1", "dense_precision": prec, "ms": ms}), flush=True)
