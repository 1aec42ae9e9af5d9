"""Projection error of the dense path (kernel 5, 3xTF32 tcgen05 GEMM on merged coefficients) against the
oracle, over many rows: max and quantiles of |p_gpu - p| / (|a| |S(v)|), the north-star tolerance being
1e-5. python tools/dense_error.py [--m M] [--rows R] [--chunk C]"""
import argparse
import json
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

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=512)
ap.add_argument("--rows", type=int, default=100_000)
ap.add_argument("--chunk", type=int, default=20_000)
ap.add_argument("--kernel", default="auto")
a = ap.parse_args()
c = configs.get("C2")
idx, A, b = fastlsh_arrays(c.n, a.m, c.k, c.w, c.seed)
P = fl.Params.from_arrays(c.n, c.w, idx, A, b)
if a.kernel != "auto":
    P.set_kernel(a.kernel)
threads = len(os.sched_getaffinity(0))
mx, hist, tot = 0.0, np.zeros(8, np.int64), 0
edges = [0, 1e-7, 3e-7, 1e-6, 2e-6, 4e-6, 6e-6, 1e-5, np.inf]
for r0 in range(0, a.rows, a.chunk):
    X = data.generate(c.data, c.n, r0, min(a.rows, r0 + a.chunk), seed=c.seed, device="cuda")
    pg = fl.fastlsh_project(P, X).cpu().numpy().astype(np.float64)
    p, s, _ = oracle.fastlsh(X.cpu().numpy(), idx, A, b, c.w, threads=threads)
    rel = np.abs(pg - p) / np.maximum(s, 1e-300)
    mx = max(mx, float(rel.max()))
    hist += np.histogram(rel, bins=edges)[0]
    tot += rel.size
print(json.dumps({"config": "C2", "m": a.m, "rows": a.rows, "kernel": fl.Params.KERNELS[P.info()["kernel"]],
                  "projections": tot, "max_rel_err": mx, "tolerance": 1e-5,
                  "hist_edges": [str(e) for e in edges], "hist": hist.tolist()}))
