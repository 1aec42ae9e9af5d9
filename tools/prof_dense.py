"""One dense-path launch for ncu (kernel 5, C2 shape): python tools/prof_dense.py [--m M] [--rows R]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2309_15479_b200 as fl  # noqa: E402
from fastlsh_inputs import configs, data  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=512)
ap.add_argument("--rows", type=int, default=262_144)
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
c = configs.get("C2")
P = fl.Params.create(c.n, a.m, c.k, c.w, seed=c.seed)
assert P.info()["kernel"] == 5
X = data.generate(c.data, c.n, 0, a.rows, seed=c.seed, device="cuda")
codes = torch.empty((a.rows, c.k), dtype=torch.int32, device="cuda")
for _ in range(a.iters):
    fl.fastlsh_hash(P, X, out=codes)
torch.cuda.synchronize()
print("ok")
