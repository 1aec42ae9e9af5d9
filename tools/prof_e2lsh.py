"""One dense E2LSH launch for ncu (K4 on C1-shaped E2LSH params): python tools/prof_e2lsh.py [--precision P] [--rows R]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2309_15479_b200 as fl  # noqa: E402
from fastlsh_inputs import configs, data  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", type=int, default=2)
ap.add_argument("--rows", type=int, default=262_144)
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
c = configs.get("C1")
P = fl.Params.e2lsh(c.n, c.k, c.w, seed=c.seed)
X = data.generate(c.data, c.n, 0, a.rows, seed=c.seed, device="cuda")
codes = torch.empty((a.rows, c.k), dtype=torch.int32, device="cuda")
for _ in range(a.iters):
    fl.e2lsh_hash(P, X, out=codes, precision=a.precision)
torch.cuda.synchronize()
print("ok")
