"""Locate K1t projection errors vs K1 (debug aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, fastlsh_arrays
name = sys.argv[1] if len(sys.argv) > 1 else "C0"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
c = configs.get(name)
idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, c.seed)
P = fl.Params.from_arrays(c.n, c.w, idx, a, b)
X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
P.set_kernel("smem"); p1 = fl.fastlsh_project(P, X).cpu().numpy()
P.set_kernel("tmem"); p2 = fl.fastlsh_project(P, X).cpu().numpy()
d = np.abs(p1 - p2) > 1e-4 * (np.abs(p1) + 1)
r, h = np.nonzero(d)
print("bad", d.sum(), "of", d.size)
print("rows mod 128 hist", np.bincount(r % 128, minlength=128).tolist())
print("rows //128 hist", np.bincount(r // 128).tolist())
print("hash hist (first 64)", np.bincount(h, minlength=c.k)[:64].tolist())
# which coordinates do bad hashes sample?
bad_h = np.unique(h)
print("n bad hashes", len(bad_h))
for hh in bad_h[:4]:
    print(hh, sorted(idx[hh].tolist()))
