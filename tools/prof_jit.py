"""One K1j launch shape for ncu: python tools/prof_jit.py [--rows R] [--mode codes|keys|keysonly] [--iters I]"""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--rows", type=int, default=8_388_608)
ap.add_argument("--mode", default="keys")
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
c = configs.get(a.config)
P = fl.Params.create(c.n, c.m, c.k, c.w, seed=c.seed)
K = fl.Keys.create(c.L or 4, c.K or 16, seed=c.seed)
P.prepare(keys=K)
X = data.generate(c.data, c.n, 0, a.rows, seed=c.seed, device="cuda")
codes = torch.empty((a.rows, c.k), dtype=torch.int32, device="cuda")
keys = torch.empty((K.L, a.rows), dtype=torch.int64, device="cuda")
for _ in range(a.iters):
    if a.mode == "codes":
        fl.fastlsh_hash(P, X, out=codes)
    elif a.mode == "keys":
        fl.hash_keys(P, K, X, codes=codes, keys_out=keys)
    else:
        fl.hash_keys(P, K, X, keys_out=keys, with_codes=False)
torch.cuda.synchronize()
print("ok")
