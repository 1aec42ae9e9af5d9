import os, sys
sys.path.insert(0, '.')
import torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data
c = configs.get("C3"); rows = 8388608
P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1); K = fl.Keys.create(c.L, c.K, seed=1)
P.prepare(keys=K)
X = data.generate(c.data, c.n, 0, rows, seed=1, device="cuda")
codes = torch.empty((rows, c.k), dtype=torch.int32, device="cuda"); keys = torch.empty((c.L, rows), dtype=torch.int64, device="cuda")
for _ in range(3): fl.hash_keys(P, K, X, codes=codes, keys_out=keys)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30): fl.hash_keys(P, K, X, codes=codes, keys_out=keys)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("FASTLSH_JIT_NOPAIR", "pair"), "%.4f ms" % (e0.elapsed_time(e1) / 30))
