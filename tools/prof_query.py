"""Time the query path on C1-sized data (1e6 rows, 50 tables) for 1e4 fresh queries."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data
c = configs.get("C1")
P = fl.Params.create(c.n, c.m, c.k, c.w, seed=c.seed)
K = fl.Keys.create(c.L, c.K, seed=c.seed)
X = data.generate(c.data, c.n, 0, c.N, seed=1, device="cuda")
keys = fl.build_keys(K, fl.fastlsh_hash(P, X))
tabs = fl.build_tables(keys)
Q = data.generate(c.data, c.n, 11_000_000, 11_010_000, seed=1, device="cuda")
qk = fl.build_keys(K, fl.fastlsh_hash(P, Q))
fl.query(X, tabs, Q, qk)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = fl.query(X, tabs, Q, qk)
e1.record(); torch.cuda.synchronize()
print(f"query kernel: {e0.elapsed_time(e1):.2f} ms for {Q.shape[0]} queries, mean candidates {r[2].double().mean().item():.0f}")
