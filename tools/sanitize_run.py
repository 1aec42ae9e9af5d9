"""Small runs of every kernel for compute-sanitizer (racecheck / synccheck / memcheck / initcheck).

  compute-sanitizer --tool racecheck python tools/sanitize_run.py [--only K1j,K1r,...]

C0-sized inputs with ragged tails; each kernel family through the C ABI (VERDICT r1
item 6): K1r (every stride class in use: C0/C3 dual 128, C1 one copy, C4 dual 8-row, C2 4-row),
K1 (plain + fused keys), K1t, K1j (codes, projections, codes+keys, keys only, flagged rows through
the slow path), K3 / K3t keys, K4 dense (1x and 3xTF32), K5 tables, K6 query, K7 transforms, probe.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data

ap = argparse.ArgumentParser()
ap.add_argument("--only", default="")
args = ap.parse_args()
only = set(x for x in args.only.split(",") if x)


def want(k):
    return not only or k in only


def X_for(c, N, seed=1):
    return data.generate(c.data, c.n, 0, N, seed=seed, device="cuda")


ran = []
if want("K1r"):
    for name, N in (("C0", 301), ("C1", 203), ("C3", 301), ("C4", 75)):
        c = configs.get(name)
        P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1).set_kernel("rows")
        X = X_for(c, N)
        fl.fastlsh_hash(P, X)
        fl.fastlsh_project(P, X)
        if c.L:
            fl.hash_keys(P, fl.Keys.create(c.L, c.K, seed=1), X)
    c = configs.get("C2")
    P = fl.Params.create(c.n, 32, c.k, c.w, seed=1).set_kernel("rows")
    fl.fastlsh_hash(P, X_for(c, 9))
    ran.append("K1r")
if want("K1"):
    c = configs.get("C1")
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1).set_kernel("smem")
    X = X_for(c, 203)
    fl.fastlsh_hash(P, X)
    Pf = fl.Params.create(c.n, c.m, c.k, c.w, seed=1).set_table_size(c.K).set_kernel("smem")
    fl.hash_keys(Pf, fl.Keys.create(c.L, c.K, seed=1), X)
    ran.append("K1")
if want("K1t"):
    c = configs.get("C1")
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1).set_kernel("tmem")
    fl.fastlsh_hash(P, X_for(c, 300))
    ran.append("K1t")
if want("K1j"):
    c = configs.get("C3")
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1).set_kernel("jit")
    K = fl.Keys.create(c.L, c.K, seed=1)
    X = X_for(c, 301)
    X[5] = float("nan")
    X[77, 3] = 1e30
    fl.fastlsh_hash(P, X)
    fl.fastlsh_project(P, X)
    fl.hash_keys(P, K, X)
    fl.hash_keys(P, K, X, with_codes=False)
    ran.append("K1j")
if want("K3"):
    for L, K, k in ((50, 10, 500), (16, 16, 256), (600, 2, 1201)):
        codes = data.random_codes(333, k, seed=3).cuda()
        fl.build_keys(fl.Keys.create(L, K, seed=1), codes)
    ran.append("K3")
if want("K4"):
    c = configs.get("C1")
    Pd = fl.Params.e2lsh(c.n, c.k, c.w, seed=1)
    X = X_for(c, 300)
    for prec in (1, 3):
        fl.e2lsh_hash(Pd, X, precision=prec)
    ran.append("K4")
if want("K5") or want("K6"):
    c = configs.get("C1")
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1)
    K = fl.Keys.create(c.L, c.K, seed=1)
    X = X_for(c, 2000)
    _, keys = fl.hash_keys(P, K, X)
    tabs = fl.build_tables(keys)
    Q = X_for(c, 20, seed=5)
    _, qk = fl.hash_keys(P, K, Q)
    fl.query(X, tabs, Q, qk, topk=10)
    ran.append("K5+K6")
if want("K7"):
    X = torch.randn((333, 37), device="cuda")
    fl.normalize_rows(X)
    kap = fl.max_row_norm(X)
    fl.mips_transform(X, kap)
    fl.mips_transform(X, query=True)
    ran.append("K7")
if want("probe"):
    a = torch.zeros(4096, dtype=torch.int32, device="cuda")
    b = torch.zeros(8192, dtype=torch.int32, device="cuda")
    fl.bandwidth_probe(a, b, 32, 512, 1024)
    ran.append("probe")
torch.cuda.synchronize()
print("sanitize_run ok:", ",".join(ran))
