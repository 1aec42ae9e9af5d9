import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, fastlsh_arrays
P61 = (1 << 61) - 1
c = configs.get("C3")
idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, 1)
P = fl.Params.from_arrays(c.n, c.w, idx, a, b).set_kernel("jit")
for L, K in ((1, 1), (2, 3), (16, 16)):
    Kobj = fl.Keys.create(L, K, seed=2)
    r = Kobj.export()
    for N, rowbad in ((1, 0), (40, 5), (40, 37)):
        X = data.generate(c.data, c.n, 0, N, seed=1, device="cuda")
        X[rowbad, :] = float("nan")
        for wc in (True, False):
            codes, keys = fl.hash_keys(P, Kobj, X, with_codes=wc)
            g = keys.cpu().numpy().view(np.uint64)[:, rowbad]
            us = []
            for l in range(L):
                S = sum(int(r[l][j + 1]) for j in range(K)) % P61
                u = (int(g[l]) - int(r[l][0])) * pow(S, P61 - 2, P61) % P61
                us.append(hex(u))
            print(L, K, N, rowbad, "codes" if wc else "keys-only", "implied u", us[:3], flush=True)
