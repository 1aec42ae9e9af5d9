import os, sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, fastlsh_arrays
from oracle import keys as okeys
c = configs.get("C3")
idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, 1)
P = fl.Params.from_arrays(c.n, c.w, idx, a, b).set_kernel("jit")
Kobj = fl.Keys.create(16, 16, seed=2)
X = data.generate(c.data, c.n, 0, 40, seed=1, device="cuda")
X[5, :] = float("nan"); X[6, 3] = 1e30
codes, keys = fl.hash_keys(P, Kobj, X)
cn = codes.cpu().numpy().astype(np.int64)
ref = okeys.build_keys(cn, Kobj.export(), 16, 16)
got = keys.cpu().numpy().view(np.uint64)
print(os.environ.get("FASTLSH_JIT_DEBUG"), "rows equal:", [(r, int((got[:, r] == ref[:, r]).sum())) for r in (4, 5, 6, 7)])
# fast-path-only reference: codes as F2I would give them (NaN->0, +ovf->INT_MAX, -ovf->INT_MIN)
p = (X.double().cpu().numpy()[:, idx] * a[None].astype(np.float64)).sum(-1)
print(" row6 gpu codes", cn[6][:8])
