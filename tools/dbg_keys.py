import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, fastlsh_arrays
from oracle import keys as okeys
c = configs.get("C3")
idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, 1)
P = fl.Params.from_arrays(c.n, c.w, idx, a, b).set_kernel("jit")
X = data.generate(c.data, c.n, 0, 3000, seed=1, device="cuda")
Kobj = fl.Keys.create(c.L, c.K, seed=2)
for flag in (False, True):
    if flag:
        X[5, :] = float("nan"); X[6, 3] = 1e30; X[2999, 7] = float("-inf")
    codes, keys = fl.hash_keys(P, Kobj, X)
    cn = codes.cpu().numpy().astype(np.int64)
    ref = okeys.build_keys(cn, Kobj.export(), c.L, c.K)
    got = keys.cpu().numpy().view(np.uint64)
    bad = np.argwhere(got != ref)
    print("flag", flag, "mismatches", len(bad), bad[:20].tolist())
    rows = sorted(set(bad[:, 1].tolist()))
    print(" rows", rows[:20])
    for r in rows[:3]:
        print(" row", r, "codes", cn[r][:20])
# what would the fast path alone have produced? (NaN -> F2I gives 0 / INT_MAX / INT_MIN)
r = Kobj.export()
for row in (5, 6, 2999):
    g = got[:, row]
    # candidate: codes with INT_MIN replaced by 0 (NaN) 
    alt = cn[row].copy(); alt[alt == -2**31] = 0
    ref0 = okeys.build_keys(alt[None, :], r, c.L, c.K)[:, 0]
    alt2 = cn[row].copy(); alt2[alt2 == -2**31] = 2**31 - 1
    ref1 = okeys.build_keys(alt2[None, :], r, c.L, c.K)[:, 0]
    print(row, "eq ref", (g == ref[:, row]).sum(), "eq nan->0", (g == ref0).sum(), "eq ->INTMAX", (g == ref1).sum())
for row in (5, 6, 2999):
    g = got[:, row]
    m = [(l, np.nonzero(ref[l] == g[l])[0][:5].tolist()) for l in range(c.L)]
    print(row, "matches of GPU key in other rows' reference keys:", m[:4])
    print("  gpu", g[:3], "ref", ref[:3, row], "x>=P?", [int(v) >= (1 << 61) - 1 for v in g[:4]])
P61 = (1 << 61) - 1
g = got[:, 5]
allmin = [(int(r[l][0]) + sum(int(r[l][j + 1]) * 0x80000000 for j in range(c.K))) % P61 for l in range(c.L)]
r0s = [int(r[l][0]) for l in range(c.L)]
print("row5 gpu", [int(x) for x in g[:4]])
print(" allmin", allmin[:4])
print(" r0", r0s[:4])
flat = r.reshape(-1)
print(" gpu in flat r?", [int(x) in set(int(v) for v in flat) for x in g[:4]])
# hypothesis: the key loop read codes from a wrong smem area; solve for sum over 16 terms with u = const
for l in range(2):
    S = sum(int(r[l][j + 1]) for j in range(c.K)) % P61
    # g = r0 + u*S mod P -> u = (g - r0) * S^-1 mod P
    u = (int(g[l]) - int(r[l][0])) * pow(S, P61 - 2, P61) % P61
    print(" l", l, "implied constant u", u, hex(u))
