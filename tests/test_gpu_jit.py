"""K1j — the params-specialised lane = row kernel (jit.cpp) vs the CPU oracle.

Same parity rule as every other kernel (tests/parity.py: north_star tolerance on projections,
codes exact outside the boundary band of DESIGN.md R5, INT32_MIN + counters for non-finite or
out-of-int32 quotients), on seeded inputs from fastlsh_inputs; keys bit-exact against Python
big integers (oracle/keys.py) evaluated on the GPU's own codes (north_star: "bit-exact given equal
codes"). K1j is the automatic choice for n <= 128 (C0, C3), so the C0/C3 cases of
test_gpu_parity.py run through it as well; here it is pinned (set_kernel("jit")).
"""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, fastlsh_arrays, philox
from oracle import keys as okeys
from parity import check_codes, check_projections, record, stats

pytestmark = pytest.mark.gpu
THREADS = max(1, min(16, len(os.sched_getaffinity(0))))
INT32_MIN = -(2 ** 31)


def _jit_params(n, m, k, w, seed=1):
    idx, a, b = fastlsh_arrays(n, m, k, w, seed)
    P = fl.Params.from_arrays(n, w, idx, a, b).set_kernel("jit")
    assert P.info()["kernel"] == 4
    return P, idx, a, b


def _check(P, idx, a, b, w, X, rows=None, tag=None):
    codes = fl.fastlsh_hash(P, X)
    proj = fl.fastlsh_project(P, X)
    torch.cuda.synchronize()
    st = P.jit_status()
    assert st["error"] == "", st
    if rows is None:
        Xh, cg, pg = X.cpu().numpy(), codes.cpu().numpy(), proj.cpu().numpy()
    else:
        ri = torch.as_tensor(rows, device=X.device)
        Xh, cg, pg = X[ri].cpu().numpy(), codes[ri].cpu().numpy(), proj[ri].cpu().numpy()
    p, scale, code = oracle.fastlsh(Xh, idx, a, b, w, threads=THREADS)
    rel = check_projections(pg, p, scale)
    amb = check_codes(cg, p, scale, code, b, w)
    if tag is not None:
        rec = dict(tag, kernel="K1j", N=int(X.shape[0]), sampled=rows is not None)
        rec.update(stats(cg, pg, p, scale, code, b, w))
        record(rec)
    return rel, amb, codes


def test_jit_is_the_automatic_choice_for_short_rows():
    for name in ("C0", "C3"):
        c = configs.get(name)
        P = fl.Params.create(c.n, c.m, c.k, c.w, seed=c.seed)
        assert P.info()["kernel"] == 4, name
    c = configs.get("C1")
    assert fl.Params.create(c.n, c.m, c.k, c.w, seed=1).info()["kernel"] == 3  # n = 960: K1r


@pytest.mark.parametrize("name,N", [("C0", None), ("C3", 4099), ("C3", 70_001)])
def test_jit_parity_configs(name, N):
    c = configs.get(name)
    N = N or c.N
    P, idx, a, b = _jit_params(c.n, c.m, c.k, c.w, c.seed)
    X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
    rows = None
    if N > 5000:
        rng = np.random.default_rng(3)
        rows = np.unique(np.concatenate([rng.choice(N, 1500, replace=False), [0, 31, 32, 33, N - 33, N - 1]]))
    rel, amb, _ = _check(P, idx, a, b, c.w, X, rows, tag={"config": name, "m": c.m, "test": "jit_pinned"})
    assert rel < 1e-6 and amb < 5e-3


@pytest.mark.parametrize("N,n,m,k,w", [(1, 128, 16, 64, 4.0), (31, 32, 5, 36, 1.5), (33, 36, 1, 4, 0.75),
                                       (1000, 100, 64, 256, 2.0), (4097, 128, 3, 128, 1.5),
                                       (65, 4, 4, 100, 1.0), (129, 64, 130, 32, 0.5), (7, 128, 128, 128, 3.0),
                                       (500, 64, 8, 96, 2.0), (333, 128, 16, 160, 4.0)])  # odd group counts: last pair half empty
def test_jit_edge_shapes(N, n, m, k, w):
    """Ragged tiles (N % 32), n % 32 != 0 (partial X boxes), k % 32 != 0 (partial code boxes),
    m = 1, m > n (replacement), non-power-of-two w (IEEE division), tiny n."""
    P, idx, a, b = _jit_params(n, m, k, w, seed=N + n + m)
    g = torch.Generator(device="cuda")
    g.manual_seed(N * 31 + n)
    X = torch.randn((N, n), generator=g, device="cuda")
    _check(P, idx, a, b, w, X)


def test_jit_flags_and_sentinels():
    """A flagged row goes through the generic slow path: INT32_MIN + counts, other rows intact."""
    c = configs.get("C3")
    P, idx, a, b = _jit_params(c.n, c.m, c.k, c.w)
    X = data.generate(c.data, c.n, 0, 3000, seed=1, device="cuda")
    ref = fl.fastlsh_hash(P, X)
    X[5, :] = float("nan")
    X[6, 3] = 1e30
    X[2999, 7] = float("-inf")
    fl.read_flags(P, reset=True)
    codes = fl.fastlsh_hash(P, X)
    cn = codes.cpu().numpy()
    assert (cn[5] == INT32_MIN).all()
    idx6 = (idx == 3).any(axis=1)
    idx7 = (idx == 7).any(axis=1)
    assert (cn[6][idx6] == INT32_MIN).all() and (cn[2999][idx7] == INT32_MIN).all()
    nf, sat = fl.read_flags(P, reset=True)
    assert nf == c.k + int(idx7.sum()) and sat == int(idx6.sum())
    keep = np.ones(3000, bool)
    keep[[5, 6, 2999]] = False
    assert torch.equal(codes[torch.as_tensor(keep, device="cuda")], ref[torch.as_tensor(keep, device="cuda")])
    # the untouched hashes of the flagged rows equal the clean run
    rn = ref.cpu().numpy()
    assert (cn[6][~idx6] == rn[6][~idx6]).all() and (cn[2999][~idx7] == rn[2999][~idx7]).all()
    # the same through the keys path: keys recomputed from the corrected codes
    Kobj = fl.Keys.create(c.L, c.K, seed=2)
    codes_k, keys_k = fl.hash_keys(P, Kobj, X)
    assert torch.equal(codes_k, codes)
    ref_keys = okeys.build_keys(cn.astype(np.int64), Kobj.export(), c.L, c.K)
    assert np.array_equal(keys_k.cpu().numpy().view(np.uint64), ref_keys)


@pytest.mark.parametrize("name,L,K,N", [("C3", 16, 16, 4099), ("C0", 5, 12, 999), ("C0", 4, 16, 2048),
                                         ("C3", 1, 256, 100)])
def test_jit_keys_bit_exact(name, L, K, N):
    """Codes + keys in one launch: codes equal the codes-only launch, keys equal Python big
    integers on those codes; keys-only (codes never written) into columns [col0, col0 + N)."""
    c = configs.get(name)
    P, idx, a, b = _jit_params(c.n, c.m, c.k, c.w, 3)
    Kobj = fl.Keys.from_arrays(philox.key_multipliers(L, K, seed=4))
    X = data.generate(c.data, c.n, 0, N, seed=5, device="cuda")
    codes_f, keys_f = fl.hash_keys(P, Kobj, X)
    codes_p = fl.fastlsh_hash(P, X)
    assert torch.equal(codes_f, codes_p)
    ref = okeys.build_keys(codes_p.cpu().numpy().astype(np.int64), Kobj.export(), L, K)
    assert np.array_equal(keys_f.cpu().numpy().view(np.uint64), ref)
    wide = torch.zeros((L, N + 77), dtype=torch.int64, device="cuda")
    none, w2 = fl.hash_keys(P, Kobj, X, keys_out=wide, with_codes=False, col0=77)
    assert none is None
    assert torch.equal(w2[:, 77:], keys_f) and (w2[:, :77] == 0).all()


def test_jit_determinism_chunking_and_host_path():
    c = configs.get("C3")
    P, idx, a, b = _jit_params(c.n, c.m, c.k, c.w)
    Kobj = fl.Keys.create(c.L, c.K, seed=1)
    X = data.generate(c.data, c.n, 0, 10_007, seed=1, device="cuda")
    c1 = fl.fastlsh_hash(P, X)
    assert torch.equal(c1, fl.fastlsh_hash(P, X))
    parts = torch.cat([fl.fastlsh_hash(P, X[i:j].contiguous()) for i, j in [(0, 4095), (4095, 4096), (4096, 10_007)]])
    assert torch.equal(c1, parts)
    codes_d, keys_d = fl.hash_keys(P, Kobj, X)
    codes_h, keys_h = fl.hash_host(P, Kobj, X.cpu().pin_memory(), chunk_rows=3000)
    assert torch.equal(codes_d.cpu(), codes_h) and torch.equal(keys_d.cpu(), keys_h)
    none, keys_h2 = fl.hash_host(P, Kobj, X.cpu().pin_memory(), chunk_rows=3000, with_codes=False)
    assert none is None and torch.equal(keys_d.cpu(), keys_h2)


def test_jit_unaligned_falls_back_in_auto_mode():
    """X not 16-byte aligned: TMA cannot stage it; the automatic choice falls back to K1 (same rule),
    the pinned kernel reports EUNSUPPORTED."""
    c = configs.get("C0")
    idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, 1)
    P = fl.Params.from_arrays(c.n, c.w, idx, a, b)
    base = torch.randn(300 * c.n + 1, device="cuda")
    X = base[1:].view(300, c.n)
    assert X.data_ptr() % 16 != 0
    codes = fl.fastlsh_hash(P, X).cpu().numpy()
    p, s, code = oracle.fastlsh(X.cpu().numpy(), idx, a, b, c.w)
    check_codes(codes, p, s, code, b, c.w)
    P.set_kernel("jit")
    with pytest.raises(fl.FastLSHError):
        fl.fastlsh_hash(P, X)


def test_jit_vs_rows_kernel_codes_agree():
    """Same Eq. 5 in fp32 with different summation orders: codes differ only at boundary ties."""
    c = configs.get("C3")
    P, idx, a, b = _jit_params(c.n, c.m, c.k, c.w)
    X = data.generate(c.data, c.n, 0, 50_000, seed=9, device="cuda")
    cj = fl.fastlsh_hash(P, X)
    P.set_kernel("rows")
    cr = fl.fastlsh_hash(P, X)
    assert (cj != cr).float().mean().item() < 1e-4
