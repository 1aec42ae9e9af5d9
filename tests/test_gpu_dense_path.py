"""The dense path for FastLSH params (kernel 5): Eq. 5 as a
3xTF32 tcgen05 GEMM against the duplicates-merged coefficient matrix. Opt-in only
(fastlsh_params_set_kernel 5): north_star reserves the tensor cores for the dense E2LSH baseline, so the
automatic choice stays on the gather kernels. Same parity rule as the gather kernels, same flags, and
the fallbacks when the GEMM cannot serve a call."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, fastlsh_arrays
from oracle import keys as okeys
from parity import check_codes, check_projections

pytestmark = pytest.mark.gpu
THREADS = max(1, min(16, len(os.sched_getaffinity(0))))


def _params(n, m, k, w, seed=1):
    idx, a, b = fastlsh_arrays(n, m, k, w, seed)
    return fl.Params.from_arrays(n, w, idx, a, b), idx, a, b


def _check(P, idx, a, b, w, X):
    codes = fl.fastlsh_hash(P, X).cpu().numpy()
    proj = fl.fastlsh_project(P, X).cpu().numpy()
    p, s, code = oracle.fastlsh(X.cpu().numpy(), idx, a, b, w, threads=THREADS)
    rel = check_projections(proj, p, s)
    amb = check_codes(codes, p, s, code, b, w)
    return rel, amb, codes


@pytest.mark.parametrize("m,N", [(512, 300), (4096, 77), (1000, 513)])
def test_pinned_dense_on_c2_shapes(m, N):
    """C2 shapes where the GEMM is the faster path: auto stays on the gather kernel (K1r), pinned
    dense meets the same parity bar."""
    c = configs.get("C2")
    P, idx, a, b = _params(c.n, m, c.k, c.w, c.seed)
    assert P.info()["kernel"] == 3
    P.set_kernel("dense")
    assert P.info()["kernel"] == 5
    X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
    rel, amb, _ = _check(P, idx, a, b, c.w, X)
    assert rel < 1e-5 and amb < 2e-2


def test_pinned_dense_on_c1_matches_gather_kernel():
    """Pinned dense on a gather-kernel shape (C1): parity holds and the codes equal K1r's wherever
    neither lies in the boundary band (the two differ only in fp32 summation order)."""
    c = configs.get("C1")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w, c.seed)
    X = data.generate(c.data, c.n, 0, 1500, seed=2, device="cuda")
    P.set_kernel("dense")
    assert P.info()["kernel"] == 5
    _, _, cd = _check(P, idx, a, b, c.w, X)
    Q, *_ = _params(c.n, c.m, c.k, c.w, c.seed)
    cr = fl.fastlsh_hash(Q, X).cpu().numpy()
    assert (cd != cr).mean() < 5e-3


def test_dense_flags_and_sentinels():
    n, m, k = 512, 64, 40
    P, idx, a, b = _params(n, m, k, 1e-3)
    P.set_kernel("dense")
    assert P.info()["kernel"] == 5
    X = torch.randn((70, n), device="cuda")
    X[3, :] = float("nan")
    X[9, 0] = float("inf")
    X[20, :] = 1e30
    fl.read_flags(P, reset=True)
    codes = fl.fastlsh_hash(P, X).cpu().numpy()
    assert (codes[3] == -(2 ** 31)).all() and (codes[20] == -(2 ** 31)).all()
    hit = np.isin(np.arange(n), [0])
    uses0 = np.array([hit[idx[i]].any() for i in range(k)])
    assert (codes[9][uses0] == -(2 ** 31)).all()
    nf, sat = fl.read_flags(P, reset=True)
    assert nf == k + int(uses0.sum()) and sat == k


def test_dense_misaligned_x_falls_back_to_a_gather_kernel():
    """X 4-byte but not 16-byte aligned: the GEMM's tensor maps cannot serve it, so the call falls
    through to the gather chain (K1 here; K0 when the packings were skipped), same parity rule."""
    n, m, k = 512, 128, 96
    P, idx, a, b = _params(n, m, k, 1.0)
    P.set_kernel("dense")
    base = torch.randn(200 * n + 1, device="cuda")
    X = base[1:].view(200, n)
    assert X.data_ptr() % 16 != 0
    rel, amb, _ = _check(P, idx, a, b, 1.0, X)
    assert rel < 1e-5


def test_dense_keys_and_host_path():
    n, m, k, L, K = 768, 128, 160, 16, 10
    P, idx, a, b = _params(n, m, k, 2.0)
    P.set_kernel("dense")
    assert P.info()["kernel"] == 5
    Kobj = fl.Keys.create(L, K, seed=3)
    X = data.generate("sparse80", n, 0, 1234, seed=5, device="cuda")
    codes, keys = fl.hash_keys(P, Kobj, X)
    cg = codes.cpu().numpy()
    kr = okeys.build_keys(cg.astype(np.int64), Kobj.export(), L, K)
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), kr)
    p, s, code = oracle.fastlsh(X.cpu().numpy(), idx, a, b, 2.0, threads=THREADS)
    check_codes(cg, p, s, code, b, 2.0)
    ch, kh = fl.hash_host(P, Kobj, X.cpu(), chunk_rows=500)
    assert np.array_equal(ch.numpy(), cg)
    assert np.array_equal(kh.numpy().view(np.uint64), kr)


def test_switching_between_dense_and_gather_kernels():
    """Python params are packed at creation (info), so pinning the dense path and back to a gather
    kernel works before and after the upload; every switch meets the parity rule."""
    n, m, k = 512, 64, 64
    P, idx, a, b = _params(n, m, k, 1.0)
    X = torch.randn((100, n), device="cuda")
    P.set_kernel("dense")
    _check(P, idx, a, b, 1.0, X)
    P.set_kernel("rows")
    assert P.info()["kernel"] == 3
    _check(P, idx, a, b, 1.0, X)
    P.set_kernel("auto")
    assert P.info()["kernel"] == 3
    P.set_kernel("dense")
    assert P.info()["kernel"] == 5
    _check(P, idx, a, b, 1.0, X)
