"""Dense E2LSH baseline (tcgen05 3xTF32 GEMM) vs the CPU oracle."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, e2lsh_arrays, fastlsh_arrays
from parity import check_codes, check_projections

pytestmark = pytest.mark.gpu
THREADS = max(1, min(16, len(os.sched_getaffinity(0))))


@pytest.mark.parametrize("N,n,k,w,recipe", [(1000, 128, 64, 4.0, "sift_u8"), (777, 960, 500, 1.0, "gist_mixture"),
                                            (300, 784, 2000, 2.0, "sparse80"), (129, 4096, 256, 0.5, "trevi_sphere"),
                                            (5, 32, 16, 1.0, "sift_u8"), (300, 100, 40, 1.0, "gist_mixture")])
@pytest.mark.parametrize("precision", [3, 2])
def test_e2lsh_3xtf32_parity(N, n, k, w, recipe, precision):
    """3xTF32 (precision 3) and 3xFP16 (precision 2: fp16 tensor cores, cross term scaled by 2^11)
    both stay within the north-star tolerance of the fp64 oracle (n = 100: ragged last K-block)."""
    idx, A, b = e2lsh_arrays(n, k, w, seed=2)
    P = fl.Params.from_arrays(n, w, idx, A, b)
    X = data.generate(recipe, n, 0, N, seed=3, device="cuda")
    proj = fl.e2lsh_project(P, X, precision=precision).cpu().numpy()
    codes = fl.e2lsh_hash(P, X, precision=precision).cpu().numpy()
    p, s, code = oracle.e2lsh(X.cpu().numpy(), A, b, w, threads=THREADS)
    check_projections(proj, p, s)
    check_codes(codes, p, s, code, b, w)


def test_e2lsh_library_params_match_identity_fastlsh():
    """e2lsh_params_create draws the same coefficients as identity-FastLSH (R11)."""
    n, k, w = 256, 128, 1.0
    P = fl.Params.e2lsh(n, k, w, seed=5)
    idx, A, b = e2lsh_arrays(n, k, w, seed=5)
    X = torch.randn((513, n), device="cuda")
    codes = fl.e2lsh_hash(P, X).cpu().numpy()
    p, s, code = oracle.e2lsh(X.cpu().numpy(), A, b, w, threads=THREADS)
    check_codes(codes, p, s, code, b, w)


def test_dense_path_on_fastlsh_params():
    """The dense GEMM on FastLSH params (duplicates-merged coefficient matrix) computes Eq. 5."""
    c = configs.get("C0")
    idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, c.seed)
    P = fl.Params.from_arrays(c.n, c.w, idx, a, b)
    X = data.generate(c.data, c.n, 0, 2000, seed=1, device="cuda")
    proj = fl.e2lsh_project(P, X).cpu().numpy()
    p, s, _ = oracle.fastlsh(X.cpu().numpy(), idx, a, b, c.w, threads=THREADS)
    check_projections(proj, p, s)


def test_plain_tf32_is_less_accurate_than_3xtf32():
    n, k, w = 960, 256, 1.0
    idx, A, b = e2lsh_arrays(n, k, w, seed=7)
    P = fl.Params.from_arrays(n, w, idx, A, b)
    X = data.generate("gist_mixture", n, 0, 512, seed=1, device="cuda")
    p, s, _ = oracle.e2lsh(X.cpu().numpy(), A, b, w, threads=THREADS)
    e3 = np.abs(fl.e2lsh_project(P, X, precision=3).cpu().numpy() - p) / s
    e1 = np.abs(fl.e2lsh_project(P, X, precision=1).cpu().numpy() - p) / s
    assert e3.max() < 1e-5
    assert e1.max() > 10 * e3.max()


def test_plain_tf32_violation_rate_c1_shape():
    """the ungated 1xTF32 comparator is reported with its violation rate — the
    fraction of projections outside the north-star band 1e-5 * |a| |S(v)| and of codes that differ
    from the oracle outside the ambiguity band. 3xTF32 has none; 1xTF32 has many."""
    c = configs.get("C1")
    idx, A, b = e2lsh_arrays(c.n, c.k, c.w, seed=c.seed)
    P = fl.Params.from_arrays(c.n, c.w, idx, A, b)
    X = data.generate(c.data, c.n, 0, 2000, seed=1, device="cuda")
    p, s, code = oracle.e2lsh(X.cpu().numpy(), A, b, c.w, threads=THREADS)
    rates = {}
    for prec in (3, 1):
        pr = fl.e2lsh_project(P, X, precision=prec).cpu().numpy()
        cg = fl.e2lsh_hash(P, X, precision=prec).cpu().numpy()
        rates[prec] = (float((np.abs(pr - p) > 1e-5 * s).mean()), float((cg != code).mean()))
    print(f"\n1xTF32 violation rate (C1 shape, 2000 rows x {c.k}): projections {rates[1][0]:.3e}, "
          f"codes {rates[1][1]:.3e}; 3xTF32: {rates[3][0]:.1e}, {rates[3][1]:.1e}")
    assert rates[3][0] == 0.0
    assert rates[1][0] > 0.01


def test_3xfp16_small_and_large_magnitudes():
    """3xFP16 keeps the tolerance where fp16 alone would not: rows scaled by 2^-20 (the low parts
    would be fp16 subnormals without the 2^11 scaling) and by 2^10 (|x| up to ~2.6e5 / 4 ... < 65504)."""
    n, k, w = 256, 128, 1.0
    idx, A, b = e2lsh_arrays(n, k, w, seed=9)
    P = fl.Params.from_arrays(n, w, idx, A, b)
    X0 = data.generate("gist_mixture", n, 0, 600, seed=4, device="cuda")
    for scale in (2.0 ** -20, 2.0 ** -8, 2.0 ** 10):
        X = (X0 * scale).contiguous()
        proj = fl.e2lsh_project(P, X, precision=2).cpu().numpy()
        p, s, _ = oracle.e2lsh(X.cpu().numpy(), A, b, w, threads=THREADS)
        check_projections(proj, p, s)


def test_3xfp16_overflow_is_flagged():
    """|x| beyond fp16's range (65504) overflows the hi part: the element comes back as the sentinel
    and counted as non-finite, never as a wrong finite code."""
    n, k, w = 64, 32, 1.0
    P = fl.Params.e2lsh(n, k, w, seed=1)
    X = torch.rand((40, n), device="cuda")
    X[7, 3] = 1.0e6
    fl.read_flags(P, reset=True)
    codes = fl.e2lsh_hash(P, X, precision=2).cpu().numpy()
    nf, _ = fl.read_flags(P, reset=True)
    assert (codes[7] == -(2 ** 31)).all() and nf == k
    keep = np.arange(40) != 7  # the other rows: the same codes as 3xTF32 away from bucket boundaries
    ref = fl.e2lsh_hash(P, X, precision=3).cpu().numpy()
    assert np.mean(codes[keep] == ref[keep]) > 0.99
