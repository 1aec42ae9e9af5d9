"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Inputs (S_i, a_i, b_i, X) come from fastlsh_inputs only; the oracle never sees a value produced
by the CUDA path. X is generated on the device by torch (plumbing) and the exact bytes hashed are
copied to the host for the oracle.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, fastlsh_arrays, e2lsh_arrays, philox
from oracle import keys as okeys
from parity import check_codes, check_projections, record, stats

pytestmark = pytest.mark.gpu
THREADS = max(1, min(16, len(os.sched_getaffinity(0))))


def _params(n, m, k, w, seed=1):
    idx, a, b = fastlsh_arrays(n, m, k, w, seed)
    return fl.Params.from_arrays(n, w, idx, a, b), idx, a, b


def _run_and_check(P, idx, a, b, w, X_dev, rows=None, tag=None, keys=None):
    """Hash X_dev on the GPU; compare all rows (rows=None) or the given row sample with the oracle.
    With `tag` (a dict naming the config) the parity statistics are recorded (parity.record); with
    `keys` the compound keys of the same launch are checked bit-exact against Python big integers
    on the GPU's codes."""
    if keys is not None:
        codes, gkeys = fl.hash_keys(P, keys, X_dev)
    else:
        codes, gkeys = fl.fastlsh_hash(P, X_dev), None
    proj = fl.fastlsh_project(P, X_dev)
    torch.cuda.synchronize()
    if rows is None:
        Xh = X_dev.cpu().numpy()
        cg, pg = codes.cpu().numpy(), proj.cpu().numpy()
        kg = gkeys.cpu().numpy().view(np.uint64) if gkeys is not None else None
    else:
        ri = torch.as_tensor(rows, device=X_dev.device)
        Xh = X_dev[ri].cpu().numpy()
        cg, pg = codes[ri].cpu().numpy(), proj[ri].cpu().numpy()
        kg = gkeys[:, ri].cpu().numpy().view(np.uint64) if gkeys is not None else None
    p, scale, code = oracle.fastlsh(Xh, idx, a, b, w, threads=THREADS)
    rel = check_projections(pg, p, scale)
    amb = check_codes(cg, p, scale, code, b, w)
    kr = None
    if keys is not None:
        kr = okeys.build_keys(cg.astype(np.int64), keys.export(), keys.L, keys.K)
        assert np.array_equal(kg, kr), "keys differ from big-integer keys on the GPU's codes"
    if tag is not None:
        rec = dict(tag)
        rec.update(kernel=fl.Params.KERNELS.get(P.info()["kernel"], "?"), N=int(X_dev.shape[0]),
                   sampled=rows is not None)
        rec.update(stats(cg, pg, p, scale, code, b, w, kg, kr))
        record(rec)
    return rel, amb, codes


def _sample_rows(N, count, seed, extra=()):
    rng = np.random.default_rng(seed)
    r = set(rng.choice(N, size=min(count, N), replace=False).tolist())
    r.update([0, N - 1, *[x for x in extra if 0 <= x < N]])
    return np.array(sorted(r), dtype=np.int64)


# ---- C0: full parity ----------------------------------------------------------------------------

def test_c0_full_parity():
    c = configs.get("C0")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w, c.seed)
    X = data.generate(c.data, c.n, 0, c.N, seed=c.seed, device="cuda")
    rel, amb, _ = _run_and_check(P, idx, a, b, c.w, X, tag={"config": "C0", "m": c.m, "test": "full"},
                                 keys=fl.Keys.create(4, 16, seed=1))
    assert rel < 1e-6
    assert amb < 5e-3


# ---- C1-C4 at small N (all rows, several tiles + ragged tail) and full N (sampled rows) ----------

SMALL = [("C1", None, 2003), ("C2", 32, 517), ("C2", 128, 261), ("C2", 512, 131), ("C2", 4096, 21),
         ("C3", None, 4099), ("C4", None, 1001)]


@pytest.mark.parametrize("name,m,N", SMALL)
def test_small_full_parity(name, m, N):
    c = configs.get(name)
    m = m or c.m
    P, idx, a, b = _params(c.n, m, c.k, c.w, c.seed)
    X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
    Kobj = fl.Keys.create(c.L, c.K, seed=1) if c.L else None
    rel, amb, _ = _run_and_check(P, idx, a, b, c.w, X, tag={"config": name, "m": m, "test": "small_all_rows"}, keys=Kobj)
    assert amb < 1e-2


FULL = [("C1", None, None, 2048), ("C2", 32, None, 1024), ("C2", 128, None, 1024), ("C2", 512, None, 512),
        ("C2", 4096, None, 256), ("C3", None, 4_000_000, 2048),
        ("C4", None, None, 2048)]


@pytest.mark.slow
@pytest.mark.parametrize("name,m,N,sample", FULL)
def test_full_size_sampled_parity(name, m, N, sample):
    """At BASELINE sizes in the bench launch configuration, sampled rows vs the oracle."""
    c = configs.get(name)
    m = m or c.m
    N = N or c.N
    P, idx, a, b = _params(c.n, m, c.k, c.w, c.seed)
    X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
    rows = _sample_rows(N, sample, seed=7, extra=[N // 2, N - 2, 4 * (N // 8) - 1])
    Kobj = fl.Keys.create(c.L, c.K, seed=1) if c.L else None
    _run_and_check(P, idx, a, b, c.w, X, rows=rows, tag={"config": name, "m": m, "test": "full_size_sampled"}, keys=Kobj)
    del X
    torch.cuda.empty_cache()


# ---- params drawn by the library from the seed == inputs-module arrays ---------------------------

def test_seeded_params_path_matches_oracle():
    c = configs.get("C0")
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=c.seed)
    idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, c.seed)
    X = data.generate(c.data, c.n, 0, 3000, seed=c.seed, device="cuda")
    _run_and_check(P, idx, a, b, c.w, X)


# ---- edge cases -----------------------------------------------------------------------------------

@pytest.mark.parametrize("N,n,m,k", [(1, 128, 16, 64), (5, 130, 7, 33), (77, 37, 50, 9), (64, 1, 5, 3),
                                     (33, 8, 1, 1), (130, 256, 200, 20), (9, 96, 64, 257), (300, 4, 4, 100)])
def test_edge_shapes(N, n, m, k):
    P, idx, a, b = _params(n, m, k, 1.5, seed=N + n)
    g = torch.Generator(device="cuda")
    g.manual_seed(N * 31 + n)
    X = torch.randn((N, n), generator=g, device="cuda")
    _run_and_check(P, idx, a, b, 1.5, X)


def test_empty_input_is_noop():
    P, *_ = _params(16, 4, 8, 1.0)
    X = torch.zeros((0, 16), device="cuda")
    out = fl.fastlsh_hash(P, X)
    assert out.shape == (0, 8)


def test_misaligned_rows_take_scalar_path():
    P, idx, a, b = _params(64, 16, 40, 1.0)
    base = torch.randn(100 * 64 + 1, device="cuda")
    X = base[1:].view(100, 64)  # 4-byte aligned, not 16-byte aligned
    assert X.data_ptr() % 16 != 0
    _run_and_check(P, idx, a, b, 1.0, X)


def test_zero_rows_give_floor_b_over_w():
    P, idx, a, b = _params(96, 16, 64, 2.0)
    X = torch.zeros((10, 96), device="cuda")
    codes = fl.fastlsh_hash(P, X).cpu().numpy()
    assert (codes == 0).all()  # b in [0, w): floor(b/w) = 0 exactly (R5)


def test_nonfinite_and_saturation_flags():
    n, m, k = 32, 8, 16
    idx = np.tile(np.arange(m, dtype=np.int32), (k, 1))
    a = np.ones((k, m), np.float32)
    b = np.zeros(k, np.float32)
    P = fl.Params.from_arrays(n, 1e-3, idx, a, b)
    X = torch.zeros((4, n), device="cuda")
    X[1, 0] = float("nan")
    X[2, 0] = float("inf")
    X[3, 0] = 1e30
    fl.read_flags(P, reset=True)
    codes = fl.fastlsh_hash(P, X).cpu().numpy()
    assert (codes[0] == 0).all()
    assert (codes[1:] == -(2 ** 31)).all()
    nf, sat = fl.read_flags(P, reset=True)
    assert nf == 2 * k and sat == k


# ---- structure: determinism, chunking, identity plan, host path -------------------------------------

def test_determinism_and_chunk_invariance():
    c = configs.get("C1")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w)
    X = data.generate(c.data, c.n, 0, 5000, seed=1, device="cuda")
    c1 = fl.fastlsh_hash(P, X)
    c2 = fl.fastlsh_hash(P, X)
    parts = [fl.fastlsh_hash(P, X[i:j].contiguous()) for i, j in [(0, 1234), (1234, 1235), (1235, 5000)]]
    assert torch.equal(c1, c2)
    assert torch.equal(c1, torch.cat(parts))
    pr1 = fl.fastlsh_project(P, X)
    pr2 = torch.cat([fl.fastlsh_project(P, X[i:j].contiguous()) for i, j in [(0, 777), (777, 5000)]])
    assert torch.equal(pr1, pr2)


def test_identity_plan_matches_e2lsh_oracle():
    n, k, w = 64, 96, 1.0
    idx, A, b = e2lsh_arrays(n, k, w, seed=4)
    P = fl.Params.from_arrays(n, w, idx, A, b)
    X = torch.randn((500, n), device="cuda")
    codes = fl.fastlsh_hash(P, X).cpu().numpy()
    proj = fl.fastlsh_project(P, X).cpu().numpy()
    p, s, code = oracle.e2lsh(X.cpu().numpy(), A, b, w)
    check_projections(proj, p, s)
    check_codes(codes, p, s, code, b, w)


@pytest.mark.parametrize("name,L,K,N,extra_k", [("C1", 50, 10, 3001, 0), ("C4", 200, 10, 1203, 0),
                                                ("C3", 16, 16, 4097, 0), ("C0", 5, 12, 999, 4)])
def test_fused_keys_equal_separate_kernels(name, L, K, N, extra_k):
    """Keys built in K1's epilogue (whole tables per CTA) == codes + the standalone key kernel."""
    c = configs.get(name)
    k = L * K + extra_k if name == "C0" else c.k
    idx, a, b = fastlsh_arrays(c.n, c.m, k, c.w, 3)
    P_fused = fl.Params.from_arrays(c.n, c.w, idx, a, b).set_table_size(K).set_kernel("smem")
    P_plain = fl.Params.from_arrays(c.n, c.w, idx, a, b).set_kernel("smem")  # the fused path is K1's
    Kobj = fl.Keys.from_arrays(philox.key_multipliers(L, K, seed=4))
    X = data.generate(c.data, c.n, 0, N, seed=5, device="cuda")
    codes_f, keys_f = fl.hash_keys(P_fused, Kobj, X)
    codes_p = fl.fastlsh_hash(P_plain, X)
    keys_p = fl.build_keys(Kobj, codes_p)
    assert torch.equal(codes_f, codes_p)
    assert torch.equal(keys_f, keys_p)


@pytest.mark.parametrize("fused", [False, True])
def test_host_entry_point_matches_device_path(fused):
    c = configs.get("C4")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w)
    if fused:
        P.set_table_size(c.K)
    K = fl.Keys.create(c.L, c.K, seed=1)
    X = data.generate(c.data, c.n, 0, 10_000, seed=1, device="cuda")
    codes_d, keys_d = fl.hash_keys(P, K, X)
    Xh = X.cpu().pin_memory()
    codes_h, keys_h = fl.hash_host(P, K, Xh, chunk_rows=3000)
    assert torch.equal(codes_d.cpu(), codes_h)
    assert torch.equal(keys_d.cpu(), keys_h)
    _, keys_h2 = fl.hash_host(P, K, Xh, chunk_rows=3000, with_codes=False)  # codes stay on the device
    assert torch.equal(keys_d.cpu(), keys_h2)


# ---- compound keys: bit-exact vs Python big integers, on seeded code matrices ------------------------

@pytest.mark.parametrize("L,K,N,ldk_pad,extra", [(50, 10, 1000, 0, 3), (16, 16, 333, 5, 3), (200, 10, 257, 0, 3),
                                                  (1, 1, 7, 0, 3), (50, 10, 1001, 0, 0), (12, 16, 777, 2, 4),
                                                  (600, 2, 1001, 0, 0)])
def test_keys_bit_exact(L, K, N, ldk_pad, extra):
    """k = L*K + extra code columns: k % 4 == 0 and rows not bank-aligned take the TMA-staged K3t
    (50x10 at k = 500, 12x16 at k = 196), others the register-batched K3 (L > 512, k % 4 != 0)."""
    r = philox.key_multipliers(L, K, seed=3)
    Kobj = fl.Keys.from_arrays(r)
    codes = data.random_codes(N, L * K + extra, seed=L + K, lo=-(2 ** 31), hi=2 ** 31 - 1)
    keys_gpu = fl.build_keys(Kobj, codes.cuda(), ldk=N + ldk_pad)[:, :N].cpu().numpy().view(np.uint64)
    ref = okeys.build_keys(codes.numpy(), r, L, K)
    assert np.array_equal(keys_gpu, ref)


def test_keys_from_oracle_codes_c1():
    c = configs.get("C1")
    idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, 1)
    X = data.generate(c.data, c.n, 0, 200, seed=1).numpy()
    _, _, code = oracle.fastlsh(X, idx, a, b, c.w, threads=THREADS)
    r = philox.key_multipliers(c.L, c.K, seed=1)
    Kobj = fl.Keys.create(c.L, c.K, seed=1)
    keys_gpu = fl.build_keys(Kobj, torch.as_tensor(code.astype(np.int32)).cuda()).cpu().numpy().view(np.uint64)
    assert np.array_equal(keys_gpu, okeys.build_keys(code, r, c.L, c.K))


# ---- K1t (tensor-memory gather, opt-in): the same parity rule on the same inputs ---------------------

TMEM_CASES = [("C0", None), ("C1", 2003), ("C3", 4099), ("C4", 1001), ("C1", 70_001)]


@pytest.mark.parametrize("name,N", TMEM_CASES)
def test_tmem_kernel_parity(name, N):
    c = configs.get(name)
    N = N or c.N
    P, idx, a, b = _params(c.n, c.m, c.k, c.w, c.seed)
    P.set_kernel("tmem")
    assert P.info()["kernel"] == 2
    X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
    rows = None if N <= 5000 else _sample_rows(N, 1500, seed=3, extra=[255, 256, N - 2])
    rel, amb, codes = _run_and_check(P, idx, a, b, c.w, X, rows=rows)
    assert amb < 1e-2
    P.set_kernel("smem")
    codes_smem = fl.fastlsh_hash(P, X)
    # both kernels compute Eq. 5 in fp32 with different summation orders: codes may differ only
    # where a projection sits within fp32 rounding of a bucket boundary
    assert (codes != codes_smem).float().mean().item() < 1e-3


@pytest.mark.parametrize("N,n,m,k", [(1, 128, 16, 64), (257, 64, 128, 7), (300, 4, 4, 100), (513, 960, 60, 130),
                                     (100, 8, 33, 1), (1000, 132, 20, 300)])
def test_tmem_kernel_edge_shapes(N, n, m, k):
    P, idx, a, b = _params(n, m, k, 1.5, seed=N + n)
    P.set_kernel("tmem")
    g = torch.Generator(device="cuda")
    g.manual_seed(N * 31 + n)
    X = torch.randn((N, n), generator=g, device="cuda")
    _run_and_check(P, idx, a, b, 1.5, X)


def test_tmem_kernel_determinism_and_flags():
    c = configs.get("C1")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w)
    P.set_kernel("tmem")
    X = data.generate(c.data, c.n, 0, 3000, seed=1, device="cuda")
    c1 = fl.fastlsh_hash(P, X)
    parts = torch.cat([fl.fastlsh_hash(P, X[i:j].contiguous()) for i, j in [(0, 999), (999, 3000)]])
    assert torch.equal(c1, fl.fastlsh_hash(P, X)) and torch.equal(c1, parts)
    X[5, :] = float("nan")
    fl.read_flags(P, reset=True)
    codes = fl.fastlsh_hash(P, X).cpu().numpy()
    assert (codes[5] == -(2 ** 31)).all()
    nf, sat = fl.read_flags(P, reset=True)
    assert nf == c.k and sat == 0


# ---- K1r (row-major stages, LDS.32; the auto choice where it applies): same rule, same inputs ---------

ROWS_CASES = [("C0", None, None), ("C1", None, 2003), ("C2", 32, 517), ("C2", 128, 261), ("C2", 512, 131),
              ("C3", None, 4099), ("C4", None, 1001), ("C1", None, 70_001)]


@pytest.mark.parametrize("name,m,N", ROWS_CASES)
def test_rows_kernel_parity(name, m, N):
    c = configs.get(name)
    m = m or c.m
    N = N or c.N
    P, idx, a, b = _params(c.n, m, c.k, c.w, c.seed)
    P.set_kernel("rows")
    assert P.info()["kernel"] == 3
    X = data.generate(c.data, c.n, 0, N, seed=c.seed, device="cuda")
    rows = None if N <= 5000 else _sample_rows(N, 1500, seed=3, extra=[7, 8, 4095, 4096, N - 2])
    rel, amb, codes = _run_and_check(P, idx, a, b, c.w, X, rows=rows)
    assert amb < 1e-2
    P.set_kernel("smem")
    codes_smem = fl.fastlsh_hash(P, X)
    # same Eq. 5 in fp32, different summation orders: codes differ only at fp32 bucket-boundary ties
    assert (codes != codes_smem).float().mean().item() < 1e-3


@pytest.mark.parametrize("N,n,m,k", [(1, 128, 16, 64), (5, 132, 7, 33), (77, 36, 50, 9), (64, 4, 5, 3),
                                     (33, 8, 1, 1), (130, 256, 200, 20), (9, 96, 64, 257), (300, 4, 4, 100),
                                     (17, 4096, 130, 6), (1000, 1000, 300, 70), (8, 2048, 64, 514)])
def test_rows_kernel_edge_shapes(N, n, m, k):
    """Ragged groups (N % 8), k % 4 != 0 (plain code stores), many parts (m > 64), every stride class."""
    P, idx, a, b = _params(n, m, k, 1.5, seed=N + n)
    P.set_kernel("rows")
    g = torch.Generator(device="cuda")
    g.manual_seed(N * 31 + n)
    X = torch.randn((N, n), generator=g, device="cuda")
    _run_and_check(P, idx, a, b, 1.5, X)


def test_rows_kernel_plain_store_path_and_offset_output():
    """The code buffer leaves through 4-byte stores when 16-byte ones cannot be used (forced here, and
    for an output that is not 16-byte aligned); results are identical to the vector path."""
    c = configs.get("C1")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w)
    P.set_kernel("rows")
    X = data.generate(c.data, c.n, 0, 3001, seed=2, device="cuda")
    ref = fl.fastlsh_hash(P, X)
    os.environ["FASTLSH_NO_VEC_STORE"] = "1"
    try:
        plain = fl.fastlsh_hash(P, X)
    finally:
        del os.environ["FASTLSH_NO_VEC_STORE"]
    assert torch.equal(ref, plain)
    buf = torch.empty(X.shape[0] * c.k + 1, dtype=torch.int32, device="cuda")
    out = buf[1:].view(X.shape[0], c.k)  # 4-byte aligned, not 16
    fl.fastlsh_hash(P, X, out=out)
    assert torch.equal(ref, out)


def test_rows_kernel_determinism_and_flags():
    c = configs.get("C1")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w)
    P.set_kernel("rows")
    X = data.generate(c.data, c.n, 0, 3000, seed=1, device="cuda")
    c1 = fl.fastlsh_hash(P, X)
    parts = torch.cat([fl.fastlsh_hash(P, X[i:j].contiguous()) for i, j in [(0, 999), (999, 3000)]])
    assert torch.equal(c1, fl.fastlsh_hash(P, X)) and torch.equal(c1, parts)
    X[5, :] = float("nan")
    X[6, 3] = 1e30
    fl.read_flags(P, reset=True)
    codes = fl.fastlsh_hash(P, X).cpu().numpy()
    assert (codes[5] == -(2 ** 31)).all()
    nf, sat = fl.read_flags(P, reset=True)
    assert nf == c.k
    # row 6: hashes that sample coordinate 3 saturate (|p| ~ 1e30 |a| / w, finite, outside int32)
    idx6 = (idx == 3).any(axis=1)
    assert sat == int(idx6.sum()) and (codes[6][idx6] == -(2 ** 31)).all()


@pytest.mark.parametrize("name,L,K,N", [("C1", 50, 10, 3001), ("C3", 16, 16, 4099), ("C0", 5, 12, 999),
                                         ("C4", 200, 10, 1203), ("C4", 60, 10, 1203), ("C4", 200, 7, 1203),
                                         ("C4", 200, 10, 1), ("C4", 200, 10, 7), ("C1", 50, 10, 5)])
def test_rows_kernel_keys_from_code_tile(name, L, K, N):
    """K1r builds the compound keys from its shared-memory code tile when every CTA hash block holds
    whole tables (C0/C1/C3: one block; C4: 4 blocks of 500 hashes, K = 10 — each block builds its 50
    tables; L = 60: the last two blocks build none); bit-exact vs codes + the standalone key kernel,
    also keys-only (which only the fused path serves) into columns [col0, col0 + N) of a wider table.
    C4 with K = 7 (tables straddle the block boundaries) takes the separate kernel, same result."""
    c = configs.get(name)
    idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, 3)
    P = fl.Params.from_arrays(c.n, c.w, idx, a, b).set_kernel("rows")  # (C0/C3 default to K1j)
    assert P.info()["kernel"] == 3
    Kobj = fl.Keys.from_arrays(philox.key_multipliers(L, K, seed=4))
    X = data.generate(c.data, c.n, 0, N, seed=5, device="cuda")
    codes_f, keys_f = fl.hash_keys(P, Kobj, X)
    codes_p = fl.fastlsh_hash(P, X)
    keys_p = fl.build_keys(Kobj, codes_p)
    assert torch.equal(codes_f, codes_p)
    assert torch.equal(keys_f, keys_p)
    rp = P.row_packing()
    ends = rp["block_h0"] + rp["block_kb"]
    whole_tables = all(h % K == 0 for h in rp["block_h0"]) and all(e % K == 0 or e >= L * K for e in ends)
    assert whole_tables == (K != 7)
    if whole_tables:
        wide = torch.zeros((L, N + 77), dtype=torch.int64, device="cuda")
        _, w2 = fl.hash_keys(P, Kobj, X, keys_out=wide, with_codes=False, col0=77)
        assert torch.equal(w2[:, 77:], keys_p) and (w2[:, :77] == 0).all()


def test_chunked_key_build_equals_whole():
    """Keys built chunk by chunk into columns [c0, c1) of one [L][N] table (the C3 bench path)."""
    c = configs.get("C3")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w)
    Kobj = fl.Keys.create(c.L, c.K, seed=1)
    X = data.generate(c.data, c.n, 0, 10_007, seed=1, device="cuda")
    whole = fl.build_keys(Kobj, fl.fastlsh_hash(P, X))
    keys = torch.empty_like(whole)
    codes = torch.empty((4096, c.k), dtype=torch.int32, device="cuda")
    for c0 in range(0, 10_007, 4096):
        c1 = min(10_007, c0 + 4096)
        cb = codes[:c1 - c0]
        fl.fastlsh_hash(P, X[c0:c1], out=cb)
        fl.build_keys(Kobj, cb, out=keys, col0=c0)
    assert torch.equal(keys, whole)


# ---- bucket tables (R15): bit-exact vs the oracle --------------------------

def _check_tables(keys_np, sk, ids, starts, nb):
    from oracle import tables as otables
    L, N = keys_np.shape
    rsk, rsi, rst = otables.build_tables(keys_np)
    assert np.array_equal(sk.cpu().numpy().view(np.uint64), rsk)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), rsi)
    nbh = nb.cpu().numpy()
    st = starts.cpu().numpy().view(np.uint32)
    for l in range(L):
        assert nbh[l] == len(rst[l])
        assert np.array_equal(st[l, :nbh[l]].astype(np.int64), rst[l])
        assert (st[l, nbh[l]:] == N).all()


@pytest.mark.parametrize("L,N,hi", [(3, 10_000, 50), (2, 4096, 2 ** 61 - 1), (5, 4097, 3), (1, 1, 9), (4, 77_777, 1000),
                                    (2, 300_001, 2 ** 61 - 1)])
def test_tables_bit_exact(L, N, hi):
    rng = np.random.default_rng(L * 1000 + N)
    keys_np = rng.integers(0, hi, size=(L, N), dtype=np.uint64)
    keys = torch.as_tensor(keys_np.view(np.int64)).cuda()
    _check_tables(keys_np, *fl.build_tables(keys))


def test_tables_from_hashed_keys_and_ldk():
    """Tables from real C1 keys (the bench path), keys read with ldk > N."""
    c = configs.get("C1")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w)
    Kobj = fl.Keys.create(c.L, c.K, seed=1)
    X = data.generate(c.data, c.n, 0, 20_000, seed=1, device="cuda")
    keys = fl.build_keys(Kobj, fl.fastlsh_hash(P, X), ldk=20_011)
    keys_np = keys[:, :20_000].cpu().numpy().view(np.uint64)
    _check_tables(keys_np, *fl.build_tables(keys, N=20_000))


def test_tables_empty():
    keys = torch.zeros((3, 0), dtype=torch.int64, device="cuda")
    sk, ids, starts, nb = fl.build_tables(keys)
    assert nb.cpu().tolist() == [0, 0, 0] and starts.cpu().numpy()[:, 0].tolist() == [0, 0, 0]


# ---- query with exact re-ranking (R16) ----------------------------------

def _check_query(ids_g, d_g, nc_g, ids_o, d_o, nc_o, X, Q, cands):
    """GPU query result vs the oracle's (R16), checked on its own terms:
    every returned id is a distinct member of the query's candidate set, its reported distance is its
    true squared distance (recomputed here in fp64 from X and Q), the list is ordered by (distance,
    id), and where the GPU's id at a rank differs from the oracle's, its TRUE distance ties the
    oracle's distance at that rank within the fp32 tolerance (a near-tie may swap ids, never admit a
    farther point)."""
    ids_g, d_g, nc_g = ids_g.cpu().numpy(), d_g.cpu().numpy().astype(np.float64), nc_g.cpu().numpy()
    X = np.asarray(X, np.float64)
    Q = np.asarray(Q, np.float64)
    assert np.array_equal(nc_g, nc_o)  # the distinct candidate counts are integers: exact
    assert np.array_equal(ids_g < 0, ids_o < 0)
    assert np.isinf(d_g[ids_g < 0]).all()
    tol = 1e-5 * np.maximum(1.0, np.abs(np.where(np.isfinite(d_o), d_o, 0.0)))  # fp32 vs double
    for q in range(ids_g.shape[0]):
        live = ids_g[q] >= 0
        got = ids_g[q][live].astype(np.int64)
        assert len(set(got.tolist())) == len(got), f"query {q}: duplicated ids {got}"
        assert set(got.tolist()) <= cands[q], f"query {q}: ids outside the candidate set"
        true = ((X[got] - Q[q]) ** 2).sum(1)
        assert (np.abs(d_g[q][live] - true) <= tol[q][live]).all(), f"query {q}: reported != true distance"
        # ordered by (distance, id): non-decreasing distances, ids ascending among equal distances
        dg = d_g[q][live]
        assert (np.diff(dg) >= 0).all(), f"query {q}: distances not sorted"
        for r in range(len(got) - 1):
            if dg[r] == dg[r + 1]:
                assert got[r] < got[r + 1], f"query {q}: equal distances not ordered by id"
        for r in np.flatnonzero(got != ids_o[q][live]):
            assert abs(true[r] - d_o[q, r]) <= 2 * tol[q, r], (q, r, true[r], d_o[q, r])


@pytest.mark.parametrize("n,N,k,m,w,L,K,topk", [(64, 6000, 24, 8, 2.0, 6, 4, 10), (128, 3000, 16, 16, 8.0, 4, 4, 32),
                                                (32, 1, 8, 4, 1.0, 2, 4, 5)])
def test_query_matches_oracle(n, N, k, m, w, L, K, topk):
    """GPU tables + query on keys from the oracle's codes (so both sides see identical keys) vs
    oracle/query.py; half the queries are data rows (they must find themselves)."""
    from oracle import query as oq
    from oracle import tables as otables
    idx, a, b = fastlsh_arrays(n, m, k, w, 3)
    g = torch.Generator().manual_seed(N + n)
    X = torch.randn((N, n), generator=g) * 2
    Qn = max(1, min(40, N))
    Q = torch.cat([X[torch.arange(Qn) * max(1, N // Qn) % N], torch.randn((40, n), generator=g) * 2])
    r = philox.key_multipliers(L, K, seed=5)
    _, _, cx = oracle.fastlsh(X.numpy(), idx, a, b, w, threads=THREADS)
    _, _, cq = oracle.fastlsh(Q.numpy(), idx, a, b, w, threads=THREADS)
    keys_o = okeys.build_keys(cx, r, L, K)
    qkeys_o = okeys.build_keys(cq, r, L, K)
    sk, si, _ = otables.build_tables(keys_o)
    ids_o, d_o, nc_o = oq.query(X.numpy(), Q.numpy(), sk, si, qkeys_o, topk)
    tables = fl.build_tables(torch.as_tensor(keys_o.view(np.int64)).cuda())
    ids_g, d_g, nc_g = fl.query(X.cuda(), tables, Q.cuda(), torch.as_tensor(qkeys_o.view(np.int64)).cuda(), topk)
    cands = [oq.candidates_brute(keys_o, qkeys_o, q) for q in range(Q.shape[0])]
    _check_query(ids_g, d_g, nc_g, ids_o, d_o, nc_o, X.numpy(), Q.numpy(), cands)
    assert (ids_g.cpu().numpy()[:Qn, 0] >= 0).all()


def test_query_end_to_end_c1_sample():
    """The product path on C1 data: hash + keys + tables + query on the GPU; queries that are data
    rows find themselves first at distance 0 (exact property, no oracle needed)."""
    c = configs.get("C1")
    P, idx, a, b = _params(c.n, c.m, c.k, c.w)
    Kobj = fl.Keys.create(c.L, c.K, seed=1)
    X = data.generate(c.data, c.n, 0, 50_000, seed=1, device="cuda")
    keys = fl.build_keys(Kobj, fl.fastlsh_hash(P, X))
    tables = fl.build_tables(keys)
    sel = torch.arange(0, 50_000, 997, device="cuda")
    qk = keys[:, sel].contiguous()
    ids, dist, nc = fl.query(X, tables, X[sel].contiguous(), qk, topk=10)
    assert torch.equal(ids[:, 0].long(), sel) and (dist[:, 0] == 0).all() and (nc >= 1).all()


# ---- extensions (R17) ------------------------------------------------

def test_transforms_match_oracle():
    from oracle import transforms as ot
    g = torch.Generator().manual_seed(4)
    X = torch.randn((3001, 37), generator=g) * torch.rand((3001, 1), generator=g) * 5
    X[7] = 0.0
    Xd = X.cuda()
    Xn = fl.normalize_rows(Xd).cpu().numpy()
    assert np.allclose(Xn, ot.normalize(X.numpy()), rtol=2e-6, atol=1e-7)
    kap = fl.max_row_norm(Xd)
    kref = ot.max_norm(X.numpy())
    assert abs(kap.item() - kref) <= 1e-6 * kref
    P = fl.mips_transform(Xd, kap).cpu().numpy().astype(np.float64)
    Pr = ot.mips_data(X.numpy(), kap.item())
    assert np.array_equal(P[:, 1:], Pr[:, 1:])  # copied coordinates are exact
    assert np.allclose(P[:, 0] ** 2, Pr[:, 0] ** 2, rtol=0, atol=2e-6 * kref ** 2)  # cancellation-aware bound
    Qt = fl.mips_transform(Xd[:50], query=True).cpu().numpy()
    assert (Qt[:, 0] == 0).all() and np.array_equal(Qt[:, 1:], X[:50].numpy())


def test_mips_pipeline_finds_max_inner_product():
    """End to end on the GPU: P/Q transforms + FastLSH keys + tables + query. Since
    ||P(v) - Q(u)||^2 = kappa^2 + 1 - 2 v.u for ||u|| = 1, the top-1 of the
    distance re-rank must be the candidate with the largest inner product (candidates recomputed
    here from the keys with torch)."""
    g = torch.Generator().manual_seed(6)
    X = (torch.randn((4000, 31), generator=g) * (1 + torch.rand((4000, 1), generator=g))).cuda()
    kap = fl.max_row_norm(X)
    PX = fl.mips_transform(X, kap)
    U = fl.normalize_rows(torch.randn((25, 31), generator=g).cuda())
    QU = fl.mips_transform(U, query=True)
    P = fl.Params.create(32, 16, 8, 2.0, seed=3)
    Kobj = fl.Keys.create(4, 2, seed=3)
    keys = fl.build_keys(Kobj, fl.fastlsh_hash(P, PX))
    qkeys = fl.build_keys(Kobj, fl.fastlsh_hash(P, QU))
    ids, dist, nc = fl.query(PX, fl.build_tables(keys), QU, qkeys, topk=1)
    ip = (U.double() @ X.double().T)
    checked = 0
    for q in range(U.shape[0]):
        cand = (keys == qkeys[:, q:q + 1]).any(dim=0).nonzero().flatten()
        assert nc[q].item() == cand.numel()
        if cand.numel() == 0:
            assert ids[q, 0].item() == -1
            continue
        best = ip[q, cand].max().item()
        got = ids[q, 0].long().item()
        assert ip[q, got].item() >= best - 1e-4 * max(1.0, abs(best))
        d_ref = kap.double().item() ** 2 + 1 - 2 * ip[q, got].item()
        assert abs(dist[q, 0].item() - d_ref) <= 1e-4 * max(1.0, d_ref)
        checked += 1
    assert checked >= 5


def test_fused_keys_only_chunked_equals_separate():
    """Keys-only fused path (codes never written), chunked into one [L][N] table with col0 offsets,
    equals codes + the key kernel (C3 shape: 16 tables of 16 codes)."""
    c = configs.get("C3")
    idx, a, b = fastlsh_arrays(c.n, c.m, c.k, c.w, 2)
    Pf = fl.Params.from_arrays(c.n, c.w, idx, a, b).set_table_size(c.K).set_kernel("smem")
    Pp = fl.Params.from_arrays(c.n, c.w, idx, a, b).set_kernel("smem")
    Kobj = fl.Keys.create(c.L, c.K, seed=7)
    N = 20_011
    X = data.generate(c.data, c.n, 0, N, seed=3, device="cuda")
    ref = fl.build_keys(Kobj, fl.fastlsh_hash(Pp, X))
    keys = torch.full_like(ref, -1)
    for c0 in range(0, N, 8192):
        c1 = min(N, c0 + 8192)
        codes, _ = fl.hash_keys(Pf, Kobj, X[c0:c1], keys_out=keys, with_codes=False, col0=c0)
        assert codes is None
    assert torch.equal(keys, ref)


# ---- K0: the generic kernel for params no specialised kernel packs (n > 4400, huge m) -------------

@pytest.mark.parametrize("N,n,m,k,w", [(257, 5000, 24, 33, 1.5), (40, 64, 20_000, 3, 4.0), (1, 8192, 7, 100, 0.5)])
def test_generic_kernel_parity(N, n, m, k, w):
    P, idx, a, b = _params(n, m, k, w, seed=N + n)
    assert P.info()["kernel"] == 0
    g = torch.Generator(device="cuda")
    g.manual_seed(n + m)
    X = torch.randn((N, n), generator=g, device="cuda")
    _run_and_check(P, idx, a, b, w, X)
    X[0, :] = float("nan")
    fl.read_flags(P, reset=True)
    codes = fl.fastlsh_hash(P, X).cpu().numpy()
    assert (codes[0] == -(2 ** 31)).all()
    assert fl.read_flags(P, reset=True) == (k, 0)
    Kobj = fl.Keys.create(1, min(k, 3), seed=1)
    c2, keys = fl.hash_keys(P, Kobj, X)
    ref = okeys.build_keys(c2.cpu().numpy().astype(np.int64), Kobj.export(), 1, min(k, 3))
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), ref)
