"""Host-side checks of libfastlsh (no GPU needed): ABI surface, params generation, packer."""
import ctypes
import os
import re
from collections import Counter

import numpy as np
import pytest

import paper_2309_15479_b200 as fl
from fastlsh_inputs import fastlsh_arrays, e2lsh_arrays, philox, configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2309_15479_b200 import build
    build.build()
    return fl.load_library()


def _declared_functions():
    with open(os.path.join(ROOT, "include", "fastlsh.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fastlsh_\w+|e2lsh_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol(lib):
    decl = _declared_functions()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), f"missing export {name}"
    assert set(decl) == set(fl.EXPORTED)
    assert lib.fastlsh_abi_version() == 1


def test_params_from_seed_match_independent_generator(lib):
    """The library's C++ Philox and fastlsh_inputs' numpy Philox implement the same spec."""
    for (n, m, k, w) in [(128, 16, 64, 4.0), (960, 60, 500, 1.0), (37, 50, 9, 0.5)]:
        p = fl.Params.create(n, m, k, w, seed=1)
        idx, a, b, ww = p.export()
        i2, a2, b2 = fastlsh_arrays(n, m, k, w, seed=1)
        assert np.array_equal(idx, i2) and np.array_equal(a, a2) and np.array_equal(b, b2)
        assert ww == np.float32(w)


def test_e2lsh_params_share_coefficient_stream(lib):
    p = fl.Params.e2lsh(24, 7, 1.0, seed=3)
    idx, a, b, _ = p.export()
    i2, a2, b2 = e2lsh_arrays(24, 7, 1.0, seed=3)
    assert np.array_equal(idx, i2) and np.array_equal(a, a2) and np.array_equal(b, b2)
    assert p.info()["is_e2lsh"] == 1


def test_keys_from_seed_match_independent_generator(lib):
    k = fl.Keys.create(50, 10, seed=1)
    assert np.array_equal(k.export(), philox.key_multipliers(50, 10, seed=1))


@pytest.mark.parametrize("args", [(0, 4, 4, 1.0), (8, 0, 4, 1.0), (8, 4, 0, 1.0), (8, 4, 4, 0.0),
                                  (8, 4, 4, -1.0), (8, 4, 4, float("nan")), (8, 4, 4, float("inf"))])
def test_invalid_params_rejected(lib, args):
    h = ctypes.c_void_p()
    assert lib.fastlsh_params_create(*args, 1, ctypes.byref(h)) == fl.EINVAL
    assert not h.value


def test_from_arrays_rejects_out_of_range_index(lib):
    idx = np.array([[0, 5]], np.int32)
    a = np.ones((1, 2), np.float32)
    b = np.zeros(1, np.float32)
    with pytest.raises(fl.FastLSHError):
        fl.Params.from_arrays(5, 1.0, idx, a, b)
    idx[0, 1] = -1
    with pytest.raises(fl.FastLSHError):
        fl.Params.from_arrays(5, 1.0, idx, a, b)


def test_keys_invalid(lib):
    h = ctypes.c_void_p()
    assert lib.fastlsh_keys_create(0, 3, 1, ctypes.byref(h)) == fl.EINVAL
    r = np.full((1, 2), (1 << 61) - 1, np.uint64)  # not reduced mod p
    assert lib.fastlsh_keys_create_from_arrays(1, 1, r.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h)) == fl.EINVAL


def test_gpu_calls_without_device_fail_loudly(lib):
    """No CPU fallback: hashing needs an uploaded params object on a B200."""
    p = fl.Params.create(16, 4, 8, 1.0, seed=1)
    rc = lib.fastlsh_hash(p._h, ctypes.c_void_p(16), 1, ctypes.c_void_p(16), None)
    assert rc in (fl.ESTATE, fl.ECUDA, fl.EUNSUPPORTED)


def test_e2lsh_precision_argument(lib):
    """e2lsh_hash / e2lsh_project: precision 1 (1xTF32), 2 (3xFP16) and 3 (3xTF32) are accepted (and
    then need a device), anything else is EINVAL before any device work."""
    p = fl.Params.e2lsh(16, 8, 1.0, seed=1)
    V = ctypes.c_void_p(16)
    for prec in (0, 4, -1, 16):
        assert lib.e2lsh_hash(p._h, V, 1, V, prec, None) == fl.EINVAL
        assert lib.e2lsh_project(p._h, V, 1, V, prec, None) == fl.EINVAL
    for prec in (1, 2, 3):
        assert lib.e2lsh_hash(p._h, V, 1, V, prec, None) in (fl.ESTATE, fl.ECUDA, fl.EUNSUPPORTED)


def _unpack(p):
    """Decode the packing into per-(hash, part) slot multisets and check its invariants."""
    pk = p.packing()
    idx, a, b, _ = p.export()
    nq, MS, W, HB, P = pk["nq"], pk["slots"], pk["warps"], pk["hash_blocks"], pk["parts"]
    offs = pk["offp"].astype(np.int64)
    assert (offs % 16 == 0).all()
    pos = offs // 16
    assert (pos < 4 * nq + 8).all()
    coef = pk["coef"]
    # bank groups: at every slot, the 8 lanes of a quarter touch distinct groups (or equal chunks)
    conflicts = 0
    for bl in range(HB):
        for w in range(W):
            for t in range(MS):
                for q in range(4):
                    ps = set(int(x) for x in pos[bl, w, t, 8 * q:8 * q + 8])
                    groups = Counter(x % 8 for x in ps)
                    conflicts += max(groups.values()) - 1
    # padding slots: zero coefficient on a zero chunk
    pad = pos >= 4 * nq
    assert (coef[pad] == 0).all()
    # every hash's multiset {(column, coefficient)} is preserved across its parts
    for bl in range(HB):
        h0, kb = int(pk["block_h0"][bl]), int(pk["block_kb"][bl])
        for hh in range(kb):
            got = Counter()
            for part in range(P):
                lane = int(pk["unit_lane"][bl, hh, part])
                w, l = divmod(lane, 32)
                for t in range(MS):
                    ps = int(pos[bl, w, t, l])
                    if ps < 4 * nq:
                        i, qd = divmod(ps, nq)
                        got[(4 * qd + i, float(coef[bl, w, t, l]))] += 1
            want = Counter((int(c), float(x)) for c, x in zip(idx[h0 + hh], a[h0 + hh]))
            assert got == want, f"hash {h0 + hh}"
    assert sum(int(x) for x in pk["block_kb"]) == p.k
    return pk, conflicts


@pytest.mark.parametrize("n,m,k", [(128, 16, 64), (960, 60, 500), (37, 50, 9), (130, 7, 33), (1, 5, 3),
                                   (784, 64, 200), (256, 200, 20)])
def test_packer_preserves_slots_and_avoids_conflicts(lib, n, m, k):
    p = fl.Params.create(n, m, k, 1.0, seed=5)
    pk, conflicts = _unpack(p)
    info = p.info()
    assert info["slots"] == pk["slots"] and info["slots"] <= 64 and info["slots"] % 2 == 0
    if info["conflict_wavefronts"] == 0:
        assert conflicts == 0
    if n >= 64 and 16 <= m <= 64 and k >= 64:
        assert info["bank_efficiency"] > 0.75


def test_bench_config_packing_quality(lib):
    c = configs.get("C1")
    p = fl.Params.create(c.n, c.m, c.k, c.w, seed=1)
    info = p.info()
    # the cost model splits m=60 into 2 parts so that 16 warps/SM fit (MS <= 32 registers); slots
    # capped at the part size leave only a few folded bank conflicts (< 2% of the wavefronts)
    stage_wavefronts = info["hash_blocks"] * info["warps_per_block"] * 4 * info["slots"]
    assert info["conflict_wavefronts"] <= 0.02 * stage_wavefronts
    assert info["slots"] <= 32 and info["warps_per_block"] == 16
    assert info["bank_efficiency"] >= 0.9


def test_kernel_selection_rules(lib, monkeypatch):
    """fastlsh_params_set_kernel: 0-5 accepted, others EINVAL; K1t needs n % 4 == 0 and m <= 128;
    auto mode never picks the dense path (5, opt-in), K1j (4) for n <= 128 shapes
    (NVRTC present), K1r (3) for other n % 4 == 0 shapes whose row packing exists, else K1;
    FASTLSH_NO_JIT=1 turns K1j off."""
    import paper_2309_15479_b200 as fl
    from fastlsh_inputs import fastlsh_arrays
    idx, a, b = fastlsh_arrays(128, 16, 64, 4.0, 1)
    P = fl.Params.from_arrays(128, 4.0, idx, a, b)
    assert P.info()["kernel"] == 4
    for k in ("smem", "tmem", "rows", "jit", "auto"):
        P.set_kernel(k)
    P.set_kernel("tmem")
    assert P.info()["kernel"] == 2 and P.info()["tmem_hash_blocks"] >= 1
    P.set_kernel("smem")
    assert P.info()["kernel"] == 1
    P.set_kernel("rows")
    assert P.info()["kernel"] == 3
    P.set_kernel("dense")
    assert P.info()["kernel"] == 5
    with pytest.raises(fl.FastLSHError):
        P.set_kernel(6)
    idx, a, b = fastlsh_arrays(130, 16, 64, 4.0, 1)   # n % 4 != 0: no TMA tensor map / bulk rows
    Q = fl.Params.from_arrays(130, 4.0, idx, a, b)
    for kern in ("tmem", "jit", "dense"):
        with pytest.raises(fl.FastLSHError):
            Q.set_kernel(kern)
    assert Q.info()["kernel"] == 1
    idx, a, b = fastlsh_arrays(960, 60, 500, 1.0, 1)  # n > 128: K1j does not apply
    assert fl.Params.from_arrays(960, 1.0, idx, a, b).info()["kernel"] == 3
    # the dense path (kernel 5) is opt-in only: north_star reserves the tensor cores for the E2LSH
    # baseline, so auto keeps the gather kernels on every shape, C2's m sweep included (k = 100 keeps
    # the packers quick)
    for m in (32, 512, 4096):
        assert fl.Params.create(4096, m, 100, 0.5, seed=1).info()["kernel"] == 3, m
    D = fl.Params.create(1000, 200, 100, 1.0, seed=1)
    D.set_kernel("dense")
    assert D.info()["kernel"] == 5
    with pytest.raises(fl.FastLSHError):
        fl.Params.create(1001, 200, 100, 1.0, seed=1).set_kernel("dense")  # n % 4 != 0
    monkeypatch.setenv("FASTLSH_NO_JIT", "1")
    idx, a, b = fastlsh_arrays(128, 16, 64, 4.0, 1)
    assert fl.Params.from_arrays(128, 4.0, idx, a, b).info()["kernel"] == 3


def test_jit_source_compiles_for_sm100a(lib):
    """K1j's generated source (C0 shape: 64 hashes x 16 samples) compiles with NVRTC for sm_100a on
    this CPU-only host; loading the module then needs a driver (ECUDA here, OK on a B200)."""
    import paper_2309_15479_b200 as fl
    from fastlsh_inputs import fastlsh_arrays
    idx, a, b = fastlsh_arrays(128, 16, 64, 4.0, 1)
    P = fl.Params.from_arrays(128, 4.0, idx, a, b)
    try:
        P.prepare()
    except fl.FastLSHError as e:
        assert e.status == fl.ECUDA
    st = P.jit_status()
    assert st["compile_seconds"] > 0, st
    assert "compile failed" not in st["error"], st


def _unpack_rows(p):
    """Decode the K1r packing (rpacker.cpp) and check its invariants; returns (packing, conflicts)."""
    pk = p.row_packing()
    assert pk is not None
    idx, a, b, _ = p.export()
    n, k = p.n, p.k
    P, MS, W, HB, S, S0, n1 = (pk[x] for x in ("parts", "slots", "warps", "hash_blocks", "S", "S0", "n1"))
    hpw = 32 // P
    assert S % 32 == 0 and S0 == 32 * ((n + 31) // 32) + 32 and MS % 2 == 0
    assert 0 <= n1 <= n and n1 % 4 == 0 and (n1 == 0 or S0 + 16 + n1 <= S)
    op = pk["offp"].astype(np.int64)
    offs = np.empty((HB, W, MS, 32), np.int64)
    offs[:, :, 0::2, :] = op & 0xFFFF
    offs[:, :, 1::2, :] = op >> 16
    assert (offs % 4 == 0).all()
    word = offs // 4
    coef = pk["coef"]
    copy1 = (word >= S0 + 16) & (word < S0 + 16 + n1)
    pad = (word >= n) & ~copy1
    assert ((word[pad] >= S0 - 32) & (word[pad] < S0)).all() and (word < S).all()  # pads read the zero tail
    assert (coef[pad] == 0).all()
    coord = np.where(copy1, word - (S0 + 16), word)  # the coordinate a (non-pad) slot reads
    # bank conflicts: distinct words at one slot position must lie in distinct banks
    conflicts = 0
    for bl in range(HB):
        for w in range(W):
            for t in range(MS):
                ws = set(int(x) for x in word[bl, w, t])
                conflicts += max(Counter(x % 32 for x in ws).values()) - 1
    # block boundaries: multiples of 4 (16-byte code runs), covering all k hashes in order
    h0s, kbs = pk["block_h0"], pk["block_kb"]
    assert int(h0s[0]) == 0 and int(kbs.sum()) == k
    assert all(int(h0s[i + 1]) == int(h0s[i] + kbs[i]) for i in range(HB - 1))
    assert all(int(x) % 4 == 0 for x in kbs[:-1])
    lh = pk["lane_hash"]
    for bl in range(HB):
        h0, kb = int(h0s[bl]), int(kbs[bl])
        seen = Counter()
        for w in range(W):
            for l in range(32):
                h = int(lh[bl, w, l])
                # parts of hash slot j = lanes j + hpw*q, and the hash is congruent to j mod hpw
                assert h == int(lh[bl, w, l % hpw])
                if h < 0:
                    assert (coef[bl, w, :, l] == 0).all()
                    continue
                assert h % hpw == l % hpw and 0 <= h < kb
                if l < hpw:
                    seen[h] += 1
        assert sorted(seen) == list(range(kb)) and set(seen.values()) == {1}
        for hh in range(kb):
            w = next(w for w in range(W) if hh in set(int(x) for x in lh[bl, w]))
            lanes = [l for l in range(32) if int(lh[bl, w, l]) == hh]
            assert len(lanes) == P
            got = Counter()
            for l in lanes:
                for t in range(MS):
                    if not pad[bl, w, t, l]:
                        got[(int(coord[bl, w, t, l]), float(coef[bl, w, t, l]))] += 1
            want = Counter((int(c), float(x)) for c, x in zip(idx[h0 + hh], a[h0 + hh]))
            assert got == want, f"hash {h0 + hh}"
    return pk, conflicts


@pytest.mark.parametrize("n,m,k", [(128, 16, 64), (960, 60, 500), (36, 50, 9), (128, 7, 33), (4, 5, 3),
                                   (784, 64, 200), (256, 200, 20), (4096, 32, 130), (1000, 130, 6)])
def test_row_packer_preserves_slots_and_banks(lib, n, m, k):
    """K1r packing: every hash's (coordinate, coefficient) multiset is kept across its parts, padding
    reads zeros, parts sit in lanes j + (32/P)q with hash = j mod 32/P, and the reported conflict
    count matches the decoded slot table (0 for these shapes unless folding was chosen)."""
    p = fl.Params.create(n, m, k, 1.0, seed=5)
    pk, conflicts = _unpack_rows(p)
    assert conflicts == pk["conflicts"]


def test_row_packer_bench_configs(lib):
    """The bench-relevant shapes pack with few padding slots (two-copy staging flattens the bank
    loads that limit a single copy) and no bank conflicts."""
    # floors: C1 sits at its bound (max bank total 1001 / 16 warps -> 63 -> MS 64), C3 at its
    # bank-pair bound (MS 18), C4 takes P = 2 (16-warp CTAs beat 8-warp MS = 72 on the GPU)
    for name, m, floor in (("C1", None, 0.91), ("C3", None, 0.88), ("C4", None, 0.8), ("C2", 32, 0.85)):
        c = configs.get(name)
        m = m or c.m
        p = fl.Params.create(c.n, m, c.k, c.w, seed=1)
        pk = p.row_packing()
        assert pk is not None, name
        useful = c.k * m
        slots = pk["hash_blocks"] * pk["warps"] * 32 * pk["slots"]
        assert useful / slots >= floor, (name, useful / slots, pk["slots"], pk["parts"])
        # C4's cheapest packing caps the slots at 64 and folds the rest (measured faster than padding)
        wavefronts = pk["hash_blocks"] * pk["warps"] * pk["slots"]
        assert pk["conflicts"] <= (0.15 * wavefronts if name == "C4" else 0), (name, pk["conflicts"])


@pytest.mark.parametrize("n,m,k", [(960, 60, 500), (784, 64, 2000), (128, 16, 256), (4096, 32, 1000), (96, 40, 37)])
def test_epilogue_partial_reads_conflict_free(lib, n, m, k):
    """The 8 consecutive hashes an epilogue quarter-warp reads have their part-q partials in 8
    distinct bank groups (lane % 8) for every part q (packer.cpp: König colouring of positions)."""
    import paper_2309_15479_b200 as fl
    from fastlsh_inputs import fastlsh_arrays
    idx, a, b = fastlsh_arrays(n, m, k, 1.0, 2)
    pk = fl.Params.from_arrays(n, 1.0, idx, a, b).packing()
    for bl in range(pk["hash_blocks"]):
        kb = int(pk["block_kb"][bl])
        ul = pk["unit_lane"][bl, :kb, :].astype(np.int64)
        for o in range(0, kb, 8):
            for q in range(pk["parts"]):
                pos = ul[o:o + 8, q] % 8
                assert len(set(pos.tolist())) == len(pos), (bl, o, q, pos)


@pytest.mark.parametrize("n,m,k", [(128, 16, 256), (128, 16, 64), (128, 16, 77)])
def test_direct_packing_warp_contiguous(lib, n, m, k):
    """One-part packings take the direct epilogue (packer.cpp, gather_impl.cuh): warp w of a block
    holds exactly the hashes [32w, 32w+32) of the block, so its code stores are contiguous runs;
    with FASTLSH_NO_DIRECT the packer may place hashes in any warp."""
    import os
    import paper_2309_15479_b200 as fl
    from fastlsh_inputs import fastlsh_arrays
    idx, a, b = fastlsh_arrays(n, m, k, 1.0, 3)
    pk = fl.Params.from_arrays(n, 1.0, idx, a, b).packing()
    assert pk["parts"] == 1
    for bl in range(pk["hash_blocks"]):
        kb = int(pk["block_kb"][bl])
        lanes = pk["unit_lane"][bl, :kb, 0].astype(np.int64)
        assert (lanes // 32 == np.arange(kb) // 32).all()
        assert len(set(lanes.tolist())) == kb
    os.environ["FASTLSH_NO_DIRECT"] = "1"
    try:
        pk2 = fl.Params.from_arrays(n, 1.0, idx, a, b).packing()
    finally:
        del os.environ["FASTLSH_NO_DIRECT"]
    assert pk2["slots"] <= pk["slots"]  # the unconstrained grouping never needs more slots


def test_table_query_transform_argument_checks(lib):
    """Size/pointer validation of the table, query and transform entry points happens before any
    device work (EINVAL, no crash); valid calls without a B200 fail loudly, never on the CPU."""
    c_size = ctypes.c_size_t()
    assert lib.fastlsh_tables_workspace(0, 10, ctypes.byref(c_size)) == fl.EINVAL
    assert lib.fastlsh_tables_workspace(3, -1, ctypes.byref(c_size)) == fl.EINVAL
    assert lib.fastlsh_tables_workspace(50, 1_000_000, ctypes.byref(c_size)) == fl.OK and c_size.value > 50 * 12e6
    V = ctypes.c_void_p(256)
    assert lib.fastlsh_build_tables(V, 0, 10, 10, V, V, V, V, V, 1 << 30, None) == fl.EINVAL   # L = 0
    assert lib.fastlsh_build_tables(V, 2, 10, 5, V, V, V, V, V, 1 << 30, None) == fl.EINVAL    # ldk < N
    assert lib.fastlsh_query_workspace(-1, 3, ctypes.byref(c_size)) == fl.EINVAL
    assert lib.fastlsh_query(V, 10, 4, V, V, 2, V, V, 3, 3, 0, V, V, V, V, 1 << 30, None) == fl.EINVAL   # topk 0
    assert lib.fastlsh_query(V, 10, 4, V, V, 2, V, V, 3, 3, 33, V, V, V, V, 1 << 30, None) == fl.EINVAL  # topk > 32
    assert lib.fastlsh_query(V, 10, 4, V, V, 2, V, V, 3, 2, 5, V, V, V, V, 1 << 30, None) == fl.EINVAL   # ldq < nq
    assert lib.fastlsh_normalize_rows(V, -1, 4, V, None) == fl.EINVAL
    assert lib.fastlsh_mips_transform(V, 5, 4, None, 0, V, None) == fl.EINVAL  # data transform needs kappa
    rc = lib.fastlsh_normalize_rows(V, 5, 4, V, None)
    assert rc in (fl.ECUDA, fl.EUNSUPPORTED)


@pytest.mark.parametrize("n,dual", [(4, True), (128, True), (256, True), (512, True), (516, False), (960, False),
                                    (4096, False)])
def test_row_packing_stage_classes(lib, n, dual):
    """Rows of n <= 512 are staged twice (second copy rotated 16 banks, n1 = n); longer rows once.
    The staged stride is a multiple of 32 words and holds copy 0, its zero tail and copy 1."""
    p = fl.Params.create(n, 16, 64, 1.0, seed=2)
    pk = p.row_packing()
    assert pk is not None
    S, S0, n1 = pk["S"], pk["S0"], pk["n1"]
    assert S % 32 == 0 and S0 == 32 * ((n + 31) // 32) + 32
    assert n1 == (n if dual else 0)
    assert (S0 + 16 + n1 <= S) if dual else (S0 <= S)


@pytest.mark.parametrize("n,m,k,w,L,K", [(128, 16, 256, 4.0, 16, 16), (36, 5, 100, 1.5, 4, 20), (64, 1, 32, 0.75, 1, 32)])
def test_jit_variants_compile(lib, n, m, k, w, L, K):
    """Every K1j variant's generated source compiles for sm_100a (NVRTC, no GPU): codes, projections,
    codes + keys, keys only, multicast keys; k % 32 == 0 (paired 3D code stores) and k % 32 != 0
    (2D boxes), power-of-two and IEEE-division w, m = 1."""
    import paper_2309_15479_b200 as fl
    from fastlsh_inputs import fastlsh_arrays
    idx, a, b = fastlsh_arrays(n, m, k, w, 5)
    P = fl.Params.from_arrays(n, w, idx, a, b)
    Kobj = fl.Keys.create(L, K, seed=2)
    assert P.jit_check(Kobj, what=0b11111) > 0
