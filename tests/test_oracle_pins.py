"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these compares the oracle with itself: each check is a paper-printed example, a hand
computation, a closed form, an invariance, a different formulation (dense matmul) or a
statistical law the hash must obey.
"""
import math
import os

import numpy as np
import pytest

import oracle
from oracle import brute, keys, theory
from fastlsh_inputs import philox, fastlsh_arrays, e2lsh_arrays

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            key, *vals = line.split()
            out[key] = [float(x) for x in vals]
    return out


# ---- P1 sampling operator -------------------------------------------------------------------

def test_paper_sampling_example():
    """v={1,3,5,7,9}, S={2,4,2} (1-based) -> S(v)={3,7,3}."""
    g = _golden("paper_sampling_example.txt")
    S = np.array([int(s) - 1 for s in g["S_1based"]], np.int32)
    assert list(oracle.apply_sampling(g["v"], S)) == g["S_v"]
    assert brute.sample(g["v"], list(S)) == g["S_v"]


def test_sampling_identity_repeated_and_n1():
    v = np.arange(7, dtype=np.float64) * 1.5
    assert list(oracle.apply_sampling(v, np.arange(7, dtype=np.int32))) == list(v)
    assert list(oracle.apply_sampling(v, np.zeros(3, np.int32))) == [0.0, 0.0, 0.0]
    assert list(oracle.apply_sampling(v, np.array([4, 4, 1], np.int32))) == [6.0, 6.0, 1.5]
    # n = 1: the only index is 0
    assert (philox.sample_indices(1, 9, 4, seed=5) == 0).all()


# ---- P2 hash formula ------------------------------------------------------------------------

def test_dyadic_hash_case():
    """Eq. 5 on the worked example with dyadic a, b, w: projection 3.5, code 1 (hand computed)."""
    g = _golden("dyadic_hash_case.txt")
    X = np.array([g["v"]], np.float32)
    idx = np.array([[int(s) - 1 for s in g["S_1based"]]], np.int32)
    a = np.array([g["a"]], np.float32)
    b = np.array(g["b"], np.float32)
    p, scale, code = oracle.fastlsh(X, idx, a, b, g["w"][0])
    assert p[0, 0] == g["projection"][0]
    assert code[0, 0] == g["code"][0]
    assert scale[0, 0] == pytest.approx(math.sqrt(1 + 0.25 + 1) * math.sqrt(9 + 49 + 9), rel=1e-15)
    assert brute.fastlsh_hash(g["v"], list(idx[0]), g["a"], g["b"][0], g["w"][0]) == (3.5, 1)


def test_zero_coefficients_and_offset_shift():
    """a = 0 gives floor(b/w) = 0 for b in [0,w); b -> b+w adds exactly 1."""
    X, idx, a, b = _case(50, 16, 8, 12, w=2.0, seed=3)
    _, _, c0 = oracle.fastlsh(X, idx, np.zeros_like(a), b, 2.0)
    assert (c0 == 0).all()
    # dyadic data so that p + b and p + b + w are exact: small integers, coefficients in 1/8ths
    Xd = np.round(X * 4).astype(np.float32)
    ad = (np.round(a * 8) / 8).astype(np.float32)
    bd = (np.round(b * 8) / 8 % 2.0).astype(np.float32)
    _, _, c1 = oracle.fastlsh(Xd, idx, ad, bd, 2.0)
    _, _, c2 = oracle.fastlsh(Xd, idx, ad, (bd + 2.0).astype(np.float32), 2.0)
    assert (c2 == c1 + 1).all()


def test_power_of_two_scaling_invariance():
    """Scaling X, b and w by 2^e leaves every code unchanged (exact in binary fp; Fact 4.5 analog)."""
    X, idx, a, b = _case(40, 32, 20, 16, w=1.5, seed=4)
    p1, _, c1 = oracle.fastlsh(X, idx, a, b, 1.5)
    for e in (-3, 2, 7):
        f = np.float32(2.0 ** e)
        p2, _, c2 = oracle.fastlsh(X * f, idx, a, b * f, 1.5 * float(f))
        assert (c1 == c2).all()
        assert np.array_equal(p2, p1 * float(f))


def test_floor_toward_minus_infinity():
    """Codes of negative quotients round toward -inf, and boundaries are half-open."""
    X = np.array([[-1.0, 0.5, 2.0]], np.float32)
    idx = np.array([[0], [1], [2]], np.int32)
    a = np.array([[1.0], [1.0], [1.0]], np.float32)
    b = np.zeros(3, np.float32)
    _, _, c = oracle.fastlsh(X, idx, a, b, 1.0)
    assert list(c[0]) == [-1, 0, 2]


# ---- P3 E2LSH special case ------------------------------------------------------------------

def test_identity_plan_equals_e2lsh_bit_exact():
    """With S = identity and m = n, Eq. 5 reduces to Eq. 1."""
    n, k = 24, 40
    idx, A, b = e2lsh_arrays(n, k, 1.0, seed=9)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((30, n)).astype(np.float32)
    pf, sf, cf = oracle.fastlsh(X, idx, A, b, 1.0)
    pe, se, ce = oracle.e2lsh(X, A, b, 1.0)
    assert np.array_equal(pf, pe) and np.array_equal(sf, se) and np.array_equal(cf, ce)


def test_projection_equals_dense_merged_matrix():
    """a.S(v) = v . A' with A'[c] = sum of a_j over slots j with idx_j = c (duplicates merged) —
    an independent formulation through a library matmul; catches index/transpose/duplicate bugs."""
    X, idx, a, b = _case(64, 37, 50, 24, w=1.0, seed=11)  # m > n: many duplicates
    p, _, _ = oracle.fastlsh(X, idx, a, b, 1.0)
    A = np.zeros((idx.shape[0], X.shape[1]))
    for i in range(idx.shape[0]):
        np.add.at(A[i], idx[i], a[i].astype(np.float64))
    ref = X.astype(np.float64) @ A.T
    assert np.allclose(p, ref, rtol=1e-12, atol=1e-12)


# ---- P9 brute force -------------------------------------------------------------------------

def test_brute_force_equals_c_oracle_bit_exact():
    X, idx, a, b = _case(20, 12, 7, 6, w=0.75, seed=21)
    p, _, c = oracle.fastlsh(X, idx, a, b, 0.75)
    bp, bc = brute.hash_all(X.tolist(), idx.tolist(), a.tolist(), b.tolist(), 0.75)
    assert np.array_equal(p, np.array(bp)) and np.array_equal(c, np.array(bc))


# ---- P4 E2LSH collision statistics ----------------------------------------------------------

def test_e2lsh_closed_form_matches_quadrature_of_eq2():
    for s in (0.3, 1.0, 2.0, 5.0):
        for w in (0.5, 1.0, 4.0):
            assert theory.p_e2lsh(s, w) == pytest.approx(theory.p_e2lsh_integral(s, w), abs=1e-10)
    assert theory.p_e2lsh(2.0, 4.0) == pytest.approx(0.609548, abs=1e-6)


def _collision_rate(codes):
    return float(np.mean(codes[0] == codes[1]))


@pytest.mark.parametrize("s,w", [(1.0, 4.0), (2.0, 4.0), (3.0, 2.0)])
def test_e2lsh_collision_rate_matches_closed_form(s, w):
    """Empirical Pr[h(v)=h(u)] over T independent E2LSH functions = Eq. 2 within 4 sigma."""
    n, T = 8, 200_000
    rng = np.random.default_rng(int(s * 10 + w))
    A = rng.standard_normal((T, n)).astype(np.float32)
    b = (rng.random(T) * w).astype(np.float32)
    d = rng.standard_normal(n)
    d = d / np.linalg.norm(d) * s
    v = rng.standard_normal(n).astype(np.float32)
    u = (v - d).astype(np.float32)
    s_true = float(np.linalg.norm(v.astype(np.float64) - u.astype(np.float64)))
    _, _, c = oracle.e2lsh(np.stack([v, u]), A, b, w, threads=4)
    p = theory.p_e2lsh(s_true, w)
    assert abs(_collision_rate(c) - p) < 4 * math.sqrt(p * (1 - p) / T)


# ---- P5 / P7 FastLSH collision statistics ---------------------------------------------------

def _fast_collisions(v, u, m, w, T, seed):
    n = len(v)
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, n, size=(T, m)).astype(np.int32)
    a = rng.standard_normal((T, m)).astype(np.float32)
    b = (rng.random(T) * w).astype(np.float32)
    _, _, c = oracle.fastlsh(np.stack([np.asarray(v, np.float32), np.asarray(u, np.float32)]), idx, a, b, w, threads=4)
    return _collision_rate(c)


@pytest.mark.parametrize("w", [1.0, 2.0, 4.0])
def test_fastlsh_collision_rate_matches_exact_enumeration(w):
    """Pr[h(v)=h(u)] = E_S[p_E2(||S(v-u)||; w)] (2-stability), enumerated over all
    5^3 multisets (with replacement). A 'without replacement' or shifted-index
    oracle would be off by >= 0.04 here, far outside 4 sigma (~0.0045)."""
    v, u, m, T = [3.0, 0.5, 0.0, 1.0, 0.0], [0.0] * 5, 3, 200_000
    p = theory.p_fastlsh_exact_enum(v, u, m, w)
    emp = _fast_collisions(v, u, m, w, T, seed=int(w * 7))
    assert abs(emp - p) < 4 * math.sqrt(p * (1 - p) / T)


def test_fastlsh_lsh_property_monotone_in_distance():
    """Collision probability decreases with distance: exact and empirical."""
    rng = np.random.default_rng(5)
    n, m, w, T = 32, 8, 2.0, 100_000
    v = rng.standard_normal(n)
    d = rng.standard_normal(n)
    d /= np.linalg.norm(d)
    exact, emp = [], []
    for t in (0.5, 1.5, 3.0, 6.0):
        u = v - t * d
        exact.append(theory.p_fastlsh_exact_mc(v, u, m, w, draws=100_000, seed=1))
        emp.append(_fast_collisions(v, u, m, w, T, seed=int(t * 10)))
    assert all(x > y for x, y in zip(exact, exact[1:]))
    assert all(x > y for x, y in zip(emp, emp[1:]))
    for e, x in zip(emp, exact):
        assert abs(e - x) < 0.01


def test_fastlsh_asymptotically_e2lsh_with_scaled_width():
    """Cor. 4.7: as m grows, p_fast(w~) -> p_E2(s; w) with w~ = sqrt(m/n) w
    (reading R7) on a smooth pair."""
    rng = np.random.default_rng(8)
    n, w = 256, 4.0
    v = rng.random(n)
    u = v + 0.15 * rng.standard_normal(n)
    s = float(np.linalg.norm(v - u))
    target = theory.p_e2lsh(s, w)
    errs = []
    for m in (4, 16, 64, 256):
        errs.append(abs(theory.p_fastlsh_exact_mc(v, u, m, theory.width_equivalent(w, m, n), seed=m) - target))
    assert errs[-1] < 0.006 and errs[2] < 0.006
    assert errs[0] > errs[-1]


def test_eq9_agrees_on_smooth_pairs_only():
    """Thm 4.4 / Eq. 9 is a CLT approximation: within 2e-3 of the exact value
    for smooth pairs (sigma/mu <= 2, m >= 16); far off for a spiky pair (reading R13)."""
    rng = np.random.default_rng(12)
    n, m, w = 128, 30, 1.0
    v = rng.random(n)
    u = v + 0.05 * rng.standard_normal(n)
    s, mu, var = theory.pair_stats(v, u)
    assert math.sqrt(var) / mu < 2.0
    assert abs(theory.p_fastlsh_eq9(v, u, m, w) - theory.p_fastlsh_exact_mc(v, u, m, w, draws=400_000)) < 2e-3
    spiky_u = v.copy()
    spiky_u[0] += 3.0
    assert abs(theory.p_fastlsh_eq9(v, spiky_u, m, w) - theory.p_fastlsh_exact_mc(v, spiky_u, m, w)) > 0.1


# ---- P6 exact moments -----------------------------------------------------------------------

def test_projection_moments_exact():
    """E[dP^2] = m s^2 / n and E[dP^4] = 3 (m sigma^2 + m^2 mu^2) (untruncated Lemma 4.8,
    PAPER.md:308-323) for dP = a.(S(v) - S(u)), estimated over T oracle hashes."""
    rng = np.random.default_rng(2)
    n, m, T = 16, 6, 400_000
    v = rng.random(n).astype(np.float32)
    u = (v + rng.standard_normal(n) * 0.5).astype(np.float32)
    idx = rng.integers(0, n, size=(T, m)).astype(np.int32)
    a = rng.standard_normal((T, m)).astype(np.float32)
    b = np.zeros(T, np.float32)
    p, _, _ = oracle.fastlsh(np.stack([v, u]), idx, a, b, 1.0, threads=4)
    dp = p[0] - p[1]
    m2, m4 = theory.exact_moments(v.astype(np.float64), u.astype(np.float64), m)
    assert np.mean(dp ** 2) == pytest.approx(m2, rel=0.01)
    assert np.mean(dp ** 4) == pytest.approx(m4, rel=0.04)


# ---- P10 keys ---------------------------------------------------------------------------------

def test_keys_hand_computed():
    r = [[5, 7]]
    assert keys.key([3], r[0], 1, 0) == 5 + 7 * 3
    assert keys.key([-1], r[0], 1, 0) == (5 + 7 * 0xFFFFFFFF) % keys.P61
    big = [[keys.P61 - 1, keys.P61 - 2, 3]]
    # (p-1) + (p-2)*2 + 3*4 = 3p + 7 - 4 ... reduce by hand: (-1) + (-2)(2) + 12 = 7 mod p
    assert keys.key([2, 4], big[0], 2, 0) == 7


def test_keys_equal_and_distinct_tuples():
    L, K = 6, 5
    r = philox.key_multipliers(L, K, seed=1)
    rng = np.random.default_rng(0)
    codes = rng.integers(-3, 3, size=(400, L * K)).astype(np.int32)
    codes[1] = codes[0]
    kk = keys.build_keys(codes, r, L, K)
    assert (kk[:, 0] == kk[:, 1]).all()
    for l in range(L):
        tuples = {}
        for v in range(codes.shape[0]):
            t = tuple(codes[v, l * K:(l + 1) * K])
            if t in tuples:
                assert kk[l, v] == kk[l, tuples[t]]
            tuples.setdefault(t, v)
        # distinct tuples -> distinct keys on this set
        assert len(set(kk[l].tolist())) == len(tuples)


def test_keys_linearity_mod_p():
    L, K = 3, 4
    r = philox.key_multipliers(L, K, seed=2)
    c1 = np.array([[1, -2, 3, 4] * L], np.int32)
    c2 = np.array([[1, -2, 3, 9] * L], np.int32)
    k1 = keys.build_keys(c1, r, L, K)
    k2 = keys.build_keys(c2, r, L, K)
    for l in range(L):
        assert (int(k2[l, 0]) - int(k1[l, 0])) % keys.P61 == (int(r[l, 4]) * 5) % keys.P61


# ---- helpers ------------------------------------------------------------------------------------

def _case(N, n, m, k, w, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((N, n)).astype(np.float32)
    idx, a, b = fastlsh_arrays(n, m, k, w, seed)
    return X, idx, a, b


# ---- bucket tables (§3.2; reading R15) ----------------------------------------

def test_tables_oracle_matches_brute_grouping():
    """build_tables (library sort) == a pure-Python dictionary grouping of (key, id) per table."""
    from oracle import tables
    rng = np.random.default_rng(5)
    L, N = 4, 600
    keys = rng.integers(0, 40, size=(L, N), dtype=np.uint64)  # many collisions
    keys[1] = rng.integers(0, 2 ** 61 - 1, size=N, dtype=np.uint64)  # (almost) all distinct
    keys[2, :] = 7  # one bucket
    sk, si, starts = tables.build_tables(keys)
    for l in range(L):
        ref = tables.buckets_brute(keys[l])
        got = {}
        bounds = list(starts[l]) + [N]
        for b in range(len(starts[l])):
            s, e = bounds[b], bounds[b + 1]
            assert (sk[l][s:e] == sk[l][s]).all()
            got[int(sk[l][s])] = [int(x) for x in si[l][s:e]]
        assert got == ref
        assert list(got.keys()) == sorted(ref.keys())  # buckets in ascending key order
        assert sorted(si[l].tolist()) == list(range(N))  # a permutation of the rows


def test_tables_oracle_hand_example():
    """Hand-written table: keys (5, 3, 5, 9, 3) -> buckets {3: [1, 4], 5: [0, 2], 9: [3]}."""
    from oracle import tables
    sk, si, starts = tables.build_tables(np.array([[5, 3, 5, 9, 3]], dtype=np.uint64))
    assert sk[0].tolist() == [3, 3, 5, 5, 9]
    assert si[0].tolist() == [1, 4, 0, 2, 3]
    assert starts[0].tolist() == [0, 2, 4]


# ---- query with exact re-ranking (reading R16) -------------------------

def test_query_oracle_candidates_and_ranking():
    """Candidates == points sharing a key with the query in some table (computed from the keys, no
    tables); the top-k == a brute-force sort of those candidates by (distance, id)."""
    from oracle import query as oq
    from oracle import tables as otables
    rng = np.random.default_rng(9)
    N, n, L, nq, topk = 400, 6, 3, 12, 5
    X = rng.standard_normal((N, n)).astype(np.float32)
    keys = rng.integers(0, 25, size=(L, N), dtype=np.uint64)
    Q = rng.standard_normal((nq, n)).astype(np.float32)
    qkeys = rng.integers(0, 30, size=(L, nq), dtype=np.uint64)  # some keys absent from every table
    sk, si, _ = otables.build_tables(keys)
    ids, dist, ncand = oq.query(X, Q, sk, si, qkeys, topk)
    for q in range(nq):
        cand = oq.candidates_brute(keys, qkeys, q)
        assert ncand[q] == len(cand)
        ref = sorted(((float(((X[c].astype(np.float64) - Q[q]) ** 2).sum()), c) for c in cand))[:topk]
        got = [(d, i) for d, i in zip(dist[q], ids[q]) if i >= 0]
        assert [i for _, i in got] == [c for _, c in ref]
        assert np.allclose([d for d, _ in got], [d for d, _ in ref], rtol=0, atol=1e-12)
        assert (ids[q][len(ref):] == -1).all() and np.isinf(dist[q][len(ref):]).all()


def test_query_oracle_point_finds_itself():
    """A query equal to a data point shares all its keys, so the point is a candidate at distance 0
    and comes first (ties at distance 0 by id)."""
    from oracle import query as oq
    from oracle import tables as otables
    rng = np.random.default_rng(2)
    X = rng.standard_normal((200, 4)).astype(np.float32)
    keys = rng.integers(0, 1 << 40, size=(4, 200), dtype=np.uint64)
    sk, si, _ = otables.build_tables(keys)
    sel = np.array([0, 17, 199])
    ids, dist, ncand = oq.query(X, X[sel], sk, si, keys[:, sel], 3)
    assert ids[:, 0].tolist() == sel.tolist() and (dist[:, 0] == 0).all()


# ---- extensions: angular and MIPS transforms (reading R17) --------

def test_transforms_oracle_pins():
    from oracle import transforms as ot
    rng = np.random.default_rng(11)
    X = rng.standard_normal((300, 7)) * rng.uniform(0.1, 3, size=(300, 1))
    X[5] = 0.0
    Xn = ot.normalize(X)
    nz = np.arange(300) != 5
    assert np.allclose(np.linalg.norm(Xn[nz], axis=1), 1.0) and (Xn[5] == 0).all()
    # hand case: (3, 4) -> (0.6, 0.8)
    assert np.allclose(ot.normalize(np.array([[3.0, 4.0]])), [[0.6, 0.8]])
    kappa = ot.max_norm(X)
    P = ot.mips_data(X, kappa)
    assert np.allclose(np.linalg.norm(P, axis=1), kappa)  # every transformed row has norm kappa
    U = rng.standard_normal((40, 7))
    U /= np.linalg.norm(U, axis=1, keepdims=True)
    Qt = ot.mips_query(U)
    # the paper's identity: argmax inner product == argmin l2 distance after P / Q (||u|| = 1)
    d = ((P[None, :, :] - Qt[:, None, :]) ** 2).sum(-1)
    assert (np.argmin(d, axis=1) == np.argmax(U @ X.T, axis=1)).all()
    # ||P(v) - Q(u)||^2 = kappa^2 + 1 - 2 v.u exactly (closed form)
    assert np.allclose(d, kappa ** 2 + 1 - 2 * (U @ X.T))
