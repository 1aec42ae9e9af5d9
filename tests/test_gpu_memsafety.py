"""Memory-safety and race checks without compute-sanitizer (closed on this GPU pool: "runs under it
have left GPUs needing a reset"; profiles/r02_sanitize_note.txt). VERDICT r1 item 6.

For every kernel family, on ragged shapes:
  * guard bands — outputs are views into larger buffers whose surroundings hold a canary; after the
    launch every canary is intact (no out-of-bounds write) and no output cell still holds the
    sentinel it was filled with (every output written: initcheck's question);
  * poisoned neighbours — the input rows sit between NaN rows; a kernel reading past its rows would
    raise the non-finite counters or change codes;
  * race stress — repeated launches while another stream keeps the GPU busy give bit-identical
    results (a shared-memory / mbarrier race shows up as run-to-run differences).
"""
import numpy as np
import pytest
import torch

import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data

pytestmark = pytest.mark.gpu
G = 4096  # guard elements on each side (16-byte multiple)
CANARY_I32 = 0x5A5A5A5A
SENT_I32 = 2 ** 31 - 2         # no code in these workloads reaches it
CANARY_I64 = 0x5A5A5A5A5A5A5A5A


def _guarded(shape, dtype, canary, sentinel):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * G,), canary, dtype=dtype, device="cuda")
    view = buf[G:G + n].view(*shape)
    view.fill_(sentinel)
    return buf, view


def _guards_ok(buf, n, canary):
    head, tail = buf[:G], buf[G + n:]
    return bool((head == canary).all()) and bool((tail == canary).all())


def _poisoned_rows(X):
    """X's rows inside a buffer with NaN rows before and after (16-byte aligned)."""
    N, n = X.shape
    pad = 64
    buf = torch.full((N + 2 * pad, n), float("nan"), device="cuda")
    buf[pad:pad + N] = X
    return buf[pad:pad + N]


SHAPES = [("C0", "jit", 1003), ("C3", "jit", 70_001), ("C0", "rows", 1003), ("C1", "rows", 2003),
          ("C3", "rows", 4099), ("C4", "rows", 1001), ("C1", "smem", 2003), ("C1", "tmem", 2003)]


@pytest.mark.parametrize("name,kernel,N", SHAPES)
def test_hash_guard_bands_and_poisoned_neighbours(name, kernel, N):
    c = configs.get(name)
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1).set_kernel(kernel)
    X = data.generate(c.data, c.n, 0, N, seed=4, device="cuda")
    ref = fl.fastlsh_hash(P, X)
    Xp = _poisoned_rows(X)
    fl.read_flags(P, reset=True)
    buf, out = _guarded((N, c.k), torch.int32, CANARY_I32, SENT_I32)
    fl.fastlsh_hash(P, Xp, out=out)
    torch.cuda.synchronize()
    assert _guards_ok(buf, N * c.k, CANARY_I32), "write outside the codes"
    assert not bool((out == SENT_I32).any()), "codes left unwritten"
    assert torch.equal(out, ref), "codes depend on rows outside X"
    assert fl.read_flags(P, reset=True) == (0, 0)
    pbuf, proj = _guarded((N, c.k), torch.float32, float("-1e38"), float("inf"))
    fl.fastlsh_project(P, Xp, out=proj)
    torch.cuda.synchronize()
    assert _guards_ok(pbuf, N * c.k, float("-1e38")) and not bool(torch.isinf(proj).any())
    if c.L:
        Kobj = fl.Keys.create(c.L, c.K, seed=2)
        ref_c, ref_k = fl.hash_keys(P, Kobj, X)
        col0, ldk = 37, N + 37 + 29
        kbuf = torch.full((c.L * ldk + 2 * G,), CANARY_I64, dtype=torch.int64, device="cuda")
        table = kbuf[G:G + c.L * ldk].view(c.L, ldk)
        cbuf, codes = _guarded((N, c.k), torch.int32, CANARY_I32, SENT_I32)
        fl.hash_keys(P, Kobj, Xp, codes=codes, keys_out=table, col0=col0)
        torch.cuda.synchronize()
        assert _guards_ok(kbuf, c.L * ldk, CANARY_I64) and _guards_ok(cbuf, N * c.k, CANARY_I32)
        assert bool((table[:, :col0] == CANARY_I64).all()) and bool((table[:, col0 + N:] == CANARY_I64).all())
        assert torch.equal(table[:, col0:col0 + N], ref_k) and torch.equal(codes, ref_c)


def test_key_kernels_guard_bands():
    for L, K, k in ((50, 10, 500), (16, 16, 256), (600, 2, 1201), (3, 7, 22)):
        N = 1337
        codes = data.random_codes(N, k, seed=L + K, lo=-(2 ** 31), hi=2 ** 31 - 1).cuda()
        Kobj = fl.Keys.create(L, K, seed=1)
        ref = fl.build_keys(Kobj, codes)
        kbuf = torch.full((L * N + 2 * G,), CANARY_I64, dtype=torch.int64, device="cuda")
        out = kbuf[G:G + L * N].view(L, N)
        out.fill_(-1)
        fl.build_keys(Kobj, codes, out=out)
        torch.cuda.synchronize()
        assert _guards_ok(kbuf, L * N, CANARY_I64) and torch.equal(out, ref), (L, K, k)


def test_dense_tables_query_transforms_guard_bands():
    c = configs.get("C1")
    X = data.generate(c.data, c.n, 0, 3001, seed=2, device="cuda")
    Pd = fl.Params.e2lsh(c.n, c.k, c.w, seed=1)
    for prec in (1, 3):
        buf, out = _guarded((3001, c.k), torch.int32, CANARY_I32, SENT_I32)
        fl.e2lsh_hash(Pd, _poisoned_rows(X), out=out, precision=prec)
        torch.cuda.synchronize()
        assert _guards_ok(buf, 3001 * c.k, CANARY_I32) and not bool((out == SENT_I32).any())
        assert torch.equal(out, fl.e2lsh_hash(Pd, X, precision=prec))
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1)
    Kobj = fl.Keys.create(c.L, c.K, seed=1)
    _, keys = fl.hash_keys(P, Kobj, X)
    tabs = fl.build_tables(keys)
    tabs2 = fl.build_tables(keys)
    assert all(torch.equal(a, b) for a, b in zip(tabs, tabs2))
    Q = data.generate(c.data, c.n, 10_000, 10_040, seed=2, device="cuda")
    _, qk = fl.hash_keys(P, Kobj, Q)
    r1 = fl.query(X, tabs, Q, qk, topk=10)
    r2 = fl.query(X, tabs, Q, qk, topk=10)
    assert all(torch.equal(a, b) for a, b in zip(r1, r2))
    Y = torch.randn((777, 37), device="cuda")
    buf = torch.full((777 * 37 + 2 * G,), -7.0, device="cuda")
    out = buf[G:G + 777 * 37].view(777, 37)
    fl.normalize_rows(Y, out=out)
    torch.cuda.synchronize()
    assert _guards_ok(buf, 777 * 37, -7.0)


@pytest.mark.parametrize("name,kernel", [("C3", "jit"), ("C1", "rows"), ("C4", "rows"), ("C1", "smem")])
def test_race_stress_bit_identical(name, kernel):
    """20 launches while a second stream runs large copies: identical codes and keys every time."""
    c = configs.get(name)
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1).set_kernel(kernel)
    Kobj = fl.Keys.create(c.L, c.K, seed=1)
    N = 50_000 if c.n <= 1000 else 5_000
    X = data.generate(c.data, c.n, 0, N, seed=6, device="cuda")
    ref_c, ref_k = fl.hash_keys(P, Kobj, X)
    side = torch.cuda.Stream()
    a = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    for i in range(20):
        with torch.cuda.stream(side):
            for _ in range(2):
                b.copy_(a)
        codes, keys = fl.hash_keys(P, Kobj, X)
        assert torch.equal(codes, ref_c) and torch.equal(keys, ref_k), f"run {i} differs"
    torch.cuda.synchronize()
