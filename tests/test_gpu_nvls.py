"""The key all-gather fused into K1j: keys written with multimem.st to
a symmetric-memory multicast table (fastlsh_hash_keys_multicast) vs the plain keys of the same rows.

Runs at world size 1 (one GPU per gpurun call): a multicast object bound to one device is still a
multicast mapping, so the multimem store path, the column offsets and the barrier are exercised; the
NCCL fallback of KeyTable is checked the same way. Skips (with the reason) where the system offers
no multicast support.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist

import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data
from paper_2309_15479_b200.distributed import KeyTable

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def pg():
    torch.cuda.set_device(0)
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["nvls", "nccl"])
def test_keytable_matches_plain_keys(pg, mode):
    c = configs.get("C3")
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1)
    K = fl.Keys.create(c.L, c.K, seed=3)
    N = 70_001
    X = data.generate(c.data, c.n, 0, N, seed=2, device="cuda")
    codes_ref, keys_ref = fl.hash_keys(P, K, X)
    try:
        table = KeyTable(c.L, N, mode=mode)
    except Exception as ex:  # noqa: BLE001
        pytest.skip(f"no NVSwitch multicast here: {ex}")
    assert table.mode == mode
    codes = torch.empty((16_384, c.k), dtype=torch.int32, device="cuda")
    for c0 in range(0, N, 16_384):
        c1 = min(N, c0 + 16_384)
        cb = table.hash_keys(fl, P, K, X[c0:c1], col0=c0, codes=codes[:c1 - c0])
        assert torch.equal(cb, codes_ref[c0:c1])
    table.finish()
    torch.cuda.synchronize()
    assert torch.equal(table.table, keys_ref)


def test_multimem_key_stores_single_device():
    """The multimem.st path of K1j on one GPU: a multicast object bound to this device alone
    (fastlsh_multicast_alloc); keys stored through the multicast address land in the table exactly as
    the plain keys, chunk by chunk at global column offsets, codes unchanged."""
    c = configs.get("C3")
    P = fl.Params.create(c.n, c.m, c.k, c.w, seed=1)
    K = fl.Keys.create(c.L, c.K, seed=3)
    N = 70_001
    X = data.generate(c.data, c.n, 0, N, seed=2, device="cuda")
    codes_ref, keys_ref = fl.hash_keys(P, K, X)
    try:
        mt = fl.MulticastTable(c.L, N + 64)
    except fl.FastLSHError as ex:
        pytest.skip(f"no multicast object on this device: {ex}")
    mt.table.fill_(-1)
    for c0 in range(0, N, 16_384):
        c1 = min(N, c0 + 16_384)
        cb = fl.hash_keys_multicast(P, K, X[c0:c1], mt.mc_ptr, N + 64, col0=32 + c0)
        assert torch.equal(cb, codes_ref[c0:c1])
    torch.cuda.synchronize()
    assert torch.equal(mt.table[:, 32:32 + N], keys_ref)
    assert bool((mt.table[:, :32] == -1).all()) and bool((mt.table[:, 32 + N:] == -1).all())
    mt.close()
