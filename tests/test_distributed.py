"""Multi-rank host logic on CPU (gloo, world size 2): sharding, key all-gather layout, timing max,
and determinism of keys across shardings (the oracle computes the reference keys)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_15479_b200.distributed import allgather_keys, alltoall_keys_by_table, max_over_ranks, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_rows_cover_and_balance():
    for N in (0, 1, 7, 10, 1000, 200_000_000):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_rows(N, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == N
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


def _worker(rank, world, port, q, N):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from fastlsh_inputs import philox
        from oracle import keys as okeys
        L, K = 5, 4
        lo, hi = shard_rows(N, world, rank)
        rng = np.random.default_rng(0)
        codes = rng.integers(-50, 50, size=(N, L * K)).astype(np.int32)  # same on every rank
        r = philox.key_multipliers(L, K, seed=9)
        # each rank computes keys of its own rows (here with the exact oracle: host logic test)
        local = okeys.build_keys(codes[lo:hi], r, L, K).view(np.int64)
        out = allgather_keys(torch.from_numpy(local.copy()), n_total=N)
        full = okeys.build_keys(codes, r, L, K).view(np.int64)
        ok_layout = np.array_equal(out.numpy(), full)
        # the bench's overlapped form: works returned unwaited, waited before the buffer is reused
        # (unequal shards: one pending object whose wait() also compacts the padded blocks)
        out2 = torch.zeros_like(out)
        works = allgather_keys(torch.from_numpy(local.copy()), out=out2, wait=False, n_total=N)
        for w in works:
            w.wait()
        ok_layout = ok_layout and len(works) == (L if N % world == 0 else 1) and np.array_equal(out2.numpy(), full)
        # the table-sharded exchange: this rank receives its tables (l % world == rank) for all rows
        mine, tab = alltoall_keys_by_table(torch.from_numpy(local.copy()), N)
        ok_layout = ok_layout and mine == [l for l in range(L) if l % world == rank]
        ok_layout = ok_layout and np.array_equal(tab.numpy(), full[mine])
        (pend,) = alltoall_keys_by_table(torch.from_numpy(local.copy()), N, wait=False)  # the overlapped form
        mine2, tab2 = pend.wait()
        ok_layout = ok_layout and mine2 == mine and np.array_equal(tab2.numpy(), full[mine])
        m = max_over_ranks(1.0 + rank)
        q.put((rank, ok_layout, m))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 12), (3, 13), (3, 2)])
def test_allgather_keys_layout_gloo(world, N):
    """World sizes 2 and 3, equal and unequal shards (N % world != 0: sizes differ by one, and a
    rank with no rows at all for N < world): the gathered [L][N] is the table-major global layout."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, N)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, m in res:
        assert ok, f"rank {rank}: gathered keys are not the table-major global layout"
        assert m == float(world)
