"""Row sharding and the key all-gather.

Rows of X are independent units (every point is hashed by the same functions), so
they shard across ranks with params replicated (each rank regenerates them from the seed — no
broadcast). The only collective on the hot path is the all-gather of compound bucket keys when the
tables are built: every rank contributes its [L][N_local] table-major keys and receives [L][N]
with rank r's rows at columns [offset_r, offset_r + N_r) of every table.

These helpers only arrange torch.distributed calls (NCCL on GPUs, gloo in the CPU tests); all
hashing arithmetic runs in libfastlsh.
"""
from __future__ import annotations


def shard_rows(N: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range [lo, hi) of `rank` for N rows over `world` ranks (sizes differ by <= 1)."""
    if world <= 0 or not (0 <= rank < world) or N < 0:
        raise ValueError("bad sharding arguments")
    base, extra = divmod(N, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def allgather_keys(keys_local, out=None, group=None, wait=True, n_total=None):
    """All-gather table-major keys [L][N_r] (int64 view of u64) into [L][N_total] with rank r's rows
    at columns [lo_r, hi_r) = shard_rows(N_total, world, r) of every table.

    Equal shards go straight into `out` with one all_gather_into_tensor per table (issued
    asynchronously back to back, waited on together, so NCCL pipelines them). Unequal shards
    (N_total % world != 0: sizes differ by one) are padded to the largest shard, gathered into a
    staging buffer and compacted into `out` on the current stream after the collective.
    n_total defaults to world * N_local (equal shards). Returns `out`, or (wait=False) the list of
    pending works: the caller waits on them later (on NCCL that makes its current stream wait),
    e.g. after overlapping the next step's hashing; with unequal shards the compaction then
    happens inside wait=True calls only, so wait=False requires equal shards.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    L, n_local = keys_local.shape
    n_total = world * n_local if n_total is None else int(n_total)
    lo, hi = shard_rows(n_total, world, rank)
    if hi - lo != n_local:
        raise ValueError(f"rank {rank} holds {n_local} rows, shard_rows gives {hi - lo}")
    if out is None:
        out = torch.empty((L, n_total), dtype=keys_local.dtype, device=keys_local.device)
    if tuple(out.shape) != (L, n_total):
        raise ValueError(f"output must be [L, N_total] = [{L}, {n_total}]")
    equal = n_total % world == 0
    if equal:
        works = [dist.all_gather_into_tensor(out[l], keys_local[l].contiguous(), group=group, async_op=True)
                 for l in range(L)]
        if not wait:
            return works
        for w in works:
            w.wait()
        return out
    if not wait:
        raise ValueError("unequal shards: the compaction after the all-gather needs wait=True")
    n_max = -(-n_total // world)
    pad = torch.zeros((L, n_max), dtype=keys_local.dtype, device=keys_local.device)
    pad[:, :n_local].copy_(keys_local)
    staged = torch.empty((L, world * n_max), dtype=keys_local.dtype, device=keys_local.device)
    works = [dist.all_gather_into_tensor(staged[l], pad[l], group=group, async_op=True) for l in range(L)]
    for w in works:
        w.wait()
    for r in range(world):
        a, b = shard_rows(n_total, world, r)
        out[:, a:b].copy_(staged[:, r * n_max:r * n_max + (b - a)])
    return out


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank timing (the multi-GPU timing rule)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])
