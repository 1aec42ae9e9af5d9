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


def allgather_keys(keys_local, out=None, group=None, wait=True):
    """All-gather table-major keys [L][N_local] (int64 view of u64) into [L][world * N_local].

    Equal shard sizes are required (all_gather_into_tensor semantics); the per-table calls are
    issued asynchronously back to back and waited on together, so NCCL pipelines them. Returns `out`,
    or (wait=False) the list of pending works: the caller waits on them later (on NCCL that makes
    its current stream wait), e.g. after overlapping the next step's hashing.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    L, n_local = keys_local.shape
    if out is None:
        out = torch.empty((L, world * n_local), dtype=keys_local.dtype, device=keys_local.device)
    if out.shape != (L, world * n_local):
        raise ValueError("output must be [L, world * N_local]")
    works = [dist.all_gather_into_tensor(out[l], keys_local[l].contiguous(), group=group, async_op=True)
             for l in range(L)]
    if not wait:
        return works
    for w in works:
        w.wait()
    return out


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank timing (the multi-GPU timing rule)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])
