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
    e.g. after overlapping the next step's hashing; with unequal shards the one pending object's
    wait() also does the compaction (so the staging buffer lives until then).
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
    n_max = -(-n_total // world)
    pad = torch.zeros((L, n_max), dtype=keys_local.dtype, device=keys_local.device)
    pad[:, :n_local].copy_(keys_local)
    staged = torch.empty((L, world * n_max), dtype=keys_local.dtype, device=keys_local.device)
    works = [dist.all_gather_into_tensor(staged[l], pad[l], group=group, async_op=True) for l in range(L)]
    pending = _CompactingWait(works, staged, out, n_total, world, n_max)
    if not wait:
        return [pending]
    pending.wait()
    return out


class _CompactingWait:
    """The pending all-gather of unequal shards: wait() waits for the collectives, then compacts the
    padded blocks into `out` (on the caller's current stream, as an NCCL work's wait orders it)."""

    def __init__(self, works, staged, out, n_total, world, n_max):
        self.works, self.staged, self.out = works, staged, out
        self.n_total, self.world, self.n_max = n_total, world, n_max

    def wait(self):
        for w in self.works:
            w.wait()
        for r in range(self.world):
            a, b = shard_rows(self.n_total, self.world, r)
            self.out[:, a:b].copy_(self.staged[:, r * self.n_max:r * self.n_max + (b - a)])
        self.works = []
        return True


def table_owner(l: int, world: int) -> int:
    """Rank that owns table l in the table-sharded exchange (round robin)."""
    return l % world


def alltoall_keys_by_table(keys_local, n_total: int, group=None, wait=True):
    """The table-sharded alternative to the all-gather ("an all-to-all by table,
    G x less ingress"): table l goes to rank l % G, which receives every rank's rows of it.

    keys_local is this rank's [L][N_r] table-major keys (rows shard_rows(n_total, G, r)); returns
    (tables, keys) with tables the list of table ids this rank owns and keys [len(tables)][n_total]
    holding them for ALL rows in global row order. Per rank the traffic is (G-1)/G of its own keys
    out and the same amount in, instead of (G-1)/G of the whole [L][N] table in (all-gather): at
    C3, G = 8, 2.8 GB vs 22.4 GB per rank and step. One all_to_all_single with split sizes (NCCL on
    GPUs, gloo in the CPU tests), then a local reorder of the received blocks. wait=False returns
    [pending] instead: pending.wait() finishes the collective, does the reorder (on the caller's
    current stream) and returns (tables, keys) — the bench overlaps it with the next step's hashing.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    L, n_local = keys_local.shape
    lo, hi = shard_rows(n_total, world, rank)
    if hi - lo != n_local:
        raise ValueError(f"rank {rank} holds {n_local} rows, shard_rows gives {hi - lo}")
    owned = [[l for l in range(L) if table_owner(l, world) == d] for d in range(world)]
    # send buffer: for destination d, its tables' rows of this rank, table after table
    send = torch.cat([keys_local[owned[d]].reshape(-1) for d in range(world)]) if L else keys_local.reshape(-1)
    in_splits = [len(owned[d]) * n_local for d in range(world)]
    sizes = [shard_rows(n_total, world, r) for r in range(world)]
    mine = owned[rank]
    out_splits = [len(mine) * (b - a) for a, b in sizes]
    recv = torch.empty(sum(out_splits), dtype=keys_local.dtype, device=keys_local.device)
    work = dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=out_splits,
                                  input_split_sizes=in_splits, group=group, async_op=True)
    pending = _ReorderWait(work, recv, send, mine, sizes, n_total)
    return [pending] if not wait else pending.wait()


class _ReorderWait:
    """The pending table-sharded exchange: wait() waits for the all-to-all, then places each source
    rank's block of the owned tables at its global rows; returns (tables, keys)."""

    def __init__(self, work, recv, send, mine, sizes, n_total):
        self.work, self.recv, self.send, self.mine, self.sizes, self.n_total = work, recv, send, mine, sizes, n_total
        self.result = None

    def wait(self):
        import torch
        if self.result is not None:
            return self.result
        self.work.wait()
        mine, recv = self.mine, self.recv
        out = torch.empty((len(mine), self.n_total), dtype=recv.dtype, device=recv.device)
        off = 0
        for a, b in self.sizes:
            out[:, a:b].copy_(recv[off:off + len(mine) * (b - a)].view(len(mine), b - a))
            off += len(mine) * (b - a)
        self.result = (mine, out)
        self.send = self.recv = None
        return self.result


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank timing (the multi-GPU timing rule)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])


class KeyTable:
    """The global [L][N_total] key table of a row-sharded build.

    mode "nvls": the table lives in torch symmetric memory with an NVSwitch multicast mapping; K1j
    writes every key with multimem.st straight into all GPUs' copies while it hashes
    (fastlsh_hash_keys_multicast), so the all-gather overlaps the hashing tile by tile and finishing
    it is one group barrier. mode "nccl": keys are built into a rank-local [L][N_r] buffer and
    all-gathered with NCCL (allgather_keys) — used when multicast is unavailable or the params are not
    served by K1j. `mode` is decided at construction ("auto" tries nvls first)."""

    def __init__(self, L: int, n_total: int, group=None, device=None, mode: str = "auto"):
        import torch
        import torch.distributed as dist
        self.L, self.n_total, self.group = L, n_total, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.lo, self.hi = shard_rows(n_total, self.world, self.rank)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.mode, self.handle, self.table, self.local = None, None, None, None
        self.why = ""
        if mode in ("auto", "nvls"):
            try:
                import torch.distributed._symmetric_memory as symm
                # ask before allocating: without multicast the [L][N_total] symmetric buffer would be wasted
                if not symm._SymmetricMemory.has_multicast_support(symm.DeviceType.CUDA, self.device.index or 0):
                    raise RuntimeError("no multicast support on this device (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED)")
                t = symm.empty((L, n_total), dtype=torch.int64, device=self.device)
                name = (group or dist.group.WORLD).group_name
                h = symm.rendezvous(t, name)
                if not getattr(h, "multicast_ptr", 0):
                    raise RuntimeError("symmetric memory has no multicast mapping on this system")
                self.mode, self.handle, self.table = "nvls", h, t
            except Exception as ex:  # noqa: BLE001 (fall back, record why)
                self.why = f"{type(ex).__name__}: {ex}"
                if mode == "nvls":
                    raise
        if self.mode is None:
            self.mode = "nccl"
            self.local = torch.empty((L, self.hi - self.lo), dtype=torch.int64, device=self.device)
            self.table = torch.empty((L, n_total), dtype=torch.int64, device=self.device)

    @property
    def multicast_ptr(self) -> int:
        return int(self.handle.multicast_ptr) if self.handle is not None else 0

    def hash_keys(self, fl, params, keys, X, col0: int, codes=None, stream=None):
        """Hash rows [col0, col0 + N) of this rank's shard (X) and place their keys (global columns
        lo + col0 ...). Returns the codes tensor (or None)."""
        if self.mode == "nvls":
            return fl.hash_keys_multicast(params, keys, X, self.multicast_ptr, self.n_total, self.lo + col0,
                                          codes=codes, with_codes=codes is not None, stream=stream)
        c, _ = fl.hash_keys(params, keys, X, codes=codes, keys_out=self.local, col0=col0,
                            with_codes=codes is not None, stream=stream)
        return c

    def finish(self, wait: bool = True):
        """Complete the exchange: nvls — a group barrier (every rank's multicast stores are visible
        afterwards); nccl — the all-gather of the local keys into the table."""
        if self.mode == "nvls":
            self.handle.barrier()
            return []
        return allgather_keys(self.local, out=self.table, group=self.group, wait=wait, n_total=self.n_total)
