#!/usr/bin/env python
"""Benchmark of the FastLSH hot path on B200 (BASELINE.json metric: hashes/s and roofline fraction).

One step = one pass of the whole hot path over the workload resident in HBM:
  K1 fastlsh_hash (stage X, gather S_i(v), project, +b, /w, floor, int32 codes)
  K3 fastlsh_build_keys (L tables of K codes -> 64-bit keys)
  (N>1 GPUs) NCCL all-gather of the keys, one all_gather_into_tensor per table.
Default workload: BASELINE.json configs[1] (C1: N=1e6, n=960, k=500, m=60, w=1, L=50 x K=10).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl reference]

Rank 0 prints ONE JSON line. See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FastLSH hashes/sec (N*k) and % of HBM/smem roofline"
SMEM_GATHERS_PER_CLK_PER_SM = 32  # one 128-B wavefront of 4-B words per SM per clock


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the measured region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.gpu), "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if r[3].replace(".", "").isdigit()), default=None)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _cores():
    return len(os.sched_getaffinity(0))


def cpu_baseline(cfg, seconds_target: float = 12.0):
    """The CPU oracle as it stands, on a bounded row sample of the same workload, all host cores."""
    import oracle
    from fastlsh_inputs import data, fastlsh_arrays
    idx, a, b = fastlsh_arrays(cfg.n, cfg.m, cfg.k, cfg.w, cfg.seed)
    cores = _cores()
    # calibrate on a small sample, then size the measured sample to ~seconds_target
    rows0 = 256
    X0 = data.generate(cfg.data, cfg.n, 0, rows0, seed=cfg.seed).numpy()
    t = time.perf_counter()
    oracle.fastlsh(X0, idx, a, b, cfg.w, threads=cores)
    dt = max(time.perf_counter() - t, 1e-4)
    rows = int(min(cfg.N, max(rows0, rows0 * seconds_target / dt)))
    X = data.generate(cfg.data, cfg.n, 0, rows, seed=cfg.seed).numpy()
    t = time.perf_counter()
    oracle.fastlsh(X, idx, a, b, cfg.w, threads=cores)
    dt = time.perf_counter() - t
    return {"value": rows * cfg.k / dt, "unit": "hashes/s", "cores": cores, "kind": "oracle",
            "sample": f"first {rows} of {cfg.N} rows ({cfg.name}), double-precision oracle, OpenMP "
                      f"{cores} threads, {dt:.2f} s (codes only; keys not included)",
            "seconds": dt}


def run_reference(args, cfg):
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    steps = []
    for _ in range(args.warmup):
        cpu_baseline(cfg, seconds_target=2.0)
    for _ in range(args.steps):
        steps.append(cpu_baseline(cfg, seconds_target=args.ref_seconds))
    vals = [s["value"] for s in steps]
    v = statistics.median(vals)
    cb = dict(steps[-1])
    cb["value"] = v
    cb.pop("seconds", None)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "hashes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(s["seconds"] for s in steps),
            "higher_is_better": True, "scaling": "strong" if cfg.name == "C3" else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_dict(cfg, world),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "hashes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _config_dict(cfg, world, n_rank=None, n_total=None, chunks=1):
    n_rank = cfg.N if n_rank is None else n_rank
    n_total = cfg.N * world if n_total is None else n_total
    d = {"workload": f"{cfg.name}: N={n_rank} rows/GPU, n={cfg.n}, k={cfg.k}, m={cfg.m}, w={cfg.w}, "
                     f"keys L={cfg.L} x K={cfg.K}, recipe {cfg.data}",
         "N_per_gpu": n_rank, "n": cfg.n, "k": cfg.k, "m": cfg.m, "w": cfg.w, "L": cfg.L, "K": cfg.K,
         "global_rows": n_total, "parallelism": f"row-sharded x{world}, params replicated",
         "l2": f"inputs {n_rank * cfg.n * 4 / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)"}
    if chunks > 1:
        d["chunks_per_step"] = chunks
    return d


def _packing_summary(P, info, fused_keys):
    """The GPU layout of the kernel that ran (K1r's row packing, else K1's)."""
    rp = P.row_packing() if info["kernel"] == 3 and not fused_keys else None
    if rp is not None:
        lanes = rp["hash_blocks"] * rp["warps"] * 32 * rp["slots"]
        return {"kernel": "K1r", "parts": rp["parts"], "slots": rp["slots"], "warps_per_block": rp["warps"],
                "hash_blocks": rp["hash_blocks"], "staged_row_words": rp["S"],
                "bank_efficiency": P.k * P.m / lanes, "conflict_wavefronts": rp["conflicts"]}
    return {"kernel": "K1", **{k: info[k] for k in ("parts", "slots", "warps_per_block", "hash_blocks",
                                                    "bank_efficiency", "conflict_wavefronts")}}


def _traffic_from_profiles(cfg, rows: int):
    """DRAM bytes per launch of the dominant kernel, from the committed `ncu --set full` capture
    (profiles/ncu_gather_full.json: dram__bytes_read + dram__bytes_write of one K1 launch on the
    same params), scaled per row to this launch's row count. None if no capture is committed."""
    path = os.path.join(ROOT, "profiles", "ncu_gather_full.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if d.get("config", "C1") != cfg.name:
            return None
        return d["dram_bytes_per_row"] * rows
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense E2LSH comparator")
    ap.add_argument("--fused-keys", action="store_true",
                    help="K1 with keys built in its epilogue (set_table_size; measured slower than K1r)")
    ap.add_argument("--keys-from-tile", action="store_true",
                    help="time the step with K1r building the keys from its code tile (one launch) instead of "
                         "codes + the key kernel; the default reports it as a side measurement")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-overlap", action="store_true",
                    help="N > 1: wait for each step's key all-gather before the next step hashes")
    ap.add_argument("--chunk-rows", type=int, default=8_388_608, help="C3: rows hashed per chunk")
    ap.add_argument("--no-tables", action="store_true", help="skip the bucket-table build and query measurements")
    ap.add_argument("--queries", type=int, default=10_000, help="queries answered in the query measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    from fastlsh_inputs import configs
    cfg = configs.get(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist
    import paper_2309_15479_b200 as fl
    from paper_2309_15479_b200.distributed import allgather_keys
    from fastlsh_inputs import data

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    P = fl.Params.create(cfg.n, cfg.m, cfg.k, cfg.w, seed=cfg.seed)
    Kobj = fl.Keys.create(cfg.L, cfg.K, seed=cfg.seed) if cfg.L else None
    if Kobj is not None and args.fused_keys:
        P.set_table_size(cfg.K)  # whole tables per CTA: keys are built in K1's epilogue
    info = P.info()
    # C3 is a fixed 2e8-row dataset sharded over the ranks (strong scaling) and hashed in chunks:
    # its codes (204.8 GB) do not fit one GPU, so only a chunk of codes lives at a time while the
    # keys of all rows are built into [L][N]. Other configs are per-GPU workloads.
    from paper_2309_15479_b200.distributed import shard_rows
    strong = cfg.name == "C3"
    if strong:
        N_total = cfg.N
        lo, hi = shard_rows(N_total, world, rank)
    else:
        lo, hi = rank * cfg.N, (rank + 1) * cfg.N
        N_total = world * cfg.N
    N = hi - lo
    chunk = min(N, args.chunk_rows) if strong else N
    bounds = [(c0, min(N, c0 + chunk)) for c0 in range(0, N, chunk)]
    X = data.generate(cfg.data, cfg.n, lo, hi, seed=cfg.seed, device=dev)
    codes = torch.empty((chunk, cfg.k), dtype=torch.int32, device=dev)
    keys = torch.empty((cfg.L, N), dtype=torch.int64, device=dev) if Kobj else None
    gathered = torch.empty((cfg.L, world * N), dtype=torch.int64, device=dev) if (Kobj and world > 1) else None
    # N > 1: the key all-gather of step j runs on NCCL's stream while step j+1 hashes into the other
    # keys buffer (double-buffered); step j+1 waits for it before launching its own all-gather
    overlap = gathered is not None and not args.no_overlap
    keys_bufs = [keys, torch.empty_like(keys)] if overlap else [keys]
    pending = []  # NCCL works of the previous step's all-gather
    step_no = [0]
    stream = torch.cuda.current_stream()

    fused_keys = bool(Kobj) and args.fused_keys
    # default: K1r builds the keys from its shared-memory code tile (one launch per chunk) when one
    # CTA hash block covers all k hashes (C1, C3)
    rp = P.row_packing() if info["kernel"] == 3 else None
    tile_keys_ok = (bool(Kobj) and not fused_keys and rp is not None and rp["hash_blocks"] == 1
                    # the library's rule (api.cu rows_keys_pay): key work small next to the gathers
                    and cfg.L * cfg.K <= 0.75 * rp["hash_blocks"] * rp["warps"] * rp["slots"])
    # Default step: K1r codes, then the key kernel, so the dominant kernel's roofline is the hashing
    # kernel's own. The one-launch variant (keys from K1r's code tile) is timed on the side.
    rows_fused = tile_keys_ok and args.keys_from_tile
    launches_per_step = len(bounds) * (1 + (1 if (Kobj and not fused_keys and not rows_fused) else 0))
    ev = []

    def step(record: bool):
        marks = []  # per chunk: (before hash, after hash, after keys)
        keys = keys_bufs[step_no[0] % len(keys_bufs)]
        step_no[0] += 1
        for c0, c1 in bounds:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if record else None
            if record:
                e[0].record(stream)
            cb = codes[:c1 - c0]
            if rows_fused:
                fl.hash_keys(P, Kobj, X[c0:c1], codes=cb, keys_out=keys, col0=c0)  # one launch: codes + keys
                if record:
                    e[1].record(stream)
            elif Kobj and args.fused_keys:
                if strong:  # keys only: the codes of the 2e8 rows never reach HBM
                    fl.hash_keys(P, Kobj, X[c0:c1], keys_out=keys, with_codes=False, col0=c0)
                else:
                    fl.hash_keys(P, Kobj, X, codes=codes, keys_out=keys)  # one launch: codes + keys
                if record:
                    e[1].record(stream)
            else:
                fl.fastlsh_hash(P, X[c0:c1], out=cb)
                if record:
                    e[1].record(stream)
                if Kobj:
                    fl.build_keys(Kobj, cb, out=keys, col0=c0)
            if record:
                e[2].record(stream)
                marks.append(e)
        ea = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if record else None
        if record:
            ea[0].record(stream)
        if gathered is not None:
            if overlap:
                for w in pending:  # the previous step's all-gather (overlapped with this step's hashing)
                    w.wait()
                pending[:] = allgather_keys(keys, out=gathered, wait=False)
            else:
                allgather_keys(keys, out=gathered)
        if record:
            ea[1].record(stream)
            ev.append((marks, ea))

    def drain():
        for w in pending:
            w.wait()
        pending.clear()

    smi_index = local
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            smi_index = int(vis.split(",")[local])
        except Exception:
            pass
    sampler = ClockSampler(smi_index)
    sampler.start()
    for _ in range(args.warmup):
        step(False)
    drain()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step(True)
    drain()  # the last step's all-gather is inside the timed region
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    total_ms = t0.elapsed_time(t1)
    hash_ms = [sum(m[0].elapsed_time(m[1]) for m in marks) for marks, _ in ev]
    keys_ms = [sum(m[1].elapsed_time(m[2]) for m in marks) for marks, _ in ev]
    ag_ms = [ea[0].elapsed_time(ea[1]) for _, ea in ev]
    tt = torch.tensor([total_ms, statistics.mean(hash_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_ms_max, hash_ms_max = float(tt[0]), float(tt[1])
    ms_per_step = total_ms_max / args.steps
    hashes_per_step = N_total * cfg.k
    value = hashes_per_step / (ms_per_step / 1e3)

    # roofline of the dominant kernel (K1): smem gathers vs the north_star bound
    peaks = _peaks()
    t_hash = statistics.mean(hash_ms) / 1e3
    gathers = N * cfg.k * cfg.m
    g_peak = 148 * SMEM_GATHERS_PER_CLK_PER_SM * peaks["sm_max_mhz"] * 1e6
    hbm_bytes = 4.0 * N * cfg.n + 4.0 * N * cfg.k
    t_roof = max(hbm_bytes / (peaks["hbm_gbs"] * 1e9), gathers / g_peak)
    t_roof_nominal = max(hbm_bytes / 8.0e12, gathers / g_peak)
    roofline = {"bound": "smem", "achieved": gathers / t_hash / 1e9, "peak": g_peak / 1e9,
                "unit": "Ggather/s", "frac": (gathers / t_hash) / g_peak,
                "traffic": _traffic_from_profiles(cfg, N),
                "kernel": ("gather_kernel (K1 fastlsh_hash, keys fused in its epilogue)" if fused_keys else
                           "rows_kernel (K1r fastlsh_hash_keys: row-major stages, LDS.32; keys built from its "
                           "shared-memory code tile)" if rows_fused else
                           {1: "gather_kernel (K1 fastlsh_hash)", 2: "tmem_gather_kernel (K1t fastlsh_hash)",
                            3: "rows_kernel (K1r fastlsh_hash: row-major stages, LDS.32)"}[info["kernel"]]),
                "algorithmic_per_launch": {"gathers": gathers, "hbm_bytes": hbm_bytes},
                "north_star_frac": t_roof / t_hash, "north_star_frac_nominal_8TBs": t_roof_nominal / t_hash,
                "hbm_achieved_gbs": hbm_bytes / t_hash / 1e9, "hbm_peak_gbs": peaks["hbm_gbs"],
                "peak_source": peaks["source"] + f"; smem peak = 148 SM x 32 x {peaks['sm_max_mhz']:.0f} MHz",
                "kernel_share_of_step": statistics.mean(hash_ms) / ms_per_step if ms_per_step else None}

    # side measurement: the same step with the keys built from K1r's code tile (one launch)
    tile_keys = None
    if tile_keys_ok and not rows_fused and not strong:
        torch.cuda.synchronize()
        for _ in range(2):
            fl.hash_keys(P, Kobj, X, codes=codes, keys_out=keys)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fl.hash_keys(P, Kobj, X, codes=codes, keys_out=keys)
        e1.record(stream)
        torch.cuda.synchronize()
        t_ms = e0.elapsed_time(e1) / args.steps
        tile_keys = {"ms_per_step": t_ms, "value": N * cfg.k / (t_ms / 1e3), "unit": "hashes/s",
                     "note": "hash + keys in one K1r launch (fastlsh_hash_keys), rank-local, same inputs; "
                             "not the headline step"}

    # bucket tables of this rank's keys: stable radix sort of
    # (key, id) per table + bucket starts — timed separately, not part of the hashing step
    tables = None
    if Kobj is not None and not args.no_tables:
        ws = None
        out_t = None
        try:
            out_t = fl.build_tables(keys)
            need = out_t  # allocate once, then time re-builds into the same buffers
            t_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize()
            t_ev[0].record(stream)
            for _ in range(3):
                fl.build_tables(keys, out=out_t, workspace=ws)
            t_ev[1].record(stream)
            torch.cuda.synchronize()
            tms = t_ev[0].elapsed_time(t_ev[1]) / 3
            entries = cfg.L * N
            tables = {"ms": tms, "entries": entries, "entries_per_s": entries / (tms / 1e3),
                      "buckets_table0": int(out_t[3][0].item()),
                      "hbm_bytes_algorithmic": entries * (8 * 8 + 8 * 24 + 8 + 4),
                      "note": "8 LSD radix passes (hist 8 B + scatter 12 B in / 12 B out per entry) + bucket starts"}
            tables["hbm_frac"] = tables["hbm_bytes_algorithmic"] / (tms / 1e3) / (_peaks()["hbm_gbs"] * 1e9)
            del out_t, need
        except Exception as ex:  # noqa: BLE001 (report, never hide a failure)
            tables = {"error": str(ex)}

    # queries: fresh rows of the same distribution are hashed,
    # keyed and answered against the tables (exact re-ranking, top-10); recall@10 against exact
    # nearest neighbours on a 100-query sample (rank 0). Timed separately from the hashing step.
    queries = None
    if Kobj is not None and not args.no_tables and not strong and rank == 0:
        try:
            nq = args.queries
            Qd = data.generate(cfg.data, cfg.n, N_total + 10_000_000, N_total + 10_000_000 + nq, seed=cfg.seed,
                               device=dev)
            tabs = fl.build_tables(keys)
            qcodes = torch.empty((nq, cfg.k), dtype=torch.int32, device=dev)

            def qstep():
                fl.fastlsh_hash(P, Qd, out=qcodes)
                qk = fl.build_keys(Kobj, qcodes)
                return fl.query(X, tabs, Qd, qk, topk=10)
            qstep()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            q0.record(stream)
            res = qstep()
            q1.record(stream)
            torch.cuda.synchronize()
            qms = q0.elapsed_time(q1)
            qids = res[0].cpu().numpy()
            ncand = res[2].double().cpu().numpy()
            # exact 10-NN of the first 100 queries (fp64 on the host) for recall@10
            ns = min(100, nq)
            Xh64 = X.cpu().numpy()
            Qh = Qd[:ns].cpu().numpy().astype(np.float64)
            xx = (Xh64.astype(np.float64) ** 2).sum(1)
            hits = 0
            for i in range(ns):
                dd = xx - 2.0 * (Xh64 @ Qh[i]) + (Qh[i] ** 2).sum()
                truth = set(np.argpartition(dd, 10)[:10].tolist())
                hits += len(truth & set(qids[i][qids[i] >= 0].tolist()))
            del Xh64
            queries = {"queries": nq, "ms": qms, "queries_per_s": nq / (qms / 1e3),
                       "mean_candidates": float(ncand.mean()), "max_candidates": float(ncand.max()),
                       "recall_at_10": hits / (10.0 * ns), "recall_sample": ns,
                       "note": "hash + keys + bucket probes + exact re-rank (top 10) of fresh rows; "
                               "recall vs exact 10-NN (fp64 host) on the first queries"}
            del tabs, Qd, qcodes, res
        except Exception as ex:  # noqa: BLE001
            queries = {"error": str(ex)}

    # on-box comparator: the dense E2LSH GEMM (tcgen05, m = n) on the same rows, k and w
    dense = None
    if not args.no_dense:
        Pd = fl.Params.e2lsh(cfg.n, cfg.k, cfg.w, seed=cfg.seed)
        dense = {}
        Nd = min(N, chunk)  # C3: the comparator runs on one chunk of rows
        Xd, cd = X[:Nd], codes[:Nd]
        for prec in (3, 1):
            fl.e2lsh_hash(Pd, Xd, out=cd, precision=prec)
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            d0.record(stream)
            for _ in range(3):
                fl.e2lsh_hash(Pd, Xd, out=cd, precision=prec)
            d1.record(stream)
            torch.cuda.synchronize()
            ms = d0.elapsed_time(d1) / 3
            kpad = (cfg.k + 255) // 256 * 256
            dense[f"tf32x{prec}"] = {"ms": ms, "rows": Nd, "hashes_per_s": Nd * cfg.k / (ms / 1e3),
                                     "mma_tflops": 2.0 * Nd * cfg.n * kpad * prec / (ms / 1e3) / 1e12,
                                     "fastlsh_hash_speedup": (ms / Nd) / (statistics.mean(hash_ms) / N)}
        dense["note"] = ("e2lsh_hash on E2LSH params (m = n) of the same k, w and rows; tf32x3 is the "
                         "parity-gated comparator (3xTF32), tf32x1 the ungated reference point")
        del Pd

    # end to end through the public host-buffer API: H2D of X, hash + keys, D2H of codes + keys
    # (C3: on a 2M-row sample of each shard; the host would need 307 GB for the whole shard at G=1)
    Ne = N if not strong else min(N, 2_097_152)
    Xh = X[:Ne].cpu().pin_memory()
    codes_h = torch.empty((Ne, cfg.k), dtype=torch.int32).pin_memory()
    keys_h = torch.empty((cfg.L, Ne), dtype=torch.int64).pin_memory() if Kobj else None
    fl.hash_host(P, Kobj, Xh, codes_h, keys_h, chunk_rows=131072)  # warm (workspace allocation)
    if world > 1:
        dist.barrier()
    te = time.perf_counter()
    for _ in range(args.e2e_steps):
        fl.hash_host(P, Kobj, Xh, codes_h, keys_h, chunk_rows=131072)
    e2e_s = (time.perf_counter() - te) / args.e2e_steps
    et = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e = {"value": world * Ne * cfg.k / float(et[0]), "unit": "hashes/s",
           "h2d_bytes_per_step": int(Xh.numel() * 4),
           "d2h_bytes_per_step": int(codes_h.numel() * 4 + (keys_h.numel() * 8 if keys_h is not None else 0)),
           "api": "fastlsh_hash_host (pinned host buffers, 2-stream chunked pipeline)", "steps": args.e2e_steps,
           "rows_per_gpu": Ne}
    del Xh, codes_h, keys_h

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(cfg)
        cb.pop("seconds", None)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "hashes/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if strong else "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, resident in HBM)",
                "config": _config_dict(cfg, world, N, N_total, len(bounds)), "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps,
                "clocks": clocks,
                "keys_fused": "K1 epilogue" if fused_keys else "K1r code tile" if rows_fused else False,
                "keys_from_code_tile": tile_keys,
                "breakdown_ms": {"hash": statistics.mean(hash_ms), "keys": statistics.mean(keys_ms),
                                 "allgather": statistics.mean(ag_ms) if gathered is not None else 0.0,
                                 "hash_max_over_ranks": hash_ms_max},
                "dense_e2lsh": dense, "tables": tables, "queries": queries,
                "packing": _packing_summary(P, info, fused_keys)}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
