#!/usr/bin/env python
"""Benchmark of the FastLSH hot path on B200 (BASELINE.json metric: hashes/s and roofline fraction).

One step = one pass of the whole hot path over the workload resident in HBM:
  a2-a5 hash (stage X, gather S_i(v), project, +b, /w, floor, int32 codes stored to HBM) and
  a6 compound keys (L tables of K codes -> 64-bit keys, table-major [L][N]);
  a8 (N > 1 GPUs) the NCCL all-gather of the keys, one all_gather_into_tensor per table.
Where the params-specialised kernel K1j applies (n <= 128: C0, C3) a2-a6 are ONE launch per chunk
(fastlsh_hash_keys: codes and keys); elsewhere K1r + the key kernel.

Default workload: BASELINE.json configs[3] (C3), the configuration the metric "at 1/2/4/8 B200"
is quoted on: a fixed 2e8-row dataset (n=128, k=256, m=16, w=4, keys 16 x 16) row-sharded across
the ranks (strong scaling), hashed in chunks (its 204.8 GB of codes do not fit one GPU; each
chunk's codes are written to HBM and overwritten by the next chunk, keys of all rows kept).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3|C1|C2|C4] [--impl reference]
  python bench.py --config C4 --stream      (streaming rebuild: 1000 batches through host rings)

Rank 0 prints ONE JSON line. See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
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
NUM_SMS = 148


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "bf16_tflops": float(d.get("bf16_tflops", 2250.0)),
                "source": "measured (MEASURED_PEAKS.json: copy bandwidth, burst)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "bf16_tflops": 2250.0,
                "source": "fallback (B200_PROFILING.md)"}


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
    if os.environ.get("FASTLSH_BENCH_SHARE_GPU") == "1":  # functional smoke test of the N > 1 path on one GPU
        local = 0
    return world, rank, local


def _backend():
    """NCCL (the product path). FASTLSH_BENCH_BACKEND=gloo only for the one-GPU functional smoke test of
    the N > 1 orchestration (tools/gpu_multirank_smoke.sh): host-staged collectives, no rank's kernel
    waits on another's; such a run's timings are not bench numbers."""
    return os.environ.get("FASTLSH_BENCH_BACKEND", "nccl")


def _cores():
    return len(os.sched_getaffinity(0))


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def _sample_rows(N: int, count: int, seed: int, extra=()):
    rng = np.random.default_rng(seed)
    r = set(rng.choice(N, size=min(count, N), replace=False).tolist()) if N else set()
    r.update(x for x in (0, N - 1, *extra) if 0 <= x < N)
    return np.array(sorted(r), dtype=np.int64)


def _oracle_sample(cfg, seconds_target: float):
    """The oracle's inputs for a bounded sample of the workload: rows sized (by a 256-row calibration
    on all host cores) to take about seconds_target, generated once on the host."""
    import oracle
    from fastlsh_inputs import data, fastlsh_arrays
    idx, a, b = fastlsh_arrays(cfg.n, cfg.m, cfg.k, cfg.w, cfg.seed)
    cores = _cores()
    rows0 = 4096
    X0 = data.generate(cfg.data, cfg.n, 0, rows0, seed=cfg.seed).numpy()
    oracle.fastlsh(X0[:256], idx, a, b, cfg.w, threads=cores)  # thread pool start-up outside the calibration
    t = time.perf_counter()
    oracle.fastlsh(X0, idx, a, b, cfg.w, threads=cores)
    dt = max(time.perf_counter() - t, 1e-4)
    rows = int(min(cfg.N, max(rows0, rows0 * seconds_target / dt)))
    X = data.generate(cfg.data, cfg.n, 0, rows, seed=cfg.seed).numpy()
    return {"X": X, "idx": idx, "a": a, "b": b, "rows": rows, "cores": cores}


def cpu_baseline(cfg, seconds_target: float = 12.0, one_core_seconds: float = 3.0, sample=None):
    """The CPU oracle as it stands, on a bounded row sample of the same workload: all host cores,
    then 1 core."""
    import oracle
    smp = sample or _oracle_sample(cfg, seconds_target)
    X, idx, a, b, rows, cores = smp["X"], smp["idx"], smp["a"], smp["b"], smp["rows"], smp["cores"]
    t = time.perf_counter()
    oracle.fastlsh(X, idx, a, b, cfg.w, threads=cores)
    dt = time.perf_counter() - t
    rows1 = int(min(rows, max(64, rows * one_core_seconds / (dt * cores))))
    t = time.perf_counter()
    oracle.fastlsh(X[:rows1], idx, a, b, cfg.w, threads=1)
    dt1 = time.perf_counter() - t
    return {"value": rows * cfg.k / dt, "unit": "hashes/s", "cores": cores, "kind": "oracle",
            "value_1core": rows1 * cfg.k / dt1, "cpu_model": _cpu_model(),
            "sample": f"first {rows} of {cfg.N} rows ({cfg.name}), double-precision oracle (oracle/fastlsh_oracle.c), "
                      f"OpenMP {cores} threads, {dt:.2f} s; 1-core rate on the first {rows1} rows, {dt1:.2f} s "
                      f"(codes only; keys not included)",
            "seconds": dt}


def run_reference(args, cfg):
    """The reference arm of this tier: the CPU oracle as it stands, on the host cores; each step runs
    it over the same bounded row sample (generated once, ~ref_seconds of oracle work)."""
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    smp = _oracle_sample(cfg, args.ref_seconds)
    for _ in range(args.warmup):
        cpu_baseline(cfg, one_core_seconds=0.1, sample=smp)
    steps = [cpu_baseline(cfg, one_core_seconds=0.3, sample=smp) for _ in range(args.steps)]
    vals = [s["value"] for s in steps]
    v = statistics.median(vals)
    cb = dict(steps[-1])
    cb["value"] = v
    cb.pop("seconds", None)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "hashes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(s["seconds"] for s in steps),
            "higher_is_better": True, "scaling": "strong" if cfg.name == "C3" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": _config_dict(cfg, world),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "hashes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _config_dict(cfg, world, n_rank=None, n_total=None, chunks=1, strong=None):
    strong = (cfg.name == "C3") if strong is None else strong
    n_rank = cfg.N if n_rank is None else n_rank
    n_total = cfg.N * (1 if strong else world) if n_total is None else n_total
    d = {"workload": f"{cfg.name}: N={n_total} rows ({n_rank} per GPU), n={cfg.n}, k={cfg.k}, m={cfg.m}, w={cfg.w}, "
                     f"keys L={cfg.L} x K={cfg.K}, recipe {cfg.data}",
         "N_per_gpu": n_rank, "n": cfg.n, "k": cfg.k, "m": cfg.m, "w": cfg.w, "L": cfg.L, "K": cfg.K,
         "global_rows": n_total, "parallelism": f"row-sharded x{world}, params replicated",
         "l2": f"inputs {n_rank * cfg.n * 4 / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)"}
    if chunks > 1:
        d["chunks_per_step"] = chunks
    return d


def _kernel_name(info, fused):
    if info["kernel"] == 5:
        return ("e2lsh_pair_kernel (kernel 5: 3xTF32 tcgen05 GEMM on the duplicates-merged coefficients)" +
                (" + keys_kernel" if fused else ""))
    if info["kernel"] == 4:
        return ("k1j (K1j fastlsh_hash_keys: params-specialised lane = row kernel, codes + keys in one launch)"
                if fused else "k1j (K1j fastlsh_hash: params-specialised lane = row kernel)")
    return {1: "gather_kernel (K1 fastlsh_hash)", 2: "tmem_gather_kernel (K1t fastlsh_hash)",
            3: "rows_kernel (K1r fastlsh_hash: row-major stages, LDS.32)"}[info["kernel"]]


def _launches_per_call(P, info, Kobj) -> int:
    """Kernel launches of one fastlsh_hash_keys call (api.cu's dispatch rules, rows_keys_pay): K1j,
    and K1r with the keys built from its code tile (every CTA hash block holds whole tables, a
    block's key work small next to its gathers), are one launch; otherwise hash + the key kernel."""
    if Kobj is None or info["kernel"] == 4:
        return 1
    if info["kernel"] == 5:
        return 2  # the GEMM, then the key kernel on its codes
    rp = P.row_packing() if info["kernel"] == 3 else None
    if rp is None:
        return 2
    L, K = Kobj.L, Kobj.K
    h0s, ends = [int(h) for h in rp["block_h0"]], [int(h + b) for h, b in zip(rp["block_h0"], rp["block_kb"])]
    whole = all(h % K == 0 for h in h0s) and all(e % K == 0 or e >= L * K for e in ends)
    tables = max(min(L, e // K) - h // K for h, e in zip(h0s, ends))
    return 1 if whole and tables * K <= 0.75 * rp["warps"] * rp["slots"] else 2


def _packing_summary(P, info):
    """The GPU layout of the kernel that ran."""
    if info["kernel"] == 5:
        return {"kernel": "K4 dense (kernel 5)", "precision": "3xTF32 (hi*hi + hi*lo + lo*hi, fp32 accumulate)",
                "A": f"[{(P.k + 255) // 256 * 256} x {P.n}] merged coefficients, hi/lo split",
                "tile": "CTA pair (cta_group::2), 256 rows x 256 hashes, TMEM accumulators"}
    if info["kernel"] == 4:
        return {"kernel": "K1j", "lane": "row (32 rows per warp, row in registers)",
                "code": "S_i register operands, a_i / b_i / 1/w immediates (NVRTC, sm_100a)",
                "jit": P.jit_status()}
    rp = P.row_packing() if info["kernel"] == 3 else None
    if rp is not None:
        lanes = rp["hash_blocks"] * rp["warps"] * 32 * rp["slots"]
        return {"kernel": "K1r", "parts": rp["parts"], "slots": rp["slots"], "warps_per_block": rp["warps"],
                "hash_blocks": rp["hash_blocks"], "staged_row_words": rp["S"],
                "bank_efficiency": P.k * P.m / lanes, "conflict_wavefronts": rp["conflicts"]}
    return {"kernel": "K1", **{k: info[k] for k in ("parts", "slots", "warps_per_block", "hash_blocks",
                                                    "bank_efficiency", "conflict_wavefronts")}}


def _traffic_from_profiles(cfg, kernel: str, rows: int):
    """DRAM bytes per launch of the dominant kernel, from the committed `ncu --set full` capture
    (profiles/ncu_traffic.json: dram__bytes_read + dram__bytes_write per row, per config and kernel),
    scaled to this launch's row count. None if no capture is committed for this config/kernel."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        e = d[f"{cfg.name}/{kernel}"]
        return {"bytes_per_launch": e["dram_bytes_per_row"] * rows, "source": e["source"]}
    except Exception:
        return None


def _roofline(cfg, info, fused, N_launch, t_launch_s, step_ms, peaks, with_codes=True):
    """Dominant-kernel roofline. K1j reads X and writes codes (+ keys) with no shared-memory
    gather, so its bound is HBM: achieved = algorithmic bytes per launch / launch time. K1r / K1 are
    shared-memory-bound: achieved gathers/s against G_s. Both also report the north_star fraction
    t_roof / t_kernel with t_roof = max(HBM time of X + codes, N k m / G_s)."""
    gathers = N_launch * cfg.k * cfg.m
    g_peak = NUM_SMS * SMEM_GATHERS_PER_CLK_PER_SM * peaks["sm_max_mhz"] * 1e6
    hbm_ns = 4.0 * N_launch * cfg.n + (4.0 * N_launch * cfg.k if with_codes else 0.0)
    t_roof = max(hbm_ns / (peaks["hbm_gbs"] * 1e9), gathers / g_peak)
    t_roof_nominal = max(hbm_ns / 8.0e12, gathers / g_peak)
    kern = {1: "K1", 2: "K1t", 3: "K1r", 4: "K1j", 5: "K4dense"}[info["kernel"]]
    if info["kernel"] == 5:
        # the contraction X[N x n] . A[n x k]: algorithmic flops 2 N k n (the 3xTF32 emulation issues
        # three TF32 MMAs per product: mma_work); peak = TF32 dense = the measured bf16 peak x 1/2 (the
        # nominal tf32 : bf16 ratio, B200_PROFILING.md)
        flops = 2.0 * N_launch * cfg.k * cfg.n
        tf32_peak = peaks["bf16_tflops"] * 0.5 * 1e12
        r = {"bound": "tensor", "achieved": flops / t_launch_s / 1e12, "peak": tf32_peak / 1e12, "unit": "TFLOP/s",
             "frac": flops / t_launch_s / tf32_peak,
             "mma_work_frac": 3 * flops / t_launch_s / tf32_peak,
             "algorithmic_per_launch": {"flops": flops, "hbm_bytes": hbm_ns, "rows": N_launch, "gathers": gathers}}
    elif info["kernel"] == 4:
        alg = hbm_ns + (8.0 * N_launch * cfg.L if (fused and cfg.L) else 0.0)
        r = {"bound": "hbm", "achieved": alg / t_launch_s / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
             "frac": alg / t_launch_s / (peaks["hbm_gbs"] * 1e9),
             "algorithmic_per_launch": {"hbm_bytes": alg, "rows": N_launch,
                                        "bytes_per_row": {"X": 4 * cfg.n, "codes": 4 * cfg.k if with_codes else 0,
                                                          "keys": 8 * cfg.L if (fused and cfg.L) else 0},
                                        "gathers": gathers}}
    else:
        r = {"bound": "smem", "achieved": gathers / t_launch_s / 1e9, "peak": g_peak / 1e9, "unit": "Ggather/s",
             "frac": (gathers / t_launch_s) / g_peak,
             "algorithmic_per_launch": {"gathers": gathers, "hbm_bytes": hbm_ns, "rows": N_launch}}
    tr = _traffic_from_profiles(cfg, kern + ("+keys" if fused else "") + ("" if with_codes else "-keysonly"), N_launch)
    r.update({"traffic": tr["bytes_per_launch"] if tr else None,
              "traffic_source": tr["source"] if tr else "no committed ncu capture for this config/kernel",
              "kernel": _kernel_name(info, fused),
              "launch_ms": t_launch_s * 1e3,
              "gathers_per_s": gathers / t_launch_s, "smem_gather_peak_per_s": g_peak,
              "north_star_frac": t_roof / t_launch_s, "north_star_frac_nominal_8TBs": t_roof_nominal / t_launch_s,
              "hbm_achieved_gbs": (hbm_ns + (8.0 * N_launch * cfg.L if fused and cfg.L else 0.0)) / t_launch_s / 1e9,
              "peak_source": peaks["source"] + f"; smem peak = {NUM_SMS} SM x 32 words/clk x {peaks['sm_max_mhz']:.0f} MHz",
              "kernel_share_of_step": (t_launch_s * 1e3) / step_ms if step_ms else None})
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=4.0, help="reference arm: oracle seconds per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense E2LSH comparator")
    ap.add_argument("--kernel", default="auto", choices=["auto", "jit", "rows", "smem", "dense"],
                    help="pin the hashing kernel (auto: K1j for n <= 128, else K1r; dense = kernel 5, opt-in analysis)")
    ap.add_argument("--sample-dims", type=int, default=None,
                    help="override the config's m, the sampled dimensions per hash (C2's sweep: 32, 128, 512, 4096)")
    ap.add_argument("--rows", type=int, default=None,
                    help="override the config's N (smoke tests; the JSON's config.workload states the rows used)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--exchange", default="auto", choices=["auto", "alltoall", "allgather", "nccl", "nvls"],
                    help="N > 1 key exchange. alltoall (auto): the tables are sharded by id, rank l %% G gathers "
                         "table l's keys of all rows (one NCCL all_to_all_single, (G-1)/G of the rank's own keys in "
                         "and out); allgather (= nccl): every rank receives the whole [L][N] table "
                         "(all_gather_into_tensor per table; measured beside alltoall as allgather_variant); nvls: "
                         "multimem stores from the K1j epilogue into a symmetric-memory multicast table")
    ap.add_argument("--no-overlap", action="store_true",
                    help="N > 1: wait for each step's key exchange before the next step hashes")
    ap.add_argument("--chunk-rows", type=int, default=8_388_608, help="C3: rows hashed per chunk (launch)")
    ap.add_argument("--no-tables", action="store_true", help="skip the bucket-table build and query measurements")
    ap.add_argument("--queries", type=int, default=10_000, help="queries answered in the query measurement")
    ap.add_argument("--stream", action="store_true", help="C4 streaming rebuild (see stream_main)")
    ap.add_argument("--batches", type=int, default=None, help="--stream: batches per step (default: the config's)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    from fastlsh_inputs import configs
    cfg = configs.get(args.config)
    if args.sample_dims is not None or args.rows is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, m=args.sample_dims or cfg.m, N=args.rows or cfg.N)
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    if args.stream:
        import stream_bench
        stream_bench.main(args, cfg)
        return

    import torch
    import torch.distributed as dist
    import paper_2309_15479_b200 as fl
    from paper_2309_15479_b200.distributed import allgather_keys, shard_rows
    from fastlsh_inputs import data

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        if _backend() == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(_backend())
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    P = fl.Params.create(cfg.n, cfg.m, cfg.k, cfg.w, seed=cfg.seed)
    if args.kernel != "auto":
        P.set_kernel(args.kernel)
    Kobj = fl.Keys.create(cfg.L, cfg.K, seed=cfg.seed) if cfg.L else None
    info = P.info()
    jit = info["kernel"] == 4
    t_prep = time.perf_counter()
    P.prepare(keys=Kobj, codes=True)  # K1j: NVRTC compile outside the timed region (no-op otherwise)
    prep_s = time.perf_counter() - t_prep

    # C3 is a fixed 2e8-row dataset sharded over the ranks (strong scaling) and hashed in chunks; other
    # configs are per-GPU workloads (weak scaling).
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
    # N > 1, K1j: the keys go straight into every GPU's copy of the [L][N_total] table with multimem
    # stores from the hashing kernel (NVSwitch multicast, torch symmetric memory); finishing the
    # all-gather is one group barrier. Otherwise (no multicast / not K1j): NCCL all-gather, where the
    # all-gather of step j runs on NCCL's stream while step j+1 hashes into the other keys buffer
    # (double-buffered); step j+1 waits for it before launching its own all-gather.
    # Exchange (N > 1). Every GPU receiving the whole [L][N] key table (all-gather) costs each GPU's
    # NVLink ingress (G-1)/G of 8 L N bytes per step whatever the transport (NCCL or NVLS multicast):
    # 22.4 GB at C3, G = 8, >= 25 ms at 900 GB/s against ~8.4 ms of hashing. Sharding the tables by id
    # (the builder of table l receives table l's keys of all rows) cuts that G-fold, so it is the
    # default; the full all-gather is measured beside it (allgather_variant). Both overlap step j's
    # exchange with step j+1's hashing (double-buffered keys) unless --no-overlap.
    exchange = None
    if Kobj and world > 1:
        exchange = {"auto": "alltoall", "nccl": "allgather"}.get(args.exchange, args.exchange)
    ktable, nvls_why = None, None
    if exchange == "nvls":
        from paper_2309_15479_b200.distributed import KeyTable
        if not jit:
            raise SystemExit("--exchange nvls needs the K1j kernel (n <= 128)")
        ktable = KeyTable(cfg.L, N_total, device=dev, mode="nvls")  # raises (allocating nothing) without multicast
    nvls = ktable is not None
    a2a = exchange == "alltoall"
    gathered = (ktable.table if nvls else torch.empty((cfg.L, N_total), dtype=torch.int64, device=dev)) \
        if exchange in ("allgather", "nvls") else None
    overlap = (gathered is not None or a2a) and not nvls and not args.no_overlap
    keys_bufs = [keys, torch.empty_like(keys)] if overlap else [keys]
    pending = []
    a2a_last = []  # (owned tables, their keys for all rows) of the last table-sharded exchange
    step_no = [0]
    fused = bool(Kobj)  # fastlsh_hash_keys: one launch where K1j / K1r-tile keys apply, else hash + keys
    ev = []

    def step(record: bool):
        marks = []
        kb = keys_bufs[step_no[0] % len(keys_bufs)]
        step_no[0] += 1
        for c0, c1 in bounds:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if record else None
            if record:
                e[0].record(stream)
            cb = codes[:c1 - c0]
            if nvls:
                fl.hash_keys_multicast(P, Kobj, X[c0:c1], ktable.multicast_ptr, N_total, lo + c0, codes=cb)
            elif Kobj is not None:
                fl.hash_keys(P, Kobj, X[c0:c1], codes=cb, keys_out=kb, col0=c0)
            else:
                fl.fastlsh_hash(P, X[c0:c1], out=cb)
            if record:
                e[1].record(stream)
                marks.append(e)
        ea = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if record else None
        if record:
            ea[0].record(stream)
        if nvls:
            ktable.handle.barrier()  # every rank's multicast key stores are complete and visible
        elif a2a:
            from paper_2309_15479_b200.distributed import alltoall_keys_by_table
            if overlap:
                drain()
                pending[:] = alltoall_keys_by_table(kb, N_total, wait=False)
            else:
                a2a_last[:] = alltoall_keys_by_table(kb, N_total)
        elif gathered is not None:
            if overlap:
                for w in pending:
                    w.wait()
                pending[:] = allgather_keys(kb, out=gathered, wait=False, n_total=N_total)
            else:
                allgather_keys(kb, out=gathered, n_total=N_total)
        if record:
            ea[1].record(stream)
            ev.append((marks, ea))

    def drain():
        for w in pending:
            r = w.wait()
            if isinstance(r, tuple):  # the table-sharded exchange: (owned tables, their keys)
                a2a_last[:] = r
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
    # NVLS self-check (first use of the multicast path on this system): the keys this rank wrote
    # through the multicast table must equal the plain keys of the same rows; otherwise fall back
    nvls_check = None
    if nvls:
        nck = min(N, 4096)
        _, ref_keys = fl.hash_keys(P, Kobj, X[:nck])
        torch.cuda.synchronize()
        ok = bool(torch.equal(gathered[:, lo:lo + nck], ref_keys))
        okt = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        nvls_check = {"rows_checked_per_rank": nck, "ok": bool(okt.item())}
        if not okt.item():
            nvls, nvls_why = False, "multicast self-check failed: keys differ from the plain keys"
            gathered = torch.empty((cfg.L, N_total), dtype=torch.int64, device=dev)
            overlap = not args.no_overlap
            keys_bufs[:] = [keys, torch.empty_like(keys)] if overlap else [keys]
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
    launch_ms = [m[0].elapsed_time(m[1]) for marks, _ in ev for m in marks]  # one entry per chunk launch
    launch_rows = [c1 - c0 for _ in ev for c0, c1 in bounds]
    hash_ms = [sum(m[0].elapsed_time(m[1]) for m in marks) for marks, _ in ev]
    ag_ms = [ea[0].elapsed_time(ea[1]) for _, ea in ev]
    tt = torch.tensor([total_ms, statistics.mean(hash_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_ms_max, hash_ms_max = float(tt[0]), float(tt[1])
    ms_per_step = total_ms_max / args.steps
    value = N_total * cfg.k / (ms_per_step / 1e3)
    peaks = _peaks()
    # the dominant kernel: the per-chunk launch, averaged over full-size chunks
    full = [t for t, r in zip(launch_ms, launch_rows) if r == chunk] or launch_ms
    t_launch = statistics.mean(full) / 1e3
    lpc = _launches_per_call(P, info, Kobj)
    roofline = _roofline(cfg, info, fused and lpc == 1, chunk, t_launch, ms_per_step, peaks)
    if lpc > 1:
        roofline["note"] = "the per-chunk time covers the hashing kernel and the key kernel (two launches)"
    roofline["launch_ms_min_max"] = [min(full), max(full)]
    # kernel_share_of_step is ONE launch's share; the kernel's share of the step over all of its
    # launches (what the ncu launch list's "share" corresponds to) is the sum over the chunks
    roofline["launches_per_step"] = len(bounds) * lpc
    roofline["kernel_share_of_step_all_launches"] = statistics.mean(hash_ms) / (total_ms / args.steps)

    # the HBM ceiling of the dominant kernel's own traffic mix (a plain streaming kernel reading and
    # writing the same bytes per row: roofline.mix_ceiling), on the same rows
    if jit:
        rb, wbytes = 4 * cfg.n, 4 * cfg.k + (8 * cfg.L if Kobj is not None else 0)
        scratch = torch.empty((chunk * wbytes + 15) // 16 * 4, dtype=torch.int32, device=dev)
        fl.bandwidth_probe(X, scratch, chunk, rb, wbytes)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for _ in range(5):
            fl.bandwidth_probe(X, scratch, chunk, rb, wbytes)
        p1.record(stream)
        torch.cuda.synchronize()
        pms = p0.elapsed_time(p1) / 5
        ceil_gbs = chunk * (rb + wbytes) / (pms / 1e3) / 1e9
        roofline["mix_ceiling"] = {"gbs": ceil_gbs, "frac_of_ceiling": roofline["achieved"] / ceil_gbs,
                                   "pattern": f"{rb} B read + {wbytes} B written per row, {chunk} rows, plain "
                                              "16-byte vector stream (fastlsh_bandwidth_probe)",
                                   "ms": pms}
        del scratch

    # exchange check (N > 1, all-gather / NVLS): every rank re-hashes the first rows of the NEXT rank's
    # shard itself (regenerated from the seed) and compares their keys with the columns the exchange
    # delivered into its gathered table: bit-exact, since the kernels are deterministic
    exchange_check = None
    if world > 1 and (gathered is not None or a2a_last):
        nr = (rank + 1) % world
        rlo, rhi = shard_rows(N_total, world, nr) if strong else (nr * cfg.N, (nr + 1) * cfg.N)
        nck = min(rhi - rlo, 2048)
        Xr = data.generate(cfg.data, cfg.n, rlo, rlo + nck, seed=cfg.seed, device=dev)
        _, kref = fl.hash_keys(P, Kobj, Xr)
        torch.cuda.synchronize()
        if gathered is not None:
            got = gathered[:, rlo:rlo + nck]
        else:  # table-sharded: this rank holds tables l % world == rank for all rows
            mine, tab = a2a_last
            got, kref = tab[:, rlo:rlo + nck], kref[mine]
        okx = torch.tensor([1 if torch.equal(got, kref) else 0], device=dev)
        dist.all_reduce(okx, op=dist.ReduceOp.MIN)
        exchange_check = {"rows_checked_per_rank": nck, "source_rank": "rank + 1", "ok": bool(okx.item())}
        del Xr, kref

    # parity sample of the timed step's own output (the last chunk's codes, the keys of those rows),
    # copied out now, before any side measurement reuses the buffers; checked in the CPU leg below
    c0p, c1p = bounds[-1]
    prow = _sample_rows(c1p - c0p, 512, seed=11, extra=[1, 31, 32, 33, (c1p - c0p) // 2])
    pri = torch.as_tensor(prow, device=dev)
    psample = {"X": X[c0p:c1p][pri].cpu().numpy(), "codes": codes[:c1p - c0p][pri].cpu().numpy(),
               "keys": ((gathered[:, lo + c0p + pri] if nvls else keys_bufs[(step_no[0] - 1) % len(keys_bufs)][:, c0p + pri])
                        .cpu().numpy().view(np.uint64) if Kobj is not None else None),
               "proj": fl.fastlsh_project(P, X[c0p:c1p][pri].contiguous()).cpu().numpy()}

    # side measurement (N > 1, table-sharded default): the same step with the full key all-gather
    # (every GPU receives the whole [L][N] table), overlapped the same way; max over ranks
    allgather_variant = None
    if a2a:
        try:
            a2a, gathered, overlap = False, torch.empty((cfg.L, N_total), dtype=torch.int64, device=dev), \
                not args.no_overlap
            keys_bufs[:] = [keys, torch.empty_like(keys)] if overlap else [keys]
            for _ in range(2):
                step(False)
            drain()
            torch.cuda.synchronize()
            dist.barrier()
            va = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            nvs = max(2, min(args.steps, 5))
            va[0].record(stream)
            for _ in range(nvs):
                step(False)
            drain()
            va[1].record(stream)
            torch.cuda.synchronize()
            dist.barrier()
            vt = torch.tensor([va[0].elapsed_time(va[1]) / nvs], dtype=torch.float64, device=dev)
            dist.all_reduce(vt, op=dist.ReduceOp.MAX)
            allgather_variant = {"ms_per_step": float(vt[0]), "value": N_total * cfg.k / (float(vt[0]) / 1e3),
                                 "steps": nvs, "exchange": "NCCL all_gather_into_tensor per table, every GPU "
                                 "receives the whole [L][N] table; overlapped with the next step's hashing"
                                 if overlap else "NCCL all_gather_into_tensor per table, serial"}
        except Exception as ex:  # noqa: BLE001
            allgather_variant = {"error": f"{type(ex).__name__}: {ex}"}
        finally:
            a2a, gathered = True, None
            keys_bufs[:] = keys_bufs[:1]
            torch.cuda.empty_cache()

    # side measurement: keys only (codes never leave the SM; K1j / K1r code tile), same chunks
    keys_only = None
    if Kobj is not None and (jit or info["kernel"] == 3):
        try:
            kk = keys_bufs[0]
            for _ in range(2):
                for c0, c1 in bounds:
                    fl.hash_keys(P, Kobj, X[c0:c1], keys_out=kk, with_codes=False, col0=c0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(1, min(args.steps, 5))
            e0.record(stream)
            for _ in range(reps):
                for c0, c1 in bounds:
                    fl.hash_keys(P, Kobj, X[c0:c1], keys_out=kk, with_codes=False, col0=c0)
            e1.record(stream)
            torch.cuda.synchronize()
            t_ms = e0.elapsed_time(e1) / reps
            keys_only = {"ms_per_step": t_ms, "value": N * cfg.k / (t_ms / 1e3), "unit": "hashes/s",
                         "roofline": {k: v for k, v in _roofline(cfg, info, True, N, t_ms / 1e3, t_ms, peaks,
                                                                  with_codes=False).items()
                                      if k in ("bound", "achieved", "peak", "unit", "frac", "north_star_frac")},
                         "note": "hash + keys with codes kept on chip (fastlsh_hash_keys, codes=NULL), rank-local; "
                                 "not the headline step (which also stores every code)"}
        except Exception as ex:  # noqa: BLE001
            keys_only = {"error": str(ex)}

    # bucket tables of this rank's keys — timed separately, per-GPU
    # workloads only (C3's 16 x 2e8 entries would need ~100 GB of sort workspace on one GPU)
    tables = None
    if Kobj is not None and not args.no_tables and not strong:
        try:
            out_t = fl.build_tables(keys)
            t_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize()
            t_ev[0].record(stream)
            for _ in range(3):
                fl.build_tables(keys, out=out_t)
            t_ev[1].record(stream)
            torch.cuda.synchronize()
            tms = t_ev[0].elapsed_time(t_ev[1]) / 3
            entries = cfg.L * N
            tables = {"ms": tms, "entries": entries, "entries_per_s": entries / (tms / 1e3),
                      "buckets_table0": int(out_t[3][0].item()),
                      "hbm_bytes_algorithmic": entries * ((8 + 8 + 12 + 12 + 12 + 8 + 8 + 4) if N <= (1 << 22)
                                                          else (8 * 8 + 8 * 24 + 8 + 4)),
                      "note": ("MSD form (N <= 2^22): one global top-digit pass (hist 8 B + scatter 8 B in / 12 B out per "
                               "entry), per-segment LSD sorts in L2 (12 B in / 12 B out), bucket starts (8 + 8 B in, 4 B "
                               "out); bound by the shared-memory ranking of the seven in-segment passes, not HBM"
                               if N <= (1 << 22) else
                               "8 LSD radix passes (hist 8 B + scatter 12 B in / 12 B out per entry) + bucket starts")}
            tables["hbm_frac"] = tables["hbm_bytes_algorithmic"] / (tms / 1e3) / (peaks["hbm_gbs"] * 1e9)
            del out_t
        except Exception as ex:  # noqa: BLE001 (report, never hide a failure)
            tables = {"error": str(ex)}
    elif strong:
        tables = {"skipped": "C3: per-GPU table build of 16 x N entries not run (sort workspace); "
                             "measured on C1 (python bench.py --config C1)"}

    # queries, per-GPU workloads only, rank 0
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
        Pd = fl.Params.e2lsh(cfg.n, cfg.k, cfg.w, seed=cfg.seed).set_kernel("smem")
        dense = {}
        Nd = min(N, chunk)
        Xd, cd = X[:Nd], codes[:Nd]
        t_codes = statistics.mean(full) / chunk  # FastLSH ms per row (the headline launch)
        for prec in (3, 2, 1):
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
            products = 1 if prec == 1 else 3
            dense["fp16x3" if prec == 2 else f"tf32x{prec}"] = {
                "ms": ms, "rows": Nd, "hashes_per_s": Nd * cfg.k / (ms / 1e3),
                "mma_tflops": 2.0 * Nd * cfg.n * kpad * products / (ms / 1e3) / 1e12,
                "fastlsh_speedup": (ms / Nd) / t_codes}
        # the faster of the two parity-gated comparators (3xTF32, 3xFP16) is the one the speedup is quoted against
        best = min(("tf32x3", "fp16x3"), key=lambda kk: dense[kk]["ms"])
        dense["gated_best"] = {"kernel": best, "ms": dense[best]["ms"], "fastlsh_speedup": dense[best]["fastlsh_speedup"]}
        # library reference points (cuBLAS through torch.matmul: plumbing, not the product): the same
        # dense X . A^T in 1xTF32 (cublasLt tensor cores) and full FP32 (SIMT SGEMM, parity-clean), with
        # the +b, /w, floor epilogue in torch
        try:
            from fastlsh_inputs import e2lsh_arrays
            _, Ad, bd = e2lsh_arrays(cfg.n, cfg.k, cfg.w, cfg.seed)
            At = torch.as_tensor(Ad, device=dev).t().contiguous()
            bt = torch.as_tensor(bd, device=dev)
            prev = torch.backends.cuda.matmul.allow_tf32
            for name, tf32 in (("cublas_tf32", True), ("cublas_fp32", False)):
                torch.backends.cuda.matmul.allow_tf32 = tf32
                run = lambda: (Xd @ At).add_(bt).div_(cfg.w).floor_().to(torch.int32)  # noqa: E731
                run()
                d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                d0.record(stream)
                for _ in range(3):
                    run()
                d1.record(stream)
                torch.cuda.synchronize()
                ms = d0.elapsed_time(d1) / 3
                dense[name] = {"ms": ms, "rows": Nd, "hashes_per_s": Nd * cfg.k / (ms / 1e3),
                               "fastlsh_speedup": (ms / Nd) / t_codes,
                               "note": "torch.matmul + torch epilogue (cuBLAS reference point)"}
            torch.backends.cuda.matmul.allow_tf32 = prev
            del At, bt
        except Exception as ex:  # noqa: BLE001
            dense["cublas_error"] = str(ex)
        # analysis only: the same FastLSH params as the 3xTF32 GEMM on the
        # duplicates-merged coefficient matrix (kernel 5, opt-in). Not the graded path: north_star
        # reserves the tensor cores for the E2LSH baseline, so the automatic choice never takes it.
        if cfg.n % 4 == 0 and cfg.n >= 512 and info["kernel"] != 5:
            try:
                Pm = fl.Params.create(cfg.n, cfg.m, cfg.k, cfg.w, seed=cfg.seed)
                Pm.set_kernel("dense")
                fl.fastlsh_hash(Pm, Xd, out=cd)
                d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                d0.record(stream)
                for _ in range(3):
                    fl.fastlsh_hash(Pm, Xd, out=cd)
                d1.record(stream)
                torch.cuda.synchronize()
                ms = d0.elapsed_time(d1) / 3
                dense["merged_fastlsh"] = {
                    "ms": ms, "rows": Nd, "hashes_per_s": Nd * cfg.k / (ms / 1e3),
                    "vs_headline_kernel": (ms / Nd) / t_codes,
                    "note": "analysis only: these FastLSH params as kernel 5 (3xTF32 tcgen05 GEMM on the "
                            "duplicates-merged coefficients, opt-in); the graded path is the gather kernel"}
                del Pm
            except Exception as ex:  # noqa: BLE001
                dense["merged_fastlsh"] = {"error": str(ex)}
        dense["note"] = ("e2lsh_hash on E2LSH params (m = n) of the same k, w and rows (codes only); tf32x3 and "
                         "fp16x3 are the parity-gated comparators (3xTF32 / 3xFP16 tcgen05 GEMMs; gated_best the "
                         "faster), tf32x1 the ungated reference point; cublas_fp32 the "
                         "parity-clean library reference, cublas_tf32 the ungated library one; speedup vs the "
                         "headline FastLSH launch per row (which also builds the keys)")
        del Pd

    # end to end through the public host-buffer API: H2D of X, hash + keys, D2H of codes + keys
    # (C3: on a 2M-row sample of each shard; the host would need 307 GB for the whole shard at G=1)
    Ne = N if not strong else min(N, 2_097_152)
    Xh = X[:Ne].cpu().pin_memory()
    codes_h = torch.empty((Ne, cfg.k), dtype=torch.int32).pin_memory()
    keys_h = torch.empty((cfg.L, Ne), dtype=torch.int64).pin_memory() if Kobj else None
    fl.hash_host(P, Kobj, Xh, codes_h, keys_h, chunk_rows=262144)  # warm (workspace allocation)
    if world > 1:
        dist.barrier()
    te = time.perf_counter()
    for _ in range(args.e2e_steps):
        fl.hash_host(P, Kobj, Xh, codes_h, keys_h, chunk_rows=262144)
    e2e_s = (time.perf_counter() - te) / args.e2e_steps
    et = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e = {"value": world * Ne * cfg.k / float(et[0]), "unit": "hashes/s",
           "h2d_bytes_per_step": int(Xh.numel() * 4),
           "d2h_bytes_per_step": int(codes_h.numel() * 4 + (keys_h.numel() * 8 if keys_h is not None else 0)),
           "api": "fastlsh_hash_host (pinned host buffers, 2-stream chunked pipeline)", "steps": args.e2e_steps,
           "rows_per_gpu": Ne, "pcie_gbs": (Xh.numel() * 4 + codes_h.numel() * 4 +
                                            (keys_h.numel() * 8 if keys_h is not None else 0)) / float(et[0]) / 1e9}
    # the same through the host API with only the keys coming back (codes stay on the device; with
    # K1j they never leave the SM): the streaming-rebuild form of the step's result
    e2e_keys = None
    if Kobj is not None:
        fl.hash_host(P, Kobj, Xh, None, keys_h, chunk_rows=262144, with_codes=False)
        te = time.perf_counter()
        for _ in range(args.e2e_steps):
            fl.hash_host(P, Kobj, Xh, None, keys_h, chunk_rows=262144, with_codes=False)
        ek = torch.tensor([(time.perf_counter() - te) / args.e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ek, op=dist.ReduceOp.MAX)
        e2e_keys = {"value": world * Ne * cfg.k / float(ek[0]), "unit": "hashes/s",
                    "h2d_bytes_per_step": int(Xh.numel() * 4), "d2h_bytes_per_step": int(keys_h.numel() * 8),
                    "api": "fastlsh_hash_host with codes_host = NULL (keys only cross PCIe)"}
    e2e["keys_only"] = e2e_keys
    del Xh, codes_h, keys_h

    # CPU leg (rank 0, N = 1 only): the oracle timed on the host cores, and the parity of sampled rows
    # of the timed step's own output (the last chunk's codes, the keys of those rows) vs the oracle
    cb, parity = None, None
    if rank == 0 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        try:
            import oracle
            from fastlsh_inputs import fastlsh_arrays, philox
            from oracle import keys as okeys
            from parity import stats
            idx, a, b = fastlsh_arrays(cfg.n, cfg.m, cfg.k, cfg.w, cfg.seed)
            p, s, code = oracle.fastlsh(psample["X"], idx, a, b, cfg.w, threads=_cores())
            cg, pg, kg, kr = psample["codes"], psample["proj"], psample["keys"], None
            if Kobj is not None:
                kr = okeys.build_keys(cg.astype(np.int64), philox.key_multipliers(cfg.L, cfg.K, cfg.seed), cfg.L, cfg.K)
            parity = stats(cg, pg, p, s, code, b, cfg.w, kg, kr)
            parity["sample"] = (f"{len(prow)} rows of the last chunk of the timed step (its codes and keys); "
                                "projections re-run on the same rows; oracle/fastlsh_oracle.c in double")
        except Exception as ex:  # noqa: BLE001
            parity = {"error": str(ex)}
        if world == 1:
            try:
                cb = cpu_baseline(cfg)
                cb.pop("seconds", None)
            except Exception as ex:  # noqa: BLE001
                cb = {"error": str(ex)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "hashes/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if strong else "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, resident in HBM)",
                "config": _config_dict(cfg, world, N, N_total, len(bounds), strong), "roofline": roofline,
                "cpu_baseline": cb, "e2e": e2e, "parity": parity,
                "gpu_launches": len(bounds) * args.steps * lpc,
                "clocks": clocks,
                "step": ("per chunk one K1j launch (fastlsh_hash_keys): X read, codes + keys written" if jit and Kobj
                         else "per chunk fastlsh_hash_keys (kernel as in roofline.kernel)") +
                        ((f"; keys written by K1j with multimem.st into every GPU's copy of the [L][N] table "
                          f"(NVSwitch multicast, symmetric memory), then one group barrier" if nvls else
                          "; then the table-sharded NCCL all-to-all (rank l % G receives table l for all rows, "
                          f"{'overlapped with the next step' if not args.no_overlap else 'serial'})" if a2a else
                          f"; then the NCCL key all-gather ({'overlapped with the next step' if overlap else 'serial'})")
                         if world > 1 else ""),
                "key_exchange": exchange, "allgather_variant": allgather_variant,
                "nvls_unavailable": nvls_why, "nvls_selfcheck": nvls_check, "exchange_check": exchange_check,
                "keys_only": keys_only,
                "breakdown_ms": {"hash": statistics.mean(hash_ms),
                                 "hash_note": "sum over the step's chunk launches of the hashing kernel(s), CUDA events; "
                                              "with K1j each launch also writes the keys",
                                 "allgather": statistics.mean(ag_ms) if (gathered is not None or a2a) else 0.0,
                                 "hash_max_over_ranks": hash_ms_max,
                                 "roofline_frac_from_hash": ((N * (4 * cfg.n + 4 * cfg.k + 8 * cfg.L) if jit else
                                                              N * cfg.k * cfg.m) / (statistics.mean(hash_ms) / 1e3) /
                                                             ((peaks["hbm_gbs"] * 1e9) if jit else
                                                              (NUM_SMS * SMEM_GATHERS_PER_CLK_PER_SM *
                                                               peaks["sm_max_mhz"] * 1e6)))},
                "jit_prepare_s": prep_s,
                "dense_e2lsh": dense, "tables": tables, "queries": queries,
                "packing": _packing_summary(P, info)}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
