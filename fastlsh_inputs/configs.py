"""The five workloads of BASELINE.json `configs` (C0..C4) as plain records.

Naming follows BASELINE.json: k = total hash functions per point, L tables of K codes each
(the paper's per-table k is our K; §3.2 — DESIGN.md reading R10).
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Config:
    name: str
    N: int            # rows (points) in the workload
    n: int            # dimensionality
    k: int            # hash functions per point
    m: int            # sampled dimensions per hash
    w: float          # bucket width
    data: str         # synthetic recipe name (fastlsh_inputs.data)
    L: int = 0        # tables of compound keys (0 = no keys in the step)
    K: int = 0        # codes per key
    seed: int = 1
    m_sweep: tuple = field(default_factory=tuple)
    batches: int = 1  # streaming batches (C4)
    note: str = ""


CONFIGS = {
    "C0": Config("C0", N=10_000, n=128, k=64, m=16, w=4.0, data="sift_u8",
                 note="Sift-shaped parity config (PAPER.md:502)"),
    "C1": Config("C1", N=1_000_000, n=960, k=500, m=60, w=1.0, data="gist_mixture", L=50, K=10,
                 note="Gist-shaped (PAPER.md:503); bench workload (BASELINE.json configs[1])"),
    "C2": Config("C2", N=1_000_000, n=4096, k=1000, m=32, w=0.5, data="trevi_sphere",
                 m_sweep=(32, 128, 512, 4096), note="Trevi-shaped (PAPER.md:500), m sweep"),
    "C3": Config("C3", N=200_000_000, n=128, k=256, m=16, w=4.0, data="sift_u8", L=16, K=16,
                 note="Sift-scale x200, row-sharded across GPUs"),
    "C4": Config("C4", N=100_000, n=784, k=2000, m=64, w=2.0, data="sparse80", L=200, K=10,
                 batches=1000, note="streaming: 1000 batches of 1e5 rows"),
}


def get(name: str) -> Config:
    return CONFIGS[name]
