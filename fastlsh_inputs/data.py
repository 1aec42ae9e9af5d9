"""Seeded synthetic datasets shaped like the paper's ANN workloads (Table 1).

The paper's datasets are not in the container; these recipes stand in for their shapes and
value ranges. They hold none of the method's arithmetic.

Rows are generated in fixed global chunks of CHUNK rows, each chunk from its own torch generator
seeded by (seed, recipe, chunk index). A row's value therefore depends only on its global index
and the device type, never on how rows are sharded across ranks or batched — so results can be
compared across 1/2/4/8 shards.
"""
from __future__ import annotations

import torch

CHUNK = 65536
_RECIPE_ID = {"sift_u8": 11, "gist_mixture": 12, "trevi_sphere": 13, "sparse80": 14}


def _gen(device, seed: int, recipe: str, chunk: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + _RECIPE_ID[recipe] * 7_919 + chunk * 104_729) % (2**63 - 1))
    return g


def _centres(n: int, seed: int, device) -> torch.Tensor:
    g = _gen(device, seed, "gist_mixture", 2**20)
    return torch.rand((100, n), generator=g, device=device, dtype=torch.float32)


def _chunk_rows(recipe: str, n: int, seed: int, chunk: int, rows: int, device, centres=None) -> torch.Tensor:
    g = _gen(device, seed, recipe, chunk)
    if recipe == "sift_u8":
        # integers uniform in [0,255], scaled by 10/255 (BASELINE.json configs[0]; R14)
        u = torch.randint(0, 256, (rows, n), generator=g, device=device, dtype=torch.int32)
        return u.to(torch.float32) * torch.tensor(10.0 / 255.0, dtype=torch.float32, device=device)
    if recipe == "gist_mixture":
        # 100-component Gaussian mixture, means U[0,1]^n, sigma 0.05, clipped at 0 (configs[1])
        z = torch.randint(0, 100, (rows,), generator=g, device=device)
        e = torch.randn((rows, n), generator=g, device=device, dtype=torch.float32)
        return torch.clamp_min(centres[z] + 0.05 * e, 0.0)
    if recipe == "trevi_sphere":
        # standard normal rows normalised to unit l2 norm (configs[2]); norm taken in double
        e = torch.randn((rows, n), generator=g, device=device, dtype=torch.float32)
        nrm = torch.linalg.vector_norm(e.to(torch.float64), dim=1, keepdim=True)
        return (e.to(torch.float64) / nrm).to(torch.float32)
    if recipe == "sparse80":
        # 80% zeros, nonzeros uniform in [0,1) (configs[4])
        keep = torch.rand((rows, n), generator=g, device=device) >= 0.8
        v = torch.rand((rows, n), generator=g, device=device, dtype=torch.float32)
        return torch.where(keep, v, torch.zeros((), device=device))
    raise ValueError(f"unknown recipe {recipe}")


def generate(recipe: str, n: int, row_begin: int, row_end: int, seed: int = 1, device="cpu",
             out: torch.Tensor | None = None) -> torch.Tensor:
    """Rows [row_begin, row_end) of the recipe's infinite synthetic dataset, f32 [rows, n]."""
    rows = row_end - row_begin
    if out is None:
        out = torch.empty((rows, n), dtype=torch.float32, device=device)
    if rows == 0:
        return out
    centres = _centres(n, seed, device) if recipe == "gist_mixture" else None
    c0 = row_begin // CHUNK
    c1 = (row_end - 1) // CHUNK
    for c in range(c0, c1 + 1):
        lo = max(row_begin, c * CHUNK)
        hi = min(row_end, (c + 1) * CHUNK)
        full = _chunk_rows(recipe, n, seed, c, CHUNK, device, centres)
        out[lo - row_begin:hi - row_begin].copy_(full[lo - c * CHUNK:hi - c * CHUNK])
        del full
    return out


def random_codes(N: int, k: int, seed: int, lo: int = -40, hi: int = 40, device="cpu") -> torch.Tensor:
    """Seeded int32 code matrices for key-builder parity (codes as inputs, not kernel outputs)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed * 7 + 3)
    return torch.randint(lo, hi, (N, k), generator=g, device=device, dtype=torch.int32)
