"""The seeded input generators: determinism and distribution."""
import math

import numpy as np
import pytest
import torch

from fastlsh_inputs import philox, data, fastlsh_arrays, configs


def test_deterministic_from_seed():
    a1 = fastlsh_arrays(128, 16, 64, 4.0, seed=1)
    a2 = fastlsh_arrays(128, 16, 64, 4.0, seed=1)
    a3 = fastlsh_arrays(128, 16, 64, 4.0, seed=2)
    for x, y in zip(a1, a2):
        assert np.array_equal(x, y)
    assert not np.array_equal(a1[0], a3[0])


def test_counter_addressing_is_order_independent():
    """Value (i, j) does not depend on how many hashes/slots were generated (prefix property)."""
    big = philox.sample_indices(960, 60, 500, seed=7)
    small = philox.sample_indices(960, 10, 20, seed=7)
    assert np.array_equal(big[:20, :10], small)
    assert np.array_equal(philox.gaussian_coefficients(60, 500, 7)[:5, :8],
                          philox.gaussian_coefficients(8, 5, 7))


def test_indices_uniform_chi_square():
    """Index frequencies over >= 1e6 draws are uniform."""
    n = 100
    idx = philox.sample_indices(n, 1000, 1000, seed=3).ravel()
    cnt = np.bincount(idx, minlength=n)
    exp = idx.size / n
    chi2 = float(((cnt - exp) ** 2 / exp).sum())
    # df = 99: mean 99, sd 14; 5 sd bound
    assert chi2 < 99 + 5 * 14
    assert idx.min() >= 0 and idx.max() < n


def test_gaussian_and_offsets_distribution():
    from scipy import stats
    a = philox.gaussian_coefficients(100, 2000, seed=4).ravel().astype(np.float64)
    assert stats.kstest(a, "norm").pvalue > 1e-4
    b = philox.uniform_offsets(100_000, 2.0, seed=4)
    assert b.min() >= 0 and b.max() < 2.0
    assert stats.kstest(b / 2.0, "uniform").pvalue > 1e-4


def test_key_multipliers_range():
    r = philox.key_multipliers(50, 10, seed=1)
    assert r.shape == (50, 11)
    assert int(r.max()) < (1 << 61) - 1


@pytest.mark.parametrize("recipe,n", [("sift_u8", 128), ("gist_mixture", 96), ("trevi_sphere", 64),
                                      ("sparse80", 80)])
def test_data_recipes_shard_independent(recipe, n):
    full = data.generate(recipe, n, 0, 700, seed=1)
    a = data.generate(recipe, n, 0, 300, seed=1)
    b = data.generate(recipe, n, 300, 700, seed=1)
    assert torch.equal(full, torch.cat([a, b]))
    if recipe == "sift_u8":
        u = full / torch.tensor(10.0 / 255.0)
        assert full.min() >= 0 and full.max() <= 10.0
        assert torch.allclose(u, torch.round(u), atol=1e-4)
    if recipe == "gist_mixture":
        assert full.min() >= 0
    if recipe == "trevi_sphere":
        assert torch.allclose(full.double().norm(dim=1), torch.ones(700, dtype=torch.float64), atol=1e-6)
    if recipe == "sparse80":
        frac = float((full == 0).float().mean())
        assert abs(frac - 0.8) < 0.01


def test_configs_match_baseline():
    c = configs.get("C1")
    assert (c.N, c.n, c.k, c.m, c.w, c.L, c.K) == (1_000_000, 960, 500, 60, 1.0, 50, 10)
    assert configs.get("C2").m_sweep == (32, 128, 512, 4096)
