"""GPU routing-surrogate sampler vs the reference's numba kernels (golden) and the C oracle."""

import os

import numpy as np
import pytest

from oracle import union_counts as uc
from paper_2510_08055_b200 import kernels as gk

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "union_counts.npz"))


def _rank_power(E, skew):
    return (np.arange(E, dtype=np.float64) + 1.0) ** (-skew)


@pytest.mark.parametrize("batch,k,E", [(1, 8, 128), (8, 8, 128), (5, 4, 32), (16, 1, 7), (3, 7, 7)])
def test_uniform_bit_exact_vs_reference(cuda, gold, batch, k, E):
    u = np.random.default_rng(42).random((500, batch, k))
    assert np.array_equal(gk.uniform_union_counts(u, batch, k, E), gold[f"uniform_{batch}_{k}_{E}"])


@pytest.mark.parametrize("batch,k,E,seed,trials", [(64, 8, 128, 7, 300), (576, 8, 128, 11, 50)])
def test_uniform_large_bit_exact(cuda, gold, batch, k, E, seed, trials):
    u = np.random.default_rng(seed).random((trials, batch, k))
    assert np.array_equal(gk.uniform_union_counts(u, batch, k, E), gold[f"uniform_{batch}_{k}_{E}_s{seed}"])


@pytest.mark.parametrize("skew", [0.0, 0.3, 1.0, 2.5])
def test_weighted_bit_exact_vs_reference(cuda, gold, skew):
    u = np.random.default_rng(9).random((400, 8, 8))
    got = gk.weighted_union_counts(u, 8, 8, 128, _rank_power(128, skew))
    assert np.array_equal(got, gold[f"weighted_{skew}"])


def test_weighted_k_equals_E(cuda, gold):
    u = np.random.default_rng(8).random((200, 3, 6))
    got = gk.weighted_union_counts(u, 3, 6, 6, _rank_power(6, 1.5))
    assert np.array_equal(got, gold["weighted_ke"])


@pytest.mark.parametrize("batch,k,E", [(8192, 8, 128), (33, 64, 64), (100, 3, 1000)])
def test_uniform_vs_c_oracle_edge_shapes(cuda, batch, k, E):
    u = np.random.default_rng(batch).random((20, batch, k))
    assert np.array_equal(gk.uniform_union_counts(u, batch, k, E), uc.uniform_union_counts(u, batch, k, E))


def test_weighted_vs_c_oracle_skewed(cuda):
    u = np.random.default_rng(5).random((50, 256, 8))
    w = _rank_power(128, 1.7)
    assert np.array_equal(gk.weighted_union_counts(u, 256, 8, 128, w), uc.weighted_union_counts(u, 256, 8, 128, w))


def test_batch_zero(cuda):
    assert gk.uniform_union_counts(np.zeros((4, 0, 8)), 0, 8, 128).tolist() == [0, 0, 0, 0]
