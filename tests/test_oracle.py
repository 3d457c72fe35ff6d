"""Pin the CPU oracle before trusting it (CPU-only).

* moe_oracle vs HF transformers 5.5.0 Qwen3MoeSparseMoeBlock outputs
  (tests/golden/hf_qwen3moe_*.npz, made by tests/golden/make_golden.py).
* union_counts.c vs the reference's own numba kernels on the reference's test
  cases (tests/golden/union_counts.npz; reference pkg/tests/test_kernels.py:33-50).
"""

import os

import numpy as np
import pytest

from oracle import moe_oracle as mo
from oracle import union_counts as uc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _hf_case(name):
    from paper_2510_08055_b200.synthetic import expert_weights, router_tokens, router_weight

    d = np.load(os.path.join(GOLD, f"hf_qwen3moe_{name}.npz"))
    T, H, I, E, k, sw, sx, tb = (int(v) for v in d["meta"])
    wr = router_weight(E, H, sw, bool(tb)).float().numpy()
    w13, w2 = expert_weights(E, H, I, sw + 1)
    x = router_tokens(T, H, sx, bool(tb)).float().numpy()
    return d, (x, wr, w13.float().numpy(), w2.float().numpy(), k)


@pytest.mark.parametrize("name", ["tiny", "e128"])
def test_oracle_matches_hf_qwen3moe(name):
    d, (x, wr, w13, w2, k) = _hf_case(name)
    r = mo.moe_forward(x, wr, w13, w2, k, renorm=True)
    assert np.array_equal(r["ids"], d["ids"])
    np.testing.assert_allclose(r["w"], d["w"], rtol=1e-5, atol=1e-7)
    assert mo.rel_l2(r["y"], d["y"]) < 1e-5


def test_dyadic_logits_exact_in_any_order():
    from paper_2510_08055_b200.synthetic import router_tokens, router_weight

    x = router_tokens(37, 2048, 1).float().numpy()
    wr = router_weight(128, 2048, 2).float().numpy()
    l32 = mo.router_logits(x, wr)
    l64 = x.astype(np.float64) @ wr.astype(np.float64).T
    assert np.array_equal(l32.astype(np.float64), l64)
    # reversed summation order, blocked partial sums: identical
    lrev = np.zeros_like(l32)
    for h0 in range(2048 - 64, -1, -64):
        lrev += x[:, h0:h0 + 64] @ wr[:, h0:h0 + 64].T
    assert np.array_equal(lrev, l32)
    # pairwise distinct per token (tie-breaker column)
    assert all(len(set(row.tolist())) == 128 for row in l32)


def test_permute_is_stable_counting_sort():
    rng = np.random.default_rng(0)
    ids = rng.integers(0, 16, size=(100, 2)).astype(np.int32)
    counts, offsets, slot_of, tok_of = mo.permute(ids, 16)
    flat = ids.reshape(-1)
    assert counts.sum() == 200 and offsets[-1] == 200
    for e in range(16):
        entries = np.nonzero(flat == e)[0]
        slots = slot_of[entries]
        assert np.array_equal(slots, np.arange(offsets[e], offsets[e + 1]))
        assert np.array_equal(tok_of[slots], entries // 2)


def test_topk_tie_break_lower_index():
    logits_x = np.zeros((1, 4), np.float32)
    wr = np.zeros((8, 4), np.float32)  # all logits tie at 0
    ids, w, _ = mo.route(logits_x, wr, 3, renorm=True)
    assert ids.tolist() == [[0, 1, 2]]
    np.testing.assert_allclose(w, 1 / 3, rtol=1e-6)


# ---------------------------------------------------------------- union counts (reference KATs)
UNIFORM_CASES = [(1, 8, 128), (8, 8, 128), (5, 4, 32), (16, 1, 7), (3, 7, 7)]


@pytest.fixture(scope="module")
def union_gold():
    return np.load(os.path.join(GOLD, "union_counts.npz"))


@pytest.mark.parametrize("batch,k,E", UNIFORM_CASES)
def test_c_oracle_uniform_matches_reference(union_gold, batch, k, E):
    u = np.random.default_rng(42).random((500, batch, k))
    assert np.array_equal(uc.uniform_union_counts(u, batch, k, E), union_gold[f"uniform_{batch}_{k}_{E}"])


@pytest.mark.parametrize("batch,k,E,seed,trials", [(64, 8, 128, 7, 300), (576, 8, 128, 11, 50)])
def test_c_oracle_uniform_large_matches_reference(union_gold, batch, k, E, seed, trials):
    u = np.random.default_rng(seed).random((trials, batch, k))
    assert np.array_equal(uc.uniform_union_counts(u, batch, k, E), union_gold[f"uniform_{batch}_{k}_{E}_s{seed}"])


def _rank_power(E, skew):  # restated from moesim/coverage.py:101-106
    return (np.arange(E, dtype=np.float64) + 1.0) ** (-skew)


@pytest.mark.parametrize("skew", [0.0, 0.3, 1.0, 2.5])
def test_c_oracle_weighted_matches_reference(union_gold, skew):
    u = np.random.default_rng(9).random((400, 8, 8))
    got = uc.weighted_union_counts(u, 8, 8, 128, _rank_power(128, skew))
    assert np.array_equal(got, union_gold[f"weighted_{skew}"])


def test_c_oracle_weighted_k_equals_E(union_gold):
    u = np.random.default_rng(8).random((200, 3, 6))
    got = uc.weighted_union_counts(u, 3, 6, 6, _rank_power(6, 1.5))
    assert np.array_equal(got, union_gold["weighted_ke"])
    assert np.all(got == 6)


def test_c_oracle_single_token_is_k():
    u = np.random.default_rng(1).random((2000, 1, 8))
    assert np.all(uc.uniform_union_counts(u, 1, 8, 128) == 8)


def test_c_oracle_closed_form_mean():
    # reference test_kernels.py:75-83: mean within 1.5e-3 of 1-(1-k/E)^B
    u = np.random.default_rng(3).random((60_000, 8, 8))
    cov = uc.uniform_union_counts(u, 8, 8, 128).mean() / 128
    assert abs(cov - (1 - (1 - 8 / 128) ** 8)) < 1.5e-3
