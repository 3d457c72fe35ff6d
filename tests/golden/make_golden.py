"""Generate the committed golden fixtures under tests/golden/.

Runs ONLY in the build container, where the reference (/root/reference, read-only)
and HF transformers 5.5.0 are importable; the fixtures it writes travel with
the repo so nothing on the GPU box needs either. Re-run with:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Fixtures (inputs are regenerated from the recorded seeds; only outputs stored):
  union_counts.npz     moesim.kernels._uniform/_weighted_union_counts_nb outputs
                       on the exact cases of the reference's tests
                       (pkg/tests/test_kernels.py:33-50, :96-101).
  hf_qwen3moe_*.npz    transformers Qwen3MoeSparseMoeBlock (fp32, weights from
                       paper_2510_08055_b200.synthetic) outputs: y, top-k ids,
                       routing weights.
  plans.json           moesim.scheduler plan streams for the planner mirror
                       (SPEC.md:404-443 worked examples + engine-driven runs).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

# ---------------------------------------------------------------- union counts
UNIFORM_CASES = [(1, 8, 128), (8, 8, 128), (5, 4, 32), (16, 1, 7), (3, 7, 7)]  # test_kernels.py:34
UNIFORM_SEED, UNIFORM_TRIALS = 42, 500
WEIGHTED_SKEWS = [0.0, 0.3, 1.0, 2.5]  # test_kernels.py:42
WEIGHTED_SEED, WEIGHTED_TRIALS = 9, 400
EXTRA_UNIFORM = [(64, 8, 128, 7, 300), (576, 8, 128, 11, 50)]  # (batch, k, E, seed, trials) larger cases
KE_CASE = (3, 6, 6, 1.5, 8, 200)  # test_kernels.py:96-101 (batch, k, E, skew, seed, trials)

# ---------------------------------------------------------------- HF layer cases
# (name, T, H, I, E, k, seed_w, seed_x, tie_break)
HF_CASES = [
    ("tiny", 64, 256, 128, 16, 2, 101, 202, True),
    ("e128", 48, 256, 128, 128, 8, 303, 404, True),
]


def make_union_counts():
    from moesim import kernels
    from moesim.coverage import rank_power_weights

    out = {}
    for batch, k, E in UNIFORM_CASES:
        u = np.random.default_rng(UNIFORM_SEED).random((UNIFORM_TRIALS, batch, k))
        out[f"uniform_{batch}_{k}_{E}"] = kernels._uniform_union_counts_nb(u, batch, k, E)
    for batch, k, E, seed, trials in EXTRA_UNIFORM:
        u = np.random.default_rng(seed).random((trials, batch, k))
        out[f"uniform_{batch}_{k}_{E}_s{seed}"] = kernels._uniform_union_counts_nb(u, batch, k, E)
    for skew in WEIGHTED_SKEWS:
        w = rank_power_weights(128, skew)
        u = np.random.default_rng(WEIGHTED_SEED).random((WEIGHTED_TRIALS, 8, 8))
        out[f"weighted_{skew}"] = kernels._weighted_union_counts_nb(u, 8, 8, 128, w)
    batch, k, E, skew, seed, trials = KE_CASE
    u = np.random.default_rng(seed).random((trials, batch, k))
    out["weighted_ke"] = kernels._weighted_union_counts_nb(u, batch, k, E, rank_power_weights(E, skew))
    np.savez_compressed(os.path.join(HERE, "union_counts.npz"), **out)
    print("union_counts.npz:", {k_: v.shape for k_, v in out.items()})


def make_hf():
    import torch
    from transformers.models.qwen3_moe.configuration_qwen3_moe import Qwen3MoeConfig
    from transformers.models.qwen3_moe.modeling_qwen3_moe import Qwen3MoeSparseMoeBlock

    from paper_2510_08055_b200.synthetic import expert_weights, router_tokens, router_weight

    for name, T, H, I, E, k, sw, sx, tb in HF_CASES:
        cfg = Qwen3MoeConfig(hidden_size=H, moe_intermediate_size=I, num_experts=E, num_experts_per_tok=k,
                             norm_topk_prob=True, hidden_act="silu")
        block = Qwen3MoeSparseMoeBlock(cfg).float().eval()
        wr = router_weight(E, H, sw, tie_break=tb).float()
        w13, w2 = expert_weights(E, H, I, sw + 1)
        x = router_tokens(T, H, sx, tie_break=tb).float()
        with torch.no_grad():
            block.gate.weight.copy_(wr)
            block.experts.gate_up_proj.copy_(w13.float())
            block.experts.down_proj.copy_(w2.float())
            logits, scores, idx = block.gate(x)
            y = block(x[None])[0]
        np.savez_compressed(os.path.join(HERE, f"hf_qwen3moe_{name}.npz"), y=y.numpy().astype(np.float32),
                            ids=idx.numpy().astype(np.int32), w=scores.numpy().astype(np.float32),
                            meta=np.array([T, H, I, E, k, sw, sx, int(tb)], np.int64))
        print(f"hf_qwen3moe_{name}.npz", y.shape)


def main():
    make_union_counts()
    make_hf()
    if os.path.exists(os.path.join(HERE, "make_plans.py")):
        from make_plans import make_plans  # noqa: E402  (sibling script)

        make_plans(os.path.join(HERE, "plans.json"))


if __name__ == "__main__":
    sys.path.insert(0, HERE)
    main()
