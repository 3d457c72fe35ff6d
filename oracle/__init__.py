"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the timed
CPU baseline. The product path (paper_2510_08055_b200) never imports it.

  moe_oracle.py   fp32 numpy restatement of the MoE layer (router/top-k,
                  permutation, SwiGLU experts, combine). Parity pinned against
                  HF transformers 5.5.0 Qwen3MoeSparseMoeBlock outputs
                  (tests/golden/hf_qwen3moe_*.npz, generator committed).
  union_counts.c  C restatement of the reference's numba routing-surrogate
                  kernels (moesim/kernels.py:73-145). Pinned against outputs of
                  the reference itself (tests/golden/union_counts.npz).
"""
