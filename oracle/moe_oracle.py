"""fp32 numpy oracle of the MoE layer — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference simulator has no numerical MoE layer (moesim SPEC.md:135: "no
weights, no numerical model execution"); it only charges its cost
(costmodel.py:57-85) at engine.py:144-154. The numerics therefore follow the
third-party model the reference's configs describe — Qwen3-30B-A3B as
implemented by HF transformers 5.5.0 (not under /root/reference):

  router  modeling_qwen3_moe.py:260-270  logits = x.Wr^T; softmax(float);
                                         topk; optional /= sum (norm_topk_prob)
  experts modeling_qwen3_moe.py:229-249  per expert: linear(x, gate_up[e]).chunk(2)
                                         -> silu(gate)*up -> linear(., down[e])
                                         -> * w -> index_add_
Pinned against that implementation by tests/golden/hf_qwen3moe_*.npz
(tests/golden/make_golden.py). Tie-break of top-k is fixed to
(logit desc, expert index asc); the expert-contiguous slot order is the stable
sort of entries t*k+j by expert, i.e. the order of HF's torch.where loop.
"""

from __future__ import annotations

import numpy as np


def router_logits(x: np.ndarray, wr: np.ndarray) -> np.ndarray:
    """fp32 logits [T, E]. Exact for the dyadic synthetic inputs in any order."""
    return np.asarray(x, np.float32) @ np.asarray(wr, np.float32).T


def route(x: np.ndarray, wr: np.ndarray, top_k: int, renorm: bool):
    """-> ids int32 [T,k], w fp32 [T,k], logits fp32 [T,E]."""
    logits = router_logits(x, wr)
    T, E = logits.shape
    # selection on logits (softmax is monotone); ties -> lower expert index
    order = np.lexsort((np.broadcast_to(np.arange(E), (T, E)), -logits), axis=-1)
    ids = order[:, :top_k].astype(np.int32)
    m = logits.max(axis=1, keepdims=True)
    p = np.exp((logits - m).astype(np.float64))
    p = (p / p.sum(axis=1, keepdims=True)).astype(np.float32)
    w = np.take_along_axis(p, ids.astype(np.int64), axis=1)
    if renorm:
        w = w / w.sum(axis=1, keepdims=True)
    return ids, w.astype(np.float32), logits


def permute(ids: np.ndarray, num_experts: int):
    """Stable counting sort of the flattened routing entries by expert.

    -> counts [E], offsets [E+1], slot_of [T*k], tok_of [T*k]
    """
    flat = ids.reshape(-1).astype(np.int64)
    k = ids.shape[1] if ids.ndim == 2 else 1
    counts = np.bincount(flat, minlength=num_experts).astype(np.int32)
    offsets = np.zeros(num_experts + 1, np.int32)
    np.cumsum(counts, out=offsets[1:])
    order = np.argsort(flat, kind="stable")          # slot -> entry
    slot_of = np.empty_like(order)
    slot_of[order] = np.arange(order.size)
    tok_of = (order // k).astype(np.int32)
    return counts, offsets, slot_of.astype(np.int32), tok_of


def silu(v: np.ndarray) -> np.ndarray:
    return v / (1.0 + np.exp(-v))


def experts(x_perm: np.ndarray, offsets: np.ndarray, w13: np.ndarray, w2: np.ndarray):
    """-> act [S, I], y_perm [S, H] in fp32."""
    S, H = x_perm.shape
    E, I2, _ = w13.shape
    I = I2 // 2
    act = np.zeros((S, I), np.float32)
    y_perm = np.zeros((S, H), np.float32)
    for e in range(E):
        a, b = int(offsets[e]), int(offsets[e + 1])
        if a == b:
            continue
        xe = np.asarray(x_perm[a:b], np.float32)
        we = np.asarray(w13[e], np.float32)
        gate = xe @ we[:I].T
        up = xe @ we[I:].T
        act[a:b] = silu(gate) * up
        y_perm[a:b] = act[a:b] @ np.asarray(w2[e], np.float32).T
    return act, y_perm


def combine(y_perm: np.ndarray, slot_of: np.ndarray, w: np.ndarray) -> np.ndarray:
    T, k = w.shape
    gathered = y_perm[slot_of.reshape(T, k)]            # [T, k, H]
    return np.einsum("tk,tkh->th", w.astype(np.float32), gathered, dtype=np.float32)


def moe_forward(x, wr, w13, w2, top_k: int, renorm: bool = True):
    """Full layer. Returns dict with every intermediate the GPU path exposes."""
    x = np.asarray(x, np.float32)
    E = wr.shape[0]
    ids, w, logits = route(x, wr, top_k, renorm)
    counts, offsets, slot_of, tok_of = permute(ids, E)
    x_perm = x[tok_of]
    act, y_perm = experts(x_perm, offsets, w13, w2)
    y = combine(y_perm, slot_of, w)
    return dict(ids=ids, w=w, logits=logits, counts=counts, offsets=offsets, slot_of=slot_of, tok_of=tok_of,
                act=act, y_perm=y_perm, y=y)


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
