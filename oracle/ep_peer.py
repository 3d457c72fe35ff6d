"""CPU restatement of the peer-memory expert-parallel protocol (test infrastructure).

Follows paper_2510_08055_b200/csrc/ep_p2p.cuh kernel by kernel (the reference,
moesim, has no multi-GPU code: SPEC.md:24). "Peer memory" is any set of per-rank
buffers every rank can index (tests use shared-memory CPU tensors across gloo
processes); barriers are the caller's. Only tests/ import this module.
"""

from __future__ import annotations

import numpy as np


def post_counts(counts: np.ndarray, inboxes: list, rank: int, layer: int) -> None:
    """k_ep_exchange, first half: inbox_d[layer & 1][rank][:] = counts (this rank's per-global-expert
    counts) for every rank d; the GPU follows it with a system-scope ready tag = layer + 1, which
    the callers here replace with a barrier."""
    for box in inboxes:
        box[layer & 1, rank, :] = counts


def plan(inbox: np.ndarray, P: int, El: int, rank: int, layer: int):
    """k_ep_exchange, second half, from this rank's OWN inbox [2][P src][E] once every source posted:
    -> dest_base [P*El] (this rank's first row per (owner d, expert el) in d's receive buffer; rows
    expert-major, source-rank-major within an expert) and off_local [El+1] (this rank's expert
    offsets over all sources)."""
    cnt = np.asarray(inbox[layer & 1]).reshape(P, P, El)  # [src, dest, el]
    dest_base = np.zeros(P * El, np.int64)
    for d in range(P):
        for el in range(El):
            dest_base[d * El + el] = cnt[:, d, :el].sum() + cnt[:rank, d, el].sum()
    per_expert = cnt[:, rank, :].sum(axis=0)  # rows rank receives per local expert
    off_local = np.zeros(El + 1, np.int64)
    np.cumsum(per_expert, out=off_local[1:])
    return dest_base, off_local


def dispatch(x: np.ndarray, ids: np.ndarray, slot_of: np.ndarray, offsets: np.ndarray, dest_base: np.ndarray,
             recv: list, El: int):
    """k_ep_dispatch: entry i = t*k + j stores x[t] into recv[d][dest_base[d*El+el] + slot_of[i] - offsets[e]]."""
    k = ids.shape[1]
    flat = ids.reshape(-1)
    dest_rank = flat // El
    row = dest_base[flat] + (slot_of - offsets[flat])
    for i in range(flat.size):
        recv[int(dest_rank[i])][int(row[i])] = x[i // k]
    return dest_rank, row


def combine(y_out: list, dest_rank: np.ndarray, dest_row: np.ndarray, w: np.ndarray) -> np.ndarray:
    """k_ep_combine: y[t] = sum_j w[t,j] * y_out[dest_rank][dest_row] in fixed j order (fp32)."""
    T, k = w.shape
    H = np.asarray(y_out[0]).shape[1]
    y = np.zeros((T, H), np.float32)
    for t in range(T):
        for j in range(k):
            i = t * k + j
            y[t] += w[t, j] * np.asarray(y_out[int(dest_rank[i])][int(dest_row[i])], np.float32)
    return y
