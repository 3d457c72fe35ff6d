"""BASELINE config 1 on the CPU: the tiny MoE (4 layers, 16 experts
top-2, d=256, ffn=128) serving one 1,024-token prompt (+8 output tokens) under layered
(G(1024)=2 groups of 2 layers) and chunked (C=512) prefill.

The serving planner/engine restatement (paper_2510_08055_b200.serving) drives a
test-only executor whose MoE layers are the fp32 numpy oracle (oracle/moe_oracle.py):
  * the final prompt hidden states of layered and chunked prefill agree (same
    per-token math; fp32 rel-L2 <= 1e-6);
  * expert bytes: the reference engine's byte model with the closed-form coverage
    (coverage.py:38-49, engine.py:137-154) gives layered 23,592,960 B vs chunked
    36,175,872 B, and the experts the oracle's routing actually touches give the
    same numbers (every 512/1,024-token layer call hits all 16 experts; a 1-token
    decode call exactly top_k = 2).
The GPU path's equivalent is tests/test_gpu_executor.py (bit-identical there).
"""

import numpy as np

from oracle import moe_oracle as mo
from paper_2510_08055_b200 import costmodel as cm
from paper_2510_08055_b200 import serving as sv
from paper_2510_08055_b200.coverage import UniformAnalytic
from paper_2510_08055_b200.synthetic import expert_weights, router_weight
from paper_2510_08055_b200.types import TINY, ModelSpec

TINY_MODEL = ModelSpec(name="tiny-moe", num_layers=4, num_experts=16, top_k=2, bytes_per_expert=196608,
                       dense_bytes_per_layer=524288, flops_per_token_per_expert=196608,
                       attn_flops_per_token_per_ctx=4096, kv_bytes_per_token=4096, hidden_dim=256)


def _rmsnorm(h, eps=1e-6):
    return h / np.sqrt(np.mean(h * h, axis=1, keepdims=True) + eps)


class OracleCost(sv.ModelledCost):
    """Modelled timing (reference formulas) + fp32 oracle hidden states, mirroring
    executor.MeasuredCost's batching: per iteration, layers with the same active row
    set run on one buffer: decode rows first, then the prefill slices."""

    def __init__(self, layers, coverage):
        super().__init__(coverage)
        self.layers = layers  # [(wr, w13, w2)] fp32
        self.stash, self.decode_row, self.final_prompt = {}, {}, {}
        self.hits = []  # experts touched per (layer call)

    def _prompt(self, st, rid):
        if rid not in self.stash:
            r = st.by_id[rid]
            self.stash[rid] = np.random.default_rng(1000 + rid).standard_normal((r.input_len, TINY.hidden),
                                                                                 dtype=np.float32)
        return self.stash[rid]

    def iteration(self, st, plan, decode_ctx):
        L = TINY_MODEL.num_layers
        for rid in [k for k in self.stash if st.by_id[k].phase == "finished"]:
            self.final_prompt[rid] = self.stash.pop(rid)
        dec = []
        for rid in plan.decode_ids:
            if rid not in self.decode_row:
                h = self.stash.pop(rid)
                self.final_prompt[rid] = h
                self.decode_row[rid] = h[-1].copy()
            dec.append(self.decode_row[rid])
        D = len(dec)
        cuts = sorted({0, L} | {a.layer_start for a in plan.prefill_assignments}
                      | {a.layer_end for a in plan.prefill_assignments})
        d = np.stack(dec) if D else np.zeros((0, TINY.hidden), np.float32)
        for l0, l1 in zip(cuts, cuts[1:]):
            act = [a for a in plan.prefill_assignments if a.layer_start <= l0 < a.layer_end]
            x = np.concatenate([d] + [self._prompt(st, a.request_id)[a.token_start:a.token_end] for a in act])
            if x.shape[0] == 0:
                continue
            for layer in range(l0, l1):  # h <- h + MoE_l(RMSNorm(h))
                wr, w13, w2 = self.layers[layer]
                out = mo.moe_forward(_rmsnorm(x), wr, w13, w2, TINY.top_k, TINY.norm_topk_prob)
                x = x + out["y"]
                self.hits.append(int((out["counts"] > 0).sum()))
            d = x[:D]
            off = D
            for a in act:
                self._prompt(st, a.request_id)[a.token_start:a.token_end] = x[off:off + a.num_tokens]
                off += a.num_tokens
        for rid, row in zip(plan.decode_ids, d):
            self.decode_row[rid] = row
        return super().iteration(st, plan, decode_ctx)


def _layers():
    out = []
    for layer in range(TINY_MODEL.num_layers):
        wr = router_weight(TINY.num_experts, TINY.hidden, 70 + layer).float().numpy()
        w13, w2 = expert_weights(TINY.num_experts, TINY.hidden, TINY.ffn, 80 + layer)
        out.append((wr, w13.float().numpy(), w2.float().numpy()))
    return out


def _serve(policy, layers):
    cost = OracleCost(layers, UniformAnalytic(TINY.top_k, TINY.num_experts))
    recs, done, _ = sv.run(TINY_MODEL, cm.H100_LIKE, sv.Planner(policy, 512, 512), [sv.Request(0, 0.0, 1024, 8)], cost)
    assert len(done) == 1 and done[0].tokens_emitted == 8
    return recs, cost


def test_c1_layered_vs_chunked_on_the_oracle():
    layers = _layers()
    lay_recs, lay = _serve("layered", layers)
    chk_recs, chk = _serve("chunked", layers)
    # the reference's byte model (closed-form coverage): 120 vs 184 expert loads of 196,608 B
    assert round(sum(r.expert_load_bytes for r in lay_recs)) == 23_592_960
    assert round(sum(r.expert_load_bytes for r in chk_recs)) == 36_175_872
    # the experts the oracle's routing really touched load the same bytes
    assert sum(lay.hits) * TINY_MODEL.bytes_per_expert == 23_592_960
    assert sum(chk.hits) * TINY_MODEL.bytes_per_expert == 36_175_872
    # same per-token math: the prompt's final hidden states agree (fp32)
    a, b = lay.final_prompt[0], chk.final_prompt[0]
    assert mo.rel_l2(a, b) <= 1e-6
    assert np.abs(a).max() > 0
