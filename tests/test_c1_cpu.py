"""BASELINE config 1 on the CPU: the tiny MoE (4 layers, 16 experts
top-2, d=256, ffn=128) serving one 1,024-token prompt (+8 output tokens) under layered
(G(1024)=2 groups of 2 layers) and chunked (C=512) prefill.

The UNMODIFIED reference engine (`moesim.engine.run`, engine.py:272-351) plans and
clocks every iteration; `refdrive.measured_costs(executor=...)` hands each BatchPlan
to a test-only executor whose MoE layers are the fp32 numpy oracle
(oracle/moe_oracle.py), exactly as the GPU run hands it to executor.LayeredExecutor:
  * the final prompt hidden states of layered and chunked prefill agree (same
    per-token math; fp32 rel-L2 <= 1e-6);
  * expert bytes: the reference engine's own byte model with the closed-form coverage
    (coverage.py:38-49, engine.py:137-154) gives layered 23,592,960 B vs chunked
    36,175,872 B, and the experts the oracle's routing actually touches — recorded by
    the reference engine itself in IterationRecord.expert_load_bytes — give the same.
The GPU path's equivalent is tests/test_gpu_executor.py (bit-identical there).
"""

import time

import numpy as np
import pytest

from oracle import moe_oracle as mo
from paper_2510_08055_b200 import refdrive
from paper_2510_08055_b200.executor import MoEIteration
from paper_2510_08055_b200.synthetic import expert_weights, router_weight
from paper_2510_08055_b200.types import TINY

if not refdrive.reference_available():
    pytest.skip("the reference (moesim) is not importable: tools/vendor_reference.sh", allow_module_level=True)
ms = refdrive.import_moesim()

TINY_MODEL = ms.types.ModelSpec(name="tiny-moe", num_layers=4, num_experts=16, top_k=2, bytes_per_expert=196608,
                                dense_bytes_per_layer=524288, flops_per_token_per_expert=196608,
                                attn_flops_per_token_per_ctx=4096, kv_bytes_per_token=4096, hidden_dim=256)
H100 = ms.types.HardwareSpec(name="h100-like", peak_flops=989e12, peak_hbm_bw=3.35e12, kv_capacity_bytes=40e9,
                             iteration_overhead_s=2e-3)  # configs/h100like.toml


def _rmsnorm(h, eps=1e-6):
    return h / np.sqrt(np.mean(h * h, axis=1, keepdims=True) + eps)


class OracleExecutor:
    """executor.LayeredExecutor's batching with fp32 oracle layers: per iteration, layers
    with the same active row set run on one buffer: decode rows first, then the slices."""

    def __init__(self, layers):
        self.layers = layers  # [(wr, w13, w2)] fp32
        self.stash, self.decode_row, self.final_prompt = {}, {}, {}
        self.hits = []  # experts touched per (layer call)

    def _prompt(self, state, rid):
        if rid not in self.stash:
            n = state.request(rid).input_len
            self.stash[rid] = np.random.default_rng(1000 + rid).standard_normal((n, TINY.hidden), dtype=np.float32)
        return self.stash[rid]

    def run_plan(self, state, plan):
        t0 = time.perf_counter()
        L = TINY_MODEL.num_layers
        for rid in [k for k in self.stash if state.request(k).phase == ms.types.Phase.FINISHED]:
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
        routed, hit = [0] * L, [0] * L
        d = np.stack(dec) if D else np.zeros((0, TINY.hidden), np.float32)
        for l0, l1 in zip(cuts, cuts[1:]):
            act = [a for a in plan.prefill_assignments if a.layer_start <= l0 < a.layer_end]
            x = np.concatenate([d] + [self._prompt(state, a.request_id)[a.token_start:a.token_end] for a in act])
            if x.shape[0] == 0:
                continue
            for layer in range(l0, l1):  # h <- h + MoE_l(RMSNorm(h))
                wr, w13, w2 = self.layers[layer]
                out = mo.moe_forward(_rmsnorm(x), wr, w13, w2, TINY.top_k, TINY.norm_topk_prob)
                x = x + out["y"]
                routed[layer], hit[layer] = x.shape[0], int((out["counts"] > 0).sum())
                self.hits.append(hit[layer])
            d = x[:D]
            off = D
            for a in act:
                self._prompt(state, a.request_id)[a.token_start:a.token_end] = x[off:off + a.num_tokens]
                off += a.num_tokens
        for rid, row in zip(plan.decode_ids, d):
            self.decode_row[rid] = row
        return MoEIteration(time.perf_counter() - t0, routed, hit)


def _layers():
    out = []
    for layer in range(TINY_MODEL.num_layers):
        wr = router_weight(TINY.num_experts, TINY.hidden, 70 + layer).float().numpy()
        w13, w2 = expert_weights(TINY.num_experts, TINY.hidden, TINY.ffn, 80 + layer)
        out.append((wr, w13.float().numpy(), w2.float().numpy()))
    return out


def _cfg(policy):
    return ms.types.SchedulerConfig(policy=ms.types.Policy(policy), chunk_size=512, group_token_target=512)


def _coverage():
    return ms.coverage.UniformAnalytic(top_k=TINY_MODEL.top_k, num_experts=TINY_MODEL.num_experts)


def _serve(policy, layers):
    ex = OracleExecutor(layers)
    reqs = [ms.types.Request(id=0, arrival_s=0.0, input_len=1024, output_len=8)]
    with refdrive.measured_costs(executor=ex):
        res = ms.engine.run(TINY_MODEL, H100, _cfg(policy), reqs, _coverage())
    assert len(res.requests) == 1 and res.requests[0].tokens_emitted == 8
    return res, ex


def test_c1_layered_vs_chunked_on_the_oracle():
    layers = _layers()
    lay, lay_ex = _serve("layered", layers)
    chk, chk_ex = _serve("chunked", layers)
    # the reference engine's own byte model (closed-form coverage, no adapter)
    for policy, want in (("layered", 23_592_960), ("chunked", 36_175_872)):
        modelled = ms.engine.run(TINY_MODEL, H100, _cfg(policy),
                                 [ms.types.Request(id=0, arrival_s=0.0, input_len=1024, output_len=8)], _coverage())
        assert round(ms.metrics.expert_load_total(modelled.records)) == want
    # the experts the oracle's routing really touched, as recorded by the reference engine
    assert ms.metrics.expert_load_total(lay.records) == 23_592_960
    assert ms.metrics.expert_load_total(chk.records) == 36_175_872
    assert sum(lay_ex.hits) * TINY_MODEL.bytes_per_expert == 23_592_960
    # same per-token math: the prompt's final hidden states agree (fp32)
    a, b = lay_ex.final_prompt[0], chk_ex.final_prompt[0]
    assert mo.rel_l2(a, b) <= 1e-6
    assert np.abs(a).max() > 0


def test_adapter_restores_the_reference():
    """measured_costs() rebinds the engine / cli call-site names only inside its with-block."""
    before = (ms.engine.iteration_runtime, ms.engine._iteration_kernels, ms.engine.moe_cost,
              ms.cli.kernel_runtime, ms.cli.moe_cost)
    with refdrive.measured_costs(coverage=_coverage(), executor=OracleExecutor(_layers())):
        assert ms.engine._iteration_kernels is not before[1]
    assert (ms.engine.iteration_runtime, ms.engine._iteration_kernels, ms.engine.moe_cost,
            ms.cli.kernel_runtime, ms.cli.moe_cost) == before


def test_measured_kernel_runtime_is_the_measured_time():
    """A measured MoE kernel charges its device seconds; other kernels keep the roofline."""
    k = refdrive.measured_moe_kernel(TINY_MODEL, [10, 10], [5, 6], 1.25e-3)
    assert k.expert_weight_bytes == 11 * TINY_MODEL.bytes_per_expert
    assert k.flops == 20 * TINY_MODEL.top_k * TINY_MODEL.flops_per_token_per_expert
    dense = ms.costmodel.dense_cost(TINY_MODEL, 10, 2)
    with refdrive.measured_costs():
        assert ms.engine.iteration_runtime([k, dense], H100) == 1.25e-3 + ms.costmodel.kernel_runtime(dense, H100)
