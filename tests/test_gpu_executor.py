"""The unmodified reference simulator drives real MoE layers on the B200.

* `moesim.engine.run` plans every iteration (scheduler.plan_for); inside
  `refdrive.measured_costs(executor=LayeredExecutor(...))` each BatchPlan runs on a
  resident layer stack. SURVEY §8(d) C1 criterion: layered and chunked prefill run
  the same per-token math, so every prompt's final hidden states must agree — on
  this GPU path they are bit-identical (per-token routing and per-column tcgen05
  accumulation do not depend on which other tokens share the batch).
* `MeasuredCoverage(layer)` as the engine's / chunk bench's CoverageModel
  (engine.py:147-153, cli.py:222-227): coverage = nnz(counts)/E of the real routing,
  MoE runtime = measured device time.
"""

import pytest
import torch

from paper_2510_08055_b200 import QWEN3_30B_A3B, refdrive
from paper_2510_08055_b200.coverage import MeasuredCoverage
from paper_2510_08055_b200.executor import LayeredExecutor, MoEModel
from paper_2510_08055_b200.moe import GpuMoE
from paper_2510_08055_b200.synthetic import expert_weights, router_weight
from paper_2510_08055_b200.types import QWEN3_30B_A3B_MODEL, TINY

pytestmark = pytest.mark.gpu

if not refdrive.reference_available():
    pytest.skip("the reference (moesim) is not importable: tools/vendor_reference.sh", allow_module_level=True)
ms = refdrive.import_moesim()

TINY_MODEL = ms.types.ModelSpec(name="tiny-moe", num_layers=4, num_experts=16, top_k=2, bytes_per_expert=196608,
                                dense_bytes_per_layer=524288, flops_per_token_per_expert=196608,
                                attn_flops_per_token_per_ctx=4096, kv_bytes_per_token=4096, hidden_dim=256)


def _cfg(policy, chunk=512, target=512):
    return ms.types.SchedulerConfig(policy=ms.types.Policy(policy), chunk_size=chunk, group_token_target=target)


def _reqs(lens, out):
    return [ms.types.Request(id=i, arrival_s=0.0, input_len=n, output_len=out) for i, n in enumerate(lens)]


def _table():
    return ms.coverage.EmpiricalTable()


@pytest.fixture(scope="module")
def stack(cuda):
    return MoEModel(TINY, 4, device=cuda, seed=3)


def _run(stack, policy, reqs, chunk=512, target=512):
    ex = LayeredExecutor(stack, keep_final_prompt=True)
    with refdrive.measured_costs(executor=ex):
        res = ms.engine.run(TINY_MODEL, refdrive.b200_hardware(), _cfg(policy, chunk, target), reqs, _table())
    return res, ex


def test_layered_equals_chunked_final_hidden(stack):
    reqs = _reqs((1024, 700, 300), 4)
    lay = _run(stack, "layered", reqs)
    chk = _run(stack, "chunked", reqs)
    hyb = _run(stack, "hybrid", reqs, chunk=256)
    for rid in range(3):
        a = lay[1].final_prompt[rid]
        assert torch.equal(a, chk[1].final_prompt[rid]), rid
        assert torch.equal(a, hyb[1].final_prompt[rid]), rid
        assert a.abs().max().item() > 0


def test_measured_iterations_follow_the_reference_plan(stack):
    reqs = _reqs((1024, 64, 64), 6)
    res, ex = _run(stack, "layered", reqs)
    ref = ms.engine.run(TINY_MODEL, refdrive.b200_hardware(), _cfg("layered"), reqs, _table())
    assert len(res.records) == len(ref.records) and len(res.requests) == 3
    assert [r.prefill_tokens for r in res.records] == [r.prefill_tokens for r in ref.records]
    assert [r.designated_group for r in res.records] == [r.designated_group for r in ref.records]
    for rec, log in zip(res.records, ex.iter_log):
        assert log["moe_s"] > 0
        # each layer's experts hit never exceed E and cover at least top_k when tokens are routed
        for n, h in zip(log["routed"], log["experts_hit"]):
            assert (h == 0) == (n == 0) and h <= 16 and (n == 0 or h >= 2)
        # the reference engine records the bytes the GPU routing really loaded (engine.py:251)
        assert rec.expert_load_bytes == sum(log["experts_hit"]) * TINY_MODEL.bytes_per_expert
        assert rec.runtime_s > log["moe_s"]  # measured MoE + modelled attention/dense


def test_decode_graphs_match_eager(cuda):
    """Per-layer CUDA graphs for decode-size segments (MoEModel(graph_tokens=...)) give the
    same hidden states, routing and expert bytes as eager calls."""
    # all arrivals at t=0: the plan stream cannot depend on the measured (graph vs eager) timings
    reqs = _reqs((700, 40, 300, 5), 7)
    eager = MoEModel(TINY, 4, device=cuda, seed=3)
    graphed = MoEModel(TINY, 4, device=cuda, seed=3, graph_tokens=16)
    res = [_run(s, "layered", reqs) for s in (eager, graphed)]
    (ra, ca), (rb, cb) = res
    assert len(graphed.graphs.graphs) > 0
    assert [r.expert_load_bytes for r in ra.records] == [r.expert_load_bytes for r in rb.records]
    assert [g["experts_hit"] for g in ca.iter_log] == [g["experts_hit"] for g in cb.iter_log]
    for rid in range(4):
        assert torch.equal(ca.final_prompt[rid], cb.final_prompt[rid]), rid
        last = [c.final_decode.get(rid, c.decode_row.get(rid)) for c in (ca, cb)]  # finished / still live
        assert last[0] is not None and torch.equal(last[0], last[1]), rid


def test_segments_above_the_call_limit_run_in_row_slices(stack):
    """A segment larger than MoEModel.max_call_tokens (a layered-prefill cohort of many prompts)
    runs each layer in row slices: hidden states and per-layer expert counts are bit-identical to
    one call per layer."""
    g = torch.Generator(device=stack.device).manual_seed(5)
    x0 = torch.randn((1000, TINY.hidden), generator=g, device=stack.device).to(torch.bfloat16)
    outs = []
    for m in (MoEModel.max_call_tokens, 96):
        stack.max_call_tokens = m
        try:
            counts = torch.zeros((4, TINY.num_experts), dtype=torch.int32, device=stack.device)
            outs.append((stack.run_segment(x0.clone(), 0, 4, counts), counts))
        finally:
            del stack.max_call_tokens  # back to the class default
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    assert int(outs[0][1].sum()) == 4 * 1000 * TINY.top_k


@pytest.fixture(scope="module")
def qwen_layer(cuda):
    s = QWEN3_30B_A3B
    w13, w2 = expert_weights(s.num_experts, s.hidden, s.ffn, 5)
    return GpuMoE(s, router_weight(s.num_experts, s.hidden, 4).to(cuda), w13.to(cuda), w2.to(cuda))


def test_reference_engine_with_measured_coverage(qwen_layer):
    """moesim.engine.run with MeasuredCoverage as its CoverageModel: every coverage query routes
    real tokens through the Qwen3-30B-A3B layer; the engine's expert bytes are nnz·bytes_per_expert
    of that routing and its MoE runtime the measured device time."""
    cov = MeasuredCoverage(qwen_layer, seed=1)
    model = refdrive.reference_model(QWEN3_30B_A3B_MODEL)
    seen = []
    orig = cov.coverage

    def spy(n, rng=None):
        c = orig(n, rng)
        seen.append((n, c, cov.last_experts_hit, cov.last_device_s))
        return c

    cov.coverage = spy
    reqs = [ms.types.Request(id=0, arrival_s=0.0, input_len=2048, output_len=3),
            ms.types.Request(id=1, arrival_s=0.0, input_len=300, output_len=4)]
    with refdrive.measured_costs(coverage=cov):
        res = ms.engine.run(model, refdrive.b200_hardware(), _cfg("layered"), reqs, cov)
    assert seen and len(res.requests) == 2
    for n, c, hit, dev_s in seen:
        assert c == hit / 128 and dev_s > 0
        assert (hit == 0) == (n == 0) and hit <= min(128, 8 * n)
    # per iteration: expert bytes = Σ_scopes nnz · 9,437,184 · layers_in_scope (costmodel.py:77)
    assert ms.metrics.expert_load_total(res.records) > 0
    for rec in res.records:
        assert rec.expert_load_bytes % model.bytes_per_expert == 0


def test_reference_chunk_bench_with_measured_coverage(qwen_layer):
    """moesim.cli.chunk_bench_rows (cli.py:211-243) with MeasuredCoverage: the MoE column is the
    measured layer time x 48 layers per chunk, the bytes column nnz·bytes_per_expert·48."""
    model = refdrive.reference_model(QWEN3_30B_A3B_MODEL)
    cov = MeasuredCoverage(qwen_layer, seed=2)
    with refdrive.measured_costs(coverage=cov):
        rows = ms.cli.chunk_bench_rows(model, refdrive.b200_hardware(), cov, 4096, [512, 4096])
    modelled = ms.cli.chunk_bench_rows(model, refdrive.b200_hardware(), ms.coverage.UniformAnalytic(8, 128), 4096,
                                       [512, 4096])
    for r, m in zip(rows, modelled):
        assert r["num_chunks"] == m["num_chunks"]
        # every 512+-token batch hits all 128 experts, as the closed form says (P(miss) ~ 1e-8)
        assert r["moe_expert_bytes"] == r["num_chunks"] * 128 * model.bytes_per_expert * 48
        assert r["moe_runtime_s"] > 0 and r["moe_runtime_s"] != m["moe_runtime_s"]
    # one 4096-token chunk streams the weights once per layer instead of 8 times
    assert rows[1]["moe_expert_bytes"] * 8 == rows[0]["moe_expert_bytes"]


def _attn_reference(att, l, xs):
    """fp32 restatement of AttentionDense.layer over a whole prompt: RMSNorm (unit gain), QKV,
    causal GQA attention, output projection, residual."""
    x = xs.float()
    xn = x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-6)
    qkv = xn @ att.wqkv[l].float().t()
    T = x.shape[0]
    q = qkv[:, :att.qd].view(T, 32, 128).transpose(0, 1)
    k = qkv[:, att.qd:att.qd + att.kd].view(T, 4, 128).transpose(0, 1).repeat_interleave(8, 0)
    v = qkv[:, att.qd + att.kd:].view(T, 4, 128).transpose(0, 1).repeat_interleave(8, 0)
    s = (q @ k.transpose(1, 2)) / 128 ** 0.5
    s = s.masked_fill(torch.triu(torch.ones(T, T, dtype=torch.bool, device=x.device), 1), float("-inf"))
    o = torch.softmax(s, -1) @ v
    return x + o.transpose(0, 1).reshape(T, att.qd) @ att.wo[l].float().t()


def test_attention_dense_chunks_and_decode_match_fp32(cuda):
    """AttentionDense: a prompt prefilled in two chunks (the second attends to the cached first) and
    then one decode row give the rows a single fp32 causal pass over the whole sequence gives."""
    from paper_2510_08055_b200.executor import AttentionDense

    att = AttentionDense(256, 2, cuda, seed=5)
    g = torch.Generator(device=cuda).manual_seed(3)
    xs = torch.randn((20, 256), generator=g, device=cuda).to(torch.bfloat16)
    ref = _attn_reference(att, 1, xs)
    a = xs[:12].clone()
    att.layer(1, a, [(7, 0, 12, 20)])          # chunk 1: positions 0..11
    b = xs[12:19].clone()
    att.layer(1, b, [(7, 12, 7, 20)])          # chunk 2: positions 12..18 over the cached 0..11
    d = xs[19:20].clone()
    att.layer(1, d, [(7, 19, 1, 20)])          # decode row at position 19
    got = torch.cat([a, b, d]).float()
    err = ((got - ref).norm() / ref.norm()).item()
    assert err < 1e-2, err


def test_attention_pooled_kv_matches_per_request(cuda):
    """Pooled KV mode (one masked SDPA for every decode row, mixed context lengths) gives the rows the
    per-request caches give: three prompts of different lengths, then two decode steps of all three."""
    from paper_2510_08055_b200.executor import AttentionDense

    outs = []
    for pool in (0, 4):
        att = AttentionDense(256, 2, cuda, seed=5, pool_slots=pool, pool_len=64)
        g = torch.Generator(device=cuda).manual_seed(4)
        lens = {1: 9, 2: 17, 3: 30}
        rows = []
        for rid, n in lens.items():
            x = torch.randn((n, 256), generator=g, device=cuda).to(torch.bfloat16)
            att.layer(0, x, [(rid, 0, n, 40)])
            rows.append(x)
        for step in range(2):
            d = torch.randn((3, 256), generator=g, device=cuda).to(torch.bfloat16)
            att.layer(0, d, [(rid, n + step, 1, 40) for rid, n in lens.items()])
            rows.append(d)
        att.drop(2)
        outs.append(torch.cat(rows).float())
        if pool:
            assert att.free == [3, 1]  # slot of request 2 returned
    err = ((outs[0] - outs[1]).norm() / outs[0].norm()).item()
    assert err < 1e-2, err


def test_layered_vs_chunked_with_measured_attention(stack):
    """With measured attention + dense projections the reference engine's layered and chunked runs
    reach the same final prompt hidden states (bf16: different chunking gives different rounding,
    so a tolerance), and the engine charges the measured time for attention too."""
    from paper_2510_08055_b200.executor import AttentionDense

    reqs = _reqs((1024, 300), 3)
    out = {}
    for policy in ("layered", "chunked"):
        att = AttentionDense(TINY.hidden, 4, stack.device, seed=9)
        ex = LayeredExecutor(stack, keep_final_prompt=True, attention=att)
        with refdrive.measured_costs(executor=ex):
            res = ms.engine.run(TINY_MODEL, refdrive.b200_hardware(), _cfg(policy), reqs, _table())
        assert all(it["moe_s"] > 0 for it in ex.iter_log)
        assert len(att.kv) <= len(reqs)  # retired requests' caches are released on the next call
        out[policy] = ex
    for rid in range(2):
        a, b = out["layered"].final_prompt[rid].float(), out["chunked"].final_prompt[rid].float()
        assert ((a - b).norm() / a.norm()).item() < 3e-2, rid


def test_iteration_graphs_match_eager_pooled_attention(stack):
    """Decode-only iterations replayed as one CUDA graph of every layer (pooled-KV attention + MoE)
    reach the decode rows the eager per-layer calls reach, bit for bit."""
    from paper_2510_08055_b200.executor import AttentionDense

    reqs = _reqs((300, 200, 100), 6)
    out = {}
    for graphs in (0, 8):
        att = AttentionDense(TINY.hidden, 4, stack.device, seed=9, pool_slots=3, pool_len=320)
        ex = LayeredExecutor(stack, keep_final_prompt=True, attention=att, iteration_graphs=graphs)
        with refdrive.measured_costs(executor=ex):
            ms.engine.run(TINY_MODEL, refdrive.b200_hardware(), _cfg("layered"), reqs, _table())
        n = sum(it["graphed"] for it in ex.iter_log)
        assert (n > 0) == (graphs > 0), n
        assert all(it["moe_s"] > 0 for it in ex.iter_log)
        out[graphs] = ex
    for rid in range(3):
        # the last iteration's rows stay in decode_row (no later call retires them)
        a, b = (out[g].final_decode.get(rid, out[g].decode_row.get(rid)) for g in (0, 8))
        assert a.abs().max().item() > 0
        assert torch.equal(a, b), (rid, (a.float() - b.float()).abs().max().item())
