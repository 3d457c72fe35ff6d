"""Host planner/engine restatement vs plan streams and summaries recorded from the
reference simulator (tests/golden/plans.json, made by tests/golden/make_plans.py)."""

import json
import os

import pytest

from paper_2510_08055_b200 import costmodel as cm
from paper_2510_08055_b200 import serving as sv
from paper_2510_08055_b200.types import ModelSpec

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "plans.json")))


def _hw(d):
    return cm.HardwareSpec(d["name"], d["peak_flops"], d["peak_hbm_bw"], d["mfu"], d["mbu"], d["kv_capacity_bytes"],
                           d["iteration_overhead_s"])


class Spy(sv.Planner):
    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.plans = []

    def plan(self, st):
        p = super().plan(st)
        self.plans.append(p)
        return p


@pytest.mark.parametrize("name", sorted(GOLD["scenarios"]))
def test_plan_stream_matches_reference(name):
    sc = GOLD["scenarios"][name]
    model = ModelSpec(**sc["model"])
    reqs = [sv.Request(i, a, li, lo) for i, a, li, lo in sc["requests"]]
    planner = Spy(sc["policy"], sc["chunk_size"], sc["group_token_target"])
    recs, done, makespan = sv.run(model, _hw(sc["hw"]), planner, reqs, seed=7)
    assert len(recs) == len(sc["iterations"])
    for p, rec, (dec, asg, runtime, eload) in zip(planner.plans, recs, sc["iterations"]):
        assert list(p.decode_ids) == dec
        assert [[a.request_id, a.token_start, a.token_end, a.layer_start, a.layer_end]
                for a in p.prefill_assignments] == asg
        assert rec.runtime_s == runtime          # bit-exact float
        assert rec.expert_load_bytes == eload
    s = sv.summarize(recs, done, makespan)
    for k in ("ttft_mean_s", "ttft_p99_s", "tbt_mean_s", "tbt_p99_s", "makespan_s", "num_iterations",
              "num_requests", "mean_decode_batch", "e2e_latency_mean_s"):
        assert s[k] == sc["summary"][k], k
    assert s["total_expert_load_bytes"] == sc["summary"]["total_expert_load_bytes"]


@pytest.mark.parametrize("policy", ["chunked", "layered"])
def test_arxiv_trace_summary_matches_reference(policy):
    model = ModelSpec(**GOLD["scenarios"]["qwen_chunked_c512_g512"]["model"])
    reqs = [sv.Request(i, a, li, lo) for i, a, li, lo in GOLD["arxiv"]["requests"]]
    recs, done, makespan = sv.run(model, cm.H100_LIKE, sv.Planner(policy, 512, 512), reqs, seed=7)
    s = sv.summarize(recs, done, makespan)
    ref = GOLD["arxiv"]["summaries"][policy]
    for k in ("ttft_mean_s", "ttft_p99_s", "tbt_mean_s", "tbt_p99_s", "num_iterations", "total_expert_load_bytes"):
        assert s[k] == ref[k], k


def test_spec_worked_examples():
    # G(8192)=16, (48,16) -> 16 groups of 3, hybrid L=1024/C=512/G=2 -> 3 steps
    assert sv.num_groups(8192, 512) == 16
    assert sv.num_groups(100_000, 512, 48) == 48
    assert sv.num_groups(1, 512) == 1
    b = sv.layer_boundaries(48, 16)
    assert len(b) == 17 and all(b[i + 1] - b[i] == 3 for i in range(16))
    assert sv.layer_boundaries(4, 2) == (0, 2, 4)
    assert sv.layer_boundaries(10, 4) == (0, 3, 6, 8, 10)  # larger groups first
    model = ModelSpec(**GOLD["scenarios"]["tiny_layered"]["model"])
    reqs = [sv.Request(0, 0.0, 1024, 2)]
    recs, done, _ = sv.run(model, cm.H100_LIKE, sv.Planner("hybrid", 512, 512), reqs)
    prefill_iters = [r for r in recs if r.prefill_tokens]
    assert len(prefill_iters) == 3  # chunks 0,1 through groups 0,1 in lockstep
    recs, done, _ = sv.run(model, cm.H100_LIKE, sv.Planner("layered", 512, 512), reqs)
    assert sum(1 for r in recs if r.prefill_tokens) == 2  # exactly G(1024)=2 layered iterations


def test_layer_token_counts():
    p = sv.BatchPlan((1, 2, 3), (sv.PrefillAssignment(9, 0, 100, 3, 6),))
    n = p.layer_token_counts(8)
    assert n == [3, 3, 3, 103, 103, 103, 3, 3]


def test_coverage_golden_values():
    # reference pkg/tests/test_coverage.py:20-29, :57-65, :88-92
    assert cm.expected_coverage_uniform(8, 8, 128) == pytest.approx(1 - 2562890625 / 4294967296, abs=1e-15)
    for b, c in cm.DEFAULT_COVERAGE_TABLE:
        assert cm.coverage_from_table(b) == c
    import math
    t = (math.log(12) - math.log(8)) / (math.log(16) - math.log(8))
    assert cm.coverage_from_table(12) == pytest.approx(0.290 + (0.445 - 0.290) * t)
    assert cm.tokens_per_expert(2048, 8, 128) == 128 and cm.tokens_per_expert(8192, 8, 128) == 512
    assert cm.coverage_from_table(0) == 0.0


def test_validation_errors():
    from paper_2510_08055_b200.types import ValidationError

    with pytest.raises(ValidationError):
        sv.Planner("bogus")
    with pytest.raises(ValidationError):
        sv.Request(0, 0.0, 0, 1)


# ---------------------------------------------------------------- trace CSV (workload.py:14, :145-178)
def test_trace_roundtrip_matches_reference_bytes(tmp_path):
    """load_trace reads the reference's export byte for byte; export_trace writes the same bytes."""
    import os

    from paper_2510_08055_b200 import serving as sv

    gold = os.path.join(os.path.dirname(__file__), "golden", "trace_arxiv10.csv")
    reqs = sv.load_trace(gold)
    assert [r.id for r in reqs] == list(range(10))
    assert reqs[0].input_len == 11567 and reqs[0].output_len == 385
    out = tmp_path / "t.csv"
    sv.export_trace(reqs, out)
    assert out.read_bytes() == open(gold, "rb").read()


def test_trace_errors_match_reference(tmp_path):
    import json
    import os

    import pytest

    from paper_2510_08055_b200 import serving as sv
    from paper_2510_08055_b200.types import ValidationError

    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "trace_errors.json")))
    for name, case in cases.items():
        p = tmp_path / f"{name}.csv"
        p.write_text(case["text"])
        with pytest.raises(ValidationError) as ei:
            sv.load_trace(str(p))
        assert str(ei.value).replace(str(p), "<path>") == case["message"]
