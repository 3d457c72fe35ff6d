"""Shape/byte constants of the hot path vs the reference's config and tests (CPU-only)."""

import pytest

from paper_2510_08055_b200.types import (QWEN3_30B_A3B, QWEN3_30B_A3B_MODEL, MoEShape, ModelSpec, ValidationError,
                                         total_expert_bytes)


def test_qwen_shape_from_reference_config():
    # configs/qwen30b.toml:12-23 -> I = 9437184 / (3*2048*2) = 768
    s = MoEShape.from_model(QWEN3_30B_A3B_MODEL)
    assert (s.hidden, s.ffn, s.num_experts, s.top_k) == (2048, 768, 128, 8)
    assert s == QWEN3_30B_A3B
    assert s.bytes_per_expert == 9_437_184 == QWEN3_30B_A3B_MODEL.bytes_per_expert
    assert s.flops_per_token_per_expert == QWEN3_30B_A3B_MODEL.flops_per_token_per_expert  # 2*3*H*I


def test_layer_and_model_expert_bytes():
    assert 128 * QWEN3_30B_A3B.bytes_per_expert == 1_207_959_552
    assert total_expert_bytes(QWEN3_30B_A3B_MODEL) == 57_982_058_496
    # reference test_types.py:93-116 window (53-58 GB) for 48x128 experts
    assert 53e9 <= total_expert_bytes(QWEN3_30B_A3B_MODEL) <= 58e9


@pytest.mark.parametrize("kw,msg", [
    (dict(hidden=100), "hidden"),
    (dict(ffn=0), "ffn"),
    (dict(num_experts=300), "num_experts"),
    (dict(top_k=0), "top_k"),
    (dict(top_k=33, num_experts=64), "top_k"),
])
def test_moeshape_validation(kw, msg):
    base = dict(hidden=2048, ffn=768, num_experts=128, top_k=8)
    base.update(kw)
    with pytest.raises(ValidationError, match=msg):
        MoEShape(**base)


def test_modelspec_validation_mirrors_reference():
    with pytest.raises(ValidationError, match="top_k out of range"):
        ModelSpec("m", 1, 4, 5, 1, 1, 1, 1, 1, 1)
    with pytest.raises(ValueError):
        ModelSpec("m", 0, 4, 2, 1, 1, 1, 1, 1, 1)
