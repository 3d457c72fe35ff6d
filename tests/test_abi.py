"""C-ABI library: loads, exports every symbol include/lpmoe.h declares, validates
arguments before touching the GPU (CPU-only; no compute launched)."""

import ctypes
import os
import re

import pytest

from paper_2510_08055_b200 import _native
from paper_2510_08055_b200.types import ValidationError

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "lpmoe.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(lp_[a-z_0-9]+)\s*\(", src, flags=re.M)


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        from paper_2510_08055_b200 import build

        build.build()
    return _native.load()


def test_header_declares_expected_api():
    fns = set(header_functions())
    assert fns == set(_native.SIGNATURES), fns ^ set(_native.SIGNATURES)


def test_library_exports_every_header_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name


def test_version(lib):
    assert "sm_100a" in _native.version()


def test_workspace_bytes_monotone_and_aligned(lib):
    prev = 0
    for T in (1, 64, 576, 8224):
        b = lib.lp_moe_workspace_bytes(T, 2048, 768, 128, 8)
        assert b > prev and b % 256 == 0
        prev = b
    # dominated by the three [T*k, *] bf16 activation buffers
    assert lib.lp_moe_workspace_bytes(576, 2048, 768, 128, 8) >= 576 * 8 * (2048 + 768 + 2048) * 2
    assert lib.lp_moe_workspace_bytes(-1, 2048, 768, 128, 8) == 0


@pytest.mark.parametrize("H,I,E,k,msg", [
    (100, 768, 128, 8, "H must be"),
    (2048, 700, 128, 8, "I must be"),
    (2048, 768, 0, 8, "E must be"),
    (2048, 768, 128, 0, "topk"),
    (2048, 768, 4, 8, "topk"),
])
def test_invalid_dims_rejected_before_launch(lib, H, I, E, k, msg):
    rc = lib.lp_moe_forward(None, None, None, None, 16, H, I, E, k, 1, None, None, None, None, None, 0, None)
    assert rc == _native.LP_EINVAL
    code, text = _native.last_error()
    assert code == _native.LP_EINVAL and msg in text
    with pytest.raises(ValidationError, match=msg):
        _native.check(rc, "lp_moe_forward")


def test_unsupported_reported(lib):
    rc = lib.lp_moe_forward(None, None, None, None, 16, 2048, 768, 512, 8, 1, None, None, None, None, None, 0, None)
    assert rc == _native.LP_EUNSUPPORTED


def test_null_pointers_rejected(lib):
    rc = lib.lp_moe_forward(None, None, None, None, 16, 2048, 768, 128, 8, 1, None, None, None, None, None, 0, None)
    assert rc == _native.LP_EINVAL and "null" in _native.last_error()[1]


def test_empty_batch_is_a_noop(lib):
    assert lib.lp_moe_forward(None, None, None, None, 0, 2048, 768, 128, 8, 1, None, None, None, None, None, 0,
                              None) == _native.LP_OK
    assert lib.lp_union_counts_uniform(None, 0, 8, 8, 128, None, None) == _native.LP_OK


def test_union_counts_domain(lib):
    assert lib.lp_union_counts_uniform(None, 4, 8, 9, 8, None, None) == _native.LP_EINVAL  # k > E
    assert lib.lp_union_counts_uniform(None, 4, 8, 65, 128, None, None) == _native.LP_EUNSUPPORTED
    assert lib.lp_union_counts_weighted(None, 4, 8, 8, 2000, None, None, None) == _native.LP_EINVAL


def test_product_fails_loudly_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(_native.NativeLibraryMissing):
        _native.load()


def test_signatures_match_ctypes_arity(lib):
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for name, (_, args) in _native.SIGNATURES.items():
        m = re.search(rf"{name}\s*\(([^)]*)\)", src)
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), name
