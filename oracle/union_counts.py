"""ctypes wrapper of oracle/union_counts.c — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
_lib = None


def build(verbose: bool = False) -> str:
    """gcc the C restatement (no FMA contraction: results must be bit-exact)."""
    import subprocess

    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           os.path.join(HERE, "union_counts.c"), "-o", LIB_PATH]
    subprocess.run(cmd, check=True, capture_output=not verbose)
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        lib = ctypes.CDLL(LIB_PATH)
        i64 = ctypes.c_int64
        p = ctypes.c_void_p
        lib.oracle_uniform_union_counts.argtypes = [p, i64, i64, i64, i64, p]
        lib.oracle_weighted_union_counts.argtypes = [p, i64, i64, i64, i64, p, p]
        _lib = lib
    return _lib


def uniform_union_counts(u: np.ndarray, batch: int, k: int, num_experts: int) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    trials = u.shape[0]
    out = np.zeros(trials, dtype=np.int64)
    if batch == 0 or trials == 0:
        return out
    rc = _load().oracle_uniform_union_counts(u.ctypes.data, trials, batch, k, num_experts, out.ctypes.data)
    assert rc == 0
    return out


def weighted_union_counts(u: np.ndarray, batch: int, k: int, num_experts: int, weights: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    trials = u.shape[0]
    out = np.zeros(trials, dtype=np.int64)
    if batch == 0 or trials == 0:
        return out
    rc = _load().oracle_weighted_union_counts(u.ctypes.data, trials, batch, k, num_experts, w.ctypes.data,
                                             out.ctypes.data)
    assert rc == 0
    return out
