"""ctypes binding of liblpmoe.so (the C ABI declared in include/lpmoe.h).

The shared library is built in-tree by `__graft_entry__.build()` (or
`python -m paper_2510_08055_b200.build`). There is no fallback: if the library
is missing or a call fails, this module raises. Error mapping mirrors the
reference's conventions: argument-domain errors are `ValidationError`
(a `ValueError`, moesim/types.py:10-16), CUDA failures are `RuntimeError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .types import ValidationError

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.environ.get("LPMOE_LIB") or os.path.join(LIB_DIR, "liblpmoe.so")  # override: trace builds

LP_OK = 0
LP_EINVAL = 1
LP_ECUDA = 2
LP_EUNSUPPORTED = 3

# (symbol, restype, argtypes) — must match include/lpmoe.h exactly.
_p = ctypes.c_void_p
_i = ctypes.c_int
_sz = ctypes.c_size_t
SIGNATURES = {
    "lp_version": (ctypes.c_char_p, []),
    "lp_last_error": (_i, [ctypes.c_char_p, _sz]),
    "lp_launch_count": (ctypes.c_uint64, []),
    "lp_moe_workspace_bytes": (_sz, [_i, _i, _i, _i, _i]),
    "lp_moe_route": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _p, _p, _sz, _p]),
    "lp_moe_permute": (_i, [_p, _p, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "lp_moe_experts": (_i, [_p, _p, _i, _p, _p, _i, _i, _i, _p, _p, _p, _sz, _p]),
    "lp_moe_experts_rows": (_i, [_p, _p, _i, _i, _p, _p, _i, _i, _i, _p, _p, _p, _sz, _p]),
    "lp_moe_combine": (_i, [_p, _p, _p, _i, _i, _i, _p, _p]),
    "lp_moe_forward": (_i, [_p, _p, _p, _p, _i, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _sz, _p]),
    "lp_union_counts_uniform": (_i, [_p, _i, _i, _i, _i, _p, _p]),
    "lp_union_counts_weighted": (_i, [_p, _i, _i, _i, _i, _p, _p, _p]),
    "lp_add_rmsnorm": (_i, [_p, _p, _p, _i, _i, ctypes.c_float, _p]),
    "lp_profile_events": (_i, [_p, _i]),
    "lp_ipc_handle": (_i, [_p, _p, _p]),
    "lp_ipc_open": (_i, [_p, _p]),
    "lp_ipc_alloc": (_i, [_sz, _p]),
    "lp_ipc_free": (_i, [_p]),
    "lp_ipc_close": (_i, [_p]),
    "lp_ep_ctl_bytes": (_sz, [_i, _i]),
    "lp_ep_barrier": (_i, [_p, _i, _i, _p]),
    "lp_ep_exchange": (_i, [_p, _p, _i, _i, _i, _p, _p, _p, _p]),
    "lp_ep_dispatch": (_i, [_p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _p, _p, _p]),
    "lp_ep_combine": (_i, [_p, _p, _p, _p, _i, _i, _i, _p, _p]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


class NativeLibraryMissing(RuntimeError):
    """liblpmoe.so has not been built; there is deliberately no fallback path."""


def load() -> ctypes.CDLL:
    """Load (once) and return the library with typed signatures."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> tuple[int, str]:
    buf = ctypes.create_string_buffer(512)
    code = load().lp_last_error(buf, len(buf))
    return code, buf.value.decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Raise the reference-style exception for a non-zero status."""
    if rc == LP_OK:
        return
    _, msg = last_error()
    if rc in (LP_EINVAL, LP_EUNSUPPORTED):
        raise ValidationError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


def version() -> str:
    return load().lp_version().decode()
