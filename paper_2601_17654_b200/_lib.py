"""ctypes binding of libkpo.so (the C ABI declared in include/kpo.h).

The product path has no CPU fallback: if the shared library is missing or a CUDA device is absent,
`lib()` raises `KpoUnavailable` and every op that needs it fails loudly.  Status codes follow
include/kpo.h: 0 = ok, negative = error class; the message comes from kpo_last_error().
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# KPO_LIB_PATH: A/B measurement tools load an alternative build of the same library (tools/*_ab.*)
LIB_PATH = os.environ.get("KPO_LIB_PATH") or os.path.join(_HERE, "libkpo.so")

KPO_OK = 0
KPO_ERR_INVALID = -1
KPO_ERR_CUDA = -2
KPO_ERR_UNSUPPORTED = -3
KPO_ERR_STATE = -4
KPO_IPC_HANDLE_BYTES = 64

_c_void_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_f32 = ctypes.c_float
_size = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/kpo.h one-to-one (tests check both directions).
SIGNATURES = {
    "kpo_last_error": (ctypes.c_char_p, []),
    "kpo_version": (_i32, []),
    "kpo_device_info": (_i32, [_i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                ctypes.POINTER(_i32)]),
    "kpo_rmsnorm_fwd": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _f32, _c_void_p]),
    "kpo_rmsnorm_bwd": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                               _i64, _i64, _c_void_p]),
    "kpo_rmsnorm_bwd_partial_rows": (_i32, [_i64, _i64, ctypes.POINTER(_i64)]),
    "kpo_colsum_f32_to_bf16": (_i32, [_c_void_p, _c_void_p, _i64, _i64, _c_void_p]),
    "kpo_rope": (_i32, [_c_void_p, _i64, _c_void_p, _i64, _i64, _i32, _i32, _f32, _i64, _i32, _c_void_p]),
    "kpo_swiglu_fwd": (_i32, [_c_void_p, _c_void_p, _i64, _i64, _c_void_p]),
    "kpo_swiglu_bwd": (_i32, [_c_void_p, _c_void_p, _c_void_p, _i64, _i64, _c_void_p]),
    "kpo_swiglu_fwd_blocked": (_i32, [_c_void_p, _c_void_p, _i64, _i64, _i32, _c_void_p]),
    "kpo_swiglu_bwd_blocked": (_i32, [_c_void_p, _c_void_p, _c_void_p, _i64, _i64, _i32, _c_void_p]),
    "kpo_gemm": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _i64, _i32, _i32, _i64, _i64,
                        _i64, _i32, _c_void_p, _c_void_p]),
    "kpo_gemm_rope": (_i32, [_c_void_p, _c_void_p, _c_void_p, _i64, _i64, _i64, _i64, _i64, _i64, _i32, _c_void_p,
                             _c_void_p, _i64, _i32, _c_void_p]),
    "kpo_gemm_swiglu": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _i64, _i64, _i64, _i64, _i64,
                               _i32, _c_void_p, _c_void_p]),
    "kpo_gemm_swiglu_bwd": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _i64, _i64, _i64, _i64,
                                   _i64, _i32, _c_void_p, _c_void_p]),
    "kpo_rope_table": (_i32, [_i64, _i32, _f32, _i64, _c_void_p, _c_void_p]),
    "kpo_attn_fwd": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _i64, _i32, _i32, _i32,
                            _i64, _i64, _i64, _i64, _f32, _i32, _c_void_p]),
    "kpo_attn_fwd_mma": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _i64, _i32, _i32, _i32,
                                _i64, _i64, _i64, _i64, _f32, _i32, _c_void_p]),
    "kpo_attn_bwd_workspace_bytes": (_i64, [_i64, _i32, _i32, _i32]),
    "kpo_attn_bwd": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                            _c_void_p, _c_void_p, _i64, _i32, _i32, _i32, _i64, _i64, _i64, _i64, _i64, _i64,
                            _i64, _f32, _i32, _c_void_p, _c_void_p]),
    "kpo_embedding_fwd": (_i32, [_c_void_p, _c_void_p, _c_void_p, _i64, _i64, _i64, _c_void_p, _c_void_p]),
    "kpo_embedding_bwd": (_i32, [_c_void_p, _c_void_p, _c_void_p, _i64, _i64, _i64, _c_void_p]),
    "kpo_cross_entropy": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _i64, _f32, _i32,
                                 _c_void_p]),
    "kpo_attn_bwd_rope": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                                 _c_void_p, _c_void_p, _i64, _i32, _i32, _i32, _i64, _i64, _i64, _i64, _i64, _i64,
                                 _i64, _f32, _i32, _c_void_p, _c_void_p, _c_void_p]),
    "kpo_comm_create": (_i32, [_i32, _i32, _i32, _size, _i32, ctypes.POINTER(_c_void_p)]),
    "kpo_comm_ipc_handle": (_i32, [_c_void_p, _c_void_p]),
    "kpo_comm_open_peers": (_i32, [_c_void_p, _c_void_p]),
    "kpo_comm_sym_ptr": (_c_void_p, [_c_void_p]),
    "kpo_comm_peer_ptr": (_c_void_p, [_c_void_p, _i32]),
    "kpo_comm_max_ctas": (_i32, [_c_void_p]),
    "kpo_comm_destroy": (_i32, [_c_void_p]),
    "kpo_all_gather": (_i32, [_c_void_p, _size, _c_void_p, _size, _i32, _c_void_p]),
    "kpo_reduce_scatter": (_i32, [_c_void_p, _size, _c_void_p, _size, _i32, _c_void_p]),
    "kpo_all_reduce": (_i32, [_c_void_p, _size, _size, _c_void_p, _size, _i32, _c_void_p]),
    "kpo_comm_trace": (_i32, [_c_void_p, _c_void_p, _i32]),
    "kpo_set_launch_completion_event": (_i32, [_c_void_p, _c_void_p]),
    "kpo_probe_launch_completion": (_i32, [_c_void_p, _c_void_p]),
    "kpo_sm_blocker": (_i32, [_i32, _i64, _c_void_p, _c_void_p]),
}


class KpoUnavailable(RuntimeError):
    """libkpo.so (the sm_100a CUDA path) is not built or cannot be loaded; there is no fallback."""


class KpoError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} failed with status {status}: {msg}")
        self.status = status


_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load and type the library without touching the GPU (safe on CPU-only hosts)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise KpoUnavailable(f"{path} not built; run __graft_entry__.build() (make -C csrc)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            if path != os.path.join(_HERE, "libkpo.so") and not hasattr(lib, name):
                continue  # an older build loaded through KPO_LIB_PATH for a same-box A/B
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    return load()


def check(name: str, status: int) -> None:
    if status != KPO_OK:
        msg = lib().kpo_last_error().decode(errors="replace")
        raise KpoError(name, status, msg)


def call(name: str, *args) -> None:
    check(name, getattr(lib(), name)(*args))


def header_symbols(header_path: str | None = None) -> list[str]:
    """Function names declared in include/kpo.h (used by the ABI tests)."""
    import re

    header_path = header_path or os.path.join(os.path.dirname(_HERE), "include", "kpo.h")
    text = open(header_path).read()
    return sorted(set(re.findall(r"\b(kpo_[a-z0-9_]+)\s*\(", text)))
