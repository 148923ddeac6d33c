"""ctypes binding of libtaub200.so (the C ABI declared in include/taub200.h).

There is no fallback: if the shared library is missing or the device is not a
B200, every entry point raises.  Build it with ``__graft_entry__.build()``
(or ``make -C paper_1704_03767_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CapacityExceededError, ConfigError, InvalidInputError

LIB_NAME = "libtaub200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
_variant = os.environ.get("TB_LIB_VARIANT")
if _variant:  # A/B experiments: an in-tree copy of this library built from a variant source
    if os.path.basename(_variant) != _variant or not _variant.startswith("libtaub200") or not _variant.endswith(".so"):
        raise ImportError(f"TB_LIB_VARIANT must name an in-tree libtaub200*.so, got {_variant!r}")
    LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), _variant)

TB_OK, TB_ERR_INVALID, TB_ERR_CAPACITY, TB_ERR_CONFIG, TB_ERR_CUDA, TB_ERR_ABORTED = 0, 1, 2, 3, 4, 5
TB_DTYPE_I32, TB_DTYPE_F32, TB_DTYPE_F64 = 0, 1, 2
TB_SIGN_I8, TB_SIGN_E4M3, TB_SIGN_E2M1, TB_SIGN_E2M1_OFS = 0, 1, 2, 3
TB_MAX_N = 65536

# Every exported symbol and its ctypes signature (kept in sync with include/taub200.h;
# tests/test_host.py::test_capi_exports_every_declared_symbol checks both directions).
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_p = ctypes.c_void_p
SIGNATURES = {
    "tb_last_error": ([], ctypes.c_char_p),
    "tb_launch_count": ([], ctypes.c_int64),
    "tb_query": ([ctypes.c_int, _p], ctypes.c_int),
    "tb_sign_k": ([_i64], _i64),
    "tb_rank_rows": ([_p, ctypes.c_int, _i64, _i64, _i64, _p, _i64, _p, _p, _p], ctypes.c_int),
    "tb_rank_dense_workspace": ([_i64, _i64, ctypes.c_int], _i64),
    "tb_rank_dense": ([_p, ctypes.c_int, _i64, _i64, _i64, _p, ctypes.c_int, _i64, _p, _p, _p, _i64, _p], ctypes.c_int),
    "tb_sign_pack": ([_p, _i64, _i64, _i64, _p, _i64, ctypes.c_int, _p], ctypes.c_int),
    "tb_abs_pack": ([_p, _i64, _i64, ctypes.c_int, _p, _p], ctypes.c_int),
    "tb_gemm_pairs": ([_p, _i64, _i64, _i64, ctypes.c_int, _i64, _i64, _i32, _p, _p], ctypes.c_int),
    "tb_gemm_pairs_fix": ([_p, _i64, _i64, _i64, ctypes.c_int, _i64, _i64, _i32, _p, _i64, _p, _p], ctypes.c_int),
    "tb_sign_pack_sums": ([_p, _i64, _i64, _i64, _p, _i64, _p, _p], ctypes.c_int),
    "tb_sign_row_sums": ([_p, _i64, _i64, _i64, _p, _p], ctypes.c_int),
    "tb_gemm_tau_b_fix": ([_p, _i64, _i64, _i64, ctypes.c_int, _i64, _i64, _i32, _p, _i64, _p, _i64, _p, _p, _p],
                          ctypes.c_int),
    "tb_gemm_pairs_simt": ([_p, _i64, _i64, _i64, _i64, _i64, _p, _p], ctypes.c_int),
    "tb_finalize": ([_p, _p, _i64, _i64, _i64, _i64, _p, _p, _p], ctypes.c_int),
    "tb_full_counts": ([_p, _p, _p, _i64, _i64, _i64, _i64, _p, _p, _p], ctypes.c_int),
    "tb_presort": ([_p, _i64, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p], ctypes.c_int),
    "tb_merge_workspace": ([_i64], _i64),
    "tb_merge_pairs": ([_p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _i64, _p], ctypes.c_int),
    "tb_records": ([_p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, _p, _p], ctypes.c_int),
    "tb_tile_cells": ([_i64, _i64, _i64, _i64], _i64),
    "tb_gemm_tau_b": ([_p, _i64, _i64, _i64, ctypes.c_int, _i64, _i64, _i32, _p, _i64, _p, _p, _p], ctypes.c_int),
    "tb_tied_counts": ([_p, _p, _i64, _p, _i64, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p], ctypes.c_int),
    "tb_records_compact": ([_p, _p, _i64, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, _p, _p], ctypes.c_int),
    "tb_records_num": ([_p, _i64, _i64, _i64, _i64, _i64, _i64, _p, _p], ctypes.c_int),
    "tb_expand_records_num": ([_p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, _p, ctypes.c_int],
                              ctypes.c_int),
    "tb_h2d_staged": ([_p, _p, _i64, _p, _p, _i64, ctypes.c_int, _p], ctypes.c_int),
    "tb_expand_store_mode": ([ctypes.c_int], ctypes.c_int),
    "tb_expand_ring": ([_p, ctypes.c_int, _p, _p, _p, _i64, _i64, _i64, _i64, _p, _i64, ctypes.c_int, _p, _i64, _i64,
                        _i64, _p, ctypes.c_int], ctypes.c_int),
    "tb_ring_wait": ([_p, _i64], ctypes.c_int),
    "tb_expand_records": ([_p, _p, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, _p, ctypes.c_int], ctypes.c_int),
}


class TbCaps(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("sm_count", ctypes.c_int32),
        ("cc_major", ctypes.c_int32),
        ("cc_minor", ctypes.c_int32),
        ("tcgen05_i8", ctypes.c_int32),
        ("smem_optin", ctypes.c_int64),
    ]


_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load (once) and return the bound library; raises if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"{LIB_NAME} is not built at {path}; run __graft_entry__.build() "
                    "(there is no CPU fallback for the device path)")
            lib = ctypes.CDLL(path)
            for name, (args, res) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


_EXC = {
    TB_ERR_INVALID: InvalidInputError,
    TB_ERR_CAPACITY: CapacityExceededError,
    TB_ERR_CONFIG: ConfigError,
    TB_ERR_CUDA: RuntimeError,
}


def check(rc: int) -> None:
    """Map a C-ABI status onto the reference exception hierarchy (errors.py:4-24)."""
    if rc == TB_OK:
        return
    msg = load().tb_last_error().decode(errors="replace")
    raise _EXC.get(rc, RuntimeError)(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def query(device: int = 0) -> TbCaps:
    caps = TbCaps()
    call("tb_query", device, ctypes.byref(caps))
    return caps
