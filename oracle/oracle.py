"""ORACLE -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

Python face of the CPU restatement in ``oracle/tau_oracle.c`` plus the numpy
restatement of the reference rank transform.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors that ``oracle/gen_golden.py`` produced by importing the
reference package (``/root/reference/pkg/src/taucorr``) itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libtauoracle.so")
_lib = None

KERNEL_SORTED = 0
KERNEL_PACKED = 1
KERNEL_NAIVE = 2


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64 = ctypes.c_int64
        p = ctypes.c_void_p
        L.orc_pair_scan.argtypes = [p, p, i64, p]
        L.orc_naive_numerator.argtypes = [p, p, i64]
        L.orc_naive_numerator.restype = i64
        L.orc_sorted_counts.argtypes = [p, p, i64, p, p]
        L.orc_packed_counts.argtypes = [p, p, i64, p, p]
        L.orc_derive_taus.argtypes = [p, p, p, i64, i64, p, p]
        L.orc_row_prefix.argtypes = [i64, i64]
        L.orc_row_prefix.restype = i64
        L.orc_job_coord.argtypes = [i64, i64, p, p]
        L.orc_all_pairs.argtypes = [p, i64, p, p, i64, ctypes.c_int, ctypes.c_int, p, p]
        L.orc_all_pairs.restype = ctypes.c_int
        _lib = L
    return _lib


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# ranks.py:37-61 restated: dense 0-based ranks through np.unique, NaN rejected.
# --------------------------------------------------------------------------
def rank_transform(values) -> np.ndarray:
    arr = np.asarray(values)
    if arr.ndim != 1 or arr.size == 0:
        raise ValueError("observations must be a non-empty 1-D array")
    if arr.dtype.kind == "f" and np.isnan(arr).any():
        raise ValueError("observations contain NaN, which has no rank")
    _, inverse = np.unique(arr, return_inverse=True)
    return np.ascontiguousarray(inverse, dtype=np.int32)


def rank_matrix(x: np.ndarray) -> np.ndarray:
    out = np.empty(x.shape, np.int32)
    for r in range(x.shape[0]):
        out[r] = rank_transform(x[r])
    return out


# --------------------------------------------------------------------------
# Per-pair counts
# --------------------------------------------------------------------------
def pair_scan(u, v) -> dict:
    """tests/conftest.py:16-66 brute force: nc, nd, n1, n2, n3, numerator."""
    u, v = _i32(u), _i32(v)
    out = np.zeros(5, np.int64)
    lib().orc_pair_scan(_ptr(u), _ptr(v), u.shape[0], _ptr(out))
    nc, nd, n1, n2, n3 = (int(x) for x in out)
    return dict(nc=nc, n_d=nd, n1=n1, n2=n2, n3=n3, numerator=nc - nd)


def naive_numerator(u, v) -> int:
    u, v = _i32(u), _i32(v)
    return int(lib().orc_naive_numerator(_ptr(u), _ptr(v), u.shape[0]))


def sorted_counts(u, v) -> tuple[int, int, int, int]:
    """kernel_sorted.py:195-212: (n_d, n1, n2, n3)."""
    u, v = _i32(u), _i32(v)
    n = u.shape[0]
    scratch = np.empty(4 * n + 16, np.int32)
    out = np.zeros(4, np.int64)
    lib().orc_sorted_counts(_ptr(u), _ptr(v), n, _ptr(scratch), _ptr(out))
    return tuple(int(x) for x in out)


def packed_counts(u, v) -> tuple[int, int, int, int]:
    """kernel_vectorized.py:507-523 semantics (scalar): (n_d, n1, n2, n3)."""
    u, v = _i32(u), _i32(v)
    n = u.shape[0]
    if n > 32767 or u.min() < 0 or v.min() < 0 or u.max() >= 1 << 15 or v.max() >= 1 << 15:
        raise ValueError("packed capacity exceeded")
    scratch = np.empty(2 * n + 16, np.int32)
    out = np.zeros(4, np.int64)
    lib().orc_packed_counts(_ptr(u), _ptr(v), n, _ptr(scratch), _ptr(out))
    return tuple(int(x) for x in out)


def numerator_from_counts(n: int, nd: int, n1: int, n2: int, n3: int) -> int:
    """result.py:42: n0 - n1 - n2 + n3 - 2*n_d."""
    n0 = n * (n - 1) // 2
    return n0 - n1 - n2 + n3 - 2 * nd


# --------------------------------------------------------------------------
# Finalize (result.py:62-82)
# --------------------------------------------------------------------------
def derive_taus(numerator, n1, n2, n: int):
    num = np.ascontiguousarray(numerator, dtype=np.int64)
    t1 = np.ascontiguousarray(n1, dtype=np.uint64)
    t2 = np.ascontiguousarray(n2, dtype=np.uint64)
    ta = np.empty(num.shape, np.float64)
    tb = np.empty(num.shape, np.float64)
    lib().orc_derive_taus(_ptr(num), _ptr(t1), _ptr(t2), num.size, n, _ptr(ta), _ptr(tb))
    return ta, tb


# --------------------------------------------------------------------------
# Geometry (pairindex.py:20-55)
# --------------------------------------------------------------------------
def row_prefix(y: int, m: int) -> int:
    return int(lib().orc_row_prefix(y, m))


def job_coord(j: int, m: int) -> tuple[int, int]:
    y = ctypes.c_int64()
    x = ctypes.c_int64()
    lib().orc_job_coord(j, m, ctypes.byref(y), ctypes.byref(x))
    return y.value, x.value


# --------------------------------------------------------------------------
# Threaded all-pairs (the CPU baseline)
# --------------------------------------------------------------------------
def all_pairs(ranks: np.ndarray, pi, pj, kernel: int = KERNEL_SORTED, threads: int | None = None,
              want_counts: bool = True):
    """Counts for the listed pairs; returns (numerator[P], counts[P,4] or None)."""
    ranks = np.ascontiguousarray(ranks, dtype=np.int32)
    pi = np.ascontiguousarray(pi, dtype=np.int64)
    pj = np.ascontiguousarray(pj, dtype=np.int64)
    P = pi.shape[0]
    num = np.empty(P, np.int64)
    counts = np.zeros((P, 4), np.int64) if want_counts else None
    if threads is None:
        threads = os.cpu_count() or 1
    lib().orc_all_pairs(_ptr(ranks), ranks.shape[1], _ptr(pi), _ptr(pj), P, kernel, threads,
                        _ptr(num), _ptr(counts) if counts is not None else None)
    return num, counts


def upper_pairs(m: int, diagonal: bool = True):
    """All (i, j) with i <= j (or i < j) in job-id order (pairindex.py:27-31)."""
    k = 0 if diagonal else 1
    ii, jj = np.triu_indices(m, k)
    return ii.astype(np.int64), jj.astype(np.int64)
