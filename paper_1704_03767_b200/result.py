"""Result record and reader-side tau derivation (src/taucorr/result.py:11-102).

These are the reference's host-side *reader* helpers (used by sinks and the
binary reader); the device finalize K5 (csrc/tb_finalize.cu) computes the same
IEEE operation sequence on the GPU and is what the hot path runs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class TauResult:
    """Integer pair counts plus derived tau values for one (u, v) pair (result.py:11-32)."""

    numerator: int
    n_d: int
    n1: int
    n2: int
    n3: int
    n0: int
    tau_a: float
    tau_b: float
    defined_b: bool


def result_from_counts(n: int, n_d: int, n1: int, n2: int, n3: int) -> TauResult:
    """numerator = n0 - n1 - n2 + n3 - 2 n_d (result.py:35-59)."""
    n0 = n * (n - 1) // 2
    numerator = n0 - n1 - n2 + n3 - 2 * n_d
    defined_b = n1 < n0 and n2 < n0
    tau_b = numerator / math.sqrt(float(n0 - n1) * float(n0 - n2)) if defined_b else math.nan
    return TauResult(int(numerator), int(n_d), int(n1), int(n2), int(n3), int(n0), numerator / n0, tau_b,
                     defined_b)


def result_tau_a_only(n: int, numerator: int) -> TauResult:
    """Quadratic-kernel result: tie counts zero, tau_b NaN (result.py:85-102)."""
    n0 = n * (n - 1) // 2
    return TauResult(int(numerator), 0, 0, 0, 0, int(n0), numerator / n0, math.nan, True)


def derive_taus(numerator, n1, n2, n: int, tau_b_valid: bool = True):
    """Vectorised tau from count arrays (result.py:62-82); NaN where the denominator vanishes."""
    n0 = n * (n - 1) // 2
    num = np.asarray(numerator, dtype=np.int64)
    t1 = np.asarray(n1, dtype=np.uint64).astype(np.float64)
    t2 = np.asarray(n2, dtype=np.uint64).astype(np.float64)
    tau_a = num / n0
    if tau_b_valid:
        denom = np.sqrt((n0 - t1) * (n0 - t2))
        with np.errstate(divide="ignore", invalid="ignore"):
            tau_b = np.where(denom > 0, num / denom, np.nan)
    else:
        tau_b = np.full(num.shape, np.nan)
    return tau_a, tau_b
