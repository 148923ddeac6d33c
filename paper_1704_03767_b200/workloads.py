"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference's published numbers were taken on GPL570/SEEK gene-expression
matrices that are not available here; these generators
stand in for them with the shapes, sizes and value distributions that
BASELINE.json names.  The draws follow SURVEY.md section 8(d) exactly
(``np.random.default_rng(170403767 + k)`` for config k, draws in the listed
order), so the oracle, the CPU baseline and the GPU consume identical bytes.

``synth_dataset`` mirrors the reference test/bench generator
(dataio.py:200-219) for host-side engine tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SEED_BASE = 170403767


@dataclass(frozen=True)
class ConfigSpec:
    k: int
    m: int
    n: int
    name: str
    path: str  # "gemm" or "merge": the numerator kernel the dispatcher picks


CONFIGS = {
    1: ConfigSpec(1, 256, 200, "m256_n200_f64_normal", "gemm"),
    2: ConfigSpec(2, 2048, 1000, "m2048_n1000_i32_uniform0to9", "gemm"),
    3: ConfigSpec(3, 16384, 500, "m16384_n500_f32_genelike", "gemm"),
    4: ConfigSpec(4, 1024, 65536, "m1024_n65536_f32_monotone_every8", "merge"),
    5: ConfigSpec(5, 65536, 1024, "m65536_n1024_f32_lowrank64", "gemm"),
}


def generate(k: int, rows: int | None = None) -> np.ndarray:
    """Return the raw value matrix X [m, n] of BASELINE config k.

    ``rows`` truncates to the first rows (same leading rows as the full draw
    for configs 1-2; configs 3-5 draw full-size factors first so a prefix is
    still a prefix of the full matrix).
    """
    rng = np.random.default_rng(SEED_BASE + k)
    if k == 1:
        x = rng.standard_normal((256, 200))
    elif k == 2:
        x = rng.integers(0, 10, (2048, 1000)).astype(np.int32)
    elif k == 3:
        w = rng.standard_normal((16384, 32))
        z = rng.standard_normal((32, 500))
        eps = rng.standard_normal((16384, 500))
        x = np.round(np.exp(w @ z + 0.5 * eps), 2).astype(np.float32)
    elif k == 4:
        x = rng.standard_normal((1024, 65536), dtype=np.float32)
        noise = rng.standard_normal((1024, 65536), dtype=np.float32)
        base = np.exp(x[0])
        for r in range(8, 1024, 8):
            x[r] = base + np.float32(0.1) * noise[r]
    elif k == 5:
        w = rng.standard_normal((65536, 64))
        z = rng.standard_normal((64, 1024))
        eps = rng.standard_normal((65536, 1024))
        x = ((w @ z + eps) / np.sqrt((w ** 2).sum(1, keepdims=True) + 1)).astype(np.float32)
    else:
        raise ValueError(f"unknown config {k}")
    if rows is not None:
        x = x[:rows]
    return np.ascontiguousarray(x)


def synth_ranks(m: int, n: int, tie_fraction: float = 0.0, seed: int = 0) -> np.ndarray:
    """Dense-rank matrix with the reference synth_dataset's draws (dataio.py:200-219)."""
    if m < 1 or n < 1:
        raise ValueError(f"dataset shape must be positive, got m={m}, n={n}")
    if not 0.0 <= tie_fraction <= 1.0:
        raise ValueError(f"tie_fraction must be in [0, 1], got {tie_fraction}")
    rng = np.random.default_rng(seed)
    distinct = max(1, math.ceil(n * (1.0 - tie_fraction)))
    base = np.arange(n, dtype=np.int32) % distinct
    ranks = np.empty((m, n), dtype=np.int32)
    for row in range(m):
        ranks[row] = rng.permutation(base)
    return ranks


def sample_pairs(m: int, count: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Seeded random i<j pairs (with replacement) for sampled parity checks."""
    rng = np.random.default_rng(seed)
    i = rng.integers(0, m, count)
    j = rng.integers(0, m, count)
    keep = i != j
    i, j = i[keep], j[keep]
    lo = np.minimum(i, j).astype(np.int64)
    hi = np.maximum(i, j).astype(np.int64)
    return lo, hi
