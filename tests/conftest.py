"""Shared test setup.

``-m "not gpu"`` tests run in the CPU dev container: the oracle against the
golden vectors, host logic, the C-ABI symbol table, gloo multi-process paths.
``-m gpu`` tests are the parity tests proper and call through the C-ABI on a
B200.  The oracle (``oracle/``) is imported here only as the checker.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libtaub200.so")


def gold_path(name: str) -> str:
    return os.path.join(GOLD, name)


def load_npz(name: str):
    return np.load(gold_path(name), allow_pickle=False)


def load_json(name: str):
    with open(gold_path(name)) as fh:
        return json.load(fh)


def split_pairs(z):
    """Yield (u, v, idx) from a concatenated golden pair file."""
    ns = z["n"]
    u = z["u"].astype(np.int32)
    v = z["v"].astype(np.int32)
    off = 0
    for k, n in enumerate(ns.tolist()):
        yield u[off:off + n], v[off:off + n], k
        off += n


@pytest.fixture(scope="session")
def oracle():
    import oracle as orc  # noqa: WPS433  (oracle/oracle.py, the checker)
    orc.lib()
    return orc


def random_rank_pair(rng, n: int, tie_fraction: float):
    """Same draws as the reference test helper (tests/conftest.py:78-89)."""
    import math
    if tie_fraction <= 0:
        return rng.permutation(n).astype(np.int32), rng.permutation(n).astype(np.int32)
    k = max(1, math.ceil(n * (1.0 - tie_fraction)))
    return rng.integers(0, k, n).astype(np.int32), rng.integers(0, k, n).astype(np.int32)
