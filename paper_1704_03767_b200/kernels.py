"""Per-pair entry points with the reference's names, arguments and errors,
computed on the device (a 2-variable dataset, job (0, 1)).

* tau_a_naive(u, v)            -- kernel_naive.py:47-62 (numerator only, tau_b NaN)
* tau_b_sorted(u, v)           -- kernel_sorted.py:254-274 (all counts)
* tau_b_vectorized(u, v, fast) -- kernel_vectorized.py:591-611 (packed capacity check)
* tie_sum / joint_tie_sum / count_discordant -- kernel_sorted.py:225-251 semantics
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidInputError
from .ranks import as_rank_array, check_pack_capacity
from .result import TauResult, result_from_counts, result_tau_a_only


def _pair(u, v) -> tuple[np.ndarray, np.ndarray]:
    ua = as_rank_array(u, "u")
    va = as_rank_array(v, "v")
    if ua.shape[0] != va.shape[0]:
        raise InvalidInputError(f"length mismatch: {ua.shape[0]} vs {va.shape[0]}")
    if ua.shape[0] < 2:
        raise InvalidInputError("need at least two observations")
    return ua, va


def _device_counts(ua: np.ndarray, va: np.ndarray, full: bool):
    import torch

    from .device import get_engine

    eng = get_engine()
    path = eng.choose_path(ua.shape[0], m=2, full_counts=full)
    x = torch.from_numpy(np.stack([ua, va])).to(eng.device)  # the device ranks them (K0 / K0w)
    res = eng.all_pairs(x, kernel=path, job_range=(1, 2),
                        tau_a=False, tau_b=False, full_counts=full)
    res.validate()
    num = int(res.numerator.item())
    if not full:
        return num, None
    n1 = res.n1_rows.cpu().tolist()
    return num, (int(res.n_d.item()), int(n1[0]), int(n1[1]), int(res.n3.item()))


def tau_a_naive(u, v) -> TauResult:
    ua, va = _pair(u, v)
    num, _ = _device_counts(ua, va, full=False)
    return result_tau_a_only(ua.shape[0], num)


def tau_b_sorted(u, v) -> TauResult:
    ua, va = _pair(u, v)
    _, (nd, n1, n2, n3) = _device_counts(ua, va, full=True)
    return result_from_counts(ua.shape[0], nd, n1, n2, n3)


def tau_b_vectorized(u, v, fast: bool = True) -> TauResult:
    ua, va = _pair(u, v)
    check_pack_capacity(ua, va)
    _, (nd, n1, n2, n3) = _device_counts(ua, va, full=True)
    return result_from_counts(ua.shape[0], nd, n1, n2, n3)
