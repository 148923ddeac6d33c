"""Randomized parity stress of the large-m GEMM features (diagnostics): multi-wave unsplit plans (the
K-lockstep throttle), offset-coded operands (forced half the time), full counts through the tie-indicator
GEMM (all rows / sparse tied rows), job sub-ranges, the fused tau_b epilogue (tau_b_bands) -- every pair
against the oracle (C restatement).  Exits 1 on the first mismatch."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as orc  # the checker only
from paper_1704_03767_b200 import _lib
from paper_1704_03767_b200.device import TauEngine

eng = TauEngine(0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
deadline = time.time() + float(os.environ.get("STRESS_SECONDS", "300"))
cases = 0
while time.time() < deadline:
    m = int(rng.integers(1500, 7000))
    n = int(rng.choice([17, 33, 64, 130, 257, 400]))
    kind = int(rng.integers(0, 4))
    if kind == 0:
        x = rng.standard_normal((m, n)).astype(np.float32)
    elif kind == 1:
        x = rng.integers(0, max(2, n // int(rng.integers(1, 20))), (m, n)).astype(np.int32)
    elif kind == 2:  # few tied rows: the sparse tied-row table
        x = rng.standard_normal((m, n)).astype(np.float32)
        t = rng.choice(m, max(1, m // 50), replace=False)
        x[t, : n // 2] = np.round(x[t, : n // 2])
    else:
        x = rng.integers(0, 3, (m, n)).astype(np.float64)
    x[0] = x[0, 0]
    ofs = bool(rng.integers(0, 2))
    eng.sign_format_override = _lib.TB_SIGN_E2M1_OFS if ofs else None
    total = m * (m + 1) // 2
    lo = int(rng.integers(0, total // 3)) if rng.integers(0, 2) else 0
    hi = int(rng.integers(2 * total // 3, total)) if lo else total
    ranks = orc.rank_matrix(x)
    xd = torch.from_numpy(x).cuda()
    res = eng.all_pairs(xd, kernel="gemm", full_counts=True, job_range=(lo, hi)).validate()
    pi, pj = orc.upper_pairs(m)
    num, counts = orc.all_pairs(ranks, pi[lo:hi], pj[lo:hi], orc.KERNEL_PACKED, threads=16, want_counts=True)
    ok = (np.array_equal(res.numerator.cpu().numpy().astype(np.int64), num)
          and np.array_equal(res.n_d.cpu().numpy(), counts[:, 0])
          and np.array_equal(res.n3.cpu().numpy(), counts[:, 3]))
    ta, tb = orc.derive_taus(num, counts[:, 1], counts[:, 2], n)
    ok = ok and np.array_equal(res.tau_a.cpu().numpy(), ta) and np.array_equal(
        np.nan_to_num(res.tau_b.cpu().numpy(), nan=9.0), np.nan_to_num(tb, nan=9.0))
    out = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
    eng.tau_b_bands(xd, [(lo, (lo + hi) // 2), ((lo + hi) // 2, hi)], out, kernel="gemm")
    torch.cuda.synchronize()
    ok = ok and np.array_equal(np.nan_to_num(out.cpu().numpy(), nan=9.0), np.nan_to_num(tb, nan=9.0))
    cases += 1
    print(f"{'ok ' if ok else 'BAD'} m={m} n={n} kind={kind} ofs={ofs} range=({lo},{hi}) fmt={res.extra.get('sign_format')}", flush=True)
    if not ok:
        sys.exit(1)
eng.sign_format_override = None
print(f"stress: {cases} cases ok")
