"""Randomized parity stress (diagnostics): random (m, n) around the kernels' size boundaries, random tie
levels, both device paths with full counts, every pair against the oracle (C restatement).  Prints one line
per case and a final count; exits 1 on the first mismatch."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as orc  # the checker only
from paper_1704_03767_b200.device import TauEngine

eng = TauEngine(0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
ns = [2, 3, 31, 64, 65, 127, 128, 129, 255, 256, 257, 1023, 1024, 1025, 2047, 2048, 2049, 3001, 4095, 4097,
      5792, 5793, 8191, 8193, 16383, 16385, 32767, 32768, 32769, 40000, 65535, 65536]
deadline = time.time() + float(os.environ.get("STRESS_SECONDS", "600"))
cases = 0
for n in ns:
    for path in ("gemm", "merge"):
        if path == "gemm" and n > 32767:
            continue
        if time.time() > deadline:
            break
        m = int(rng.integers(2, 24 if n > 20000 else (40 if n > 4096 else 130)))
        kind = rng.integers(0, 4)
        if kind == 0:
            x = rng.standard_normal((m, n)).astype(np.float32)
        elif kind == 1:
            x = rng.integers(0, max(2, n // int(rng.integers(1, 50))), (m, n)).astype(np.int32)
        elif kind == 2:
            x = rng.integers(0, 3, (m, n)).astype(np.float64)
        else:
            x = np.stack([rng.permutation(n) if r % 2 else np.arange(n)[::-1] for r in range(m)]).astype(np.float32)
        x[0] = x[0, 0]  # a constant row
        ranks = orc.rank_matrix(x)
        res = eng.all_pairs(torch.from_numpy(x).cuda(), kernel=path, full_counts=True).validate()
        pi, pj = orc.upper_pairs(m)
        num, counts = orc.all_pairs(ranks, pi, pj, orc.KERNEL_SORTED, threads=16)
        ok = (np.array_equal(res.numerator.cpu().numpy().astype(np.int64), num)
              and np.array_equal(res.n_d.cpu().numpy(), counts[:, 0])
              and np.array_equal(res.n3.cpu().numpy(), counts[:, 3]))
        ta, tb = orc.derive_taus(num, counts[:, 1], counts[:, 2], n)
        ok = ok and np.array_equal(res.tau_a.cpu().numpy(), ta) and np.array_equal(
            np.nan_to_num(res.tau_b.cpu().numpy(), nan=9.0), np.nan_to_num(tb, nan=9.0))
        cases += 1
        print(f"{'ok ' if ok else 'BAD'} path={path} m={m} n={n} kind={kind} fmt={res.extra.get('sign_format')}", flush=True)
        if not ok:
            sys.exit(1)
print(f"stress: {cases} cases ok")
