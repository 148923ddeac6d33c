"""Wall time of the reference-compatible API compute_all_pairs (48-byte CELL_DTYPE records in tile order,
sink protocol) on config 2, vs the device-only step (diagnostics)."""
import os, sys, time, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import numpy as np
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.engine import Dataset, compute_all_pairs
from paper_1704_03767_b200.ranks import rank_transform
x = workloads.generate(2)
ranks = np.stack([rank_transform(r) for r in x])
ds = Dataset([f"v{i}" for i in range(ranks.shape[0])], ranks)
for kernel in ("gemm", "auto"):
    for _ in range(2):
        compute_all_pairs(ds, kernel, sink=None)
    ts = []
    nrec = [0]
    def sink(v):
        nrec[0] += len(v)
    for _ in range(5):
        nrec[0] = 0
        t0 = time.perf_counter()
        s = compute_all_pairs(ds, kernel, sink=sink)
        ts.append(time.perf_counter() - t0)
    print(f"compute_all_pairs(kernel={kernel!r}): {min(ts)*1e3:.1f} ms best of 5, {nrec[0]} records "
          f"({nrec[0] / min(ts):.3g} cells/s); summary {s}", flush=True)
