"""Run one device path on (a row prefix of) a BASELINE config, for ncu/sanitizer targets.

    python tools/run_path.py --config 4 --rows 64 --reps 3
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1704_03767_b200 import workloads  # noqa: E402
from paper_1704_03767_b200.device import TauEngine  # noqa: E402
from paper_1704_03767_b200.ranks import rank_transform  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--rows", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--path", default="auto")
a = ap.parse_args()
x = workloads.generate(a.config, rows=a.rows)
eng = TauEngine(0)
path = eng.choose_path(x.shape[1]) if a.path == "auto" else a.path
if path == "merge":
    x = np.stack([rank_transform(r) for r in x])
xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
for _ in range(a.reps):
    res = eng.all_pairs(xd, kernel=path)
torch.cuda.synchronize()
res.validate()
print("ok", path, x.shape, float(res.tau_b[:4].sum()))
