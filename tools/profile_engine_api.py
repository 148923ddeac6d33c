import os, sys, cProfile, pstats, io
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.engine import Dataset, compute_all_pairs
from paper_1704_03767_b200.ranks import rank_transform
x = workloads.generate(2)
ranks = np.stack([rank_transform(r) for r in x])
ds = Dataset([f"v{i}" for i in range(ranks.shape[0])], ranks)
for _ in range(3):
    compute_all_pairs(ds, "gemm", sink=lambda v: None)
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    compute_all_pairs(ds, "gemm", sink=lambda v: None)
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25); print(s.getvalue())
