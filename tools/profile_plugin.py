"""Where a small compute_all_pairs call spends its time (config 2 / 1): wall time of repeated calls, then
cProfile of one call (top entries by cumulative time)."""
import cProfile, os, pstats, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import paper_1704_03767_b200 as tb
from paper_1704_03767_b200 import workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
x = workloads.generate(cfg)
ds = tb.Dataset(labels=[str(i) for i in range(x.shape[0])], ranks=np.stack([tb.rank_transform(r) for r in x]))
got = [0]
def sink(r):
    got[0] += r.shape[0]
for _ in range(3):
    tb.compute_all_pairs(ds, "vectorized", sink=sink)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    tb.compute_all_pairs(ds, "vectorized", sink=sink)
    ts.append(time.perf_counter() - t0)
print(f"config {cfg}: compute_all_pairs {min(ts) * 1e3:.2f} ms (min of 5), median {sorted(ts)[2] * 1e3:.2f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
tb.compute_all_pairs(ds, "vectorized", sink=sink)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
