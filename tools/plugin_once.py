"""One config-5 compute_all_pairs call with a counting sink (ncu launch-list target)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import paper_1704_03767_b200 as tb
from paper_1704_03767_b200 import workloads

x = workloads.generate(int(os.environ.get("CFG", "5")))
ds = tb.Dataset(labels=[str(i) for i in range(x.shape[0])], ranks=np.stack([tb.rank_transform(r) for r in x]))
got = [0]
def sink(r):
    got[0] += r.shape[0]
import gc
if os.environ.get("NOGC") == "1":
    gc.disable()
if os.environ.get("FREEZE") == "1":
    gc.collect(); gc.freeze()
for _ in range(int(os.environ.get("CALLS", "1"))):
    t0 = time.perf_counter()
    tb.compute_all_pairs(ds, "vectorized", sink=sink, overlap=os.environ.get("OVERLAP", "1") == "1")
    print(f"call {1e3 * (time.perf_counter() - t0):.1f} ms, records {got[0]}", flush=True)
