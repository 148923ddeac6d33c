"""compute_all_pairs (the reference plugin call) on a BASELINE config: wall time per call, records
delivered, for slot-size / slot-count variants (engine.SLOT_BYTES / PASS_SLOTS)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import paper_1704_03767_b200 as tb
from paper_1704_03767_b200 import engine, workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
x = workloads.generate(cfg)
t0 = time.perf_counter()
ds = tb.Dataset(labels=[str(i) for i in range(x.shape[0])], ranks=np.stack([tb.rank_transform(r) for r in x]))
print(f"config {cfg}: host ranks {time.perf_counter() - t0:.1f} s", flush=True)
got = [0]
def sink(r):
    got[0] += r.shape[0]
for slot_mb, slots, overlap in [(256, 3, True), (512, 3, True), (256, 4, True), (128, 6, True)]:
    engine.SLOT_BYTES, engine.PASS_SLOTS = slot_mb << 20, slots
    tb.compute_all_pairs(ds, "vectorized", sink=sink, overlap=overlap)
    ts = []
    for _ in range(2):
        got[0] = 0
        t0 = time.perf_counter()
        s = tb.compute_all_pairs(ds, "vectorized", sink=sink, overlap=overlap)
        ts.append(time.perf_counter() - t0)
    assert got[0] == s.total_cells
    print(f"slot {slot_mb} MiB x {slots}, overlap {overlap}: {min(ts):.3f} s per call, {s.total_cells} records "
          f"({s.total_cells * 48 / min(ts) / 1e9:.1f} GB/s of records), {len(s.passes)} passes, "
          f"device wait {s.device_seconds:.3f} s", flush=True)
t0 = time.perf_counter()
s = tb.compute_all_pairs(ds, "vectorized", sink=None)
print(f"sink=None: {time.perf_counter() - t0:.3f} s", flush=True)
