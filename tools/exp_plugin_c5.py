"""Config-5 plugin call (compute_all_pairs, 103 GB of records) broken down on the consumer thread: time
waiting for batch events, time expanding compact batches on host threads, per-pass Python (views, sink
hand-off), for each record-path mix (TB_RECORDS_FULL_EVERY) and pass size."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import paper_1704_03767_b200 as tb
from paper_1704_03767_b200 import engine, workloads

x = workloads.generate(int(os.environ.get("CFG", "5")))
ds = tb.Dataset(labels=[str(i) for i in range(x.shape[0])], ranks=np.stack([tb.rank_transform(r) for r in x]))
got = [0]


def sink(r):
    got[0] += r.shape[0]


acc = {"expand": 0.0, "n": 0}
orig = engine._DevicePipe.expand


def timed_expand(self, batch, slot):
    t0 = time.perf_counter()
    orig(self, batch, slot)
    acc["expand"] += time.perf_counter() - t0
    acc["n"] += 1


engine._DevicePipe.expand = timed_expand
orig_ring = engine._DevicePipe.expand_ring


def timed_ring(self, batch, slot):
    t0 = time.perf_counter()
    orig_ring(self, batch, slot)
    acc["expand"] += time.perf_counter() - t0
    acc["n"] += 1


engine._DevicePipe.expand_ring = timed_ring
print("ring slots", engine.RING_SLOTS, "expand threads", engine.EXPAND_THREADS, "pass slots", engine.PASS_SLOTS, flush=True)
wjs = [int(a) for a in os.environ.get("WJ", str(engine.WINDOW_JOBS)).split(",")]
for wj in wjs:
    for _ in range(2):
        tb.compute_all_pairs(ds, "vectorized", sink=None, window_jobs=wj)
    t0 = time.perf_counter()
    tb.compute_all_pairs(ds, "vectorized", sink=None, window_jobs=wj)
    print(f"window_jobs {wj}: sink=None {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
for fe in [int(a) for a in (sys.argv[1:] or ["1", "1000000"])]:
    engine.FULL_EVERY = fe
    for pt in [int(a) for a in os.environ.get("PT", "4096").split(",")]:
        for _ in range(2):
            tb.compute_all_pairs(ds, "vectorized", sink=sink, pass_tiles=pt, window_jobs=wjs[-1])
        reps = 1 if x.shape[0] > 20000 else 10
        best = None
        for _ in range(reps):
            acc.update(expand=0.0, n=0)
            t0 = time.perf_counter()
            s = tb.compute_all_pairs(ds, "vectorized", sink=sink, pass_tiles=pt, window_jobs=wjs[-1])
            wall = time.perf_counter() - t0
            if best is None or wall < best[0]:
                best = (wall, s, dict(acc))
        wall, s, accb = best
        acc.update(accb)
        wr = sum(p.write_seconds for p in s.passes)
        print(f"full_every {fe:8d} pass_tiles {pt:6d}: wall {1e3 * wall:7.1f} ms, event waits {1e3 * s.device_seconds:7.1f} ms, "
              f"expand {1e3 * acc['expand']:7.1f} ms ({acc['n']} batches), submit {1e3 * wr:6.1f} ms, passes {len(s.passes)}",
              flush=True)
