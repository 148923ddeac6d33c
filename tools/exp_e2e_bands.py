"""Config-2 end-to-end time (all_pairs_host, pinned host buffers, L2 flushed) vs row-band fractions."""
import os, sys, statistics, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
eng = TauEngine(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
xh = torch.from_numpy(workloads.generate(cfg)).pin_memory()
m = xh.shape[0]
out = torch.empty(m * (m + 1) // 2, dtype=torch.float64).pin_memory()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
def geo(k, r):  # k bands, each r times the previous one's share of the pairs
    w = [r ** i for i in range(k)]
    return tuple(x / sum(w) for x in w)


VARIANTS = {
    2: (((0.7, 0.3), 2), ((0.65, 0.25, 0.10), 2), ((0.8, 0.2), 2), ((0.6, 0.4), 2), ((1.0,), 2)),
    3: ((geo(6, 0.7), 2), (geo(7, 0.77), 2)),
    5: ((geo(12, 0.82), 2), (geo(10, 0.8), 2)),
}
iters = 12 if cfg != 5 else 5
for fr, hc in VARIANTS.get(cfg, VARIANTS[2]):
    ts = []
    for it in range(iters):
        with torch.cuda.stream(st):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            r = eng.all_pairs_host(xh, out, band_fracs=fr, stream=st, h2d_chunks=hc)
            e.record(st)
        torch.cuda.synchronize()
        if it >= (2 if iters > 5 else 1):
            ts.append(s.elapsed_time(e))
        del r
    print(f"bands {len(fr)} first {fr[0]:.3f} last {fr[-1]:.3f} h2d_chunks {hc}: median {statistics.median(ts):.3f} ms  min {min(ts):.3f}", flush=True)
