"""Device-resident step: one all_pairs call over every job id vs the same job range cut into row bands
(separate GEMM + finalize launches per band), config 5 by default (diagnostics)."""
import os, sys, statistics, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
eng = TauEngine(0)
x = torch.from_numpy(workloads.generate(cfg)).cuda()
m = x.shape[0]
total = m * (m + 1) // 2
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()

def run(nb):
    if nb == 1:
        r = eng.all_pairs(x, kernel="gemm", stream=st)
        return [r]
    fr = TauEngine.default_band_fracs(total) if nb == 0 else tuple([1.0 / nb] * nb)
    cuts = eng.bands(m, len(fr), fracs=fr)
    out = []
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        lo, hi = r0 * (2 * m - r0 + 1) // 2, r1 * (2 * m - r1 + 1) // 2
        out.append(eng.all_pairs(x, kernel="gemm", job_range=(lo, hi), stream=st))
    return out

for nb in tuple(int(a) for a in sys.argv[2].split(",")) if len(sys.argv) > 2 else (1, 0, 4):
    ts = []
    for it in range(4):
        with torch.cuda.stream(st):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            rs = run(nb)
            e.record(st)
        torch.cuda.synchronize()
        if it >= 1:
            ts.append(s.elapsed_time(e))
        del rs
        torch.cuda.empty_cache()
    print(f"config {cfg} bands {nb if nb else 'default'}: median {statistics.median(ts):.2f} ms  min {min(ts):.2f}", flush=True)
