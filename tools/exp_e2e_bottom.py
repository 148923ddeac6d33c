"""(Reverted experiment; needs the all_pairs_host(bottom_first=...) option from git history.) Config-2
top-band shares (diagnostics; checks the output against the default schedule)."""
import os, sys, statistics, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
eng = TauEngine(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
xh = torch.from_numpy(workloads.generate(cfg)).pin_memory()
m = xh.shape[0]
out = torch.empty(m * (m + 1) // 2, dtype=torch.float64).pin_memory()
ref = torch.empty_like(out).pin_memory()
eng.all_pairs_host(xh, ref); torch.cuda.synchronize()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
for bf, fr in ((0.0, None), (0.5, (0.6, 0.4)), (0.5, (1.0,)), (0.5, (0.5, 0.3, 0.2)), (0.375, (0.6, 0.4)),
               (0.625, (0.6, 0.4)), (0.625, (1.0,)), (0.75, (0.6, 0.4))):
    ts = []
    for it in range(14):
        with torch.cuda.stream(st):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            r = eng.all_pairs_host(xh, out, band_fracs=fr, stream=st, bottom_first=bf)
            e.record(st)
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(s.elapsed_time(e))
        del r
    same = torch.equal(out.view(torch.int64), ref.view(torch.int64))
    print(f"bottom_first {bf} top bands {fr}: median {statistics.median(ts):.3f} ms  min {min(ts):.3f}  same {same}", flush=True)
