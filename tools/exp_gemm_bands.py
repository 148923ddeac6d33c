"""Device-resident all_pairs with the numerator GEMM launched over 1..k equal-pair row bands
(TauEngine.gemm_bands), prepare (rank + sign pack) once (diagnostics)."""
import os, sys, statistics, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
bands = tuple(int(a) for a in sys.argv[2].split(",")) if len(sys.argv) > 2 else (1, 4, 8)
eng = TauEngine(0)
x = torch.from_numpy(workloads.generate(cfg)).cuda()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
ref = None
for nb in bands:
    eng.gemm_bands = nb
    ts = []
    for it in range(4):
        with torch.cuda.stream(st):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            r = eng.all_pairs(x, kernel="gemm", stream=st, tau_a=False)
            e.record(st)
        torch.cuda.synchronize()
        if it >= 1:
            ts.append(s.elapsed_time(e))
        if it == 3:
            h = torch.sum(r.numerator.to(torch.int64)).item()
            ref = h if ref is None else ref
            same = h == ref
        del r
        torch.cuda.empty_cache()
    print(f"config {cfg} gemm bands {nb}: median {statistics.median(ts):.2f} ms  min {min(ts):.2f}  checksum-same {same}", flush=True)
