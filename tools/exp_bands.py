"""Config 3 device step vs band count of the overlapped GEMM/finalize path (diagnostics)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
import paper_1704_03767_b200.device as dv
eng = dv.TauEngine(0)
x = torch.from_numpy(workloads.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 3)).cuda()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for mb in (0, 2, 4, 8):
    if mb == 0:
        dv.FIN_OVERLAP_MIN_PAIRS = 1 << 40
    else:
        dv.FIN_OVERLAP_MIN_PAIRS = 16 << 20
        dv.FIN_OVERLAP_MAX_BANDS = mb
    for _ in range(2):
        r = eng.all_pairs(x, kernel="gemm"); del r
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); r = eng.all_pairs(x, kernel="gemm"); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e)); del r
    ts.sort()
    print(f"max bands {mb}: step {ts[2]:.3f} ms", flush=True)
