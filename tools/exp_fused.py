"""Config 3 step: sequential GEMM + finalize vs tb_gemm_taus (overlapped finalize)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
import paper_1704_03767_b200.device as dv
eng = dv.TauEngine(0)
x = torch.from_numpy(workloads.generate(3)).cuda()
for thr in (1 << 40, 1, 1 << 40, 1):
    dv.FUSED_FINALIZE_MIN_PAIRS = thr
    for _ in range(2):
        r = eng.all_pairs(x, kernel="gemm"); del r
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); r = eng.all_pairs(x, kernel="gemm", _events=(g0, g1)); e.record(); torch.cuda.synchronize()
        ts.append((s.elapsed_time(e), g0.elapsed_time(g1))); del r
    ts.sort()
    print(f"fused={thr == 1}: step {ts[2][0]:.3f} ms  gemm(+fin) {ts[2][1]:.3f} ms", flush=True)
