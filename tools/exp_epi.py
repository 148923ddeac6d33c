import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
eng = TauEngine(0)
for k in [int(a) for a in (sys.argv[1:] or ["2", "3"])]:
    x = torch.from_numpy(workloads.generate(k)).cuda()
    for skip in ("0",):
        os.environ["TB_EXP_SKIP_EPI"] = skip
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            eng.all_pairs(x, kernel="gemm", tau_a=False, tau_b=False, _events=(s, e))
            torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        print(f"config {k} skip_epilogue={skip}: gemm ms {sorted(ts)[2]:.3f}", flush=True)
    eng.release(); del x; torch.cuda.empty_cache()
