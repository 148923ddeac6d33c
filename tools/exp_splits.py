"""GEMM stage time of a config for forced uniform split counts (tb_gemm_pairs splits argument) and the
automatic plan; CUDA events around the numerator launches, L2 flushed, median of 20."""
import os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
eng = TauEngine(0)
x = torch.from_numpy(workloads.generate(cfg)).cuda()
m = x.shape[0]
total = m * (m + 1) // 2
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
num = torch.empty(total, dtype=torch.int32, device="cuda")
with eng.session() as st:
    prep = eng.prepare(x, "gemm")
    for s in [int(a) for a in os.environ.get('SPLITS', '0,1,2,3,4,5,6,8').split(',')]:
        ts = []
        for it in range(23):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            eng.numerators(prep, 0, total, num, splits=s)
            b.record(st)
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b))
        print(f"config {cfg} TB_PLAN_EPI={os.environ.get('TB_PLAN_EPI', '100')} splits={s or 'auto'}: "
              f"{1e3 * statistics.median(ts):.1f} us", flush=True)
