"""TB_TRACE=1 of the config-1 GEMM (diagnostics)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
eng = TauEngine(0)
x = torch.from_numpy(workloads.generate(1)).cuda()
for _ in range(3):
    r = eng.all_pairs(x); torch.cuda.synchronize(); del r
