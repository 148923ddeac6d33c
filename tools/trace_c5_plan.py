import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
eng = TauEngine(0)
x = torch.from_numpy(workloads.generate(5)).cuda()
for nb in (1, 8):
    eng.gemm_bands = nb
    r = eng.all_pairs(x, kernel="gemm", tau_a=False, tau_b=False); torch.cuda.synchronize(); del r
    print("=== bands", nb, flush=True)
    r = eng.all_pairs(x, kernel="gemm", tau_a=False, tau_b=False); torch.cuda.synchronize(); del r
