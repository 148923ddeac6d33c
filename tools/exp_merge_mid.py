"""Merge-path (K4) time per job id at mid-size n (several pairs per CTA), for library A/B runs (TB_LIB_VARIANT)."""
import os, sys, statistics
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200.device import TauEngine
eng = TauEngine(0)
rng = np.random.default_rng(0)
for n in (2048, 4096, 8192, 16384, 32767, 65536):
    m = 192
    x = torch.from_numpy(rng.standard_normal((m, n)).astype(np.float32)).cuda()
    ts = []
    for it in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); r = eng.all_pairs(x, kernel="merge", tau_a=False, tau_b=False); e.record(); torch.cuda.synchronize()
        if it: ts.append(s.elapsed_time(e))
    jobs = m * (m + 1) // 2
    print(f"{os.environ.get('TB_LIB_VARIANT', 'default')}: n={n} {1e6 * statistics.median(ts) / jobs:.1f} ns per job", flush=True)
