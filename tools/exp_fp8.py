"""Experiment: is tcgen05 kind::f8f6f4 (e4m3 +-1/0, f32 accumulate) exact for the sign GEMM?"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads  # noqa: E402
from paper_1704_03767_b200.device import TauEngine  # noqa: E402

eng = TauEngine(0)


from paper_1704_03767_b200 import _lib  # noqa: E402

FMTS = {None: _lib.TB_SIGN_I8, "f8": _lib.TB_SIGN_E4M3, "f4": _lib.TB_SIGN_E2M1}


def run(x, kind):
    eng.sign_format_override = FMTS[kind]
    for _ in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        res = eng.all_pairs(x, kernel="gemm", tau_a=False, tau_b=False, _events=(s, e))
        torch.cuda.synchronize()
    return res.numerator.clone(), s.elapsed_time(e)


for k in [int(a) for a in sys.argv[1:]] or [2, 3, 5]:
    x = torch.from_numpy(workloads.generate(k)).cuda()
    a, ta = run(x, None)
    b, tb = run(x, "f8")
    c, tc = run(x, "f4")
    print(f"config {k}: gemm int8 {ta:.3f} ms, fp8 {tb:.3f} ms, fp4 {tc:.3f} ms; mismatches fp8 {(a != b).sum().item()} "
          f"fp4 {(a != c).sum().item()} of {a.numel()}, max|num| {a.abs().max().item()}", flush=True)
    del a, b, c, x
    eng.release()
    torch.cuda.empty_cache()
# adversarial: identical / reversed rows at the largest K the GEMM path takes (n = 8192 -> K ~ 3.4e7 > 2^24)
for n in (4096, 5770, 8192):
    base = torch.randperm(n, device="cuda").to(torch.int32)
    x = torch.stack([base, base, n - 1 - base, torch.randperm(n, device="cuda").to(torch.int32)])
    a, _ = run(x, None)
    b, _ = run(x, "f8")
    c, _ = run(x, "f4") if n <= 5770 else (a, 0)
    print(f"n={n}: K={n*(n-1)//2} int8 {a.tolist()} fp8 {b.tolist()} fp4 {c.tolist()}", flush=True)
