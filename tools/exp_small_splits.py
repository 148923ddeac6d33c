"""GEMM time vs forced split count on small workloads (CUDA-graph replays, diagnostics)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads, _lib
from paper_1704_03767_b200.device import TauEngine, _ptr, _stream_ptr, PairResult

eng = TauEngine(0)
for cfg in (1,):
    x = torch.from_numpy(workloads.generate(cfg)).cuda()
    m, n = x.shape
    res = eng.all_pairs(x, kernel="gemm")
    S, K, ldS, fmt = eng._gemm_prepare(x, res, _stream_ptr(None))
    total = m * (m + 1) // 2
    num = torch.empty(total, dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    for s in (0, 1, 2, 3, 4, 6, 8, 12, 16, 20, 32):
        with torch.cuda.stream(st):
            for _ in range(3):
                _lib.call("tb_gemm_pairs", _ptr(S), m, K, ldS, fmt, 0, total, s, _ptr(num), _stream_ptr(st))
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
            for _ in range(20):
                _lib.call("tb_gemm_pairs", _ptr(S), m, K, ldS, fmt, 0, total, s, _ptr(num), _stream_ptr(st))
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                a.record(st); g.replay(); b.record(st)
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b) / 20 * 1e3)
        ok = torch.equal(num, res.numerator)
        print(f"config {cfg} splits {s:3d}: {sorted(ts)[2]:7.2f} us per GEMM call  exact={ok}", flush=True)

# whole step: tensor-core FP4 vs SIMT dp4a (int8 S), graph replays
for cfg in (1,):
    x = torch.from_numpy(workloads.generate(cfg)).cuda()
    st = torch.cuda.Stream()
    for simt in (False, True):
        for _ in range(3):
            eng.all_pairs(x, kernel="gemm", simt=simt, stream=st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
            for _ in range(10):
                r = eng.all_pairs(x, kernel="gemm", simt=simt, stream=st)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                a.record(st); g.replay(); b.record(st)
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b) / 10 * 1e3)
        print(f"config {cfg} step simt={simt}: {sorted(ts)[2]:7.2f} us", flush=True)
