"""Config-2 GEMM time vs forced uniform split count (CUDA-graph replays, diagnostics)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads, _lib
from paper_1704_03767_b200.device import TauEngine, _ptr, _stream_ptr
eng = TauEngine(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
x = torch.from_numpy(workloads.generate(cfg)).cuda()
m, n = x.shape
res = eng.all_pairs(x, kernel="gemm")
S, K, ldS, fmt = eng._gemm_prepare(x, res, _stream_ptr(None))
total = m * (m + 1) // 2
num = torch.empty(total, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
for s in (0, 1, 2, 3, 4, 5, 6):
    with torch.cuda.stream(st):
        for _ in range(2):
            _lib.call("tb_gemm_pairs", _ptr(S), m, K, ldS, fmt, 0, total, s, _ptr(num), _stream_ptr(st))
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            _lib.call("tb_gemm_pairs", _ptr(S), m, K, ldS, fmt, 0, total, s, _ptr(num), _stream_ptr(st))
            b.record(st)
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ok = torch.equal(num, res.numerator)
    print(f"config {cfg} splits {s}: {sorted(ts)[3]*1e3:8.1f} us  exact={ok}", flush=True)
