"""K5 finalize variants timed with CUDA events on config-3/5-sized synthetic counts (diagnostics)."""
import os, sys, torch, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import _lib
from paper_1704_03767_b200.device import _ptr, _stream_ptr
for m, n in ((16384, 500), (2048, 1000)):
    total = m * (m + 1) // 2
    n0 = n * (n - 1) // 2
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    num = torch.randint(-n0, n0, (total,), dtype=torch.int32, device="cuda", generator=g)
    n1 = torch.randint(0, n0 // 4, (m,), dtype=torch.int64, device="cuda", generator=g)
    ta = torch.empty(total, dtype=torch.float64, device="cuda"); tb = torch.empty_like(ta)
    ref = None
    for var in ("-",):
        os.environ["TB_FIN_VARIANT"] = var
        ts = []
        for it in range(8):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            _lib.call("tb_finalize", _ptr(num), _ptr(n1), m, n, 0, total, _ptr(ta), _ptr(tb), _stream_ptr(None))
            e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        out = torch.cat([ta, tb])
        same = True if ref is None else bool(torch.equal(out.view(torch.int64), ref.view(torch.int64)))
        ref = out if ref is None else ref
        ts.sort()
        gb = total * 20 / 1e9
        print(f"m={m} n={n} variant {var}: {ts[3]*1e3:8.1f} us  {gb/ts[3]*1e3:6.0f} GB/s  same={same}", flush=True)
    del num, ta, tb, ref, out
    torch.cuda.empty_cache()
