"""Host enqueue time of the public calls vs their GPU time (is the step host-bound?)."""
import os, sys, time, statistics, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
eng = TauEngine(0)
x = workloads.generate(2)
xd = torch.from_numpy(x).cuda()
xh = torch.from_numpy(x).pin_memory()
m = x.shape[0]
out = torch.empty(m * (m + 1) // 2, dtype=torch.float64).pin_memory()
st = torch.cuda.Stream()
for name, fn in (("all_pairs", lambda: eng.all_pairs(xd, stream=st)),
                 ("all_pairs_host", lambda: eng.all_pairs_host(xh, out, stream=st))):
    for _ in range(5):
        r = fn(); torch.cuda.synchronize(); del r
    host, gpu = [], []
    for _ in range(20):
        torch.cuda.synchronize()
        # a long GPU-side delay first, so the enqueue never waits on the GPU
        with torch.cuda.stream(st):
            torch.cuda._sleep(2_000_000)
            s = torch.cuda.Event(enable_timing=True); s.record(st)
        t0 = time.perf_counter()
        r = fn()
        t1 = time.perf_counter()
        with torch.cuda.stream(st):
            e = torch.cuda.Event(enable_timing=True); e.record(st)
        torch.cuda.synchronize()
        host.append((t1 - t0) * 1e3)
        gpu.append(s.elapsed_time(e))
        del r
    print(f"{name}: host enqueue median {statistics.median(host):.3f} ms, GPU time median {statistics.median(gpu):.3f} ms", flush=True)
