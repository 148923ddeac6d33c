"""H2D copy behaviour on the box: per-copy event timings, pinned (torch) vs cudaHostRegister'd memory."""
import torch, ctypes
dev = torch.device("cuda:0")
torch.cuda.init()
st = torch.cuda.Stream()
for mb in (1, 2, 4, 8, 16):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    ts = []
    for it in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            s.record(st); d.copy_(h, non_blocking=True); e.record(st)
        torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    print(f"H2D {mb:2d} MiB pinned: min {ts[0]:7.1f} med {ts[10]:7.1f} max {ts[-1]:7.1f} us  -> {n/ts[10]/1e3:5.1f} GB/s (med)", flush=True)
    # back-to-back without sync between copies
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        s.record(st)
        for _ in range(10): d.copy_(h, non_blocking=True)
        e.record(st)
    torch.cuda.synchronize()
    print(f"    10 back-to-back: {s.elapsed_time(e)*1e3/10:7.1f} us each", flush=True)
