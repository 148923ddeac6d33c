"""Pinned device->host copy bandwidth vs copy size, sustained pattern (median of back-to-back copies)."""
import statistics
import torch
dev = torch.device("cuda:0")
for mb in (1, 2, 4, 8, 11, 17):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); h.copy_(d, non_blocking=True); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    med = statistics.median(ts)
    print(f"D2H {mb:3d} MiB: min {min(ts)*1e3:8.1f} med {med*1e3:8.1f} us -> {n/med/1e6:6.1f} GB/s (med)", flush=True)
    # the same bytes in 2 MiB pieces, back to back on one stream
    piece = 2 << 20
    ts = []
    for _ in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for o in range(0, n, piece):
            h[o:o + piece].copy_(d[o:o + piece], non_blocking=True)
        e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    med = statistics.median(ts)
    print(f"    in 2 MiB pieces: med {med*1e3:8.1f} us -> {n/med/1e6:6.1f} GB/s", flush=True)
