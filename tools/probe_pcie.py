"""Pinned host <-> device copy bandwidth on this box (e2e floor for bench's host entry point)."""
import torch
dev = torch.device("cuda:0")
for mb in (2, 8, 17, 64):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for name, f in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(3): f()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); f(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
        print(f"{name} {mb:3d} MiB: {best*1e3:8.1f} us  {n/best/1e6:6.1f} GB/s", flush=True)
# concurrent H2D + D2H on two streams
n = 64 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device=dev); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
e.record(); torch.cuda.synchronize()
print(f"concurrent H2D+D2H 64 MiB each: {s.elapsed_time(e)*1e3:.1f} us  {2*n/s.elapsed_time(e)/1e6:.1f} GB/s total")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max", "--format=csv"], capture_output=True, text=True).stdout)
