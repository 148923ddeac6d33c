"""HBM write-only and read-only streaming bandwidth (torch fill_ / sum over 32 GB): the ceiling of a
write-dominated kernel like K5 (4 B read + 16 B written per cell) next to the copy figure in
MEASURED_PEAKS.json."""
import torch
x = torch.empty(4 << 30, dtype=torch.float64, device="cuda")  # 32 GiB
for name, fn, nbytes in (("write (fill_)", lambda: x.fill_(1.0), x.numel() * 8),
                         ("read (sum)", lambda: x.sum(), x.numel() * 8),
                         ("copy (half -> half)", lambda: x[: x.numel() // 2].copy_(x[x.numel() // 2:]), x.numel() * 8)):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    print(f"{name}: {nbytes / best / 1e12:.2f} TB/s", flush=True)
