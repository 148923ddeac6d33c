"""Sustained D2H into rotating pinned buffers (the compute_all_pairs record stream pattern): GB/s for
chunk sizes 16..512 MiB, one or two copy streams, ~40 GB moved per variant."""
import sys, time
import torch

dev = torch.device("cuda", 0)
src = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
for mb in (16, 64, 256, 512):
    nb = mb << 20
    pins = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(4)]
    for nstreams in (1, 2):
        sts = [torch.cuda.Stream(device=dev) for _ in range(nstreams)]
        total = 40 << 30
        count = total // nb
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(count):
            st = sts[i % nstreams]
            with torch.cuda.stream(st):
                pins[i % 4].copy_(src[(i * nb) % (1 << 30) // nb * nb:][:nb], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"D2H {mb:4d} MiB chunks x {count}, {nstreams} stream(s): {count * nb / dt / 1e9:.1f} GB/s", flush=True)
    del pins
