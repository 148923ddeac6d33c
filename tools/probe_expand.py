"""Host record expansion rate (tb_expand_records): 48-byte records rebuilt from the 8-byte compact stream on
host threads, alone and while the copy engine streams D2H into other pinned memory (the hybrid record
pipeline's two paths at once).  Config-5 geometry (m = 65536, q = 8), ~256 MiB of records per call."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import _lib
from paper_1704_03767_b200.pairindex import JobSpace

lib = _lib.load()
m, q, n = 65536, 8, 1024
space = JobSpace(m, q)
ntiles = 5592405 // 36 * 1  # ~5.6M records: 36 cells per full tile
lo = 1000
cells = int(lib.tb_tile_cells(m, q, lo, lo + ntiles))
print("cores", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), "records", cells, "MiB", cells * 48 / 2**20)
compact = torch.empty(cells * 8, dtype=torch.uint8).pin_memory()
compact.numpy()[:] = np.random.default_rng(0).integers(0, 255, cells * 8, dtype=np.uint8)
n1 = np.zeros(m, np.uint64)
outs = [torch.empty(cells * 48, dtype=torch.uint8).pin_memory() for _ in range(2)]


def expand(nt, k=0):
    rc = lib.tb_expand_records(compact.data_ptr(), n1.ctypes.data, m, n, q, lo, ntiles, 0, outs[k].data_ptr(), nt)
    assert rc == 0


for nt in (1, 2, 4, 8, 12, 16, 24, 32):
    if nt > os.cpu_count():
        break
    expand(nt)
    ts = []
    for r in range(5):
        t0 = time.perf_counter(); expand(nt, r % 2); ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"threads {nt:2d}: {1e3 * t:.1f} ms  {cells * 48 / t / 1e9:.1f} GB/s of records  {cells / t / 1e9:.2f} G rec/s")

# concurrently with D2H into other pinned memory
dev = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
host = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
st = torch.cuda.Stream()
for _ in range(2):
    with torch.cuda.stream(st):
        host.copy_(dev, non_blocking=True)
    st.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(st):
    host.copy_(dev, non_blocking=True)
st.synchronize()
t_d2h = time.perf_counter() - t0
print(f"D2H alone: {2**30 / t_d2h / 1e9:.1f} GB/s")
for nt in (8, 12, 16):
    if nt > os.cpu_count():
        break
    with torch.cuda.stream(st):
        for _ in range(4):
            host.copy_(dev, non_blocking=True)
    t0 = time.perf_counter()
    ne = 0
    while not st.query():
        expand(nt, ne % 2)
        ne += 1
    t1 = time.perf_counter()
    st.synchronize()
    print(f"threads {nt:2d} + D2H: {ne} expansions in {1e3 * (t1 - t0):.0f} ms -> {ne * cells * 48 / (t1 - t0) / 1e9:.1f} GB/s "
          f"records, D2H {4 * 2**30 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
