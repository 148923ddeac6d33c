"""Host record expansion into a small ring of pass buffers (cache-resident) vs large slots (DRAM-bound):
tb_expand_records_num with streaming or plain stores, per pass size, ring depth and thread count.
Config-5 geometry (m = 65536, q = 8)."""
import os, subprocess, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import _lib

lib = _lib.load()
print(subprocess.run("lscpu | egrep 'Model name|Socket|Core|Thread|L2|L3|NUMA|^CPU\\(s\\)'", shell=True,
                     capture_output=True, text=True).stdout)
m, q, n = 65536, 8, 1024
lo = 1000
total_tiles = 40 * 4096  # ~5.9M records, 283 MB of records per sweep point
cells_total = int(lib.tb_tile_cells(m, q, lo, lo + total_tiles))
nums = torch.empty(cells_total * 4, dtype=torch.uint8).pin_memory()
nums.numpy()[:] = np.random.default_rng(0).integers(0, 255, cells_total * 4, dtype=np.uint8)
n1 = np.zeros(m, np.uint64)
ring_buf = torch.empty(1 << 29, dtype=torch.uint8).pin_memory()
print("cores", os.cpu_count(), "records", cells_total)


def sweep(pass_tiles, R, nt, plain, reps=3):
    lib.tb_expand_store_mode(1 if plain else 0)
    npass = total_tiles // pass_tiles
    pcells = int(lib.tb_tile_cells(m, q, lo, lo + pass_tiles)) + 64
    assert R * pcells * 48 <= ring_buf.numel()
    best = 1e9
    for _ in range(reps):
        off = 0
        t0 = time.perf_counter()
        for p in range(npass):
            t_lo = lo + p * pass_tiles
            c = int(lib.tb_tile_cells(m, q, t_lo, t_lo + pass_tiles))
            rc = lib.tb_expand_records_num(nums.data_ptr() + 4 * off, n1.ctypes.data, None, None, 0, m, n, q, t_lo,
                                           pass_tiles, 0, ring_buf.data_ptr() + (p % R) * pcells * 48, nt)
            assert rc == 0
            off += c
        best = min(best, time.perf_counter() - t0)
    lib.tb_expand_store_mode(0)
    return off * 48 / best / 1e9, 1e6 * best / npass


for plain in (0, 1):
    for pass_tiles in (512, 1024, 2048, 4096, 8192, 40960):
        for R in (2, 4):
            row = []
            for nt in (4, 8, 12, 16):
                if nt > os.cpu_count():
                    continue
                gbs, us = sweep(pass_tiles, R, nt, plain)
                row.append(f"t{nt}: {gbs:6.1f} GB/s ({us:7.1f} us/pass)")
            print(f"{'plain ' if plain else 'stream'} pass_tiles {pass_tiles:6d} ({pass_tiles * 64 * 48 / 2**20:6.1f} MiB) ring {R}: " + "  ".join(row), flush=True)
