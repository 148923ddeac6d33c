"""H2D from write-combined vs ordinary pinned host memory (cudaHostAlloc flags), sustained pattern."""
import ctypes, numpy as np, torch
torch.cuda.init()
dev = torch.device("cuda:0")
cudart = None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        cudart = ctypes.CDLL(name); break
    except OSError:
        pass
if cudart is None:
    import glob, os
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    cudart = ctypes.CDLL(cands[0])

def host_alloc(nbytes, flags):
    p = ctypes.c_void_p()
    rc = cudart.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(nbytes), ctypes.c_uint(flags))
    assert rc == 0, rc
    buf = (ctypes.c_uint8 * nbytes).from_address(p.value)
    return torch.from_numpy(np.frombuffer(buf, dtype=np.uint8))

st = torch.cuda.Stream()
for mb in (4, 8, 16):
    n = mb << 20
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    dd = torch.empty(4 * n, dtype=torch.uint8, device=dev)
    hd = torch.empty(4 * n, dtype=torch.uint8).pin_memory()
    for label, h in (("torch pinned", torch.empty(n, dtype=torch.uint8).pin_memory()),
                     ("cudaHostAlloc default", host_alloc(n, 0)),
                     ("cudaHostAlloc WC", host_alloc(n, 4))):
        h.fill_(7)
        print(label, "is_pinned", h.is_pinned(), flush=True)
        ts = []
        for it in range(12):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                s.record(st); d.copy_(h, non_blocking=True); e.record(st)
                hd.copy_(dd, non_blocking=True)  # the e2e pattern: a D2H of 4x the bytes after each upload
            torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
        ts.sort()
        print(f"  H2D {mb:2d} MiB {label:22s}: min {ts[0]:7.1f} med {ts[6]:7.1f} max {ts[-1]:7.1f} us -> {n/ts[6]/1e3:5.1f} GB/s", flush=True)
