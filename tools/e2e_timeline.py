"""Event timeline of TauEngine.all_pairs_host on config 2 (diagnostics)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
import paper_1704_03767_b200.device as dv

eng = TauEngine(0)
xh = torch.from_numpy(workloads.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 2)).pin_memory()
m = xh.shape[0]
out = torch.empty(m * (m + 1) // 2, dtype=torch.float64).pin_memory()
marks = []
orig_call = dv._lib.call
def call(name, *a):
    r = orig_call(name, *a)
    e = torch.cuda.Event(enable_timing=True); e.record(torch.cuda.current_stream()); marks.append((name, e))
    return r
dv._lib.call = call
verbose = os.environ.get("TL_VERBOSE") == "1"
for fr in [(0.65, 0.25, 0.1)]:
  for pb in (4 << 20,):
    for hc in (2,):
        tt = []
        for it in range(8):
            marks.clear()
            s = torch.cuda.Event(enable_timing=True); s.record()
            eng.all_pairs_host(xh, out, band_fracs=fr, h2d_chunks=hc, h2d_piece_bytes=pb)
            e = torch.cuda.Event(enable_timing=True); e.record(); torch.cuda.synchronize()
            tt.append(s.elapsed_time(e))
        tt.sort()
        print(f"bands {fr} piece {pb >> 20} MiB h2d_chunks {hc}: median {tt[4]:.3f} ms  min {tt[0]:.3f}", flush=True)
        if verbose:
            for name, ev in marks:
                print(f"   {name:22s} done at {s.elapsed_time(ev):.3f}")
