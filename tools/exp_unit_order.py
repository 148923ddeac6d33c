"""GEMM unit-order experiment on config 5: the full device step (8 row-band GEMM launches) timed with
CUDA events for the unit-order knobs in the environment (TB_GEMM_GR / TB_GEMM_WIN / TB_GEMM_SERP),
with the SM clock sampled during the timed loop (power cap)."""
import os, statistics, subprocess, sys, threading, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eng = TauEngine(0)
if os.environ.get("GB"):
    eng.gemm_bands = int(os.environ["GB"])
x = torch.from_numpy(workloads.generate(5)).cuda()
st = torch.cuda.Stream()
for _ in range(2):
    r = eng.all_pairs(x, stream=st, tau_a=False); del r
torch.cuda.synchronize()
clk = []
proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                         "-lms", "100"], stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [clk.append(l) for l in proc.stdout], daemon=True).start()
ts, gs = [], []
for _ in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        s.record(st)
        r = eng.all_pairs(x, stream=st, tau_a=False, _events=(g0, g1))
        e.record(st)
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e)); gs.append(g0.elapsed_time(g1)); del r
proc.terminate()
mhz = [float(l.split(",")[0]) for l in clk if l.strip()]
pw = [float(l.split(",")[1]) for l in clk if l.strip()]
tag = f"GB={os.environ.get('GB', '-')} " + " ".join(f"{k}={os.environ.get(k, '-')}" for k in ("TB_GEMM_GR", "TB_GEMM_WIN", "TB_GEMM_SERP", "TB_GEMM_LEAD", "TB_GEMM_LAGQ"))
print(f"{tag}: step {statistics.median(ts):.1f} ms, gemm {statistics.median(gs):.1f} ms "
      f"(min {min(gs):.1f}), sm clock median {statistics.median(mhz) if mhz else 0:.0f} MHz, "
      f"power median {statistics.median(pw) if pw else 0:.0f} W", flush=True)
