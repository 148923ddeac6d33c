"""Does the power-capped GEMM rate depend on the operand bit patterns?  Config 5's S is overwritten with
e2m1 nibble patterns (the results are meaningless; only time, SM clock and power are read):
  real   : the sign matrix K2 built (+1 = 0x2, -1 = 0xA, few zeros)
  zeros  : every element 0
  ones   : every element +1
  pm1    : random +1 / -1
  b01    : random 0 / +1   (the {0,1} indicator encoding B = (S + 1) / 2)
  b01q   : 0 / +1 with P(1) = 1/4
"""
import os, statistics, subprocess, sys, threading
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
pats = sys.argv[2].split(",") if len(sys.argv) > 2 else ["real", "zeros", "ones", "pm1", "b01", "b01q", "real"]
eng = TauEngine(0)
x = torch.from_numpy(workloads.generate(5)).cuda()
m, n = x.shape
total = m * (m + 1) // 2
st = torch.cuda.Stream()


def fill(S, pat):
    if pat == "real":
        return
    if pat == "zeros":
        S.zero_(); return
    if pat == "ones":
        S.fill_(0x22); return
    step = 1 << 30
    for o in range(0, S.numel(), step):
        c = S[o:o + step]
        if pat == "pm1":
            r = torch.randint(0, 256, (c.numel(),), dtype=torch.uint8, device=c.device)
            v = ((r & 0x88) | 0x22)
        elif pat == "b01":
            r = torch.randint(0, 256, (c.numel(),), dtype=torch.uint8, device=c.device)
            v = (r & 0x22)
        elif pat.startswith("nib"):  # random 0 / nibble value, e.g. nib1 = 0.5, nib2 = 1.0, nib4 = 2.0, nib6 = 4.0
            v0 = int(pat[3:], 16)
            r = torch.randint(0, 256, (c.numel(),), dtype=torch.uint8, device=c.device)
            v = (r & 0x11) * v0
        elif pat == "b01q":
            r = torch.randint(0, 256, (c.numel(),), dtype=torch.uint8, device=c.device)
            r2 = torch.randint(0, 256, (c.numel(),), dtype=torch.uint8, device=c.device)
            v = (r & r2 & 0x22)
        else:
            raise SystemExit(pat)
        c.copy_(v.view(torch.int8))
        del r, v


with eng.session(st):
    prep = eng.prepare(x, "gemm")
    num = torch.empty(total, dtype=torch.int32, device="cuda")
    for pat in pats:
        if pat == "real":
            prep = eng.prepare(x, "gemm")
        fill(prep.S, pat)
        torch.cuda.synchronize()
        eng.numerators(prep, 0, total, num)
        torch.cuda.synchronize()
        clk = []
        proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        threading.Thread(target=lambda: [clk.append(l) for l in proc.stdout], daemon=True).start()
        ts = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            eng.numerators(prep, 0, total, num)
            e.record(st)
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        proc.terminate()
        mhz = [float(l.split(",")[0]) for l in clk if l.strip()]
        pw = [float(l.split(",")[1]) for l in clk if l.strip()]
        print(f"pattern {pat}: gemm {statistics.median(ts):.1f} ms (min {min(ts):.1f}), sm clock median "
              f"{statistics.median(mhz) if mhz else 0:.0f} MHz, power median {statistics.median(pw) if pw else 0:.0f} W",
              flush=True)
