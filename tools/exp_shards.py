"""8-GPU strong-scaling projection on one GPU, gather included.  Each rank's step of `bench.py --gpus P`
(balanced job-id shard, shrinking row bands, tb_finalize per band) is timed alone on this GPU (CUDA
events, L2 flushed); the banded gather to rank 0 overlaps later bands, so what it adds is the transfer
of every rank's LAST band into rank 0 (ingress-bound: (P - 1) x last-band bytes at the measured 770 GB/s
NVLink peer bandwidth, B200_PROFILING.md), provided rank 0's total ingress ((P - 1)/P of tau_b) fits in
its compute time.  projected speedup = full N = 1 step / max over ranks (shard step + gather tail)."""
import os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import get_engine
from paper_1704_03767_b200.multi import balanced_job_shards, gather_band_fracs, shard_bands

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
NB = int(sys.argv[3]) if len(sys.argv) > 3 else 0        # bands per rank (0: bench.py's automatic count)
RATIO = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5  # band share ratio
NVLINK = 770e9
eng = get_engine(0)
x = torch.from_numpy(workloads.generate(cfg)).cuda()
m, n = x.shape
total = m * (m + 1) // 2
path = eng.choose_path(n, m=m)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()


def timed(bands, reps=3):
    out = torch.empty(bands[-1][1] - bands[0][0], dtype=torch.float64, device="cuda")
    ts = []
    for it in range(reps + 1):
        with torch.cuda.stream(st):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
        eng.tau_b_bands(x, bands, out, kernel=path, stream=st)
        e.record(st)
        torch.cuda.synchronize()
        if it:
            ts.append(s.elapsed_time(e) / 1e3)
    del out
    return statistics.median(ts)


full = timed([(0, total)])
shards = balanced_job_shards(P, m, path)
nb = NB or int(min(4, max(1, (shards[0][1] - shards[0][0]) >> 26)))  # bench.py's automatic band count
fr = gather_band_fracs(nb, RATIO)
print(f"config {cfg}: N=1 step {1e3 * full:.2f} ms; P={P} shards, {nb} bands per rank, shares {[round(f, 3) for f in fr]}",
      flush=True)
worst = 0.0
for r, (lo, hi) in enumerate(shards):
    bands = shard_bands(lo, hi, m, nb, fr)
    t = timed(bands)
    last = bands[-1][1] - bands[-1][0]
    tail = (P - 1) * last * 8 / NVLINK
    ingress = (total - (hi - lo)) * 8 / NVLINK if r == 0 else 0.0
    worst = max(worst, t + tail)
    print(f"  shard {r}/{P}: {hi - lo} job ids, step {1e3 * t:.2f} ms, gather tail {1e3 * tail:.2f} ms"
          + (f", rank-0 ingress {1e3 * ingress:.1f} ms (overlapped)" if r == 0 else ""), flush=True)
print(f"projected {P}-GPU strong scaling, gather included: {full / worst:.2f}x", flush=True)
