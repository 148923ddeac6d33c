"""Strong-scaling projection on one GPU: the device-resident step of each of P contiguous job-id shards
(pairindex.job_shard_range) of a config, timed alone (CUDA events, L2 flushed).  max(shard) vs the
full range bounds the P-GPU strong-scaling efficiency from compute alone (no collective)."""
import os, sys, statistics, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
from paper_1704_03767_b200.pairindex import job_shard_range
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
eng = TauEngine(0)
x = torch.from_numpy(workloads.generate(cfg)).cuda()
m = x.shape[0]
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()

def timed(jr, reps=3):
    ts = []
    for it in range(reps + 1):
        with torch.cuda.stream(st):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            r = eng.all_pairs(x, stream=st, job_range=jr)
            e.record(st)
        torch.cuda.synchronize()
        if it:
            ts.append(s.elapsed_time(e))
        del r

    return statistics.median(ts)

full = timed(None)
shards = [timed(job_shard_range(r, P, m)) for r in range(P)]
print(f"config {cfg}: full range {full:.2f} ms", flush=True)
for r, t in enumerate(shards):
    print(f"  shard {r}/{P}: {t:.2f} ms", flush=True)
print(f"projected {P}-GPU strong scaling (compute only): {full / max(shards):.2f}x "
      f"(sum of shards {sum(shards):.1f} ms)", flush=True)
