"""TB_TRACE of one job-id shard's device step (diagnostics): python tools/trace_shard.py CFG P R"""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import workloads
from paper_1704_03767_b200.device import TauEngine
from paper_1704_03767_b200.pairindex import job_shard_range
cfg, P, R = (int(a) for a in sys.argv[1:4])
eng = TauEngine(0)
x = torch.from_numpy(workloads.generate(cfg)).cuda()
m = x.shape[0]
jr = job_shard_range(R, P, m)
print("job range", jr, flush=True)
for _ in range(2):
    r = eng.all_pairs(x, job_range=jr); torch.cuda.synchronize(); del r
marks = []
import paper_1704_03767_b200.device as dv
orig = dv._lib.call
def call(name, *a):
    s = torch.cuda.Event(enable_timing=True); s.record()
    rr = orig(name, *a)
    e = torch.cuda.Event(enable_timing=True); e.record(); marks.append((name, s, e))
    return rr
dv._lib.call = call
r = eng.all_pairs(x, job_range=jr); torch.cuda.synchronize()
for name, s, e in marks:
    print(f"  {name:18s} {s.elapsed_time(e):8.3f} ms", flush=True)
