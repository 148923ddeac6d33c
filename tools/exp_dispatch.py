"""Dispatcher measurement (north star (3): numerator kernel per shape from measured throughput): for each
n, time the GEMM path (K0/K0w ranks + K2 sign pack, then the K3 GEMM over every job id) and the merge
path (K0w ranks + K1 presort, then K4 over every job id) on B200, CUDA events, and print per-unit costs:
pack seconds per row, GEMM seconds per job id, presort seconds per row, merge seconds per job id."""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_1704_03767_b200 import _lib
from paper_1704_03767_b200.device import TauEngine

eng = TauEngine(0)
free = torch.cuda.mem_get_info()[0]
ns = [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096, 5792, 6144, 8192, 12288, 16384, 24576, 32767]


def timed(fn, reps=3):
    best = None
    for _ in range(reps + 1):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e) / 1e3
        best = t if best is None else min(best, t)
    return best


for n in ns:
    rng = np.random.default_rng(n)
    out = {"n": n}
    if n <= 32767:
        K, fmt, ldS, _ = eng._gemm_layout(n)
        mg = int(max(64, min(2048, 0.35 * free / ldS)))
        x = torch.from_numpy(rng.standard_normal((mg, n), dtype=np.float32)).cuda()
        total = mg * (mg + 1) // 2
        num = torch.empty(total, dtype=torch.int32, device="cuda")
        with eng.session() as st:
            prep = eng.prepare(x, "gemm")
            torch.cuda.synchronize()
            tp = timed(lambda: eng.prepare(x, "gemm"))
            tn = timed(lambda: eng.numerators(prep, 0, total, num))
        out.update(fmt="e2m1" if fmt == _lib.TB_SIGN_E2M1 else "i8", m_gemm=mg, gemm_pack_s_per_row=tp / mg,
                   gemm_s_per_job=tn / total, gemm_tops=2 * K * total / tn / 1e12)
        del x, num, prep
        eng.release()
        torch.cuda.empty_cache()
    mm = 256 if n <= 16384 else 128
    x = torch.from_numpy(rng.standard_normal((mm, n), dtype=np.float32)).cuda()
    total = mm * (mm + 1) // 2
    num = torch.empty(total, dtype=torch.int32, device="cuda")
    with eng.session() as st:
        prep = eng.prepare(x, "merge")
        torch.cuda.synchronize()
        tp = timed(lambda: eng.prepare(x, "merge"))
        tn = timed(lambda: eng.numerators(prep, 0, total, num), reps=2)
    out.update(m_merge=mm, merge_prep_s_per_row=tp / mm, merge_s_per_job=tn / total)
    del x, num, prep
    eng.release()
    torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)
