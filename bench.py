"""Benchmark: all-pairs Kendall tau-b variable-pairs/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config k] [--impl ours|reference]

A "step" is one full pass of the hot path over the configured workload
(BASELINE config 2 by default: m=2048 x n=1000 int32 0..9, every i<j pair):
K0 rank -> K2 sign pack -> K3 tcgen05 sign GEMM (kind::mxf4, e2m1 signs) ->
K5 fp64 finalize (tau_a, tau_b).

* value: pairs/s with inputs resident in HBM, CUDA-event timed on the launching
  stream, L2 flushed (256 MiB write) before every timed step, max over ranks.
* e2e: the same metric through the public host API (TauEngine.all_pairs_host)
  with pinned HOST buffers: H2D of the values, the full path, D2H of tau_b for
  every job id, all inside the events.
* roofline: the GEMM (dominant kernel), algorithmic ops 2K per i<j pair
  (K = n(n-1)/2 sample pairs), per-launch CUDA-event duration vs the dense
  tensor peak of the MMA kind it runs (FP4: nominal 9 PFLOP/s, B200_PROFILING.md;
  int8: measured here with torch._int_mm since MEASURED_PEAKS.json has no int8).
* cpu_baseline: the oracle port (C restatement of the reference packed/VSE
  merge kernel, pthreads over all host cores) on a bounded sample (rank 0, N=1).

``--impl reference`` times that CPU implementation alone on the host cores
(oracle port: the reference is Python/numba and does not travel to the box).
Multi-GPU (torchrun): every rank computes its own copy of the workload
(independent objects, no collective) -> "scaling": "weak"; ``--scaling strong``
shards the job-id range instead (contiguous shards concatenate, pairindex.py:68-80);
``--gather`` adds the path's only collective (all-gather of the tau_b shards) to every
timed strong-scaling step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

with open(os.path.join(ROOT, "BASELINE.json")) as _fh:
    METRIC = json.load(_fh)["metric"]
UNIT = "pairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--gather", action="store_true",
                    help="strong scaling: all-gather every rank's tau_b shard inside the timed step "
                         "(multi.gather_shards: NCCL all_gather over NVLink)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay the device step as one CUDA graph (auto: config 1, whose step is launch-bound)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU legs
# SURVEY 8(d) CPU protocol: configs 1 and 2 run every pair; configs 3 and 5 a seeded subset of m' = 2048
# variables (every pair among them), config 4 m' = 64, drawn with np.random.default_rng(99).choice(m, m').
CPU_SUBSET = {1: None, 2: None, 3: 2048, 4: 64, 5: 2048}


def cpu_subset(k: int, m: int, size: int | None = None) -> np.ndarray:
    """Row indices of the CPU-timed variable subset of config k (sorted; all rows for configs 1-2)."""
    sz = CPU_SUBSET.get(k) if size is None else size
    if sz is None or sz >= m:
        return np.arange(m)
    return np.sort(np.random.default_rng(99).choice(m, sz, replace=False))


def cpu_pairs_rate(x: np.ndarray, rows: np.ndarray, threads: int):
    """Time the oracle port on every i<j pair of the variable subset ``rows`` of the raw values ``x``
    (ranked first, outside the timer like the reference's rank_transform); returns
    (pairs/s, kernel name, pair count, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc  # CPU baseline leg only

    sub = np.ascontiguousarray(host_ranks(x[rows]))
    ms, n = sub.shape
    kernel = orc.KERNEL_PACKED if (n <= 32767 and sub.max() < 1 << 15) else orc.KERNEL_SORTED
    pi, pj = orc.upper_pairs(ms, diagonal=False)
    t0 = time.perf_counter()
    orc.all_pairs(sub, pi, pj, kernel, threads=threads, want_counts=True)
    dt = time.perf_counter() - t0
    kname = "packed (VSE semantics, kernel_vectorized.py:507-523)" if kernel == orc.KERNEL_PACKED else \
        "sorted (GSE, kernel_sorted.py:195-212)"
    return pi.shape[0] / dt, kname, int(pi.shape[0]), dt


def cpu_sample_text(k: int, m: int, rows: np.ndarray, count: int, dt: float, kname: str, threads: int) -> str:
    what = (f"every i<j pair of all {m} variables" if rows.shape[0] == m else
            f"every i<j pair of a {rows.shape[0]}-variable subset (np.random.default_rng(99).choice({m}, "
            f"{rows.shape[0]}, replace=False), SURVEY 8(d))")
    return (f"{count} pairs = {what}; oracle port of the reference {kname} with all counts "
            f"(n_d, n1, n2, n3), {threads} threads, {dt:.1f} s")


def workload(k: int):
    from paper_1704_03767_b200 import workloads
    spec = workloads.CONFIGS[k]
    x = workloads.generate(k)
    return spec, x


def host_ranks(x: np.ndarray) -> np.ndarray:
    """Dense ranks per row for the CPU legs (the reference ranks outside its timer, dataio.py:194-196)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc  # CPU legs only
    return orc.rank_matrix(x)


def run_reference(args):
    """The reference's CPU path (oracle port, all host threads) on this arm's workload: every step times
    every pair of the SURVEY 8(d) variable subset (shrunk if the whole run would exceed ~3 min)."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    spec, x = workload(args.config)
    threads = os.cpu_count() or 1
    m, n = x.shape
    total_steps = args.steps + args.warmup
    rows = cpu_subset(args.config, m)
    # probe one step; shrink the subset (pairs ~ m'^2) so that all steps fit the budget
    rate0, _, cnt0, dt0 = cpu_pairs_rate(x, rows, threads)
    budget = 180.0 / max(total_steps, 1)
    if dt0 > budget and rows.shape[0] > 64:
        keep = max(64, int(rows.shape[0] * (budget / dt0) ** 0.5))
        rows = cpu_subset(args.config, m, keep)
    times = []
    for s in range(total_steps):
        rate, kname, count, dt = cpu_pairs_rate(x, rows, threads)
        if s >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = count * len(times) / tot
    sample = cpu_sample_text(args.config, m, rows, count, tot / len(times), kname, threads) + " per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"config{args.config}_{spec.name}", "m": m, "n": n,
                   "pairs_timed_per_step": count, "path": "cpu",
                   "outputs": "numerator + n_d/n1/n2/n3 per pair (the reference's CELL_DTYPE fields)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def measure_int8_peak(torch, dev):
    """Dense int8 tensor peak via cuBLASLt (torch._int_mm 8192^3, best of 10)."""
    try:
        a = torch.randint(-3, 3, (8192, 8192), dtype=torch.int8, device=dev)
        b = torch.randint(-3, 3, (8192, 8192), dtype=torch.int8, device=dev).t()
        for _ in range(3):
            torch._int_mm(a, b)
        best = float("inf")
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch._int_mm(a, b)
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e) / 1e3)
        del a, b
        return 2 * 8192 ** 3 / best
    except Exception as exc:  # noqa: BLE001
        print(f"# int8 peak probe failed: {exc}", file=sys.stderr)
        return None


def measure_fp4_peak(torch, dev):
    """Library MXFP4 GEMM throughput: cuBLASLt block-scaled e2m1 (torch.nn.functional.scaled_mm,
    BlockWise1x32 ue8m0 scales) 8192 x 8192 x 32768, best of 5 -- the attainable FP4 tensor rate
    a stock library reaches on this GPU (tools/probe_fp4_peak.py, profiles/r01_fp4_library_peak.json)."""
    try:
        import torch.nn.functional as F
        M = N = 8192
        K = 32768
        a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        sa = torch.full((M, K // 32), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)
        sb = torch.full((N, K // 32), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)

        def f():
            return F.scaled_mm(a, b.t(), sa, F.ScalingType.BlockWise1x32, sb, F.ScalingType.BlockWise1x32,
                               swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                               output_dtype=torch.bfloat16)
        for _ in range(3):
            f()
        best = float("inf")
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            f()
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e) / 1e3)
        del a, b, sa, sb
        return 2.0 * M * N * K / best
    except Exception as exc:  # noqa: BLE001
        print(f"# fp4 library peak probe failed: {exc}", file=sys.stderr)
        return None


def measure_mxf4_ceiling():
    """FLOP/s of the GEMM's own MMA stream (tcgen05 kind::mxf4, 2-SM, M=256, two N=240 accumulators
    alternating) issued back to back with no operand traffic (csrc/tb_probe.cu): the practical tensor
    ceiling for the numerator GEMM on this GPU."""
    try:
        import ctypes
        lib = ctypes.CDLL(os.path.join(ROOT, "paper_1704_03767_b200", "libtbprobe.so"))
        lib.tb_probe_mxf4_flops.restype = ctypes.c_double
        lib.tb_probe_mxf4_flops.argtypes = [ctypes.c_int]
        v = float(lib.tb_probe_mxf4_flops(3))
        return v if v > 0 else None
    except OSError as exc:
        print(f"# mxf4 probe unavailable: {exc}", file=sys.stderr)
        return None


def measure_int32_peak():
    """INT32 lane-ops/s of dependency-free IADD3/LOP3 chains on all SMs (csrc/tb_probe.cu)."""
    try:
        import ctypes
        lib = ctypes.CDLL(os.path.join(ROOT, "paper_1704_03767_b200", "libtbprobe.so"))
        lib.tb_probe_int32_ops.restype = ctypes.c_double
        lib.tb_probe_int32_ops.argtypes = [ctypes.c_int]
        v = float(lib.tb_probe_int32_ops(5))
        return v if v > 0 else None
    except OSError as exc:
        print(f"# int32 probe unavailable: {exc}", file=sys.stderr)
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, local, world = dist_env()
    # TB_BENCH_SHARE_GPU=1 (plumbing check only, never a measurement): ranks share the visible GPUs and
    # talk over gloo, so the N > 1 code path can be exercised on a one-GPU box
    share = os.environ.get("TB_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    red_dev = torch.device("cpu") if share else dev  # all_reduce tensors live where the backend wants them
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.device import TauEngine
    from paper_1704_03767_b200.pairindex import job_shard_range

    spec, x = workload(args.config)
    m, n = x.shape
    total_jobs = m * (m + 1) // 2
    job_range = job_shard_range(rank, world, m) if args.scaling == "strong" else (0, total_jobs)
    eng = TauEngine(local)
    stream = torch.cuda.Stream(device=dev)
    path = eng.choose_path(n)
    xin = x  # raw values: both paths rank on the device (K0 / K0w)
    xd = torch.from_numpy(np.ascontiguousarray(xin)).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    K = n * (n - 1) // 2

    # pairs (i<j) this rank computes
    def strict_pairs(lo, hi):
        # job ids include the diagonal; count diagonal cells in [lo, hi)
        ys = np.arange(m, dtype=np.int64)
        dj = ys * (2 * m - ys + 1) // 2
        return (hi - lo) - int(((dj >= lo) & (dj < hi)).sum())

    my_pairs = strict_pairs(*job_range)

    # instrumented step: events around the GEMM (dominant kernel) on the launching stream
    gemm_events = []

    gather = args.gather and args.scaling == "strong" and world > 1
    if gather:
        from paper_1704_03767_b200.multi import gather_shards

    def step(instrument=False):
        with torch.cuda.stream(stream):
            if instrument:
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                res = eng.all_pairs(xd, kernel=path, job_range=job_range, stream=stream,
                                    _events=(s, e))
                gemm_events.append((s, e))
            else:
                res = eng.all_pairs(xd, kernel=path, job_range=job_range, stream=stream)
            if gather:  # the only collective of the path: tau_b shards -> every rank (stream-ordered)
                tb = res.tau_b if not share else res.tau_b.cpu()
                full = gather_shards(tb, m)
                if rank == 0:
                    res.extra["tau_b_full"] = full
        return res

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    res.validate()
    launches_per_step = res.launches
    sign_format = res.extra.get("sign_format")
    del res

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    times = []
    use_graph = args.graph == "on" or (args.graph == "auto" and args.config == 1)
    graph = None
    if use_graph:
        # config 1 is launch-bound; time back-to-back replays of the whole step captured
        # in one CUDA graph.  The dominant kernel's time still comes from eager instrumented steps.
        for _ in range(min(args.steps, 50)):
            step(instrument=True)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream, capture_error_mode="relaxed"):
            res_graph = eng.all_pairs(xd, kernel=path, job_range=job_range, stream=stream)
        torch.cuda.synchronize()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
        if graph is not None:
            with torch.cuda.stream(stream):
                graph.replay()
        else:
            res = step(instrument=True)
        e.record(stream)
        times.append((s, e))
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if graph is not None:
        res = res_graph
        res.validate()
    gather_check = None
    if gather and rank == 0:  # the gathered stream equals one device computing every job id
        full_ref = eng.all_pairs(xd, kernel=path, stream=stream)
        torch.cuda.synchronize()
        got = res.extra["tau_b_full"].to(dev)
        gather_check = bool(torch.equal(got.view(torch.int64), full_ref.tau_b.view(torch.int64)))
        del full_ref, got
    if world > 1:
        dist.barrier()
    t_total = sum(s.elapsed_time(e) for s, e in times) / 1e3
    gemm_s = [s.elapsed_time(e) / 1e3 for s, e in gemm_events]
    gemm_avg = sum(gemm_s) / len(gemm_s)
    t_max = t_total
    if world > 1:
        tt = torch.tensor([t_total], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    total_pairs = my_pairs * world
    value = total_pairs * args.steps / t_max
    ms_per_step = 1e3 * t_max / args.steps
    del res

    # ---- e2e through the public API with pinned host buffers: H2D values -> device path -> tau_b D2H
    xh = torch.from_numpy(np.ascontiguousarray(xin)).pin_memory()
    out_tb = torch.empty(total_jobs, dtype=torch.float64).pin_memory()
    e2e_times = []
    e2e_launches = 0
    for it in range(args.e2e_steps + 2):
        with torch.cuda.stream(stream):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            r = eng.all_pairs_host(xh, out_tb, kernel=path, stream=stream)
            e.record(stream)
        if it >= 2:
            e2e_times.append((s, e))
        e2e_launches = r.launches
        del r
    torch.cuda.synchronize()
    e2e_t = sum(s.elapsed_time(e) for s, e in e2e_times) / 1e3
    if world > 1:
        tt = torch.tensor([e2e_t], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())
    # every rank runs the full host entry point: weak scaling counts each rank's copy, strong scaling
    # (one shared job range) does not shard this leg, so it counts the pairs once
    e2e_pairs = strict_pairs(0, total_jobs) * (world if args.scaling == "weak" else 1)
    e2e_value = e2e_pairs * len(e2e_times) / e2e_t if e2e_times else None  # --e2e-steps 0: leg skipped
    h2d = xh.numel() * xh.element_size()
    d2h = total_jobs * 8

    out = None
    if rank == 0:
        peak = measure_int8_peak(torch, dev) if path == "gemm" else None
        algo = 2 * K * my_pairs if path == "gemm" else 4 * n * int(np.ceil(np.log2(n))) * my_pairs
        achieved = algo / gemm_avg
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as fh:
                tj = json.load(fh)
            traffic = tj.get(f"config{args.config}", {}).get("dram_bytes_per_launch")
        if path == "gemm":
            fp4 = sign_format == _lib.TB_SIGN_E2M1
            fp4_lib = measure_fp4_peak(torch, dev) if fp4 else None
            mma_ceiling = measure_mxf4_ceiling() if fp4 else None
            if fp4:
                pk, src = 9.0e15, "nominal dense FP4 (kind::mxf4) 9 PFLOP/s, B200_PROFILING.md table (no measured FP4 entry)"
            else:
                pk = peak or 4.5e15
                src = ("measured here: torch._int_mm int8 8192^3 best-of-10 (cuBLASLt)" if peak
                       else "nominal 4.5 POPS dense int8 (probe failed)")
            roof = {"bound": "tensor", "achieved": achieved / 1e12, "peak": pk / 1e12,
                    "unit": "TFLOP/s", "frac": achieved / pk, "traffic": traffic,
                    "kernel": "gemm_fp4_kernel (tcgen05.mma kind::mxf4, 2-SM)" if fp4
                    else "gemm_tc2_kernel (tcgen05.mma kind::i8, 2-SM)",
                    "peak_source": src,
                    "frac_of_measured_int8_peak": (achieved / peak) if peak else None,
                    "measured_fp4_library_tflops": fp4_lib / 1e12 if fp4_lib else None,
                    "frac_of_measured_fp4_library": (achieved / fp4_lib) if fp4_lib else None,
                    "measured_mma_ceiling_tflops": mma_ceiling / 1e12 if mma_ceiling else None,
                    "frac_of_measured_mma_ceiling": (achieved / mma_ceiling) if mma_ceiling else None,
                    "measured_int8_peak_tops": peak / 1e12 if peak else None,
                    "algorithmic": f"2*K ops per i<j pair, K=n(n-1)/2={K} sample pairs; {my_pairs} pairs per launch",
                    "kernel_ms": 1e3 * gemm_avg, "kernel_share_of_step": gemm_avg / (t_total / args.steps)}
        else:
            # INT32 issue peak measured here: dependency-free IADD3/LOP3 chains on every SM
            # (csrc/tb_probe.cu); the nominal 128 lanes/clk/SM x SMs x max clock is reported beside it
            props = torch.cuda.get_device_properties(dev)
            nominal = 128 * props.multi_processor_count * 1.965e9
            measured = measure_int32_peak()
            int32_peak = measured or nominal
            roof = {"bound": "int32", "achieved": achieved / 1e12, "peak": int32_peak / 1e12, "unit": "TOP/s",
                    "frac": achieved / int32_peak, "traffic": traffic, "kernel": "merge_pairs_kernel",
                    "peak_source": ("measured here: IADD3/LOP3 microbenchmark, best of 5 (libtbprobe.so)" if measured
                                    else "nominal INT32 issue 128 lanes/clk/SM x SMs x 1.965 GHz (probe failed)"),
                    "nominal_int32_tops": nominal / 1e12,
                    "algorithmic": f"4*n*ceil(log2 n) INT32 ops per i<j pair, n={n}; {my_pairs} pairs per launch",
                    "kernel_ms": 1e3 * gemm_avg, "kernel_share_of_step": gemm_avg / (t_total / args.steps)}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            rows = cpu_subset(args.config, m)
            rate, kname, count, dt = cpu_pairs_rate(x, rows, threads)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": cpu_sample_text(args.config, m, rows, count, dt, kname, threads)}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": ("e2m1" if sign_format == _lib.TB_SIGN_E2M1 else "i8") if path == "gemm" else "int32",
            "data": "synthetic",
            "config": {"workload": f"config{args.config}_{spec.name}", "m": m, "n": n,
                       "pairs_per_rank": my_pairs, "path": path,
                       "l2": "flushed before every timed step (256 MiB write, untimed)",
                       "step": "one CUDA graph replay" if use_graph else "eager launches",
                       "outputs": "numerator i32 + tau_a f64 + tau_b f64 in job-id order"
                       + ("; tau_b shards all-gathered to every rank inside the step" if gather else "")},
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * e2e_t / len(e2e_times) if e2e_times else None,
                    "api": "TauEngine.all_pairs_host (pinned host values in, tau_b f64 for every job id out; "
                           "row bands overlap D2H with compute)", "gpu_launches_per_step": e2e_launches},
            "clocks": clocks, "gpu_launches": launches_per_step * args.steps,
            "abi": _lib.TB_MAX_N and "libtaub200.so",
        }
        if gather:
            out["gather_check"] = gather_check
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
