"""Device-level all-pairs tau: the hot path, composed from the C-ABI kernels.

``TauEngine.all_pairs(x)`` takes a [m, n] device tensor (raw values or dense
ranks) and returns device tensors for one contiguous job-id range
(pairindex.py:27-31 numbering, diagonal included):

* GEMM path (small n):  K2 sign pack -> K3 tcgen05 int8 GEMM -> K5 finalize
  (optionally the |S| GEMM + full counts for n_d / n3);
* merge path (large n): K1 presort -> K4 Knight merge-inversion -> K5 finalize.

Everything runs on the caller's current CUDA stream; nothing here touches the
host except the optional ``validate()`` (one 4-byte flag read).
"""

from __future__ import annotations

import contextlib
import ctypes
import math
import os
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import CapacityExceededError, ConfigError, InvalidInputError
from .pairindex import job_coord

# Dispatcher (north star (3): the numerator kernel per shape from measured throughput; the reference's
# analogue is the capacity-driven kernel switch, engine.py:338-346).  Per-unit costs measured on B200 by
# tools/exp_dispatch.py (profiles/r02_dispatch_table.jsonl): for n, the GEMM path's sign-pack seconds per
# row (K0/K0w + K2) and GEMM seconds per job id (K3: e2m1 kind::mxf4 up to n = 5792, int8 above; measured
# at the largest m whose S fits, given as m_gemm), and the merge path's K0w + K1 seconds per row and K4
# seconds per job id.  A shape (m, n) takes the path with the smaller m * per_row + J * per_job
# (J = m(m+1)/2 job ids), the GEMM only while its sign matrix fits the free device memory.
DISPATCH_TABLE = (
    # n, gemm pack s/row, gemm s/job, m_gemm, merge prep s/row, merge s/job  (tools/exp_dispatch.py on a B200,
    # profiles/r02_dispatch_table.jsonl; e2m1 GEMM at every n, merge with several pairs per CTA for n <= 32768)
    (1024, 1.109e-07, 2.017e-10, 2048, 3.289e-07, 9.204e-08),
    (2048, 3.726e-07, 9.795e-10, 2048, 4.082e-07, 1.134e-08),
    (4096, 1.108e-06, 7.872e-09, 2048, 5.305e-07, 2.459e-08),
    (5792, 2.325e-06, 1.575e-08, 2048, 6.819e-07, 5.314e-08),
    (6144, 2.494e-06, 1.768e-08, 2048, 6.968e-07, 5.264e-08),
    (8192, 3.725e-06, 3.141e-08, 2048, 9.226e-07, 5.415e-08),
    (12288, 6.698e-06, 7.267e-08, 1769, 1.142e-06, 1.149e-07),
    (16384, 1.232e-05, 1.517e-07, 995, 1.665e-06, 1.184e-07),
    (24576, 2.774e-05, 3.989e-07, 442, 2.782e-06, 2.505e-07),
    (32767, 6.850e-05, 1.002e-06, 248, 4.336e-06, 2.635e-07),
)
D2H_PIECE_BYTES = 256 << 20
FP4_WIDE = os.environ.get("TB_FP4_WIDE", "1") != "0"
# offset-coded GEMM operands (TB_SIGN_E2M1_OFS, see TauEngine.sign_format): "auto" | "1" | "0"
SIGN_OFS = os.environ.get("TB_SIGN_OFS", "auto")
FUSED_ROW_SUMS = os.environ.get("TB_FUSED_ROW_SUMS", "1") != "0"  # 0: tb_sign_pack + tb_sign_row_sums (cross-check)
OFS_MIN_WORK = 1e13  # m^2 K from which the GEMM runs long enough to be power-capped (config 3: 3.3e13)
TIED_SPARSE_FRAC = 0.35  # |S| GEMM over the tied rows only while they are at most this share of the rows
GEMM_MAX_N = 14000  # the crossover for shapes of unknown m (large m: the GEMM's per-job cost decides): e2m1
# GEMM vs merge with several pairs per CTA, n = 12288: 73 vs 115 ns per job, n = 16384: 152 vs 118 ns
RANK_ROWS_MAX_N = 8192  # tb_rank_rows' row limit; wider GEMM-path rows are ranked by tb_rank_dense
SIGN_MAX_N = 32767      # tb_sign_pack: 15-bit ranks
PATHS = ("gemm", "merge")


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream_ptr(stream: torch.cuda.Stream | None = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.int32:
        return _lib.TB_DTYPE_I32
    if t.dtype == torch.float32:
        return _lib.TB_DTYPE_F32
    if t.dtype == torch.float64:
        return _lib.TB_DTYPE_F64
    raise InvalidInputError(f"unsupported value dtype {t.dtype}; use int32, float32 or float64")


def row_prefix(y: int, m: int) -> int:
    return y * (2 * m - y + 1) // 2


@dataclass
class PairResult:
    """Per-pair device outputs for job ids [job_lo, job_hi)."""

    m: int
    n: int
    job_lo: int
    job_hi: int
    path: str
    numerator: torch.Tensor            # int32 [count]
    n1_rows: torch.Tensor              # int64 [m] (tie pairs per variable; n2 of a pair is n1 of its x)
    tau_a: torch.Tensor | None = None  # float64 [count]
    tau_b: torch.Tensor | None = None  # float64 [count]
    n_d: torch.Tensor | None = None    # int64 [count]
    n3: torch.Tensor | None = None     # int64 [count]
    flags: torch.Tensor | None = None  # int32 [1] device status (NaN / bad ranks)
    launches: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def count(self) -> int:
        return self.job_hi - self.job_lo

    def validate(self) -> "PairResult":
        """Raise InvalidInputError if a kernel flagged the input (syncs the stream)."""
        if self.flags is not None:
            f = int(self.flags.item())
            if f & 1:
                raise InvalidInputError("observations contain NaN, which has no rank")
            if f & 2:
                raise InvalidInputError("ranks must be dense integers in [0, n)")
        return self


@dataclass
class Prepared:
    """Device operands of one dataset (TauEngine.prepare): what every job range's numerator reads."""

    path: str
    m: int
    n: int
    full: bool
    n1_rows: torch.Tensor             # int64 [m]
    flags: torch.Tensor               # int32 [1]
    simt: bool = False
    S: torch.Tensor | None = None     # GEMM: sign matrix [m, ldS] bytes
    A: torch.Tensor | None = None     # GEMM full counts: |S|
    K: int = 0
    ldS: int = 0
    fmt: int = 0
    fix: torch.Tensor | None = None      # TB_SIGN_E2M1_OFS: int32 [m] row sums of S (tb_sign_row_sums)
    fix_abs: torch.Tensor | None = None  # ... and n1 per row as int32 (the tie-indicator GEMM's correction)
    row_lo: int = 0
    any_ties: bool | None = None      # GEMM full counts: does any row >= row_lo have ties (read lazily)
    tied_rows: np.ndarray | None = None   # sparse full counts: the tied rows >= row_lo (host, ascending)
    tied_dev: torch.Tensor | None = None  # ... on the device (int32)
    absdot_t: torch.Tensor | None = None  # |S_a|.|S_b| over the tied rows' own job ids (int32)
    keys: torch.Tensor | None = None  # merge: K1 presort outputs
    pos: torch.Tensor | None = None
    srt: torch.Tensor | None = None
    maxgrp: torch.Tensor | None = None
    groups: torch.Tensor | None = None
    ngroups: torch.Tensor | None = None

    def validate(self) -> "Prepared":
        PairResult.validate(self)  # same flag bits
        return self


class TauEngine:
    """Owns device workspaces; one instance per device.  Calls from several host threads serialise on
    ``lock``; every kernel launches on this engine's device."""

    def __init__(self, device: int | torch.device | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("TauEngine needs a CUDA device (B200, sm_100a); there is no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   (device.index if isinstance(device, torch.device) else device))
        _lib.load()
        self.caps = _lib.query(self.device.index)
        if not self.caps.tcgen05_i8:
            raise RuntimeError(f"device cc {self.caps.cc_major}.{self.caps.cc_minor} is not sm_100 (B200)")
        self._ws: dict[str, torch.Tensor] = {}
        self._events = None
        self._stream = None
        # One call at a time owns the workspaces (S, |S|, ranks, presort arrays): host threads serialise on
        # the lock, and a call on another stream first waits for the previous call's stream work (_tail),
        # so a workspace is never overwritten while kernels of an earlier call may still read it.
        self.lock = threading.RLock()
        self._tail: torch.cuda.Event | None = None

    @contextlib.contextmanager
    def _session(self, stream: torch.cuda.Stream | None):
        """Enter this engine's device and stream (kernels launch on the current device: the C ABI uses
        cudaGetDevice), holding the workspace lock; orders the stream after the previous call."""
        with self.lock, torch.cuda.device(self.device):
            st = stream if stream is not None else torch.cuda.current_stream(self.device)
            if st.device != self.device:
                raise ConfigError(f"stream is on {st.device}, engine on {self.device}")
            capturing = torch.cuda.is_current_stream_capturing()
            if self._tail is not None and not capturing:
                st.wait_event(self._tail)
            self._stream, self._events = st, None
            try:
                with torch.cuda.stream(st):
                    yield st
            finally:
                if not capturing:  # (a graph replay is ordered by the stream it is replayed on)
                    ev = torch.cuda.Event()
                    ev.record(st)
                    self._tail = ev

    # -------------------------------------------------------------- workspaces
    def _buf(self, name: str, numel: int, dtype: torch.dtype) -> torch.Tensor:
        t = self._ws.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            if t is not None:
                del self._ws[name]
                t = None
            try:
                t = torch.empty(max(numel, 1), dtype=dtype, device=self.device)
            except torch.OutOfMemoryError as exc:  # e.g. S = m x K/2 bytes beyond this GPU's HBM
                nbytes = numel * torch.empty(0, dtype=dtype).element_size()
                raise CapacityExceededError(
                    f"device workspace {name!r} needs {nbytes / 2**30:.1f} GiB, more than is free on "
                    f"{self.device}; split the variables into blocks (fewer rows per call) or use the merge "
                    f"path (kernel='merge', O(m n) memory)") from exc
            self._ws[name] = t
        return t[:numel]

    def release(self):
        self._ws.clear()

    def _mark(self, which: int):
        if self._events is not None:
            self._events[which].record(self._stream)

    sign_format_override: int | None = None  # tests / experiments: force TB_SIGN_*
    force_abs_gemm: bool = False  # tests: run the |S| GEMM even when no variable has ties
    # full counts with tied variables: "auto" runs the |S| GEMM over the tied rows only when they are at
    # most TIED_SPARSE_FRAC of the rows (n3 = 0 for every pair with an untied variable), else over all rows
    tied_mode: str = "auto"
    # tau_b-only callers (tau_b_bands, all_pairs_host(numerators=False)) on the GEMM path go through
    # tb_gemm_tau_b: one-launch plans write tau_b from the GEMM epilogue (no numerator round trip, no
    # finalize launch; TB_FUSE_EPILOGUE=0 restores numerators + tb_finalize), split plans finalize straight
    # from the f32 workspace (one launch instead of convert + finalize)
    fuse_finalize: bool = os.environ.get("TB_FUSE_FINALIZE", "1") != "0"

    def sign_format(self, K: int, m: int | None = None) -> int:
        """e2m1 (kind::mxf4) for every K: beyond 2^24 the FP4 GEMM splits each unit into items whose f32
        sums stay exact and adds them as int32 (twice the int8 rate, half its S bytes).  TB_FP4_WIDE=0
        restores int8 (kind::i8) for K >= 2^24.

        While 4 K < 2^24 (n <= 2896) and the GEMM is long enough to run into the board's power cap
        (m^2 K >= OFS_MIN_WORK, or TB_SIGN_OFS=1), the operands are offset-coded (TB_SIGN_E2M1_OFS: S + 1,
        non-negative and half zero): the same MMA stream toggles fewer bits, the capped SM clock rises
        (config 5: 1.31 -> 1.54 GHz) and the GEMM is ~12% faster (profiles/r02_power_pattern.log)."""
        if self.sign_format_override is not None:
            return self.sign_format_override
        if K >= (1 << 24) and not FP4_WIDE:
            return _lib.TB_SIGN_I8
        if 4 * K < (1 << 24) and (SIGN_OFS == "1" or (SIGN_OFS == "auto" and m is not None
                                                     and m * m * K >= OFS_MIN_WORK)):
            return _lib.TB_SIGN_E2M1_OFS
        return _lib.TB_SIGN_E2M1

    @staticmethod
    def path_costs(m: int, n: int) -> dict:
        """Modelled seconds of each device path for an m x n all-pairs job (DISPATCH_TABLE, log-log
        interpolation in n; below the table the GEMM scales with K ~ n^2, the merge with n log n)."""
        tab = DISPATCH_TABLE
        ns = [r[0] for r in tab]
        J = m * (m + 1) / 2

        def interp(col: int) -> float:
            if n <= ns[0]:
                v = tab[0][col]
                return v * ((n / ns[0]) ** 2 if col in (1, 2) else (n * math.log2(max(n, 2))) / (ns[0] * 10.0))
            if n >= ns[-1]:
                return tab[-1][col] * (n / ns[-1]) ** (2 if col in (1, 2) else 1)
            for a, b in zip(tab, tab[1:]):
                if a[0] <= n <= b[0]:
                    f = math.log(n / a[0]) / math.log(b[0] / a[0])
                    return math.exp(math.log(a[col]) * (1 - f) + math.log(b[col]) * f)
            raise AssertionError
        out = {"merge": m * interp(4) + J * interp(5)}
        if n <= SIGN_MAX_N:
            out["gemm"] = m * interp(1) + J * interp(2)
        return out

    def choose_path(self, n: int, m: int | None = None, full_counts: bool = False) -> str:
        """The numerator path for an (m x n) job on this device (module-level choose_path)."""
        return choose_path(n, m=m, full_counts=full_counts, eng=self)

    # -------------------------------------------------------------- the hot path
    def all_pairs(self, x: torch.Tensor, kernel: str = "auto", job_range: tuple[int, int] | None = None,
                  tau_a: bool = True, tau_b: bool = True, full_counts: bool = False, splits: int = 0,
                  stream: torch.cuda.Stream | None = None, simt: bool = False,
                  _events: tuple | None = None) -> PairResult:
        """All pairs of the job range.  ``_events=(start, end)`` brackets the numerator kernel
        (GEMM or merge) with CUDA events on the launching stream (bench instrumentation)."""
        if x.device.type != "cuda":
            raise InvalidInputError("x must be a CUDA tensor (use the host API for numpy input)")
        if x.dim() != 2:
            raise InvalidInputError(f"values must be 2-D (variables x observations), got {x.dim()}-D")
        m, n = x.shape
        if m < 1 or n < 1:
            raise InvalidInputError("dataset is empty")
        if n < 2:
            raise InvalidInputError("need at least two observations per variable")
        if n > _lib.TB_MAX_N:
            raise CapacityExceededError(f"n={n} exceeds the device limit {_lib.TB_MAX_N}")
        if x.stride(1) != 1:
            x = x.contiguous()
        total = m * (m + 1) // 2
        job_lo, job_hi = (0, total) if job_range is None else (int(job_range[0]), int(job_range[1]))
        if not 0 <= job_lo <= job_hi <= total:
            raise ConfigError(f"job range [{job_lo}, {job_hi}) outside [0, {total})")
        path = self.choose_path(n, m=m, full_counts=full_counts) if kernel == "auto" else kernel
        if path not in PATHS:
            raise ConfigError(f"unknown device path {kernel!r}, expected one of {PATHS + ('auto',)}")
        if x.device != self.device:
            raise InvalidInputError(f"x is on {x.device}, engine on {self.device}")
        with self._session(stream) as st_t:
            self._events = _events
            return self._run(x, path, m, n, job_lo, job_hi, _stream_ptr(st_t), tau_a, tau_b, full_counts,
                             splits, simt)

    def _run(self, x, path, m, n, job_lo, job_hi, st, tau_a, tau_b, full_counts, splits, simt) -> PairResult:
        count = job_hi - job_lo
        dev = self.device
        c0 = _lib.load().tb_launch_count()
        row_lo = job_coord(job_lo, m)[0] if job_hi > job_lo else m
        prep = self.prepare(x, path, full_counts=full_counts, row_lo=row_lo, simt=simt)
        res = PairResult(m=m, n=n, job_lo=job_lo, job_hi=job_hi, path=path,
                         numerator=torch.empty(count, dtype=torch.int32, device=dev),
                         n1_rows=prep.n1_rows, flags=prep.flags)
        res.extra["sign_format"] = prep.fmt if path == "gemm" else None
        if path == "merge" or full_counts:
            res.n_d = torch.empty(count, dtype=torch.int64, device=dev)
            res.n3 = torch.empty(count, dtype=torch.int64, device=dev)
        self._mark(0)
        self.numerators(prep, job_lo, job_hi, res.numerator, res.n_d, res.n3, splits=splits, _mark_after_num=True)
        if tau_a or tau_b:
            res.tau_a = torch.empty(count, dtype=torch.float64, device=dev) if tau_a else None
            res.tau_b = torch.empty(count, dtype=torch.float64, device=dev) if tau_b else None
            _lib.call("tb_finalize", _ptr(res.numerator), _ptr(res.n1_rows), m, n, job_lo, job_hi,
                      _ptr(res.tau_a), _ptr(res.tau_b), st)
        res.launches = _lib.load().tb_launch_count() - c0
        return res

    # -------------------------------------------------------------- prepared operands + job-range numerators
    def session(self, stream: torch.cuda.Stream | None = None):
        """Context manager for callers composing prepare() / numerators() themselves (the engine's
        compute_all_pairs pipeline): this device, the workspace lock, ``stream`` (default: the device's
        current stream) current and ordered after the previous call; yields the stream."""
        return self._session(stream)

    def prepare(self, x: torch.Tensor, path: str, full_counts: bool = False, row_lo: int = 0,
                simt: bool = False, all_rows: bool = True) -> "Prepared":
        """Per-dataset device operands, once per call (inside session()): ranks and n1 of every row (of rows
        >= row_lo only with all_rows=False: a job range starting in row row_lo never reads the others), then
        the sign matrix S of rows >= row_lo on the GEMM path, or the K1 presort on the merge path.
        Workspaces are the engine's (valid until the next prepare on this engine)."""
        m, n = x.shape
        st = _stream_ptr(self._stream)
        prep = Prepared(path=path, m=m, n=n, full=full_counts, simt=simt,
                        n1_rows=(torch.empty if all_rows else torch.zeros)(m, dtype=torch.int64, device=self.device),
                        flags=torch.zeros(1, dtype=torch.int32, device=self.device))
        stub = PairResult(m=m, n=n, job_lo=row_prefix(min(row_lo, m), m), job_hi=m * (m + 1) // 2, path=path,
                          numerator=None, n1_rows=prep.n1_rows, flags=prep.flags)
        prep.row_lo = min(row_lo, m)
        if path == "gemm":
            prep.S, prep.K, prep.ldS, prep.fmt = self._gemm_prepare(x, stub, st, simt, all_rows=all_rows)
            prep.fix = stub.extra.get("fix")
        else:
            prep.pos, prep.srt, prep.keys, (prep.maxgrp, prep.groups, prep.ngroups) = \
                self._merge_prepare(x.contiguous(), stub, st, row_from=0 if all_rows else prep.row_lo)
        return prep

    def numerators(self, prep: "Prepared", lo: int, hi: int, num: torch.Tensor, nd: torch.Tensor | None = None,
                   n3: torch.Tensor | None = None, splits: int = 0, _mark_after_num: bool = False) -> None:
        """Numerator (and n_d / n3 when given) of job ids [lo, hi) into num[0:hi-lo] etc. (inside session())."""
        if hi <= lo:
            return
        m, n = prep.m, prep.n
        st = _stream_ptr(self._stream)
        if prep.path == "merge":
            ws, wsb = self._merge_ws(n)
            _lib.call("tb_merge_pairs", _ptr(prep.keys), _ptr(prep.pos), _ptr(prep.srt), _ptr(prep.n1_rows),
                      _ptr(prep.maxgrp), _ptr(prep.groups), _ptr(prep.ngroups), m, n, lo, hi, _ptr(num),
                      _ptr(nd), _ptr(n3), _ptr(ws), wsb, st)
            if _mark_after_num:
                self._mark(1)
            return
        n0 = n * (n - 1) // 2
        for a, b in self._gemm_ranges(m, lo, hi):
            self._gemm_numerator(prep.S, num[a - lo:b - lo], m, prep.K, prep.ldS, prep.fmt, a, b, st, splits,
                                 prep.simt, fix=prep.fix, fix_c=n0)
        if _mark_after_num:
            self._mark(1)
        if nd is not None or n3 is not None:
            if not prep.full:
                raise ConfigError("n_d / n3 on the GEMM path need prepare(..., full_counts=True)")
            if prep.any_ties is None:
                # one read per prepare (a host sync): with no tied variable among the rows the range touches,
                # |S_y|.|S_x| = n0 - n1_y - n1_x and the |S| GEMM (as long as the numerator GEMM) is skipped;
                # with few tied variables only their pairs need it (n3 = 0 whenever one variable is untied)
                tied = np.flatnonzero(prep.n1_rows[prep.row_lo:].cpu().numpy() > 0) + prep.row_lo
                prep.any_ties = tied.size > 0
                sparse = self.tied_mode == "sparse" or (
                    self.tied_mode == "auto" and tied.size <= TIED_SPARSE_FRAC * (m - prep.row_lo))
                if prep.any_ties and sparse:
                    prep.tied_rows = tied
            absdot = None
            if prep.tied_rows is not None and not self.force_abs_gemm:
                self._tied_counts(prep, lo, hi, num, nd, n3, st, splits)
                return
            if prep.any_ties or self.force_abs_gemm:
                if prep.A is None:
                    y0 = prep.row_lo
                    prep.A = self._buf("A", m * prep.ldS, torch.int8)
                    _lib.call("tb_abs_pack", _ptr(prep.S[y0 * prep.ldS:]), m - y0, prep.ldS, prep.fmt,
                              _ptr(prep.A[y0 * prep.ldS:]), st)
                if prep.fix is not None and prep.fix_abs is None:
                    # offset operands: A is the tie indicator Z, |S_y|.|S_x| = n0 - n1_y - n1_x + Z_y.Z_x
                    prep.fix_abs = prep.n1_rows.to(torch.int32)
                absdot = self._buf("absdot", hi - lo, torch.int32)
                for a, b in self._gemm_ranges(m, lo, hi):
                    self._gemm_numerator(prep.A, absdot[a - lo:b - lo], m, prep.K, prep.ldS, prep.fmt, a, b, st,
                                         splits, prep.simt, fix=prep.fix_abs, fix_c=-n0)
            _lib.call("tb_full_counts", _ptr(num), _ptr(absdot), _ptr(prep.n1_rows), m, n, lo, hi, _ptr(nd),
                      _ptr(n3), st)

    def _tied_counts(self, prep: "Prepared", lo: int, hi: int, num, nd, n3, st, splits: int = 0) -> None:
        """Sparse full counts: the closed form for every pair, then n_d / n3 of tied x tied pairs from the
        |S| GEMM over the tied rows (computed once per prepare, in the tied rows' own job-id order)."""
        m, n = prep.m, prep.n
        T = prep.tied_rows
        nt = int(T.size)
        if prep.absdot_t is None:
            prep.tied_dev = torch.from_numpy(T.astype(np.int32)).to(self.device)
            S2 = prep.S[: m * prep.ldS].view(m, prep.ldS)
            St = self._buf("S_tied", nt * prep.ldS, torch.int8)
            torch.index_select(S2, 0, prep.tied_dev.long(), out=St[: nt * prep.ldS].view(nt, prep.ldS))
            At = self._buf("A_tied", nt * prep.ldS, torch.int8)
            _lib.call("tb_abs_pack", _ptr(St), nt, prep.ldS, prep.fmt, _ptr(At), st)
            tt = nt * (nt + 1) // 2
            prep.absdot_t = torch.empty(tt, dtype=torch.int32, device=self.device)
            # offset operands: At is the tied rows' tie indicator Z (see numerators)
            fix_t = None if prep.fix is None else prep.n1_rows[prep.tied_dev.long()].to(torch.int32)
            for a, b in self._gemm_ranges(nt, 0, tt):
                self._gemm_numerator(At, prep.absdot_t[a:b], nt, prep.K, prep.ldS, prep.fmt, a, b, st, splits,
                                     prep.simt, fix=fix_t, fix_c=-(n * (n - 1) // 2))
        _lib.call("tb_full_counts", _ptr(num), None, _ptr(prep.n1_rows), m, n, lo, hi, _ptr(nd), _ptr(n3), st)
        # tied rows a whose row T[a] meets the job range: rows y_lo .. y_hi
        y_lo, y_hi = job_coord(lo, m)[0], job_coord(hi - 1, m)[0]
        a0, a1 = int(np.searchsorted(T, y_lo, "left")), int(np.searchsorted(T, y_hi, "right"))
        if a1 > a0:
            tj_lo, tj_hi = a0 * (2 * nt - a0 + 1) // 2, a1 * (2 * nt - a1 + 1) // 2
            _lib.call("tb_tied_counts", _ptr(prep.absdot_t), _ptr(prep.tied_dev), nt, _ptr(prep.n1_rows), m, n, lo,
                      hi, tj_lo, tj_hi, _ptr(num), _ptr(nd), _ptr(n3), st)

    def _fused_tau_b(self, prep: "Prepared") -> bool:
        return self.fuse_finalize and prep.path == "gemm" and not prep.simt

    def _gemm_tau_b(self, S, num, tb, n1_rows, m, n, K, ldS, fmt, lo, hi, st, fix=None) -> None:
        """tau_b of job ids [lo, hi) into tb[0:hi-lo] from the GEMM epilogue (num: fallback workspace)."""
        for a, b in self._gemm_ranges(m, lo, hi):
            _lib.call("tb_gemm_tau_b_fix", _ptr(S), m, K, ldS, fmt, a, b, 0, _ptr(fix), n * (n - 1) // 2,
                      _ptr(n1_rows), n, _ptr(num[a - lo:b - lo]), _ptr(tb[a - lo:b - lo]), st)

    def _gemm_layout(self, n: int, simt: bool = False, m: int | None = None):
        """(K, sign format, row stride of S in bytes, row stride of R) for n samples."""
        K = int(_lib.load().tb_sign_k(n))  # padded diagonal layout, >= n(n-1)/2 elements
        fmt = self.sign_format(K, m) if not simt else _lib.TB_SIGN_I8
        kbytes = K // 2 if fmt in (_lib.TB_SIGN_E2M1, _lib.TB_SIGN_E2M1_OFS) else K
        return K, fmt, (kbytes + 15) // 16 * 16, (n + 7) // 8 * 8

    def _gemm_prepare(self, x, res: PairResult, st, simt: bool = False, row_chunks=None, all_rows: bool = True):
        """K0 rank transform + K2 sign pack of every row: the GEMM operand S (m x K signs).

        ``row_chunks`` = [(r0, r1, wait_fn)]: prepare rows [r0, r1) after ``wait_fn()`` (the
        host entry point waits for each chunk's H2D copy); default one chunk of all rows."""
        m, n = res.m, res.n
        K, fmt, ldS, ldr = self._gemm_layout(n, simt, m)
        R = self._buf("R", m * ldr, torch.int16)
        S = self._buf("S", m * ldS, torch.int8)
        fix = self._buf("fix", m, torch.int32) if fmt == _lib.TB_SIGN_E2M1_OFS else None
        res.extra["fix"] = fix
        # every job id of [job_lo, job_hi) pairs rows >= y_lo (the row of job_lo): rows above it need no sign
        # vector -- a late job-range shard (multi-GPU strong scaling) packs only its own share of S -- and
        # with all_rows=False they are not ranked either (their n1 stays 0)
        y_lo = job_coord(res.job_lo, m)[0] if res.job_hi > res.job_lo else m
        for r0, r1, wait in (row_chunks or [(0, m, None)]):
            if wait is not None:
                wait()
            if not all_rows:
                r0 = max(r0, y_lo)
                if r0 >= r1:
                    continue
            if n <= RANK_ROWS_MAX_N:  # K0: shared-memory / register sorts
                _lib.call("tb_rank_rows", _ptr(x[r0:r1]), _dtype_code(x), r1 - r0, n, x.stride(0),
                          _ptr(R[r0 * ldr:]), ldr, _ptr(res.n1_rows[r0:]), _ptr(res.flags), st)
            else:  # K0w: wide rows (uint16 ranks out)
                code = _dtype_code(x)
                wsb = int(_lib.load().tb_rank_dense_workspace(r1 - r0, n, code))
                ws = self._buf("rank_ws", wsb, torch.uint8)
                _lib.call("tb_rank_dense", _ptr(x[r0:r1]), code, r1 - r0, n, x.stride(0), _ptr(R[r0 * ldr:]), 1, ldr,
                          _ptr(res.n1_rows[r0:]), _ptr(res.flags), _ptr(ws), wsb, st)
            p0 = max(r0, y_lo)
            if p0 < r1:
                if fix is not None and FUSED_ROW_SUMS:  # the pack sums what it writes (no extra pass over S)
                    _lib.call("tb_sign_pack_sums", _ptr(R[p0 * ldr:]), r1 - p0, n, ldr, _ptr(S[p0 * ldS:]), ldS,
                              _ptr(fix[p0:]), st)
                else:
                    _lib.call("tb_sign_pack", _ptr(R[p0 * ldr:]), r1 - p0, n, ldr, _ptr(S[p0 * ldS:]), ldS, fmt, st)
                    if fix is not None:
                        _lib.call("tb_sign_row_sums", _ptr(S[p0 * ldS:]), r1 - p0, ldS, n, _ptr(fix[p0:]), st)
        res.extra["sign_format"] = fmt
        return S, K, ldS, fmt

    def _gemm_numerator(self, src, out, m, K, ldS, fmt, job_lo, job_hi, st, splits=0, simt=False, fix=None,
                        fix_c=0):
        if simt:
            _lib.call("tb_gemm_pairs_simt", _ptr(src), m, K, ldS, job_lo, job_hi, _ptr(out), st)
        elif fix is not None:  # offset operands: out = dot - fix[y] - fix[x] - fix_c
            _lib.call("tb_gemm_pairs_fix", _ptr(src), m, K, ldS, fmt, job_lo, job_hi, splits, _ptr(fix), fix_c,
                      _ptr(out), st)
        else:
            _lib.call("tb_gemm_pairs", _ptr(src), m, K, ldS, fmt, job_lo, job_hi, splits, _ptr(out), st)

    # GEMM launches per call for very large job ranges (see _gemm_ranges); None = automatic
    gemm_bands: int | None = None

    def _gemm_ranges(self, m: int, job_lo: int, job_hi: int) -> list[tuple[int, int]]:
        """Job sub-ranges the numerator GEMM is launched over.  Ranges of >= 2^30 job ids run as ~8
        row bands of equal pair counts (aligned to the 256-row block): measured on config 5
        (tools/exp_value_bands.py) a single 2.1e9-id launch takes 468-482 ms, eight band launches
        436-443 ms; smaller ranges stay one launch (config 3 slows down when banded)."""
        nb = self.gemm_bands
        if nb is None:
            nb = 8 if job_hi - job_lo >= (1 << 30) else 1
        if nb <= 1:
            return [(job_lo, job_hi)]
        cuts = self.bands(m, nb)
        out = []
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            lo = max(job_lo, r0 * (2 * m - r0 + 1) // 2)
            hi = min(job_hi, r1 * (2 * m - r1 + 1) // 2)
            if lo < hi:
                out.append((lo, hi))
        return out

    def tau_b_bands(self, x: torch.Tensor, bands: list, out: torch.Tensor, kernel: str = "auto", on_band=None,
                    stream: torch.cuda.Stream | None = None, timing: list | None = None) -> Prepared:
        """tau_b of the consecutive job ranges ``bands`` (one rank's shard, multi.shard_bands) into
        ``out`` (indexed from bands[0][0]), band by band -- one numerator launch and one finalize each --
        calling ``on_band(b, out_slice)`` after band b's finalize is enqueued (multi.BandGather.band ships
        it while band b+1 computes).  Asynchronous on ``stream``; ``timing`` collects (start, end) CUDA
        events around each band's numerator kernels (bench instrumentation)."""
        m, n = x.shape
        path = self.choose_path(n, m=m) if kernel == "auto" else kernel
        if not bands:
            return None
        base = bands[0][0]
        with self._session(stream) as st_t:
            st = _stream_ptr(st_t)
            prep = self.prepare(x, path, row_lo=job_coord(base, m)[0], all_rows=False)
            num = self._buf("num_band", max(hi - lo for lo, hi in bands), torch.int32)
            fused = self._fused_tau_b(prep)
            for b, (lo, hi) in enumerate(bands):
                if timing is not None:  # (start, end) events around the band's numerator kernels
                    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    ev[0].record(st_t)
                tb = out[lo - base:hi - base]
                if fused:
                    self._gemm_tau_b(prep.S, num, tb, prep.n1_rows, m, n, prep.K, prep.ldS, prep.fmt, lo, hi, st,
                                     fix=prep.fix)
                else:
                    self.numerators(prep, lo, hi, num)
                if timing is not None:
                    ev[1].record(st_t)
                    timing.append(ev)
                if not fused:
                    _lib.call("tb_finalize", _ptr(num), _ptr(prep.n1_rows), m, n, lo, hi, None, _ptr(tb), st)
                if on_band is not None:
                    on_band(b, tb)
        return prep

    # -------------------------------------------------------------- host-buffer entry point
    @staticmethod
    def bands(m: int, nbands: int = 3, align: int = 256, fracs: tuple | None = None) -> list[int]:
        """Row boundaries splitting the pair triangle into bands holding the given fractions of the
        pairs (default: equal), aligned to the GEMM row block."""
        if fracs is None:
            fracs = (1.0 / nbands,) * nbands
        cuts, acc = [0], 0.0
        for fr in fracs[:-1]:
            acc += fr
            r = int(round(m * (1.0 - (1.0 - min(acc, 1.0)) ** 0.5) / align)) * align
            if cuts[-1] < r < m:
                cuts.append(r)
        cuts.append(m)
        return cuts

    @staticmethod
    def default_band_fracs(total: int) -> tuple:
        """Row-band shares of the pairs for all_pairs_host: more, geometrically shrinking bands as the
        job grows, so the tau_b copy of every band but a small last one hides behind later bands'
        kernels while each band stays large enough for an efficient GEMM launch.  Measured
        (tools/exp_e2e_bands.py, profiles/r01_e2e_band_sweep_v3.log): config 2 (2.1 M job ids) two bands
        0.850 ms (three: 0.876); config 3 (134 M) six-seven bands 22.5 ms (three: 24.4); config 5 (2.1 G)
        twelve bands 417-427 ms (three: 627)."""
        if total <= (8 << 20):
            return (0.7, 0.3)
        k = int(min(14, 2 + round(1.25 * math.log2(total / (8 << 20)))))
        r = 0.7 + 0.01 * k
        w = [r ** i for i in range(k)]
        return tuple(x / sum(w) for x in w)

    def all_pairs_host(self, x_host: torch.Tensor, tau_b_out: torch.Tensor, kernel: str = "auto",
                       band_fracs: tuple | None = None, stream: torch.cuda.Stream | None = None,
                       copy_stream: torch.cuda.Stream | None = None, h2d_chunks: int = 2,
                       h2d_piece_bytes: int = 4 << 20, job_range: tuple[int, int] | None = None,
                       numerators: bool = True) -> PairResult:
        """End-to-end from host buffers: H2D of the values, the device path, tau_b back to host.

        The job range (default: every job id; a rank's shard under multi-GPU strong scaling) is cut into
        row bands; band i's tau_b copy (on ``copy_stream``) overlaps band i+1's numerator kernel.
        ``tau_b_out[j - job_lo]`` receives job id j.  ``x_host`` and ``tau_b_out`` should be pinned; the
        call is asynchronous on ``stream`` (which finally waits for the copies).
        """
        m, n = x_host.shape
        total = m * (m + 1) // 2
        jlo, jhi = (0, total) if job_range is None else (int(job_range[0]), int(job_range[1]))
        if not 0 <= jlo <= jhi <= total:
            raise ConfigError(f"job range [{jlo}, {jhi}) outside [0, {total})")
        if tau_b_out.numel() < jhi - jlo:
            raise ConfigError(f"tau_b_out holds {tau_b_out.numel()} values, need {jhi - jlo}")
        path = self.choose_path(n, m=m) if kernel == "auto" else kernel
        with self._session(stream) as st_t:
            cp_t = copy_stream if copy_stream is not None else self._copy_stream()
            st = _stream_ptr(st_t)
            # H2D in row chunks on the copy stream; rank + sign pack of chunk i overlap chunk i+1's copy
            x = self._buf("x_dev", m * n, x_host.dtype).view(m, n)
            nchunk = max(1, min(h2d_chunks, m // 256)) if path == "gemm" else 1
            cuts_h = [m * i // nchunk // 8 * 8 for i in range(nchunk)] + [m]
            cp_t.wait_stream(st_t)  # the previous call's kernels are done with x
            chunks = []
            row_bytes = n * x_host.element_size()
            piece_rows = max(1, h2d_piece_bytes // max(1, row_bytes))
            for r0, r1 in zip(cuts_h[:-1], cuts_h[1:]):
                with torch.cuda.stream(cp_t):
                    # copies of >= 8 MiB run at ~13 GB/s on the pool's hosts in a sustained pattern
                    # (tools/probe_h2d*.py), <= 4 MiB at ~50 GB/s: upload in pieces
                    for p0 in range(r0, r1, piece_rows):
                        p1 = min(r1, p0 + piece_rows)
                        x[p0:p1].copy_(x_host[p0:p1], non_blocking=True)
                    ev_c = torch.cuda.Event()
                    ev_c.record(cp_t)
                chunks.append((r0, r1, ev_c))
            c0 = _lib.load().tb_launch_count()
            res = PairResult(m=m, n=n, job_lo=jlo, job_hi=jhi, path=path,
                             numerator=self._buf("num_all", jhi - jlo, torch.int32),
                             n1_rows=torch.empty(m, dtype=torch.int64, device=self.device),
                             flags=torch.zeros(1, dtype=torch.int32, device=self.device))
            res.tau_b = self._buf("taub_all", jhi - jlo, torch.float64)
            if path == "gemm":
                S, K, ldS, fmt = self._gemm_prepare(
                    x, res, st, row_chunks=[(r0, r1, (lambda e=ev: st_t.wait_event(e))) for r0, r1, ev in chunks])
            else:
                for _, _, ev in chunks:
                    st_t.wait_event(ev)
                pos, srt, keys, maxgrp = self._merge_prepare(x, res, st)
            if band_fracs is None:
                band_fracs = self.default_band_fracs(jhi - jlo)
            y0 = job_coord(jlo, m)[0] if jhi > jlo else 0
            # row bands of the job range's own rows (equal shares of its pairs)
            sub = [y0 + c for c in self.bands(m - y0, len(band_fracs), fracs=band_fracs)]
            for r0, r1 in zip(sub[:-1], sub[1:]):
                lo, hi = max(jlo, r0 * (2 * m - r0 + 1) // 2), min(jhi, r1 * (2 * m - r1 + 1) // 2)
                if hi <= lo:
                    continue
                num = res.numerator[lo - jlo:hi - jlo]
                tb = res.tau_b[lo - jlo:hi - jlo]
                fused = path == "gemm" and not numerators and self.fuse_finalize
                if fused:  # tau_b from the GEMM epilogue; res.numerator is not filled
                    self._gemm_tau_b(S, num, tb, res.n1_rows, m, n, K, ldS, fmt, lo, hi, st, fix=res.extra.get("fix"))
                elif path == "gemm":
                    self._gemm_numerator(S, num, m, K, ldS, fmt, lo, hi, st, fix=res.extra.get("fix"),
                                         fix_c=n * (n - 1) // 2)
                else:
                    ws, wsb = self._merge_ws(n)
                    _lib.call("tb_merge_pairs", _ptr(keys), _ptr(pos), _ptr(srt), _ptr(res.n1_rows), _ptr(maxgrp[0]),
                              _ptr(maxgrp[1]), _ptr(maxgrp[2]), m, n, lo, hi, _ptr(num), None, None, _ptr(ws), wsb,
                              st)
                if not fused:
                    _lib.call("tb_finalize", _ptr(num), _ptr(res.n1_rows), m, n, lo, hi, None, _ptr(tb), st)
                ev = torch.cuda.Event()
                ev.record(st_t)
                cp_t.wait_event(ev)
                with torch.cuda.stream(cp_t):
                    # D2H in 256 MiB pieces (the record pipeline's slot size: 51-56 GB/s sustained); one copy of
                    # several GB ran at ~30 GB/s on some hosts (profiles/r02_bench_config5_final_b.json)
                    step = D2H_PIECE_BYTES // 8
                    for p0 in range(lo, hi, step):
                        p1 = min(hi, p0 + step)
                        tau_b_out[p0 - jlo:p1 - jlo].copy_(res.tau_b[p0 - jlo:p1 - jlo], non_blocking=True)
            st_t.wait_stream(cp_t)
            res.launches = _lib.load().tb_launch_count() - c0
        return res

    def _copy_stream(self) -> torch.cuda.Stream:
        cs = getattr(self, "_cs", None)
        if cs is None:
            cs = torch.cuda.Stream(device=self.device)
            self._cs = cs
        return cs

    def _merge_ws(self, n: int):
        """K4's scratch for pairs with large u tie groups (tb_merge_workspace bytes)."""
        wsb = int(_lib.load().tb_merge_workspace(n))
        return self._buf("merge_ws", wsb, torch.uint8), wsb

    def _merge_prepare(self, x, res: PairResult, st, row_from: int = 0):
        """K0w dense ranks of the raw values (any dtype, any n), then the K1 presort of every variable
        (u-order positions, sorted ranks, min-rank merge keys, n1, tie groups) -- of rows >= row_from."""
        m, n = res.m, res.n
        r0 = min(max(row_from, 0), m - 1)
        mr = m - r0
        code = _dtype_code(x)
        ranks = self._buf("R32", m * n, torch.int32)
        wsb = int(_lib.load().tb_rank_dense_workspace(mr, n, code))
        ws = self._buf("rank_ws", wsb, torch.uint8)
        _lib.call("tb_rank_dense", _ptr(x[r0:]), code, mr, n, x.stride(0), _ptr(ranks[r0 * n:]), 0, n,
                  _ptr(res.n1_rows[r0:]), _ptr(res.flags), _ptr(ws), wsb, st)
        pos = self._buf("pos", m * n, torch.int32)
        srt = self._buf("sorted", m * n, torch.int32)
        keys = self._buf("mkeys", m * n, torch.int16)
        work = self._buf("work", m * n, torch.int32)
        maxgrp = self._buf("maxgrp", m, torch.int32)
        ngroups = self._buf("ngroups", m, torch.int32)
        _lib.call("tb_presort", _ptr(ranks[r0 * n:]), mr, n, _ptr(pos[r0 * n:]), _ptr(srt[r0 * n:]),
                  _ptr(keys[r0 * n:]), _ptr(res.n1_rows[r0:]), _ptr(maxgrp[r0:]), _ptr(work[r0 * n:]),
                  _ptr(ngroups[r0:]), _ptr(res.flags), st)
        return pos, srt, keys, (maxgrp, work, ngroups)


def choose_path(n: int, m: int | None = None, full_counts: bool = False, eng: "TauEngine | None" = None) -> str:
    """The numerator path for an (m x n) job: the cheaper of the measured cost models (TauEngine.path_costs),
    the GEMM only while its sign matrix (and |S| for full counts) fits 80% of the device's free memory.
    Without m or a device, the large-m crossover GEMM_MAX_N decides."""
    if m is None or eng is None:
        return "gemm" if n <= GEMM_MAX_N else "merge"
    costs = TauEngine.path_costs(m, n)
    if "gemm" not in costs:
        return "merge"
    K, fmt, ldS, _ = eng._gemm_layout(n, m=m)
    need = m * ldS * (2 if full_counts else 1)
    have = eng._ws["S"].numel() if "S" in eng._ws else 0  # a cached S workspace is reusable
    free = torch.cuda.mem_get_info(eng.device)[0] + have
    if need > 0.8 * free:
        return "merge"
    return "gemm" if costs["gemm"] <= costs["merge"] else "merge"


_ENGINES: dict[int, TauEngine] = {}


def get_engine(device: int | None = None) -> TauEngine:
    idx = torch.cuda.current_device() if device is None else int(device)
    eng = _ENGINES.get(idx)
    if eng is None:
        eng = TauEngine(idx)
        _ENGINES[idx] = eng
    return eng
