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

import math

import ctypes
from dataclasses import dataclass, field

import torch

from . import _lib
from .errors import CapacityExceededError, ConfigError, InvalidInputError
from .pairindex import job_coord

# Dispatcher crossover (numerator kernel per shape).  The GEMM costs 2K = n(n-1)
# int8 ops per pair at tensor-core rate; the merge costs ~4 n log2 n INT32 ops
# per pair at CUDA-core rate -- SURVEY 7 step 5.  Above this n the sign matrix
# is also too large to materialise (m * n^2 / 2 bytes).
GEMM_MAX_N = 8192  # also the device rank transform's row limit (tb_rank_rows)
PATHS = ("gemm", "merge")


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream_ptr(stream: torch.cuda.Stream | None):
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


class TauEngine:
    """Owns device workspaces; one instance per device/stream user."""

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

    def sign_format(self, K: int) -> int:
        """e2m1 (kind::mxf4) while the f32 sums stay exact (K < 2^24), else int8 (kind::i8)."""
        if self.sign_format_override is not None:
            return self.sign_format_override
        return _lib.TB_SIGN_E2M1 if K < (1 << 24) else _lib.TB_SIGN_I8

    @staticmethod
    def choose_path(n: int) -> str:
        return "gemm" if n <= GEMM_MAX_N else "merge"

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
        path = self.choose_path(n) if kernel == "auto" else kernel
        if path not in PATHS:
            raise ConfigError(f"unknown device path {kernel!r}, expected one of {PATHS + ('auto',)}")
        st = _stream_ptr(stream)
        self._events = _events
        self._stream = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(self._stream):
            return self._run(x, path, m, n, job_lo, job_hi, st, tau_a, tau_b, full_counts, splits, simt)

    def _run(self, x, path, m, n, job_lo, job_hi, st, tau_a, tau_b, full_counts, splits, simt) -> PairResult:
        count = job_hi - job_lo
        dev = self.device
        c0 = _lib.load().tb_launch_count()
        res = PairResult(m=m, n=n, job_lo=job_lo, job_hi=job_hi, path=path,
                         numerator=torch.empty(count, dtype=torch.int32, device=dev),
                         n1_rows=torch.empty(m, dtype=torch.int64, device=dev),
                         flags=torch.zeros(1, dtype=torch.int32, device=dev))
        if path == "gemm":
            self._gemm_path(x, res, st, full_counts, splits, simt)
        else:
            self._merge_path(x, res, st)
        if tau_a or tau_b:
            res.tau_a = torch.empty(count, dtype=torch.float64, device=dev) if tau_a else None
            res.tau_b = torch.empty(count, dtype=torch.float64, device=dev) if tau_b else None
            _lib.call("tb_finalize", _ptr(res.numerator), _ptr(res.n1_rows), m, n, job_lo, job_hi,
                      _ptr(res.tau_a), _ptr(res.tau_b), st)
        res.launches = _lib.load().tb_launch_count() - c0
        return res

    def _gemm_layout(self, n: int, simt: bool = False):
        """(K, sign format, row stride of S in bytes, row stride of R) for n samples."""
        K = int(_lib.load().tb_sign_k(n))  # padded diagonal layout, >= n(n-1)/2 elements
        fmt = self.sign_format(K) if not simt else _lib.TB_SIGN_I8
        kbytes = K // 2 if fmt == _lib.TB_SIGN_E2M1 else K
        return K, fmt, (kbytes + 15) // 16 * 16, (n + 7) // 8 * 8

    def _gemm_prepare(self, x, res: PairResult, st, simt: bool = False, row_chunks=None):
        """K0 rank transform + K2 sign pack of every row: the GEMM operand S (m x K signs).

        ``row_chunks`` = [(r0, r1, wait_fn)]: prepare rows [r0, r1) after ``wait_fn()`` (the
        host entry point waits for each chunk's H2D copy); default one chunk of all rows."""
        m, n = res.m, res.n
        K, fmt, ldS, ldr = self._gemm_layout(n, simt)
        R = self._buf("R", m * ldr, torch.int16)
        S = self._buf("S", m * ldS, torch.int8)
        # every job id of [job_lo, job_hi) pairs rows >= y_lo (the row of job_lo): rows above it are ranked
        # (their n1 is part of the result) but need no sign vector -- a late job-range shard (multi-GPU
        # strong scaling) packs only its own share of S
        y_lo = job_coord(res.job_lo, m)[0] if res.job_hi > res.job_lo else m
        for r0, r1, wait in (row_chunks or [(0, m, None)]):
            if wait is not None:
                wait()
            _lib.call("tb_rank_rows", _ptr(x[r0:r1]), _dtype_code(x), r1 - r0, n, x.stride(0),
                      _ptr(R[r0 * ldr:]), ldr, _ptr(res.n1_rows[r0:]), _ptr(res.flags), st)
            p0 = max(r0, y_lo)
            if p0 < r1:
                _lib.call("tb_sign_pack", _ptr(R[p0 * ldr:]), r1 - p0, n, ldr, _ptr(S[p0 * ldS:]), ldS, fmt, st)
        res.extra["sign_format"] = fmt
        return S, K, ldS, fmt

    def _gemm_numerator(self, src, out, m, K, ldS, fmt, job_lo, job_hi, st, splits=0, simt=False):
        if simt:
            _lib.call("tb_gemm_pairs_simt", _ptr(src), m, K, ldS, job_lo, job_hi, _ptr(out), st)
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

    def _gemm_path(self, x, res: PairResult, st, full_counts: bool, splits: int, simt: bool):
        m, n = res.m, res.n
        S, K, ldS, fmt = self._gemm_prepare(x, res, st, simt)
        self._mark(0)
        for lo, hi in self._gemm_ranges(m, res.job_lo, res.job_hi):
            num = res.numerator[lo - res.job_lo:hi - res.job_lo]
            self._gemm_numerator(S, num, m, K, ldS, fmt, lo, hi, st, splits, simt)
        self._mark(1)
        if full_counts:
            A = self._buf("A", m * ldS, torch.int8)
            _lib.call("tb_abs_pack", _ptr(S), m, ldS, fmt, _ptr(A), st)
            absdot = self._buf("absdot", res.count, torch.int32)
            self._gemm_numerator(A, absdot, m, K, ldS, fmt, res.job_lo, res.job_hi, st, splits, simt)
            res.n_d = torch.empty(res.count, dtype=torch.int64, device=self.device)
            res.n3 = torch.empty(res.count, dtype=torch.int64, device=self.device)
            _lib.call("tb_full_counts", _ptr(res.numerator), _ptr(absdot), _ptr(res.n1_rows), m, n,
                      res.job_lo, res.job_hi, _ptr(res.n_d), _ptr(res.n3), st)

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
                       h2d_piece_bytes: int = 4 << 20) -> PairResult:
        """End-to-end from host buffers: H2D of the values, the device path, tau_b back to host.

        The job range is cut into row bands; band i's tau_b copy (on ``copy_stream``) overlaps
        band i+1's numerator kernel.  ``x_host`` and ``tau_b_out`` should be pinned; the call is
        asynchronous on ``stream`` (which finally waits for the copies).
        """
        st_t = stream if stream is not None else torch.cuda.current_stream()
        cp_t = copy_stream if copy_stream is not None else self._copy_stream()
        m, n = x_host.shape
        total = m * (m + 1) // 2
        if tau_b_out.numel() < total:
            raise ConfigError(f"tau_b_out holds {tau_b_out.numel()} values, need {total}")
        path = self.choose_path(n) if kernel == "auto" else kernel
        st = _stream_ptr(st_t)
        self._events, self._stream = None, st_t
        if path == "merge" and x_host.dtype != torch.int32:
            raise InvalidInputError("the merge path takes dense int32 ranks (rank_transform output)")
        with torch.cuda.stream(st_t):
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
            res = PairResult(m=m, n=n, job_lo=0, job_hi=total, path=path,
                             numerator=self._buf("num_all", total, torch.int32),
                             n1_rows=torch.empty(m, dtype=torch.int64, device=self.device),
                             flags=torch.zeros(1, dtype=torch.int32, device=self.device))
            res.tau_b = self._buf("taub_all", total, torch.float64)
            if path == "gemm":
                S, K, ldS, fmt = self._gemm_prepare(
                    x, res, st, row_chunks=[(r0, r1, (lambda e=ev: st_t.wait_event(e))) for r0, r1, ev in chunks])
            else:
                for _, _, ev in chunks:
                    st_t.wait_event(ev)
                pos, srt, keys, maxgrp = self._merge_prepare(x, res, st)
            if band_fracs is None:
                band_fracs = self.default_band_fracs(total)
            cuts = self.bands(m, len(band_fracs), fracs=band_fracs)
            for r0, r1 in zip(cuts[:-1], cuts[1:]):
                lo, hi = r0 * (2 * m - r0 + 1) // 2, r1 * (2 * m - r1 + 1) // 2
                num = res.numerator[lo:hi]
                if path == "gemm":
                    self._gemm_numerator(S, num, m, K, ldS, fmt, lo, hi, st)
                else:
                    _lib.call("tb_merge_pairs", _ptr(keys), _ptr(pos), _ptr(srt), _ptr(res.n1_rows), _ptr(maxgrp[0]),
                              _ptr(maxgrp[1]), _ptr(maxgrp[2]), m, n, lo, hi, _ptr(num), None, None, st)
                tb = res.tau_b[lo:hi]
                _lib.call("tb_finalize", _ptr(num), _ptr(res.n1_rows), m, n, lo, hi, None, _ptr(tb), st)
                ev = torch.cuda.Event()
                ev.record(st_t)
                cp_t.wait_event(ev)
                with torch.cuda.stream(cp_t):
                    tau_b_out[lo:hi].copy_(tb, non_blocking=True)
            st_t.wait_stream(cp_t)
            res.launches = _lib.load().tb_launch_count() - c0
        return res

    def _copy_stream(self) -> torch.cuda.Stream:
        cs = getattr(self, "_cs", None)
        if cs is None:
            cs = torch.cuda.Stream(device=self.device)
            self._cs = cs
        return cs

    def _merge_prepare(self, x, res: PairResult, st):
        """K1 presort of every variable (u-order positions, sorted ranks, min-rank merge keys, n1,
        tie groups)."""
        m, n = res.m, res.n
        if x.dtype != torch.int32:
            raise InvalidInputError("the merge path takes dense int32 ranks (rank_transform output)")
        pos = self._buf("pos", m * n, torch.int32)
        srt = self._buf("sorted", m * n, torch.int32)
        keys = self._buf("mkeys", m * n, torch.int16)
        work = self._buf("work", m * n, torch.int32)
        maxgrp = self._buf("maxgrp", m, torch.int32)
        ngroups = self._buf("ngroups", m, torch.int32)
        _lib.call("tb_presort", _ptr(x), m, n, _ptr(pos), _ptr(srt), _ptr(keys), _ptr(res.n1_rows),
                  _ptr(maxgrp), _ptr(work), _ptr(ngroups), _ptr(res.flags), st)
        return pos, srt, keys, (maxgrp, work, ngroups)

    def _merge_path(self, x, res: PairResult, st):
        m, n = res.m, res.n
        x = x.contiguous()
        pos, srt, keys, (maxgrp, groups, ngroups) = self._merge_prepare(x, res, st)
        res.n_d = torch.empty(res.count, dtype=torch.int64, device=self.device)
        res.n3 = torch.empty(res.count, dtype=torch.int64, device=self.device)
        self._mark(0)
        _lib.call("tb_merge_pairs", _ptr(keys), _ptr(pos), _ptr(srt), _ptr(res.n1_rows), _ptr(maxgrp), _ptr(groups),
                  _ptr(ngroups), m, n,
                  res.job_lo, res.job_hi, _ptr(res.numerator), _ptr(res.n_d), _ptr(res.n3), st)
        self._mark(1)


_ENGINES: dict[int, TauEngine] = {}


def get_engine(device: int | None = None) -> TauEngine:
    idx = torch.cuda.current_device() if device is None else int(device)
    eng = _ENGINES.get(idx)
    if eng is None:
        eng = TauEngine(idx)
        _ENGINES[idx] = eng
    return eng
