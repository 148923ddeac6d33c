"""Multi-GPU plumbing: one process per GPU, contiguous job-id shards, banded gather to one consumer.

Every pair is independent, so ranks never exchange data while computing: rank r of p computes a
contiguous job-id range (the reference's contiguous shard rule, pairindex.py:68-80, applied to job ids;
PAPER.md:538), and the shards concatenate to the full job-id stream.  The only collective is the gather
of result bands (tau_b) to one consumer rank, pipelined with the compute:

* ``balanced_job_shards`` cuts the job range so every rank's *cost* is equal, not just its pair count:
  on the GEMM path a shard also sign-packs every row from its first one to m, so early shards do more
  packing per pair (cost model: pairs + ROW_COST_PAIRS x rows packed).
* ``shard_bands`` splits a shard into row-aligned bands of equal pair counts; a rank finishes band b,
  then hands it to ``BandGather.band``: point-to-point sends to the consumer (NCCL over NVLink on a B200
  box: ncclSend/ncclRecv grouped per band; gloo in the CPU tests), issued right after the band's
  finalize on the compute stream, so band b crosses NVLink while band b+1 is computed.  The consumer
  posts the matching receives into its full-size output.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

from .pairindex import job_shard_range

# Cost model of one rank's shard on the GEMM path, in units of one pair's GEMM time: every pair costs 1
# (one-GPU timings of row-block-aligned config-5 shards: 0.19-0.21 ns per pair whatever the rows, within
# the run-to-run noise, profiles/r02_strong_scaling_projection.log -- the width dependence seen before the
# alignment was the duplicated boundary row blocks), and every row the shard sign-packs (all rows from its
# first one to m) costs ROW_PACK_COST pairs (K2: 42 ns per 1024-sample row against 0.196 ns per pair).
ROW_WIDTH_COST = 0.0
ROW_PACK_COST = float(os.environ.get("TB_ROW_PACK_COST", "214"))


def _row_prefix(y: int, m: int) -> int:
    return y * (2 * m - y + 1) // 2


def _row_of(j: int, m: int) -> int:
    """Row of job id j (integer bisection; exact for any m)."""
    lo, hi = 0, m - 1
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if _row_prefix(mid, m) <= j:
            lo = mid
        else:
            hi = mid - 1
    return lo


def _weighted_rows(y0: int, y1: int, m: int) -> float:
    """sum over full rows y in [y0, y1) of w (1 + ROW_WIDTH_COST w / m), w = m - y (closed form)."""
    if y1 <= y0:
        return 0.0
    a, b = m - y1 + 1, m - y0  # widths a..b

    def s1(k):
        return k * (k + 1) / 2

    def s2(k):
        return k * (k + 1) * (2 * k + 1) / 6
    return (s1(b) - s1(a - 1)) + ROW_WIDTH_COST / m * (s2(b) - s2(a - 1))


def shard_cost(lo: int, hi: int, m: int, path: str = "gemm") -> float:
    """Modelled cost of job ids [lo, hi) (GEMM path: width-weighted pairs + sign-pack rows; merge: pairs)."""
    if hi <= lo:
        return 0.0
    if path != "gemm":
        return float(hi - lo)
    y0, y1 = _row_of(lo, m), _row_of(hi - 1, m)
    wt = lambda y: 1.0 + ROW_WIDTH_COST * (m - y) / m  # noqa: E731
    if y0 == y1:
        c = (hi - lo) * wt(y0)
    else:
        c = (_row_prefix(y0 + 1, m) - lo) * wt(y0) + _weighted_rows(y0 + 1, y1, m) + (hi - _row_prefix(y1, m)) * wt(y1)
    return c + ROW_PACK_COST * (m - y0)


GEMM_ROW_BLOCK = 256  # the GEMM's unit height: a job range that cuts a row block computes all of it


def balanced_job_shards(world: int, m: int, path: str = "gemm", align: int | None = None) -> list[tuple[int, int]]:
    """Contiguous job-id shards of equal modelled cost covering [0, m(m+1)/2) (bisection on the per-shard
    cost target; the merge path's cost is its pair count, i.e. job_shard_range).  On the GEMM path the
    boundaries are row-block starts (``align`` rows, default the GEMM's 256 when m is large enough): a
    boundary inside a row block would make both neighbouring shards run that block's full units."""
    total = m * (m + 1) // 2
    if world < 1:
        raise ValueError("world must be >= 1")
    if path != "gemm" or world == 1:
        return [job_shard_range(r, world, m) for r in range(world)]
    if align is None:
        align = GEMM_ROW_BLOCK if m >= 8 * GEMM_ROW_BLOCK * world else 1
    cand = [_row_prefix(y, m) for y in range(0, m, align)] + [total] if align > 1 else None

    def largest_hi(lo: int, target: float) -> int:
        if cand is None:
            a, b = lo, total
            while a < b:
                mid = (a + b + 1) // 2
                if shard_cost(lo, mid, m, path) <= target:
                    a = mid
                else:
                    b = mid - 1
            return a
        import bisect
        i0 = bisect.bisect_left(cand, lo)
        a, b = i0, len(cand) - 1
        while a < b:
            mid = (a + b + 1) // 2
            if shard_cost(lo, cand[mid], m, path) <= target:
                a = mid
            else:
                b = mid - 1
        return cand[a]

    def cut(target: float):
        bounds, lo = [0], 0
        for _ in range(world - 1):
            lo = largest_hi(lo, target)
            bounds.append(lo)
        bounds.append(total)
        return bounds

    t_lo, t_hi = 0.0, shard_cost(0, total, m, path)
    for _ in range(200):
        t = 0.5 * (t_lo + t_hi)
        b = cut(t)
        if shard_cost(b[-2], b[-1], m, path) <= t:
            t_hi = t
        else:
            t_lo = t
        if t_hi - t_lo < 1.0:
            break
    b = cut(t_hi)
    return list(zip(b[:-1], b[1:]))


def gather_band_fracs(nbands: int, ratio: float = 0.5) -> tuple:
    """Shares of a shard's pairs per band for the banded gather: geometrically shrinking (ratio 0.5), so
    the last band -- whose transfer to the consumer is the only part not hidden behind compute -- is
    small while the first bands stay large enough for efficient GEMM launches."""
    if nbands <= 1:
        return (1.0,)
    w = [ratio ** i for i in range(nbands)]
    return tuple(x / sum(w) for x in w)


def shard_bands(lo: int, hi: int, m: int, nbands: int, fracs: tuple | None = None,
                align: int = GEMM_ROW_BLOCK) -> list[tuple[int, int]]:
    """[lo, hi) split into <= nbands contiguous sub-ranges holding the given shares of its pairs (default:
    equal), cut at row starts -- row-block starts (multiples of ``align``) when the range spans enough of
    them, so no GEMM row block is split between two launches."""
    if hi <= lo:
        return []
    if fracs is None:
        fracs = (1.0 / nbands,) * nbands
    y_lo, y_hi = _row_of(lo, m), _row_of(hi - 1, m)
    if y_hi - y_lo < 4 * align * nbands:
        align = 1
    cuts, acc = [lo], 0.0
    for fr in fracs[:-1]:
        acc += fr
        j = lo + int((hi - lo) * min(acc, 1.0))
        y = _row_of(j, m)
        if align > 1:
            y = (y + align // 2) // align * align
        r = _row_prefix(min(y, m - 1), m)
        j = r if r > cuts[-1] else j
        if cuts[-1] < j < hi:
            cuts.append(j)
    cuts.append(hi)
    return list(zip(cuts[:-1], cuts[1:]))


def my_job_range(m: int, rank: int | None = None, world: int | None = None) -> tuple[int, int]:
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    return job_shard_range(rank, world, m)


class BandGather:
    """Stream every rank's shard bands to ``dst`` as they finish.

    All ranks know every rank's shard and band plan (deterministic), so the consumer posts exactly the
    matching receives: for band b, one receive per other rank into ``out[band]`` (job-id offsets).  On
    NCCL the sends / receives of one band are one grouped launch (batch_isend_irecv) that waits for the
    band's finalize on the current stream and runs on the communicator's stream, overlapping the next
    band's kernels; ``finish()`` makes the current stream wait for all of them.  ``host_staging`` copies
    device bands through host memory (gloo plumbing runs)."""

    def __init__(self, shards: list[tuple[int, int]], m: int, nbands: int, out: torch.Tensor | None = None,
                 dst: int = 0, group=None, host_staging: bool = False, fracs: tuple | None = None):
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if len(shards) != self.world:
            raise ValueError(f"{len(shards)} shards for {self.world} ranks")
        self.shards, self.m, self.dst, self.group = shards, m, dst, group
        self.bands = [shard_bands(lo, hi, m, nbands, fracs) for lo, hi in shards]
        self.nb = max(len(b) for b in self.bands)
        self.out = out
        self.host = host_staging
        self.works: list = []
        self._keep: list = []
        self._pending: list = []
        self._nccl = dist.get_backend(group) == "nccl"
        self._next = 0  # next band index this rank ships (the consumer posts receives up to nb in finish)
        if self.rank == dst and out is None:
            raise ValueError("the consumer rank needs an output tensor")

    def band(self, b: int, local: torch.Tensor) -> None:
        """Rank's band b (job ids self.bands[rank][b]) is finished on the current stream: ship it."""
        ops = []
        self._next = b + 1
        if self.rank == self.dst:
            if local is not None and b < len(self.bands[self.rank]):
                blo, bhi = self.bands[self.rank][b]
                dst_view = self.out[blo:bhi]
                if local.data_ptr() != dst_view.data_ptr():
                    dst_view.copy_(local, non_blocking=True)
            for r in range(self.world):
                if r == self.rank or b >= len(self.bands[r]):
                    continue
                blo, bhi = self.bands[r][b]
                view = self.out[blo:bhi]
                if self.host:
                    buf = torch.empty(bhi - blo, dtype=self.out.dtype)
                    self._pending.append((view, buf))
                    view = buf
                ops.append(dist.P2POp(dist.irecv, view, r, self.group))
        elif b < len(self.bands[self.rank]):
            t = local
            if self.host:
                t = local.cpu()
                self._keep.append(t)
            ops.append(dist.P2POp(dist.isend, t, self.dst, self.group))
        if not ops:
            return
        if self._nccl:
            self.works.extend(dist.batch_isend_irecv(ops))
        else:
            for op in ops:
                self.works.append(op.op(op.tensor, op.peer, op.group))

    def finish(self) -> None:
        """Post the consumer's receives for bands it had none of its own for, then make the current
        stream (NCCL) / the host (gloo) wait for every transfer."""
        if self.rank == self.dst:
            for b in range(self._next, self.nb):
                self.band(b, None)
        self._next = 0
        for w in self.works:
            w.wait()
        for view, buf in self._pending:
            view.copy_(buf)
        self.works, self._keep, self._pending = [], [], []


def gather_shards(local: torch.Tensor, m: int, dst: int = 0, group=None) -> torch.Tensor | None:
    """Concatenate every rank's job_shard_range shard on rank ``dst`` (None elsewhere): one
    all_gather_into_tensor of equal padded chunks (the simple, un-pipelined form of BandGather)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    total = m * (m + 1) // 2
    chunk = -(-total // world)
    lo, hi = job_shard_range(rank, world, m)
    if local.numel() != hi - lo:
        raise ValueError(f"rank {rank}: shard has {local.numel()} entries, expected {hi - lo}")
    padded = torch.zeros(chunk, dtype=local.dtype, device=local.device)
    padded[: local.numel()] = local
    out = torch.empty(chunk * world, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    if rank != dst:
        return None
    parts = []
    for r in range(world):
        a, b = job_shard_range(r, world, m)
        parts.append(out[r * chunk: r * chunk + (b - a)])
    return torch.cat(parts)
