"""World-size-2 gloo test of the multi-GPU host logic on CPU: job-range shards
computed independently per rank (the oracle stands in for the device compute)
gather to exactly the single-process result."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, n, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    import oracle as orc
    from paper_1704_03767_b200.multi import gather_shards, my_job_range

    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    ranks = np.stack([orc.rank_transform(rng.integers(0, n // 2, n)) for _ in range(m)])
    lo, hi = my_job_range(m)
    pi, pj = orc.upper_pairs(m)
    num, _ = orc.all_pairs(ranks, pi[lo:hi], pj[lo:hi], orc.KERNEL_SORTED, threads=1, want_counts=False)
    full = gather_shards(torch.from_numpy(num), m)
    if rank == 0:
        ref, _ = orc.all_pairs(ranks, pi, pj, orc.KERNEL_SORTED, threads=2, want_counts=False)
        np.save(out_path, np.stack([full.numpy(), ref]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [1, 7, 40])
def test_gloo_two_rank_shards_gather(tmp_path, m):
    out = str(tmp_path / "res.npy")
    port = _free_port()
    mp.spawn(_worker, args=(2, port, m, 33, out), nprocs=2, join=True)
    got, ref = np.load(out)
    np.testing.assert_array_equal(got, ref)


def _band_worker(rank, world, port, m, nbands, out_path):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    from paper_1704_03767_b200.multi import BandGather, balanced_job_shards, shard_bands

    dist.init_process_group("gloo", rank=rank, world_size=world)
    shards = balanced_job_shards(world, m, "gemm")
    lo, hi = shards[rank]
    total = m * (m + 1) // 2
    out = torch.full((total,), -1.0, dtype=torch.float64) if rank == 0 else None
    local = out[lo:hi] if rank == 0 else torch.empty(hi - lo, dtype=torch.float64)
    from paper_1704_03767_b200.multi import gather_band_fracs
    fr = gather_band_fracs(nbands)
    g = BandGather(shards, m, nbands, out=out, fracs=fr)
    for step in range(2):  # the gather object is reused across steps
        for b, (blo, bhi) in enumerate(shard_bands(lo, hi, m, nbands, fr)):
            # "compute" band b: job id j -> j + 0.5 * step (what the device finalize would write)
            local[blo - lo:bhi - lo] = torch.arange(blo, bhi, dtype=torch.float64) + 0.5 * step
            g.band(b, local[blo - lo:bhi - lo])
        g.finish()
        if rank == 0:
            ok = torch.equal(out, torch.arange(total, dtype=torch.float64) + 0.5 * step)
            np.save(out_path + f".{step}.npy", np.array([ok]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,nbands", [(2, 1, 3), (2, 40, 4), (3, 300, 5), (4, 7, 8)])
def test_gloo_banded_gather(tmp_path, world, m, nbands):
    """BandGather over gloo (world 2-4): every rank ships its shard's bands as they finish, the consumer
    assembles the full job-id stream, also when ranks have different band counts (tiny shards)."""
    out = str(tmp_path / "ok")
    mp.spawn(_band_worker, args=(world, _free_port(), m, nbands, out), nprocs=world, join=True)
    for step in range(2):
        assert bool(np.load(out + f".{step}.npy")[0])


def test_balanced_shards_partition_and_balance():
    from paper_1704_03767_b200.multi import balanced_job_shards, shard_bands, shard_cost
    for m in (1, 5, 300, 65536):
        total = m * (m + 1) // 2
        for world in (1, 2, 3, 8):
            for path in ("gemm", "merge"):
                sh = balanced_job_shards(world, m, path)
                assert len(sh) == world and sh[0][0] == 0 and sh[-1][1] == total
                assert all(a[1] == b[0] for a, b in zip(sh, sh[1:])) and all(lo <= hi for lo, hi in sh)
                for lo, hi in sh:
                    bands = shard_bands(lo, hi, m, 4)
                    assert (not bands and lo == hi) or (bands[0][0] == lo and bands[-1][1] == hi)
                    assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(bands, bands[1:]))
    from paper_1704_03767_b200.multi import _row_of, _row_prefix, gather_band_fracs
    sh = balanced_job_shards(8, 65536, "gemm", align=1)
    costs = [shard_cost(lo, hi, 65536) for lo, hi in sh]
    assert max(costs) / min(costs) < 1.001
    assert sh[0][1] - sh[0][0] < sh[-1][1] - sh[-1][0]  # early shards pack more rows: fewer pairs
    # default: boundaries at GEMM row-block starts (no row block split between two shards or two bands)
    sh = balanced_job_shards(8, 65536, "gemm")
    costs = [shard_cost(lo, hi, 65536) for lo, hi in sh]
    assert max(costs) / min(costs) < 1.06
    for lo, hi in sh:
        y = _row_of(lo, 65536)
        assert y % 256 == 0 and _row_prefix(y, 65536) == lo
        for a, _ in shard_bands(lo, hi, 65536, 3, gather_band_fracs(3)):
            ya = _row_of(a, 65536)
            assert ya % 256 == 0 and _row_prefix(ya, 65536) == a
