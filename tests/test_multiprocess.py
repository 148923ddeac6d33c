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
