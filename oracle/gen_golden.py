"""Generate tests/golden/ fixtures by running the REFERENCE package itself.

Run in the dev container only (needs /root/reference and numba):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden.py

Nothing at test/bench time reads /root/reference; the fixtures written here
are the committed pins for both the CPU oracle (oracle/) and the GPU path.
Every fixture names the reference function that produced it.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = os.path.join(ROOT, "tests", "golden")

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, ROOT)

import taucorr  # noqa: E402  (the reference)
from taucorr.kernel_sorted import sorted_counts  # noqa: E402
from taucorr.kernel_vectorized import vectorized_counts, LANE_WIDTH  # noqa: E402
from conftest import brute_reference, random_rank_pair  # noqa: E402  (reference test helpers)

from paper_1704_03767_b200 import workloads  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_counts(u, v):
    n = u.shape[0]
    u = np.ascontiguousarray(u, np.int32)
    v = np.ascontiguousarray(v, np.int32)
    if n <= 32767 and u.max() < 1 << 15 and v.max() < 1 << 15:
        pa, pb = np.empty(n, np.int32), np.empty(n, np.int32)
        la, lb = np.empty(LANE_WIDTH, np.int32), np.empty(LANE_WIDTH, np.int32)
        nd, n1, n2, n3 = vectorized_counts(u, v, pa, pb, la, lb, True)
    else:
        s = [np.empty(n, np.int32) for _ in range(4)]
        nd, n1, n2, n3 = sorted_counts(u, v, *s)
    r = taucorr.result_from_counts(n, int(nd), int(n1), int(n2), int(n3))
    return r


def gen_kats():
    out = {}
    r = taucorr.tau_b_sorted([1, 1, 2], [1, 2, 2])
    out["tied_example"] = dict(u=[1, 1, 2], v=[1, 2, 2], n0=r.n0, n1=r.n1, n2=r.n2, n3=r.n3,
                               n_d=r.n_d, numerator=r.numerator, tau_b=r.tau_b, tau_a=r.tau_a)
    r = taucorr.tau_b_sorted([0, 1, 2, 3], [3, 2, 1, 0])
    out["reversal4"] = dict(u=[0, 1, 2, 3], v=[3, 2, 1, 0], n_d=r.n_d, numerator=r.numerator,
                            tau_a=r.tau_a, tau_b=r.tau_b)
    r = taucorr.tau_b_sorted([0, 1, 2, 3], [0, 1, 2, 3])
    out["identity4"] = dict(u=[0, 1, 2, 3], v=[0, 1, 2, 3], n_d=r.n_d, numerator=r.numerator,
                            tau_a=r.tau_a, tau_b=r.tau_b)
    r = taucorr.tau_a_naive([0, 1, 2], [0, 2, 1])
    out["third"] = dict(u=[0, 1, 2], v=[0, 2, 1], numerator=r.numerator, tau_a=r.tau_a)
    r = taucorr.tau_b_sorted([4, 4, 4, 4], [0, 1, 2, 3])
    out["constant"] = dict(u=[4, 4, 4, 4], v=[0, 1, 2, 3], defined_b=r.defined_b,
                           numerator=r.numerator, n1=r.n1, n_d=r.n_d)
    out["tie_sum"] = [[[1, 1, 2, 2, 2], taucorr.tie_sum([1, 1, 2, 2, 2])],
                      [[5, 5, 5, 5], taucorr.tie_sum([5, 5, 5, 5])]]
    out["joint_tie_sum"] = [[[3, 3, 3], [3, 3, 3], taucorr.joint_tie_sum([3, 3, 3], [3, 3, 3])]]
    out["count_discordant"] = [[[0, 1, 2], [0, 2, 1], taucorr.count_discordant([0, 1, 2], [0, 2, 1])[0]],
                               [[0, 1, 2, 3], [3, 2, 1, 0],
                                taucorr.count_discordant([0, 1, 2, 3], [3, 2, 1, 0])[0]]]
    rt_cases = [[3.2, 1.1, 3.2, 5.0], [0.0, -0.0, 1.0, -1.0], [float("inf"), -float("inf"), 0.0, 2.0, 2.0],
                [7, 7, 7], [2, 0, 1]]
    out["rank_transform"] = [[c, taucorr.rank_transform(np.array(c)).tolist()] for c in rt_cases]
    out["bijection"] = dict(
        job_id_2_3_4=taucorr.job_id(2, 3, 4),
        job_coord_5_4=list(taucorr.job_coord(5, 4)),
        tile_id_1_2_3=taucorr.tile_id(1, 2, 3),
        shard_ranges=[[m, q, p, [list(taucorr.shard_range(i, p, taucorr.JobSpace(m, q))) for i in range(p)]]
                      for (m, q, p) in [(21, 4, 3), (3, 8, 5), (100, 8, 7), (1000, 16, 8)]],
    )
    with open(os.path.join(GOLD, "kats.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def gen_corpus():
    """test_acceptance.py:44-52 corpus (seed 20240512) + boundary (seed 77, :74-100)."""
    rng = np.random.default_rng(20240512)
    ties = (0.0, 0.3, 0.9)
    ns, us, vs, cnt, brute = [], [], [], [], []
    for k in range(1000):
        n = int(rng.integers(2, 513))
        u, v = random_rank_pair(rng, n, ties[k % 3])
        r = taucorr.tau_b_sorted(u, v)
        b = brute_reference(u, v)
        ns.append(n)
        us.append(u)
        vs.append(v)
        cnt.append([r.n_d, r.n1, r.n2, r.n3, r.numerator])
        brute.append([b.nc, b.n_d, b.n1, b.n2, b.n3])
        assert (r.n_d, r.n1, r.n2, r.n3, r.numerator) == (b.n_d, b.n1, b.n2, b.n3, b.numerator)
    taus = [taucorr.tau_b_sorted(u, v) for u, v in zip(us, vs)]
    np.savez_compressed(
        os.path.join(GOLD, "corpus.npz"),
        n=np.array(ns, np.int64), u=np.concatenate(us).astype(np.int16), v=np.concatenate(vs).astype(np.int16),
        counts=np.array(cnt, np.int64), brute=np.array(brute, np.int64),
        tau_a=np.array([t.tau_a for t in taus]), tau_b=np.array([t.tau_b for t in taus]),
        source=np.array("taucorr.tau_b_sorted + conftest.brute_reference, rng 20240512"),
    )
    rng = np.random.default_rng(77)
    ns, us, vs, cnt, ta, tb = [], [], [], [], [], []
    for n in (15, 16, 17, 31, 32, 33, 32767):
        for tie in (0.0, 0.3, 0.9):
            u, v = random_rank_pair(rng, n, tie)
            r = taucorr.tau_b_sorted(u, v)
            rv = taucorr.tau_b_vectorized(u, v)
            assert (r.n_d, r.n1, r.n2, r.n3) == (rv.n_d, rv.n1, rv.n2, rv.n3)
            ns.append(n)
            us.append(u)
            vs.append(v)
            cnt.append([r.n_d, r.n1, r.n2, r.n3, r.numerator])
            ta.append(r.tau_a)
            tb.append(r.tau_b)
    np.savez_compressed(
        os.path.join(GOLD, "boundary.npz"),
        n=np.array(ns, np.int64), u=np.concatenate(us).astype(np.int16), v=np.concatenate(vs).astype(np.int16),
        counts=np.array(cnt, np.int64), tau_a=np.array(ta), tau_b=np.array(tb),
        source=np.array("taucorr.tau_b_sorted == tau_b_vectorized, rng 77, test_acceptance.py:85"),
    )


def gen_configs():
    """Sampled reference counts for each BASELINE config (SURVEY 8(d) generators)."""
    plan = {1: None, 2: 3000, 3: 1500, 4: 120, 5: 1500}
    for k, count in plan.items():
        t0 = time.time()
        x = workloads.generate(k)
        spec = workloads.CONFIGS[k]
        ranks = np.empty(x.shape, np.int32)
        for r in range(x.shape[0]):
            ranks[r] = taucorr.rank_transform(x[r])
        n = x.shape[1]
        if count is None:
            # full run through the reference engine (records in tile order, q=8)
            ds = taucorr.Dataset(labels=[f"V{i}" for i in range(x.shape[0])], ranks=ranks)
            chunks = []
            taucorr.compute_all_pairs(ds, "vectorized", workers=8, tile_size=8,
                                      sink=lambda rec: chunks.append(rec.copy()))
            rec = np.sort(np.concatenate(chunks), order=["i", "j"])
            pi = rec["i"].astype(np.int64)
            pj = rec["j"].astype(np.int64)
            counts = np.stack([rec["n_d"], rec["n1"], rec["n2"], rec["n3"]], 1).astype(np.int64)
            num = rec["numerator"].astype(np.int64)
            ta, tb = taucorr.derive_taus(rec["numerator"], rec["n1"], rec["n2"], n)
        else:
            pi, pj = workloads.sample_pairs(spec.m, count, seed=1000 + k)
            if k == 4:
                # correlated row 0 vs every 8th row, plus pairs inside the correlated family
                extra_i = np.array([0] * 8 + [8, 16, 504], np.int64)
                extra_j = np.array([8, 16, 24, 512, 1016, 1, 2, 3, 16, 1016, 1016], np.int64)
                pi = np.concatenate([extra_i, pi])
                pj = np.concatenate([extra_j, pj])
            counts, num, ta, tb = [], [], [], []
            for i, j in zip(pi.tolist(), pj.tolist()):
                r = ref_counts(ranks[i], ranks[j])
                counts.append([r.n_d, r.n1, r.n2, r.n3])
                num.append(r.numerator)
                ta.append(r.tau_a)
                tb.append(r.tau_b)
            counts = np.array(counts, np.int64)
            num = np.array(num, np.int64)
            ta = np.array(ta)
            tb = np.array(tb)
        n1_rows = np.array([taucorr.tie_sum(np.sort(ranks[r])) for r in range(ranks.shape[0])], np.int64)
        np.savez_compressed(
            os.path.join(GOLD, f"config{k}.npz"),
            x_sha256=np.array(sha(x)), ranks_sha256=np.array(sha(ranks)),
            m=np.int64(x.shape[0]), n=np.int64(n), pi=pi, pj=pj,
            counts=counts, numerator=num, tau_a=ta, tau_b=tb, n1_rows=n1_rows,
            ranks_head=ranks[:4].astype(np.int32),
            source=np.array("taucorr rank_transform + vectorized_counts/sorted_counts "
                            "(config1: compute_all_pairs full) on workloads.generate(k)"),
        )
        print(f"config {k}: {len(pi)} pairs in {time.time() - t0:.1f}s", flush=True)


def gen_engine():
    """BinaryWriter byte streams (test_acceptance.py:281-331, test_engine.py)."""
    out = {}
    for (m, n, tie, seed) in [(64, 48, 0.3, 512), (13, 10, 0.2, 1), (512, 48, 0.3, 512)]:
        ds = taucorr.synth_dataset(m, n, tie_fraction=tie, seed=seed)
        for q in (1, 3, 4, 8):
            s = io.BytesIO()
            taucorr.compute_all_pairs(ds, "sorted", workers=1, tile_size=q, pass_tiles=4096,
                                      sink=taucorr.BinaryWriter(s, ds.n))
            blob = s.getvalue()
            key = f"m{m}_n{n}_t{tie}_s{seed}_q{q}"
            out[key] = hashlib.sha256(blob).hexdigest()
            if m <= 64 and q == 4:
                with open(os.path.join(GOLD, f"stream_{key}.bin"), "wb") as fh:
                    fh.write(blob)
            if m == 512 and q == 4:
                parts = b"".join(
                    (lambda s2: (taucorr.compute_all_pairs(
                        ds, "sorted", workers=2, tile_size=4, shard=(i, 4),
                        sink=taucorr.BinaryWriter(s2, ds.n)), s2.getvalue())[1])(io.BytesIO())
                    for i in range(4))
                assert parts == blob
        ranks = taucorr.synth_dataset(m, n, tie_fraction=tie, seed=seed).ranks
        out[f"synth_m{m}_n{n}_t{tie}_s{seed}_sha256"] = sha(ranks)
    # TSV lines for a small run
    ds = taucorr.synth_dataset(6, 9, tie_fraction=0.4, seed=12)
    s = io.StringIO()
    taucorr.compute_all_pairs(ds, "sorted", tile_size=2, sink=taucorr.TsvWriter(s, ds.labels, ds.n))
    out["tsv_m6_n9_t0.4_s12_q2"] = s.getvalue()
    with open(os.path.join(GOLD, "engine_streams.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def gen_bijection():
    rng = np.random.default_rng(17941)
    res = {}
    for m in (17941, 10 ** 6, 65536, 2 ** 21 + 7):
        total = m * (m + 1) // 2
        js = np.concatenate([rng.integers(0, total, 2000), [0, total - 1, total // 2]]).astype(np.int64)
        yx = np.array([taucorr.job_coord(int(j), m) for j in js], np.int64)
        res[f"m{m}_j"] = js
        res[f"m{m}_yx"] = yx
    np.savez_compressed(os.path.join(GOLD, "bijection.npz"), **res)


if __name__ == "__main__":
    os.makedirs(GOLD, exist_ok=True)
    which = sys.argv[1:] or ["kats", "corpus", "bijection", "engine", "configs"]
    for w in which:
        t0 = time.time()
        globals()[f"gen_{w}"]()
        print(f"{w}: {time.time() - t0:.1f}s", flush=True)
