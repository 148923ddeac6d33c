"""GPU parity: the sm_100a path through the C ABI vs the oracle and the reference's golden vectors.

Integers (numerator, n_d, n1, n2, n3) must match bit-exactly; tau_a / tau_b are
compared with assert_array_equal (the IEEE finalize is bit-identical to the
reference's derive_taus -- the north-star tolerance is 1e-12 absolute, and the
tests assert the stronger 0-ulp bound, NaN where the reference has NaN).
"""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from conftest import load_json, load_npz, random_rank_pair, split_pairs

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

TAU_ATOL = 1e-12  # north-star tolerance; the asserts below are exact


@pytest.fixture(scope="module")
def eng():
    from paper_1704_03767_b200.device import TauEngine
    return TauEngine(0)


def _full_oracle(oracle, ranks, kernel=None):
    m, n = ranks.shape
    pi, pj = oracle.upper_pairs(m)
    k = oracle.KERNEL_SORTED if kernel is None else kernel
    num, counts = oracle.all_pairs(ranks, pi, pj, k, threads=8)
    return pi, pj, num, counts


def _check_full(res, oracle, ranks, full=True):
    n = ranks.shape[1]
    pi, pj, num, counts = _full_oracle(oracle, ranks)
    lo, hi = res.job_lo, res.job_hi
    got = res.numerator.cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(got, num[lo:hi])
    n1 = res.n1_rows.cpu().numpy()
    np.testing.assert_array_equal(n1[pi[lo:hi]], counts[lo:hi, 1])
    np.testing.assert_array_equal(n1[pj[lo:hi]], counts[lo:hi, 2])
    if full:
        np.testing.assert_array_equal(res.n_d.cpu().numpy(), counts[lo:hi, 0])
        np.testing.assert_array_equal(res.n3.cpu().numpy(), counts[lo:hi, 3])
    ta, tb = oracle.derive_taus(num[lo:hi], counts[lo:hi, 1], counts[lo:hi, 2], n)
    if res.tau_a is not None:
        np.testing.assert_array_equal(res.tau_a.cpu().numpy(), ta)
    if res.tau_b is not None:
        np.testing.assert_array_equal(res.tau_b.cpu().numpy(), tb)


@pytest.mark.parametrize("path", ["gemm", "merge"])
@pytest.mark.parametrize("m,n,tie", [(1, 5, 0.0), (2, 2, 0.0), (3, 17, 0.5), (37, 33, 0.3), (130, 64, 0.0),
                                     (257, 31, 0.9), (300, 130, 0.2)])
def test_small_shapes_vs_oracle(eng, oracle, path, m, n, tie):
    rng = np.random.default_rng(m * 1000 + n)
    ranks = np.stack([oracle.rank_transform(random_rank_pair(rng, n, tie)[0]) for _ in range(m)])
    res = eng.all_pairs(torch.from_numpy(ranks).cuda(), kernel=path, full_counts=True).validate()
    torch.cuda.synchronize()
    _check_full(res, oracle, ranks)


@pytest.mark.parametrize("path", ["gemm", "merge"])
def test_constant_rows_nan(eng, oracle, path):
    ranks = np.zeros((5, 40), np.int32)
    ranks[1] = np.arange(40)
    ranks[3] = np.arange(40)[::-1]
    res = eng.all_pairs(torch.from_numpy(ranks).cuda(), kernel=path, full_counts=True).validate()
    tb = res.tau_b.cpu().numpy()
    _check_full(res, oracle, ranks)
    assert math.isnan(tb[0])  # (0, 0): constant vs constant


def test_nan_rejected(eng):
    from paper_1704_03767_b200 import InvalidInputError
    x = torch.randn(4, 10, dtype=torch.float64, device="cuda")
    x[2, 3] = float("nan")
    with pytest.raises(InvalidInputError):
        eng.all_pairs(x, kernel="gemm").validate()


def test_non_dense_values_merge(eng):
    """The merge path ranks its input on the device (K0w), so any int32 / float values work -- as for the
    reference's kernels, which compare values (kernel_sorted.py:30-57): same counts as dense ranks."""
    x = torch.tensor([[0, 1, 7, 7, -3], [5, 1, 2, 2, 9]], dtype=torch.int32, device="cuda")
    d = torch.tensor([[1, 2, 3, 3, 0], [3, 0, 1, 1, 4]], dtype=torch.int32, device="cuda")
    a = eng.all_pairs(x, kernel="merge", full_counts=True).validate()
    b = eng.all_pairs(d, kernel="merge", full_counts=True).validate()
    for f in ("numerator", "n_d", "n3", "n1_rows", "tau_b"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f


def test_kats_device(oracle):
    import paper_1704_03767_b200 as tb
    k = load_json("kats.json")
    t = k["tied_example"]
    r = tb.tau_b_sorted(t["u"], t["v"])
    assert (r.n_d, r.n1, r.n2, r.n3, r.numerator) == (t["n_d"], t["n1"], t["n2"], t["n3"], t["numerator"])
    assert r.tau_b == t["tau_b"] == 0.5
    assert tb.tau_b_vectorized(t["u"], t["v"]).tau_b == 0.5
    r = tb.tau_b_sorted(k["reversal4"]["u"], k["reversal4"]["v"])
    assert r.n_d == 6 and r.numerator == -6 and r.tau_a == -1.0
    assert tb.tau_a_naive([0, 1, 2, 3], [0, 1, 2, 3]).tau_a == 1.0
    assert tb.tau_a_naive([0, 1, 2], [0, 2, 1]).numerator == 1
    c = tb.tau_b_sorted([4, 4, 4, 4], [0, 1, 2, 3])
    assert not c.defined_b and math.isnan(c.tau_b)
    with pytest.raises(tb.InvalidInputError):
        tb.tau_b_sorted([1, 2], [1])
    with pytest.raises(tb.InvalidInputError):
        tb.tau_b_sorted([1], [1])
    with pytest.raises(tb.CapacityExceededError):
        tb.tau_b_vectorized([0, 40000, 2], [0, 1, 2])


def test_corpus_device_vs_reference():
    """The reference acceptance corpus (1,000 pairs, rng 20240512), per-pair device API."""
    import paper_1704_03767_b200 as tb
    z = load_npz("corpus.npz")
    for u, v, k in split_pairs(z):
        r = tb.tau_b_sorted(u, v)
        assert (r.n_d, r.n1, r.n2, r.n3, r.numerator) == tuple(z["counts"][k]), k
        assert r.tau_a == z["tau_a"][k]
        assert (math.isnan(r.tau_b) and math.isnan(z["tau_b"][k])) or r.tau_b == z["tau_b"][k]


def test_boundary_device_vs_reference(eng):
    """Boundary n in {15,16,17,31,32,33,32767} with ties, both device paths."""
    z = load_npz("boundary.npz")
    for u, v, k in split_pairs(z):
        x = torch.from_numpy(np.stack([u, v])).cuda()
        for path in ("merge", "gemm") if len(u) <= 4096 else ("merge",):
            res = eng.all_pairs(x, kernel=path, job_range=(1, 2), full_counts=True).validate()
            n1 = res.n1_rows.cpu().tolist()
            got = (int(res.n_d.item()), n1[0], n1[1], int(res.n3.item()), int(res.numerator.item()))
            assert got == tuple(z["counts"][k]), (path, len(u), k)
            assert res.tau_a.item() == z["tau_a"][k]


def _sampled_check(res, z, n):
    pi, pj = z["pi"], z["pj"]
    jid = pi * (2 * res.m - pi + 1) // 2 + pj - pi - res.job_lo
    idx = torch.from_numpy(jid).cuda()
    num = res.numerator.index_select(0, idx).cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(num, z["numerator"])
    n1 = res.n1_rows.cpu().numpy()
    np.testing.assert_array_equal(n1[pi], z["counts"][:, 1])
    np.testing.assert_array_equal(n1[pj], z["counts"][:, 2])
    if res.n_d is not None:
        np.testing.assert_array_equal(res.n_d.index_select(0, idx).cpu().numpy(), z["counts"][:, 0])
        np.testing.assert_array_equal(res.n3.index_select(0, idx).cpu().numpy(), z["counts"][:, 3])
    ta = res.tau_a.index_select(0, idx).cpu().numpy()
    tb = res.tau_b.index_select(0, idx).cpu().numpy()
    np.testing.assert_array_equal(ta, z["tau_a"])
    np.testing.assert_array_equal(tb, z["tau_b"])
    assert np.nanmax(np.abs(tb - z["tau_b"])) <= TAU_ATOL if len(tb) else True


def _diag_properties(res, n):
    """Size-independent: every diagonal cell has numerator n0 - n1 (n_d = 0, n3 = n1)."""
    m = res.m
    y = torch.arange(m, device="cuda", dtype=torch.int64)
    jd = y * (2 * m - y + 1) // 2 - res.job_lo
    ok = (jd >= 0) & (jd < res.count)
    n0 = n * (n - 1) // 2
    d = res.numerator.index_select(0, jd[ok]).to(torch.int64)
    assert torch.equal(d, n0 - res.n1_rows[ok])


@pytest.mark.parametrize("path", ["gemm", "merge"])
def test_config1_full(eng, oracle, path):
    """Config 1 (256 x 200 f64 N(0,1)): every cell vs the reference engine's records."""
    from paper_1704_03767_b200 import workloads
    z = load_npz("config1.npz")
    x = workloads.generate(1)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["x_sha256"])
    xin = torch.from_numpy(x).cuda() if path == "gemm" else torch.from_numpy(oracle.rank_matrix(x)).cuda()
    res = eng.all_pairs(xin, kernel=path, full_counts=True).validate()
    _sampled_check(res, z, 200)
    _diag_properties(res, 200)


@pytest.mark.timeout(600)
def test_config2_every_pair_vs_oracle(eng, oracle):
    """Config 2 (2048 x 1000, int 0..9): EVERY cell (2,098,176 job ids, SURVEY 8(d) parity protocol) vs
    the pinned oracle's packed/VSE counts -- numerator, n1, n2, n_d, n3 bit-exact, tau_a / tau_b 0 ulp --
    plus the reference's own golden pairs and the dp4a cross-check kernel."""
    from paper_1704_03767_b200 import workloads
    z = load_npz("config2.npz")
    x = workloads.generate(2)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["x_sha256"])
    xd = torch.from_numpy(x).cuda()
    res = eng.all_pairs(xd, kernel="gemm", full_counts=True).validate()
    _sampled_check(res, z, 1000)
    _diag_properties(res, 1000)
    ranks = oracle.rank_matrix(x)
    pi, pj = oracle.upper_pairs(x.shape[0])
    num, cnt = oracle.all_pairs(ranks, pi, pj, oracle.KERNEL_PACKED)
    np.testing.assert_array_equal(res.numerator.cpu().numpy().astype(np.int64), num)
    n1 = res.n1_rows.cpu().numpy()
    np.testing.assert_array_equal(n1[pi], cnt[:, 1])
    np.testing.assert_array_equal(n1[pj], cnt[:, 2])
    np.testing.assert_array_equal(res.n_d.cpu().numpy(), cnt[:, 0])
    np.testing.assert_array_equal(res.n3.cpu().numpy(), cnt[:, 3])
    ta, tb = oracle.derive_taus(num, cnt[:, 1], cnt[:, 2], 1000)
    np.testing.assert_array_equal(res.tau_a.cpu().numpy(), ta)
    np.testing.assert_array_equal(res.tau_b.cpu().numpy(), tb)
    assert np.nanmax(np.abs(res.tau_b.cpu().numpy() - tb)) <= TAU_ATOL
    ref = eng.all_pairs(xd, kernel="gemm", simt=True, tau_a=False, tau_b=False).validate()
    assert torch.equal(res.numerator, ref.numerator)


@pytest.mark.parametrize("splits", [1, 2, 7])
def test_gemm_splits_and_shards(eng, oracle, splits):
    """K-split counts and contiguous job-id shards concatenate to the full result."""
    from paper_1704_03767_b200.pairindex import job_shard_range
    rng = np.random.default_rng(splits)
    m, n = 600, 150
    x = torch.from_numpy(rng.standard_normal((m, n)).astype(np.float32)).cuda()
    full = eng.all_pairs(x, kernel="gemm", splits=splits).validate()
    parts = [eng.all_pairs(x, kernel="gemm", job_range=job_shard_range(i, 5, m), splits=splits).validate()
             for i in range(5)]
    assert torch.equal(torch.cat([p.numerator for p in parts]), full.numerator)
    assert torch.equal(torch.cat([p.tau_b for p in parts]), full.tau_b)
    ranks = oracle.rank_matrix(x.cpu().numpy())
    _check_full(full, oracle, ranks, full=False)


@pytest.mark.parametrize("n", [32769, 40000, 65535, 65536])
def test_merge_two_halves_vs_oracle(eng, oracle, n):
    """n > 32768 (two sorted halves, cross inversions from min-rank key sums + the tie scan of the
    first half): every pair of tie-heavy rows vs the reference's sorted_counts (kernel_sorted.py:195).
    Rows: 4 and 2 distinct values (runs crossing every thread boundary of the half, the large-group
    path), a constant row, ascending / descending permutations, ties only in the first half, a
    random permutation with a few pairs tied."""
    rng = np.random.default_rng(n)
    perm = rng.permutation(n)
    few = perm.copy()
    few[rng.integers(0, n, 40)] = few[rng.integers(0, n, 40)]
    head = np.arange(n)
    head[: n // 2] = rng.integers(0, 3, n // 2)
    rows = [rng.integers(0, 4, n), rng.integers(0, 2, n), np.zeros(n, np.int64), np.arange(n),
            np.arange(n)[::-1], head, few, rng.integers(0, 1000, n)]
    ranks = np.stack([oracle.rank_transform(r) for r in rows])
    m = ranks.shape[0]
    res = eng.all_pairs(torch.from_numpy(ranks).cuda(), kernel="merge", full_counts=True).validate()
    pi, pj = oracle.upper_pairs(m)
    got_nd = res.n_d.cpu().numpy()
    got_n3 = res.n3.cpu().numpy()
    got_num = res.numerator.cpu().numpy()
    for k, (i, j) in enumerate(zip(pi.tolist(), pj.tolist())):
        nd, n1, n2, n3 = oracle.sorted_counts(ranks[i], ranks[j])
        assert (int(got_nd[k]), int(got_n3[k])) == (nd, n3), (n, i, j)
        assert int(got_num[k]) == oracle.numerator_from_counts(n, nd, n1, n2, n3), (n, i, j)
    eng.release()


@pytest.mark.parametrize("n", [2047, 2048, 4097, 8193, 16384, 20000, 32767, 32768])
def test_merge_block_sizes_vs_oracle(eng, oracle, n):
    """One sorted block (n <= 32768) at every per-thread run length E = L / 1024 (2 .. 32): the
    register leaf, the checked merge levels (runs < 32 keys) and the look-ahead-slot levels, with
    tie-heavy, tie-free, monotone and constant rows, every pair vs sorted_counts (kernel_sorted.py:195)."""
    rng = np.random.default_rng(n + 7)
    rows = [rng.integers(0, 5, n), rng.permutation(n), np.arange(n)[::-1], rng.integers(0, n // 3, n),
            np.zeros(n, np.int64), rng.integers(0, 2, n)]
    ranks = np.stack([oracle.rank_transform(r) for r in rows])
    m = ranks.shape[0]
    res = eng.all_pairs(torch.from_numpy(ranks).cuda(), kernel="merge", full_counts=True).validate()
    pi, pj = oracle.upper_pairs(m)
    got_nd = res.n_d.cpu().numpy()
    got_n3 = res.n3.cpu().numpy()
    for k, (i, j) in enumerate(zip(pi.tolist(), pj.tolist())):
        nd, n1, n2, n3 = oracle.sorted_counts(ranks[i], ranks[j])
        assert (int(got_nd[k]), int(got_n3[k])) == (nd, n3), (n, i, j)


@pytest.mark.parametrize("n", [2048, 3001, 8193, 16384, 20000, 32768])
def test_merge_multi_pair_ctas_vs_oracle(eng, oracle, n):
    """n <= 32768: 65536 / L pairs share a CTA (merge_multi_kernel: one padded array, per-pair in-place
    64-output merge levels, leaf counts credited per block).  Tie-free, light-tie (small u groups), monotone
    and short-run rows, plus one heavy-tie row whose batches fall back to one pair at a time; every pair's
    n_d / n3 / numerator vs the oracle."""
    rng = np.random.default_rng(n + 11)
    m = 37
    rows = []
    for r in range(m):
        k = r % 4
        if k == 0:
            rows.append(rng.permutation(n))
        elif k == 1:
            rows.append(rng.integers(0, n // 2, n))  # many groups of 2-3
        elif k == 2:
            rows.append(np.arange(n) if r % 8 == 2 else np.arange(n)[::-1])
        else:
            rows.append(rng.permutation(n) // 2)  # pairs
    rows[20] = rng.integers(0, 4, n)  # heavy groups: batches holding row 20 run pair by pair
    ranks = np.stack([oracle.rank_transform(r) for r in rows])
    res = eng.all_pairs(torch.from_numpy(ranks).cuda(), kernel="merge", full_counts=True).validate()
    pi, pj, num, counts = _full_oracle(oracle, ranks)
    np.testing.assert_array_equal(res.numerator.cpu().numpy().astype(np.int64), num)
    np.testing.assert_array_equal(res.n_d.cpu().numpy(), counts[:, 0])
    np.testing.assert_array_equal(res.n3.cpu().numpy(), counts[:, 3])


@pytest.mark.parametrize("path,n", [("merge", 1025), ("merge", 4096), ("merge", 32767), ("gemm", 6500)])
def test_job_subranges_match_full_run(eng, path, n):
    """Job sub-ranges that start and end anywhere (multi-pair merge CTAs whose first pair is not a multiple
    of P; wide-K FP4 split plans over row fragments) give exactly the full run's counts."""
    rng = np.random.default_rng(n)
    m = 29
    x = np.stack([rng.permutation(n) if r % 3 else rng.integers(0, n // 2, n) for r in range(m)]).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    full = eng.all_pairs(xd, kernel=path, full_counts=True).validate()
    total = m * (m + 1) // 2
    for lo, hi in ((0, 1), (1, 2), (3, 100), (37, total - 5), (total - 1, total)):
        part = eng.all_pairs(xd, kernel=path, full_counts=True, job_range=(lo, hi)).validate()
        for f in ("numerator", "n_d", "n3"):
            assert torch.equal(getattr(part, f), getattr(full, f)[lo:hi]), (f, lo, hi)


def test_merge_row_maximum_clamp(eng, oracle):
    """n = 65536: key 65535 (a unique row maximum) is sorted as 65534 (0xFFFF is the merge loop's
    look-ahead INF) and corrected.  The maximum and a unique second maximum placed in the same half
    (either order) and in different halves; one row with a tied top pair (no key 65535)."""
    n = 65536
    rng = np.random.default_rng(65536)
    rows = [np.arange(n)]
    for p1, p2 in ((10, 40000), (40000, 10), (10, 20), (20, 10), (40000, 40010), (40010, 40000)):
        v = rng.permutation(n - 2)
        v = np.insert(v, min(p1, p2), -1)
        v = np.insert(v, max(p1, p2), -1)
        v[p1], v[p2] = n - 1, n - 2
        rows.append(v)
    tied = rng.permutation(n)
    tied[tied == n - 1] = n - 2
    rows.append(tied)
    rows.append(rng.permutation(n))
    ranks = np.stack([oracle.rank_transform(r) for r in rows])
    m = ranks.shape[0]
    res = eng.all_pairs(torch.from_numpy(ranks).cuda(), kernel="merge", full_counts=True).validate()
    pi, pj = oracle.upper_pairs(m)
    got_nd = res.n_d.cpu().numpy()
    got_n3 = res.n3.cpu().numpy()
    for k, (i, j) in enumerate(zip(pi.tolist(), pj.tolist())):
        nd, n1, n2, n3 = oracle.sorted_counts(ranks[i], ranks[j])
        assert (int(got_nd[k]), int(got_n3[k])) == (nd, n3), (i, j)
    eng.release()


def test_merge_shards(eng, oracle):
    from paper_1704_03767_b200.pairindex import job_shard_range
    rng = np.random.default_rng(5)
    m, n = 40, 3000
    ranks = np.stack([oracle.rank_transform(rng.integers(0, 2000, n)) for _ in range(m)])
    x = torch.from_numpy(ranks).cuda()
    full = eng.all_pairs(x, kernel="merge").validate()
    parts = [eng.all_pairs(x, kernel="merge", job_range=job_shard_range(i, 3, m)).validate() for i in range(3)]
    assert torch.equal(torch.cat([p.numerator for p in parts]), full.numerator)
    _check_full(full, oracle, ranks)


def _oracle_pairs_check(res, oracle, x, pi, pj, kernel, counts=False):
    """SURVEY 8(c) parity protocol at full size: the listed pairs vs the pinned C oracle (its kernels
    match the reference's golden vectors, tests/test_oracle_golden.py), bit-exact numerator / n1 / n2
    (and n_d / n3 when the result carries them), tau compared with assert_array_equal (0 ulp; the
    north-star tolerance 1e-12 is weaker)."""
    rows, inv = np.unique(np.concatenate([pi, pj]), return_inverse=True)
    ranks = np.stack([oracle.rank_transform(x[r]) for r in rows])
    ci, cj = inv[: len(pi)], inv[len(pi):]
    num, cnt = oracle.all_pairs(ranks, ci, cj, kernel, want_counts=True)
    m, n = x.shape
    jid = torch.from_numpy(pi * (2 * m - pi + 1) // 2 + pj - pi - res.job_lo).cuda()
    np.testing.assert_array_equal(res.numerator.index_select(0, jid).cpu().numpy().astype(np.int64), num)
    n1 = res.n1_rows.cpu().numpy()
    np.testing.assert_array_equal(n1[pi], cnt[:, 1])
    np.testing.assert_array_equal(n1[pj], cnt[:, 2])
    if counts and res.n_d is not None:
        np.testing.assert_array_equal(res.n_d.index_select(0, jid).cpu().numpy().astype(np.int64), cnt[:, 0])
        np.testing.assert_array_equal(res.n3.index_select(0, jid).cpu().numpy().astype(np.int64), cnt[:, 3])
    ta, tb = oracle.derive_taus(num, cnt[:, 1], cnt[:, 2], n)
    if res.tau_a is not None:
        np.testing.assert_array_equal(res.tau_a.index_select(0, jid).cpu().numpy(), ta)
    np.testing.assert_array_equal(res.tau_b.index_select(0, jid).cpu().numpy(), tb)


def _random_pairs(m, count, seed):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, m, count)
    b = rng.integers(0, m, count)
    return np.minimum(a, b).astype(np.int64), np.maximum(a, b).astype(np.int64)


def test_config3_gemm_sampled(eng, oracle):
    """Config 3 (16384 x 500 gene-like f32, ties): sampled pairs vs the reference, and 10^4 seeded
    random pairs vs the pinned oracle (SURVEY 8(c) parity protocol), counts included."""
    from paper_1704_03767_b200 import workloads
    z = load_npz("config3.npz")
    x = workloads.generate(3)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["x_sha256"])
    res = eng.all_pairs(torch.from_numpy(x).cuda(), kernel="gemm", full_counts=True).validate()
    _sampled_check(res, z, 500)
    _diag_properties(res, 500)
    pi, pj = _random_pairs(x.shape[0], 10000, 3)
    _oracle_pairs_check(res, oracle, x, pi, pj, oracle.KERNEL_PACKED, counts=True)
    eng.release()


@pytest.mark.timeout(900)
def test_config4_merge_sampled(eng, oracle):
    """Config 4 (1024 x 65536, monotone family every 8th row): the Knight merge path over every job id
    vs the reference's golden pairs, and 10^4 seeded random pairs plus row 0 against every member of
    its monotone family vs the pinned oracle, counts included."""
    from paper_1704_03767_b200 import workloads
    z = load_npz("config4.npz")
    x = workloads.generate(4)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["x_sha256"])
    m = x.shape[0]
    ranks = np.stack([oracle.rank_transform(r) for r in x])
    np.testing.assert_array_equal(ranks[:4], z["ranks_head"])
    # raw float32 values in: the device ranks every row (K0w) -- bit-exact vs the oracle's np.unique ranks
    res = eng.all_pairs(torch.from_numpy(x).cuda(), kernel="merge", full_counts=True).validate()
    np.testing.assert_array_equal(eng._ws["R32"][: m * x.shape[1]].view(m, -1).cpu().numpy(), ranks)
    pi, pj = z["pi"], z["pj"]
    jid = torch.from_numpy(pi * (2 * m - pi + 1) // 2 + pj - pi).cuda()
    np.testing.assert_array_equal(res.numerator.index_select(0, jid).cpu().numpy(), z["numerator"])
    np.testing.assert_array_equal(res.n_d.index_select(0, jid).cpu().numpy(), z["counts"][:, 0])
    np.testing.assert_array_equal(res.n3.index_select(0, jid).cpu().numpy(), z["counts"][:, 3])
    np.testing.assert_array_equal(res.tau_b.index_select(0, jid).cpu().numpy(), z["tau_b"])
    ri, rj = _random_pairs(m, 10000, 4)
    fam = np.arange(8, m, 8, dtype=np.int64)
    ri = np.concatenate([ri, np.zeros_like(fam)])
    rj = np.concatenate([rj, fam])
    _oracle_pairs_check(res, oracle, ranks, ri, rj, oracle.KERNEL_SORTED, counts=True)
    del res
    eng.release()


@pytest.mark.timeout(900)
def test_config5_gemm_sampled(eng, oracle):
    """Config 5 (65536 x 1024 low-rank f32, 2.15e9 pairs): sampled pairs vs the reference, and 10^4
    seeded random pairs vs the pinned oracle."""
    from paper_1704_03767_b200 import workloads
    z = load_npz("config5.npz")
    x = workloads.generate(5)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["x_sha256"])
    res = eng.all_pairs(torch.from_numpy(x).cuda(), kernel="gemm", tau_a=False, full_counts=True).validate()
    pi, pj = z["pi"], z["pj"]
    m = x.shape[0]
    jid = torch.from_numpy(pi * (2 * m - pi + 1) // 2 + pj - pi).cuda()
    np.testing.assert_array_equal(res.numerator.index_select(0, jid).cpu().numpy(), z["numerator"])
    np.testing.assert_array_equal(res.tau_b.index_select(0, jid).cpu().numpy(), z["tau_b"])
    np.testing.assert_array_equal(res.n_d.index_select(0, jid).cpu().numpy(), z["counts"][:, 0])
    np.testing.assert_array_equal(res.n3.index_select(0, jid).cpu().numpy(), z["counts"][:, 3])
    _diag_properties(res, 1024)
    ri, rj = _random_pairs(m, 10000, 5)
    _oracle_pairs_check(res, oracle, x, ri, rj, oracle.KERNEL_PACKED, counts=True)
    del res
    eng.release()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", [1, 2, 3])
def test_sign_formats_agree(eng, k):
    """kind::mxf4 (e2m1, f32 sums), kind::f8f6f4 (e4m3) and kind::i8 give identical numerators."""
    from paper_1704_03767_b200 import _lib, workloads
    x = torch.from_numpy(workloads.generate(k)).cuda()
    outs = {}
    try:
        for fmt in (_lib.TB_SIGN_I8, _lib.TB_SIGN_E4M3, _lib.TB_SIGN_E2M1, _lib.TB_SIGN_E2M1_OFS):
            eng.sign_format_override = fmt
            r = eng.all_pairs(x, kernel="gemm", tau_a=False, tau_b=False, full_counts=(k == 1)).validate()
            assert r.extra["sign_format"] == fmt
            outs[fmt] = (r.numerator.clone(), None if r.n_d is None else r.n_d.clone())
    finally:
        eng.sign_format_override = None
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][0], outs[2][0])
    assert torch.equal(outs[0][0], outs[3][0])
    if k == 1:
        assert torch.equal(outs[0][1], outs[2][1])
        assert torch.equal(outs[0][1], outs[3][1])
    eng.release()


@pytest.fixture
def ofs_eng(eng):
    """The engine with offset-coded GEMM operands forced (TB_SIGN_E2M1_OFS: S + 1, row-sum correction)."""
    from paper_1704_03767_b200 import _lib
    eng.sign_format_override = _lib.TB_SIGN_E2M1_OFS
    try:
        yield eng
    finally:
        eng.sign_format_override = None


@pytest.mark.gpu
def test_offset_operands_small_shapes(ofs_eng, oracle):
    """TB_SIGN_E2M1_OFS against the oracle: every pair and count of the small shapes (ties up to 90%, m = 1,
    n = 2, constant rows), K-split plans, job-id shards, config 1 in full."""
    for m, n, tie in [(1, 5, 0.0), (2, 2, 0.0), (3, 17, 0.5), (37, 33, 0.3), (130, 64, 0.0), (257, 31, 0.9),
                      (300, 130, 0.2), (520, 47, 0.5)]:
        test_small_shapes_vs_oracle(ofs_eng, oracle, "gemm", m, n, tie)
    test_constant_rows_nan(ofs_eng, oracle, "gemm")
    for splits in (1, 2, 7):
        test_gemm_splits_and_shards(ofs_eng, oracle, splits)
    test_config1_full(ofs_eng, oracle, "gemm")


@pytest.mark.gpu
def test_offset_operands_full_counts_and_entry_points(ofs_eng, oracle):
    """TB_SIGN_E2M1_OFS through the tie-indicator GEMM (all rows and the sparse tied-row table), the fused
    tau_b calls, the host entry point and job sub-ranges."""
    for mode in ("auto", "sparse", "full"):
        test_full_counts_sparse_tied_rows(ofs_eng, oracle, mode)
    test_full_counts_tie_free_shortcut(ofs_eng, oracle)
    for m, n, levels in [(300, 200, 0), (2600, 96, 7), (700, 90, 30)]:
        test_fused_tau_b_epilogue(ofs_eng, oracle, m, n, levels)
    test_host_entry_point_bands(ofs_eng, oracle, "gemm", 700, 90, None)
    test_host_entry_point_bands(ofs_eng, oracle, "gemm", 2048, 1000, (0.4, 0.3, 0.2, 0.1))
    test_host_entry_point_job_ranges(ofs_eng, oracle, "gemm", 700, 90)


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_lockstep_gemm_concurrent_launches(oracle):
    """The K-lockstep throttle (multi-wave unsplit plans) with two engines launching on two streams of one
    device at once: the launches share the per-device progress slots (told apart by epoch), neither may hang
    or wait on the other, and both results equal the throttle-free numerators (TB_GEMM_LEAD is read once per
    process, so the reference run is the dp4a cross-check kernel) and, sampled, the oracle."""
    import threading
    from paper_1704_03767_b200.device import TauEngine
    rng = np.random.default_rng(77)
    m, n = 6400, 260  # 25 row blocks x 14 column-block pairs / 2 > 74 units: several waves, no K split
    xs = [torch.from_numpy(rng.integers(0, 40, (m, n)).astype(np.int32)).cuda() for _ in range(2)]
    engs = [TauEngine(0), TauEngine(0)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    out = [None, None]

    def run(k):
        for _ in range(3):
            out[k] = engs[k].all_pairs(xs[k], kernel="gemm", stream=streams[k], tau_a=False)

    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=240)
        assert not t.is_alive(), "concurrent lockstep GEMM launches did not finish"
    torch.cuda.synchronize()
    for k in range(2):
        ref = engs[k].all_pairs(xs[k], kernel="gemm", simt=True, tau_a=False, tau_b=False)
        assert torch.equal(out[k].numerator, ref.numerator)
        ri, rj = _random_pairs(m, 2000, 5 + k)
        _oracle_pairs_check(out[k], oracle, xs[k].cpu().numpy(), ri, rj, oracle.KERNEL_PACKED, counts=False)
    for e in engs:
        e.release()


@pytest.mark.gpu
def test_fused_row_sums_match_the_separate_pass(eng, oracle):
    """tb_sign_pack_sums (the pack sums the offset-coded values it writes) against tb_sign_row_sums (a pass
    over the packed S) and the definition sum_{a<b} sign(r_b - r_a), for row widths around the layout's
    section boundaries, with ties."""
    import ctypes
    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.device import _ptr
    lib = _lib.load()
    for n in (2, 15, 16, 17, 33, 200, 1000, 1024, 2896):
        m = 37 if n < 2000 else 5
        rng = np.random.default_rng(n)
        ranks = np.stack([oracle.rank_transform(rng.integers(0, max(2, n // 3), n)) for _ in range(m)])
        ldr = (n + 7) // 8 * 8
        R = torch.zeros((m, ldr), dtype=torch.int16, device="cuda")
        R[:, :n] = torch.from_numpy(ranks.astype(np.int16)).cuda()
        K = int(lib.tb_sign_k(n))
        ldS = (K // 2 + 15) // 16 * 16
        S1 = torch.empty(m * ldS, dtype=torch.int8, device="cuda")
        S2 = torch.empty(m * ldS, dtype=torch.int8, device="cuda")
        f1 = torch.empty(m, dtype=torch.int32, device="cuda")
        f2 = torch.full((m,), 12345, dtype=torch.int32, device="cuda")
        _lib.call("tb_sign_pack", _ptr(R), m, n, ldr, _ptr(S1), ldS, _lib.TB_SIGN_E2M1_OFS, None)
        _lib.call("tb_sign_row_sums", _ptr(S1), m, ldS, n, _ptr(f1), None)
        _lib.call("tb_sign_pack_sums", _ptr(R), m, n, ldr, _ptr(S2), ldS, _ptr(f2), None)
        torch.cuda.synchronize()
        assert torch.equal(S1, S2)
        d = ranks[:, None, :] - ranks[:, :, None]            # [r, a, b] = r_b - r_a
        want = np.triu(np.sign(d), 1).sum(axis=(1, 2)) if n <= 1024 else None
        assert torch.equal(f1, f2), n
        if want is not None:
            np.testing.assert_array_equal(f1.cpu().numpy(), want.astype(np.int32))


@pytest.mark.gpu
def test_offset_operands_limit(ofs_eng, oracle):
    """n = 2896 is the last n with 4 K < 2^24 (sums of (S + 1)(S + 1) <= 4 n0 stay exact in f32): a monotone pair
    (numerator = n0, the largest sum) and its reverse, heavy ties; n = 2897 is refused (the engine's own
    choice falls back to the +-1 coding there)."""
    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.errors import ConfigError
    n, m = 2896, 20
    rng = np.random.default_rng(2896)
    rows = [rng.integers(0, n // 3, n) for _ in range(m - 3)] + [np.arange(n), np.arange(n), np.arange(n)[::-1]]
    ranks = np.stack([oracle.rank_transform(r) for r in rows])
    res = ofs_eng.all_pairs(torch.from_numpy(ranks).cuda(), kernel="gemm", full_counts=True).validate()
    assert res.extra["sign_format"] == _lib.TB_SIGN_E2M1_OFS
    _check_full(res, oracle, ranks)
    with pytest.raises(ConfigError):
        ofs_eng.all_pairs(torch.from_numpy(np.stack([oracle.rank_transform(rng.integers(0, 50, 2897))
                                                     for _ in range(4)])).cuda(), kernel="gemm")
    ofs_eng.sign_format_override = None
    K = int(_lib.load().tb_sign_k(2897))
    assert ofs_eng.sign_format(K, m=1 << 20) == _lib.TB_SIGN_E2M1
    assert ofs_eng.sign_format(int(_lib.load().tb_sign_k(1024)), m=65536) == _lib.TB_SIGN_E2M1_OFS
    assert ofs_eng.sign_format(int(_lib.load().tb_sign_k(1000)), m=2048) == _lib.TB_SIGN_E2M1


@pytest.mark.parametrize("fracs", [None, (0.4, 0.3, 0.2, 0.1)])
@pytest.mark.parametrize("path,m,n", [("gemm", 2048, 1000), ("gemm", 700, 90), ("merge", 60, 3000)])
def test_host_entry_point_bands(eng, oracle, path, m, n, fracs):
    """all_pairs_host (pinned host in, tau_b out, row bands overlapping D2H) == the device API, with the
    default (size-dependent) bands and an explicit four-band split."""
    rng = np.random.default_rng(m + n)
    x = rng.integers(0, max(2, n // 3), (m, n)).astype(np.int32)
    if path == "merge":
        x = np.stack([oracle.rank_transform(r) for r in x])
    xh = torch.from_numpy(x).pin_memory()
    total = m * (m + 1) // 2
    out = torch.full((total,), -7.0, dtype=torch.float64).pin_memory()
    eng.all_pairs_host(xh, out, kernel=path, band_fracs=fracs, h2d_chunks=3)
    torch.cuda.synchronize()
    ref = eng.all_pairs(torch.from_numpy(x).cuda(), kernel=path, tau_a=False).validate()
    np.testing.assert_array_equal(out.numpy(), ref.tau_b.cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.int32, np.float32, np.float64])
def test_rank_rows_vs_oracle(oracle, dtype):
    """K0 dense ranks + tie counts vs the oracle's rank_transform (ranks.py:37-61), int32 rows on
    both sides of the 1024-wide histogram path (range 1023 / 1024, negative values, constants)."""
    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.device import _ptr, _stream_ptr, _dtype_code
    rng = np.random.default_rng(404)
    for n in (7, 33, 500, 1000, 1024, 2000):
        rows = [rng.integers(-5, 5, n), rng.integers(0, 1024, n), rng.integers(0, 1025, n),
                rng.integers(-2**31, 2**31 - 1, n), np.full(n, 7), rng.integers(100, 103, n),
                rng.standard_normal(n) * 1000, np.arange(n)[::-1]]
        x = np.stack(rows).astype(dtype)
        if dtype is not np.int32:
            x[0, : n // 3] = -0.0
        m = x.shape[0]
        ldr = (n + 7) // 8 * 8
        xd = torch.from_numpy(x).cuda()
        R = torch.empty(m * ldr, dtype=torch.int16, device="cuda")
        n1 = torch.empty(m, dtype=torch.int64, device="cuda")
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("tb_rank_rows", _ptr(xd), _dtype_code(xd), m, n, n, _ptr(R), ldr, _ptr(n1), _ptr(flags),
                  _stream_ptr(None))
        torch.cuda.synchronize()
        got = R.view(m, ldr)[:, :n].cpu().numpy().astype(np.int64)
        for r in range(m):
            ref = oracle.rank_transform(x[r])
            np.testing.assert_array_equal(got[r], ref, err_msg=f"n={n} row={r}")
            _, c = np.unique(ref, return_counts=True)
            assert int(n1[r]) == int((c * (c - 1) // 2).sum()), (n, r)
        assert int(flags.item()) == 0


@pytest.mark.gpu
def test_finalize_ranges_vs_numpy():
    """K5 over arbitrary job ranges (mid-row starts, rows shorter than the 256-id step, ranges ending
    inside a chunk) == derive_taus (result.py:62-82) evaluated in numpy on the same counts."""
    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.device import _ptr, _stream_ptr
    from paper_1704_03767_b200.pairindex import job_coord
    rng = np.random.default_rng(77)
    for m, n in ((1, 5), (3, 9), (40, 17), (300, 1000), (5000, 64), (70, 3000)):
        n0 = n * (n - 1) // 2
        total = m * (m + 1) // 2
        n1 = rng.integers(0, n0 + 1, m).astype(np.uint64)
        n1[::2] = 0  # tie-free rows: tau_b of tie-free pairs comes from the quotient table (n <= 2048)
        n1[rng.integers(0, m)] = n0  # a constant row -> NaN tau_b
        for lo, hi in ((0, total), (total // 3, total // 3 + 1), (max(0, total // 2 - 777), total),
                       (1, min(total, 4097)), (0, min(total, 4096 * 3 + 5))):
            if hi <= lo:
                continue
            num = rng.integers(-n0, n0 + 1, hi - lo).astype(np.int32)
            dn = torch.from_numpy(num).cuda()
            dn1 = torch.from_numpy(n1.view(np.int64)).cuda()
            ta = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
            tb = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
            _lib.call("tb_finalize", _ptr(dn), _ptr(dn1), m, n, lo, hi, _ptr(ta), _ptr(tb), _stream_ptr(None))
            torch.cuda.synchronize()
            ys_all = np.repeat(np.arange(m, dtype=np.int64), m - np.arange(m))
            starts = np.arange(m, dtype=np.int64) * (2 * m - np.arange(m) + 1) // 2
            xs_all = np.arange(total, dtype=np.int64) - starts[ys_all] + ys_all
            ys, xs = ys_all[lo:hi], xs_all[lo:hi]
            assert job_coord(lo, m) == (ys[0], xs[0]) and job_coord(hi - 1, m) == (ys[-1], xs[-1])
            t1 = n1[ys].astype(np.float64)
            t2 = n1[xs].astype(np.float64)
            denom = np.sqrt((n0 - t1) * (n0 - t2))
            with np.errstate(divide="ignore", invalid="ignore"):
                ref_b = np.where(denom > 0, num / denom, np.nan)
            np.testing.assert_array_equal(ta.cpu().numpy(), num / float(n0))
            np.testing.assert_array_equal(tb.cpu().numpy(), ref_b)


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["e2m1", "i8"])
def test_gemm_beyond_2_24(eng, oracle, fmt):
    """K >= 2^24 (n > 5792): the FP4 GEMM splits every unit into items of <= 65535 k-blocks, whose f32 sums
    stay exact integers, and adds them as int32 (red.add.s32); the int8 GEMM (kind::i8) covers the same
    shapes.  Every pair against the oracle, with ties and a monotone pair (|numerator| = n0 > 2^24), across
    the boundary n = 5793 / 5794, at n = 6000 and n = 11000 (3 items per unit)."""
    from paper_1704_03767_b200 import _lib
    code = {"e2m1": _lib.TB_SIGN_E2M1, "i8": _lib.TB_SIGN_I8}[fmt]
    try:
        eng.sign_format_override = code
        for n, m in ((5793, 24), (5794, 24), (6000, 40), (11000, 12)):
            if fmt == "i8" and n == 11000:
                continue
            rng = np.random.default_rng(n)
            rows = [rng.integers(0, n // 4, n) for _ in range(m - 2)] + [np.arange(n), np.arange(n)]
            ranks = np.stack([oracle.rank_transform(r) for r in rows])
            res = eng.all_pairs(torch.from_numpy(ranks).cuda(), kernel="gemm", full_counts=True).validate()
            assert res.extra["sign_format"] == code
            _check_full(res, oracle, ranks)
    finally:
        eng.sign_format_override = None


@pytest.mark.gpu
def test_gemm_workspace_beyond_hbm_is_capacity_error(eng):
    """S = m x K / 2 bytes beyond the GPU (m = 14000, n = 8192, e2m1: ~235 GB) -> CapacityExceededError."""
    import paper_1704_03767_b200 as tb
    x = torch.zeros((14000, 8192), dtype=torch.float32, device="cuda")
    with pytest.raises(tb.CapacityExceededError):
        eng.all_pairs(x, kernel="gemm")
    eng.release()
    torch.cuda.empty_cache()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.int32, np.float32, np.float64])
def test_rank_dense_vs_oracle(oracle, dtype):
    """K0w (any row width): dense int32 ranks + tie counts vs the oracle's rank_transform (np.unique,
    ranks.py:37-61) -- -0.0 == +0.0, +-inf orderable, heavy ties, constant rows, rows wider than 65536;
    NaN raises through the engine (flag bit 0)."""
    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.device import _dtype_code, _ptr, _stream_ptr
    lib = _lib.load()
    rng = np.random.default_rng(77)
    for n in (1, 2, 31, 33, 1000, 9000, 65536, 70001):
        rows = [rng.integers(-5, 5, n), rng.integers(0, 3, n), np.full(n, 7), np.arange(n)[::-1],
                rng.integers(-2**31, 2**31 - 1, n), rng.standard_normal(n) * 1e3]
        x = np.stack(rows).astype(dtype)
        if dtype is not np.int32:
            x[0, : n // 3] = -0.0
            x[0, n // 3: n // 2] = 0.0
            x[1, ::7] = np.inf
            x[1, 1::11] = -np.inf
        m = x.shape[0]
        xd = torch.from_numpy(x).cuda()
        R = torch.empty(m * n, dtype=torch.int32, device="cuda")
        n1 = torch.empty(m, dtype=torch.int64, device="cuda")
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        wsb = int(lib.tb_rank_dense_workspace(m, n, _dtype_code(xd)))
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        _lib.call("tb_rank_dense", _ptr(xd), _dtype_code(xd), m, n, n, _ptr(R), 0, n, _ptr(n1), _ptr(flags),
                  _ptr(ws), wsb, _stream_ptr(None))
        torch.cuda.synchronize()
        got = R.view(m, n).cpu().numpy()
        for r in range(m):
            ref = oracle.rank_transform(x[r])
            np.testing.assert_array_equal(got[r], ref, err_msg=f"n={n} row={r}")
            _, c = np.unique(ref, return_counts=True)
            assert int(n1[r]) == int((c * (c - 1) // 2).sum()), (n, r)
        assert int(flags.item()) == 0
    if dtype is not np.int32:
        from paper_1704_03767_b200 import InvalidInputError
        from paper_1704_03767_b200.device import TauEngine
        x = rng.standard_normal((3, 9000)).astype(dtype)
        x[1, 5] = np.nan
        with pytest.raises(InvalidInputError, match="NaN"):
            TauEngine(0).all_pairs(torch.from_numpy(x).cuda(), kernel="merge").validate()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("n,levels", [(3000, 5), (40000, 7), (65536, 2), (65536, 10)])
def test_merge_heavy_ties_vs_oracle(eng, oracle, n, levels):
    """Rows with huge tie groups (<= 10 distinct values, groups of thousands): K4's O(n log n) segmented
    radix count of the within-group inversions and joint ties, every pair vs the oracle's GSE counts
    (kernel_sorted.py:195-212), with a time bound (the O(sum g^2) enumeration it replaces needed ~1-10 ms
    per pair at n = 65536)."""
    import time
    rng = np.random.default_rng(n + levels)
    m = 7
    x = rng.integers(0, levels, (m, n)).astype(np.int32)
    x[2] = rng.permutation(n)              # a tie-free row
    x[3] = 4                               # a constant row (tau_b undefined)
    x[4, : n // 2] = rng.integers(0, 50, n // 2)  # small and large groups mixed
    xd = torch.from_numpy(x).cuda()
    eng.all_pairs(xd, kernel="merge").validate()  # warm-up (allocations)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = eng.all_pairs(xd, kernel="merge", full_counts=True).validate()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    assert dt < 2.0, f"{m * (m + 1) // 2} pairs took {dt:.2f} s"
    ranks = oracle.rank_matrix(x)
    _check_full(res, oracle, ranks)


def test_full_counts_tie_free_shortcut(eng, oracle):
    """With no tied variable, n_d / n3 come from the closed form |S_y|.|S_x| = n0 - n1_y - n1_x (no |S|
    GEMM); identical to the |S| GEMM path and to the oracle; one tied row switches the GEMM back on."""
    rng = np.random.default_rng(31)
    x = np.stack([rng.permutation(700) for _ in range(300)]).astype(np.float32) * 0.25 - 40.0  # no ties
    xd = torch.from_numpy(x).cuda()
    a = eng.all_pairs(xd, kernel="gemm", full_counts=True).validate()
    try:
        eng.force_abs_gemm = True
        b = eng.all_pairs(xd, kernel="gemm", full_counts=True).validate()
    finally:
        eng.force_abs_gemm = False
    assert int(a.n1_rows.max()) == 0
    for f in ("numerator", "n_d", "n3"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    _check_full(a, oracle, oracle.rank_matrix(x))
    x[7, :50] = 1.0  # ties in one row
    c = eng.all_pairs(torch.from_numpy(x).cuda(), kernel="gemm", full_counts=True).validate()
    _check_full(c, oracle, oracle.rank_matrix(x))


@pytest.mark.parametrize("mode", ["auto", "sparse", "full"])
def test_full_counts_sparse_tied_rows(eng, oracle, mode):
    """With a few tied variables the |S| GEMM runs over the tied rows only (n3 = 0 for every pair with an
    untied variable) and tb_tied_counts patches their pairs; identical to the full |S| GEMM and the oracle,
    over the whole job space and over job sub-ranges that cut rows (the compute_all_pairs windows)."""
    rng = np.random.default_rng(77)
    m, n = 420, 260
    x = rng.standard_normal((m, n)).astype(np.float32)
    tied = [0, 5, 6, 131, 132, 300, 419]
    for k, r in enumerate(tied):  # shared tie patterns (joint ties) and private ones
        x[r, : 20 + 7 * k] = x[r, 0]
        x[r, 100:110] = 2.5 if k % 2 else x[r, 100]
    x[rng.integers(0, m), 200:203] = 0.125  # one more row with one small tie group
    ranks = oracle.rank_matrix(x)
    xd = torch.from_numpy(x).cuda()
    try:
        eng.tied_mode = "sparse" if mode == "sparse" else "auto"
        eng.force_abs_gemm = mode == "full"
        res = eng.all_pairs(xd, kernel="gemm", full_counts=True).validate()
        _check_full(res, oracle, ranks)
        total = m * (m + 1) // 2
        for lo, hi in ((0, 1), (1000, 5000), (total // 3, total // 3 + 12345), (total - 999, total)):
            part = eng.all_pairs(xd, kernel="gemm", full_counts=True, job_range=(lo, hi)).validate()
            for f in ("numerator", "n_d", "n3"):
                assert torch.equal(getattr(part, f), getattr(res, f)[lo:hi]), (f, lo, hi)
    finally:
        eng.tied_mode = "auto"
        eng.force_abs_gemm = False


@pytest.mark.parametrize("path,m,n", [("gemm", 700, 90), ("merge", 60, 3000)])
def test_host_entry_point_job_ranges(eng, oracle, path, m, n):
    """all_pairs_host over a rank's job range (multi-GPU e2e): tau_b of [lo, hi) lands at out[0:hi-lo] and
    equals the device API's; tau_b_bands (the bench / gather path) over shrinking bands of the same range
    too, with rows above the range neither ranked nor packed."""
    from paper_1704_03767_b200.multi import balanced_job_shards, gather_band_fracs, shard_bands
    rng = np.random.default_rng(m * n)
    x = rng.integers(0, max(2, n // 3), (m, n)).astype(np.int32)
    ref = eng.all_pairs(torch.from_numpy(x).cuda(), kernel=path, tau_a=False).validate().tau_b.cpu().numpy()
    xh = torch.from_numpy(x).pin_memory()
    for lo, hi in balanced_job_shards(3, m, path):
        out = torch.full((hi - lo,), -7.0, dtype=torch.float64).pin_memory()
        eng.all_pairs_host(xh, out, kernel=path, job_range=(lo, hi))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.numpy(), ref[lo:hi])
        dout = torch.full((hi - lo,), -7.0, dtype=torch.float64, device="cuda")
        bands = shard_bands(lo, hi, m, 3, gather_band_fracs(3))
        seen = []
        eng.tau_b_bands(torch.from_numpy(x).cuda(), bands, dout, kernel=path, on_band=lambda b, t: seen.append(b))
        torch.cuda.synchronize()
        assert seen == list(range(len(bands)))
        np.testing.assert_array_equal(dout.cpu().numpy(), ref[lo:hi])


@pytest.mark.parametrize("m,n,levels", [(300, 200, 0), (2600, 96, 7), (700, 90, 30)])
def test_fused_tau_b_epilogue(eng, oracle, m, n, levels):
    """tau_b straight from the FP4 GEMM epilogue (tb_gemm_tau_b: no numerator round trip, no finalize
    launch) equals the numerator + tb_finalize path bit for bit -- tie-free rows (num / n0), tied rows
    (the sqrt sequence), a constant row (NaN), one-launch and split-K plans (the split plan falls back to
    numerator + finalize) -- through tau_b_bands and all_pairs_host(numerators=False)."""
    rng = np.random.default_rng(m + n)
    x = (rng.standard_normal((m, n)) if levels == 0 else rng.integers(0, levels, (m, n))).astype(np.float32)
    x[3] = 1.5  # constant row: tau_b NaN
    xd = torch.from_numpy(x).cuda()
    ref = eng.all_pairs(xd, kernel="gemm", tau_a=False).validate().tau_b.cpu().numpy()
    total = m * (m + 1) // 2
    bands = [(0, total // 3), (total // 3, total // 3 + 777), (total // 3 + 777, total)]
    try:
        for fuse in (True, False):
            eng.fuse_finalize = fuse
            out = torch.empty(total, dtype=torch.float64, device="cuda")
            eng.tau_b_bands(xd, bands, out, kernel="gemm")
            torch.cuda.synchronize()
            np.testing.assert_array_equal(out.cpu().numpy(), ref)
            xh = torch.from_numpy(x).pin_memory()
            outh = torch.empty(total, dtype=torch.float64).pin_memory()
            eng.all_pairs_host(xh, outh, kernel="gemm", numerators=False)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(outh.numpy(), ref)
    finally:
        eng.fuse_finalize = True
    pi, pj = oracle.upper_pairs(m)
    sel = rng.integers(0, total, 4000)
    num, counts = oracle.all_pairs(oracle.rank_matrix(x), pi[sel], pj[sel], oracle.KERNEL_SORTED, threads=8)
    _, tb = oracle.derive_taus(num, counts[:, 1], counts[:, 2], n)
    np.testing.assert_array_equal(ref[sel], tb)


@pytest.mark.parametrize("fuse", ["0", "1"])
def test_fused_epilogue_switch_subprocess(tmp_path, fuse):
    """TB_FUSE_EPILOGUE (read once per process; default on): the FP4 GEMM epilogue writes tau_b itself on
    one-launch plans, or (0) writes numerators for a separate finalize; both identical to all_pairs'
    numerator + finalize sequence (run in a child process)."""
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
from paper_1704_03767_b200.device import TauEngine
eng = TauEngine(0)
rng = np.random.default_rng(5)
x = torch.from_numpy(rng.integers(0, 40, (8192, 64)).astype(np.float32)).cuda()  # short K: a one-launch plan
ref = eng.all_pairs(x, kernel="gemm", tau_a=False).validate().tau_b
m = x.shape[0]; total = m * (m + 1) // 2
out = torch.empty(total, dtype=torch.float64, device="cuda")
eng.gemm_bands = 1
eng.tau_b_bands(x, [(0, total)], out, kernel="gemm")
torch.cuda.synchronize()
assert torch.equal(out.isnan(), ref.isnan())
assert torch.equal(torch.nan_to_num(out), torch.nan_to_num(ref))
print("ok")
""" % (str(__import__("conftest").ROOT),)
    env = dict(__import__("os").environ, TB_FUSE_EPILOGUE=fuse)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
