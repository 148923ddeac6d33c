"""CPU-only tests: host geometry vs the reference's golden vectors, engine validation,
record-order planning, and the C-ABI symbol table (no compute calls without a GPU)."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_json, load_npz


def test_bijection_kats():
    import paper_1704_03767_b200 as tb
    k = load_json("kats.json")["bijection"]
    assert tb.job_id(2, 3, 4) == k["job_id_2_3_4"] == 8
    assert list(tb.job_coord(5, 4)) == k["job_coord_5_4"] == [1, 2]
    assert tb.tile_id(1, 2, 3) == k["tile_id_1_2_3"] == 4
    for m, q, p, ranges in k["shard_ranges"]:
        space = tb.JobSpace(m, q)
        assert [list(tb.shard_range(i, p, space)) for i in range(p)] == ranges


def test_bijection_exhaustive_and_sampled():
    import paper_1704_03767_b200 as tb
    for m in range(1, 120):
        j = 0
        for y in range(m):
            for x in range(y, m):
                assert tb.job_id(y, x, m) == j
                assert tb.job_coord(j, m) == (y, x)
                j += 1
    z = load_npz("bijection.npz")
    for key in z.files:
        if key.endswith("_j"):
            m = int(key[1:-2])
            for j, yx in zip(z[key].tolist(), z[key[:-2] + "_yx"].tolist()):
                assert tb.job_coord(j, m) == tuple(yx)


def test_vectorised_tile_order_matches_tile_cells():
    import paper_1704_03767_b200 as tb
    for m in (1, 2, 7, 13, 40):
        for q in (1, 2, 3, 8, 9):
            space = tb.JobSpace(m, q)
            expected = []
            for t in range(space.total_tiles):
                expected.extend(space.tile_cells(*tb.tile_coord(t, space.w)))
            ii, jj = space.cells_in_tile_order(0, space.total_tiles)
            assert list(zip(ii.tolist(), jj.tolist())) == expected
            assert len(expected) == m * (m + 1) // 2


def test_plan_passes_exact():
    import paper_1704_03767_b200 as tb
    space = tb.JobSpace(m=4, q=1)
    plans = tb.plan_passes(space, (0, 10), 4)
    assert [(p.tile_lo, p.tile_hi) for p in plans] == [(0, 4), (4, 8), (8, 10)]
    space = tb.JobSpace(m=23, q=4)
    for pass_tiles in (1, 3, 7):
        plans = tb.plan_passes(space, (0, space.total_tiles), pass_tiles)
        for p in plans:
            assert p.cells == sum(space.tile_cell_count(*tb.tile_coord(t, space.w))
                                  for t in range(p.tile_lo, p.tile_hi))
    with pytest.raises(tb.ConfigError):
        tb.plan_passes(space, (0, 10), 0)


def test_job_shards_partition():
    import paper_1704_03767_b200 as tb
    for m in (1, 5, 100, 65536):
        for p in (1, 2, 3, 8):
            rs = [tb.job_shard_range(i, p, m) for i in range(p)]
            assert rs[0][0] == 0 and rs[-1][1] == m * (m + 1) // 2
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))


def test_engine_config_errors_before_device():
    import paper_1704_03767_b200 as tb
    ds = tb.synth_dataset(4, 6, seed=9)
    for kw in [dict(kernel="fancy"), dict(workers=0), dict(tile_size=0), dict(pass_tiles=0), dict(shard=(2, 2))]:
        kernel = kw.pop("kernel", "sorted")
        with pytest.raises(tb.ConfigError):
            tb.compute_all_pairs(ds, kernel, **kw)
    with pytest.raises(tb.InvalidInputError):
        tb.compute_all_pairs(tb.Dataset(labels=["a", "b"], ranks=np.zeros((2, 1), np.int32)), "sorted")
    with pytest.raises(tb.InvalidInputError):
        tb.Dataset(labels=["a", "a"], ranks=np.zeros((2, 3), np.int32))
    with pytest.raises(tb.InvalidInputError):
        tb.Dataset(labels=[], ranks=np.zeros((0, 3), np.int32))


def test_rank_and_pack_kats():
    import paper_1704_03767_b200 as tb
    for vals, expected in load_json("kats.json")["rank_transform"]:
        assert tb.rank_transform(np.array(vals)).tolist() == expected
    with pytest.raises(tb.InvalidInputError):
        tb.rank_transform([1.0, float("nan")])
    p = tb.pack_pairs([1, 2], [3, 4])
    u, v = tb.unpack_pairs(p)
    assert u.tolist() == [1, 2] and v.tolist() == [3, 4]
    with pytest.raises(tb.CapacityExceededError):
        tb.pack_pairs([0, 1 << 15], [0, 1])


def test_record_writers_roundtrip():
    import io
    import paper_1704_03767_b200 as tb
    rec = np.zeros(3, tb.CELL_DTYPE)
    rec["i"] = [0, 0, 1]
    rec["j"] = [0, 1, 1]
    rec["numerator"] = [6, -2, 0]
    rec["n1"] = [0, 0, 6]
    rec["n2"] = [0, 6, 6]
    s = io.BytesIO()
    tb.BinaryWriter(s, 4)(rec)
    back, ta, tbb = tb.read_binary(io.BytesIO(s.getvalue()), 4)
    assert np.isnan(tbb[1]) and np.isnan(tbb[2]) and tbb[0] == 1.0


def _header_symbols():
    with open(os.path.join(ROOT, "include", "taub200.h")) as fh:
        txt = fh.read()
    return set(re.findall(r"^(?:int|int64_t|const char \*)\s*(tb_\w+)\(", txt, re.M))


def test_capi_exports_every_declared_symbol():
    from paper_1704_03767_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libtaub200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _header_symbols()
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name), name
    loaded = _lib.load()
    assert loaded.tb_last_error() is not None


def test_no_oracle_in_product_path():
    """The package must not import the oracle (the checker) anywhere."""
    pkg = os.path.join(ROOT, "paper_1704_03767_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert "import oracle" not in src and "tau_oracle" not in src and "libtauoracle" not in src, f


def test_sign_k_block_layout():
    """tb_sign_k(n): 16 x (chunks of the block layout), >= n(n-1)/2 with < 16 * (n / 16 + 16) slack."""
    from paper_1704_03767_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libtaub200.so not built")
    lib = _lib.load()
    for n in list(range(2, 70)) + [255, 256, 500, 1000, 1024, 5793, 8192, 32767]:
        nbf, nt = divmod(n, 16)
        chunks = 16 * (nbf * (nbf - 1) // 2) + 7 * nbf + (nbf + 1) // 2 + nt * nbf + max(nt - 1, 0)
        k = int(lib.tb_sign_k(n))
        assert k == 16 * chunks, n
        assert n * (n - 1) // 2 <= k < n * (n - 1) // 2 + 16 * (nbf + 16), n
    assert int(lib.tb_sign_k(1000)) == 499584


def test_band_plans_cover_the_job_range():
    """Host logic of the banded launches: row bands (aligned to the 256-row GEMM block) and the
    size-dependent default shares of all_pairs_host; the GEMM sub-ranges of a (shard) job range are
    contiguous and cover it exactly."""
    import types

    from paper_1704_03767_b200.device import TauEngine
    from paper_1704_03767_b200.pairindex import job_shard_range

    for total in (3, 2_098_176, 134_225_920, 2_147_516_416):
        fr = TauEngine.default_band_fracs(total)
        assert abs(sum(fr) - 1.0) < 1e-9 and all(a >= b for a, b in zip(fr, fr[1:]))
        assert len(fr) == (2 if total <= (8 << 20) else len(fr)) and 2 <= len(fr) <= 14
    for m in (1, 255, 256, 700, 2048, 16384, 65536):
        for nb in (1, 2, 3, 7, 8, 12):
            cuts = TauEngine.bands(m, nb)
            assert cuts[0] == 0 and cuts[-1] == m and cuts == sorted(set(cuts))
            assert all(c % 256 == 0 for c in cuts[1:-1])
    for m in (300, 2048, 65536):
        total = m * (m + 1) // 2
        for nb in (1, 8):
            eng = types.SimpleNamespace(gemm_bands=nb, bands=TauEngine.bands)
            for p in (1, 3, 8):
                for r in range(p):
                    lo, hi = job_shard_range(r, p, m)
                    rr = TauEngine._gemm_ranges(eng, m, lo, hi)
                    if lo == hi:
                        assert rr == []
                        continue
                    assert rr[0][0] == lo and rr[-1][1] == hi
                    assert all(a[1] == b[0] for a, b in zip(rr, rr[1:])) and all(a < b for a, b in rr)
        auto = types.SimpleNamespace(gemm_bands=None, bands=TauEngine.bands)
        assert len(TauEngine._gemm_ranges(auto, m, 0, total)) == (8 if total >= (1 << 30) else 1)


def test_closed_form_cell_counts_and_pass_spans():
    """Pass planning in O(1) per pass (the reference plans with a per-tile Python loop,
    engine.py:147-167): closed-form per-tile counts, cells before a tile, the job span a pass touches, and
    the C ABI's tb_tile_cells, all against brute-force enumeration of tile_cells."""
    import numpy as np

    import paper_1704_03767_b200 as tb
    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.engine import _cells_before, _pass_job_span, _tile_cells_vec, _window_groups

    lib = _lib.load() if os.path.exists(_lib.LIB_PATH) else None
    for m in (1, 2, 7, 13, 40, 97):
        for q in (1, 2, 3, 8, 9, 100):
            space = tb.JobSpace(m, q)
            tt = space.total_tiles
            brute = [space.tile_cell_count(*tb.tile_coord(t, space.w)) for t in range(tt)]
            assert _tile_cells_vec(space, 0, tt).tolist() == brute
            before = np.concatenate([[0], np.cumsum(brute)])
            assert _cells_before(space, np.arange(tt + 1)).tolist() == before.tolist()
            for pass_tiles in (1, 3, 7, 4096):
                plans = tb.plan_passes(space, (0, tt), pass_tiles)
                assert sum(p.cells for p in plans) == m * (m + 1) // 2
                for p in plans:
                    ii, jj = space.cells_in_tile_order(p.tile_lo, p.tile_hi)
                    jid = ii * (2 * m - ii + 1) // 2 + jj - ii
                    assert _pass_job_span(space, p) == (int(jid.min()), int(jid.max()) + 1)
                    if lib is not None:
                        assert lib.tb_tile_cells(m, q, p.tile_lo, p.tile_hi) == p.cells
                for wj in (1, 50, 1 << 25):
                    groups = _window_groups(space, plans, wj)
                    assert [p for _, ps in groups for p in ps] == plans
                    for (lo, hi), ps in groups:
                        spans = [_pass_job_span(space, p) for p in ps]
                        assert lo == spans[0][0] and hi == spans[-1][1]
                        assert len(ps) == 1 or hi - lo <= wj
    # config-5 scale: 33.6 M tiles planned without per-tile host arrays
    space = tb.JobSpace(65536, 8)
    plans = tb.plan_passes(space, (0, space.total_tiles), 4096)
    assert sum(p.cells for p in plans) == 65536 * 65537 // 2


def test_dispatcher_cost_model(monkeypatch):
    """The measured cost model picks the GEMM for the BASELINE GEMM configs and the merge for config 4
    and for large n with few rows; the GEMM is refused when S does not fit the free memory."""
    import types

    import torch

    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.device import DISPATCH_TABLE, TauEngine, choose_path

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libtaub200.so not built")
    eng = types.SimpleNamespace(_ws={}, device=None, sign_format_override=None)
    eng.sign_format = lambda K, m=None: TauEngine.sign_format(eng, K, m)
    eng._gemm_layout = lambda n, simt=False, m=None: TauEngine._gemm_layout(eng, n, simt, m)
    monkeypatch.setattr(torch.cuda, "mem_get_info", lambda dev=None: (170 << 30, 180 << 30))
    for (m, n), want in {(256, 200): "gemm", (2048, 1000): "gemm", (16384, 500): "gemm", (65536, 1024): "gemm",
                         (1024, 65536): "merge", (128, 32767): "merge", (4, 9000): "merge",
                         (2000, 8192): "gemm", (1000, 12288): "gemm", (1000, 16384): "merge"}.items():
        assert choose_path(n, m=m, eng=eng) == want, (m, n)
    assert choose_path(1000) == "gemm" and choose_path(15000) == "merge"  # no shape: the large-m crossover
    monkeypatch.setattr(torch.cuda, "mem_get_info", lambda dev=None: (1 << 30, 180 << 30))
    assert choose_path(1024, m=65536, eng=eng) == "merge"  # S = 17 GB does not fit 1 GiB
    for n, *_ in DISPATCH_TABLE:  # the model is finite and increasing in m
        c1, c2 = TauEngine.path_costs(100, n), TauEngine.path_costs(1000, n)
        assert all(0 < c1[k] < c2[k] for k in c1)


def test_bench_helpers():
    """bench.py's pair counting and the SURVEY 8(d) CPU subset draw."""
    import importlib.util

    import numpy as np
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for m in (1, 2, 5, 300):
        total = m * (m + 1) // 2
        assert bench._strict_pairs(m, 0, total) == m * (m - 1) // 2
        assert sum(bench._strict_pairs(m, a, b) for a, b in ((0, total // 3), (total // 3, total))) == m * (m - 1) // 2
    rows = bench.cpu_subset(5, 65536)
    assert rows.shape == (2048,) and np.array_equal(rows, np.sort(np.random.default_rng(99).choice(65536, 2048, replace=False)))
    assert bench.cpu_subset(2, 2048).shape == (2048,) and bench.cpu_subset(4, 1024).shape == (64,)


@pytest.mark.parametrize("m,q,naive", [(1, 8, 0), (37, 8, 0), (64, 8, 1), (101, 4, 0), (300, 16, 0), (257, 3, 0)])
def test_expand_records_host(m, q, naive):
    """tb_expand_records (host threads, no device) rebuilds the 48-byte CELL_DTYPE stream of tb_records from
    the 8-byte (numerator, n3) compact stream: i, j from the tile order, n1/n2 per row, n_d from result.py:42,
    for any tile sub-range and thread count."""
    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.engine import CELL_DTYPE
    from paper_1704_03767_b200.pairindex import JobSpace

    rng = np.random.default_rng(m * 31 + q)
    n = 50
    n0 = n * (n - 1) // 2
    space = JobSpace(m, q)
    n1 = rng.integers(0, n0 // 3, m).astype(np.uint64)
    n1[rng.integers(0, m)] = n0  # a constant row
    lib = _lib.load()
    tt = space.total_tiles
    for lo, hi in ((0, tt), (tt // 3, tt // 3 + max(1, tt // 4)), (tt - 1, tt)):
        ii, jj = space.cells_in_tile_order(lo, hi)
        k = ii.size
        n3 = rng.integers(0, 40, k).astype(np.int64)
        nd = rng.integers(0, 200, k).astype(np.int64)
        num = (n0 - n1[ii].astype(np.int64) - n1[jj].astype(np.int64) + n3 - 2 * nd).astype(np.int32)
        exp = np.zeros(k, CELL_DTYPE)
        exp["i"], exp["j"], exp["numerator"] = ii, jj, num
        if not naive:
            exp["n_d"], exp["n1"], exp["n2"], exp["n3"] = nd, n1[ii], n1[jj], n3
        compact = np.empty((k, 2), np.uint32)
        compact[:, 0] = num.view(np.uint32)
        compact[:, 1] = 0 if naive else n3
        for nthreads in (1, 4):
            buf = np.zeros(k * 48 + 16, np.uint8)
            off = (-buf.ctypes.data) % 16
            out = buf[off:off + k * 48]
            rc = lib.tb_expand_records(compact.ctypes.data, n1.ctypes.data, m, n, q, lo, hi - lo, naive,
                                       out.ctypes.data, nthreads)
            assert rc == 0, lib.tb_last_error()
            assert out.tobytes() == exp.tobytes(), (lo, hi, nthreads)


def test_expand_ring_host():
    """tb_expand_ring (host threads, no device): a compact stream expanded pass by pass into a ring of pass
    buffers, in two batches, while a consumer takes each pass (tb_ring_wait) and releases its slot -- the
    concatenated passes are the reference CELL_DTYPE stream; the abort flag ends a blocked call."""
    import threading
    import time

    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.engine import CELL_DTYPE
    from paper_1704_03767_b200.pairindex import JobSpace

    lib = _lib.load()
    m, q, n = 301, 4, 50
    n0 = n * (n - 1) // 2
    rng = np.random.default_rng(1)
    space = JobSpace(m, q)
    n1 = rng.integers(0, n0 // 3, m).astype(np.uint64)
    lo, hi = 5, space.total_tiles
    ii, jj = space.cells_in_tile_order(lo, hi)
    k = ii.size
    n3 = rng.integers(0, 40, k).astype(np.int64)
    nd = rng.integers(0, 200, k).astype(np.int64)
    num = (n0 - n1[ii].astype(np.int64) - n1[jj].astype(np.int64) + n3 - 2 * nd).astype(np.int32)
    exp = np.zeros(k, CELL_DTYPE)
    exp["i"], exp["j"], exp["numerator"] = ii, jj, num
    exp["n_d"], exp["n1"], exp["n2"], exp["n3"] = nd, n1[ii], n1[jj], n3
    compact = np.empty((k, 2), np.uint32)
    compact[:, 0] = num.view(np.uint32)
    compact[:, 1] = n3
    bounds = np.array(list(range(lo, hi, 37)) + [hi], np.int64)
    npass = bounds.size - 1
    cells = [int(lib.tb_tile_cells(m, q, int(a), int(b))) for a, b in zip(bounds[:-1], bounds[1:])]
    assert sum(cells) == k
    slot = (max(cells) * 48 + 63) // 64 * 64
    for R, nthreads in ((1, 1), (3, 4)):
        raw = np.zeros(R * slot + 64, np.uint8)
        off = (-raw.ctypes.data) % 64
        ring = raw[off:off + R * slot]
        ctl = np.zeros(3, np.int64)
        got = []

        def consumer():
            for p in range(npass):
                assert lib.tb_ring_wait(ctl.ctypes.data, p) == 0
                got.append(ring[(p % R) * slot:(p % R) * slot + cells[p] * 48].tobytes())
                time.sleep(0.0002)
                ctl[1] = p + 1

        t = threading.Thread(target=consumer)
        t.start()
        h = npass // 2
        args = (n1.ctypes.data, None, None, 0, m, n, q)
        rc = lib.tb_expand_ring(compact.ctypes.data, 8, *args, bounds.ctypes.data, h, 0, ring.ctypes.data, slot, R, 0,
                                ctl.ctypes.data, nthreads)
        assert rc == 0, lib.tb_last_error()
        rc = lib.tb_expand_ring(compact.ctypes.data + 8 * sum(cells[:h]), 8, *args, bounds[h:].ctypes.data, npass - h, 0,
                                ring.ctypes.data, slot, R, h, ctl.ctypes.data, nthreads)
        assert rc == 0, lib.tb_last_error()
        t.join()
        assert b"".join(got) == exp.tobytes()
    # nobody releases: the call blocks on a full ring until the abort flag is raised
    ctl = np.zeros(3, np.int64)
    threading.Timer(0.05, lambda: ctl.__setitem__(2, 1)).start()
    rc = lib.tb_expand_ring(compact.ctypes.data, 8, n1.ctypes.data, None, None, 0, m, n, q, bounds.ctypes.data, npass, 0,
                            ring.ctypes.data, slot, R, 0, ctl.ctypes.data, 4)
    assert rc == _lib.TB_ERR_ABORTED
    assert lib.tb_ring_wait(ctl.ctypes.data, 10 ** 6) == _lib.TB_ERR_ABORTED
    # a pass larger than the ring slot is refused
    ctl[:] = 0
    rc = lib.tb_expand_ring(compact.ctypes.data, 8, n1.ctypes.data, None, None, 0, m, n, q, bounds.ctypes.data, npass, 0,
                            ring.ctypes.data, 48, R, 0, ctl.ctypes.data, 1)
    assert rc == _lib.TB_ERR_CAPACITY


def test_expand_records_after_fork():
    """The host expansion pool survives fork(): a child process that expands after the parent did builds its
    own workers instead of waiting on the parent's (which it does not have)."""
    import multiprocessing as mp

    from paper_1704_03767_b200 import _lib
    lib = _lib.load()
    m, q, n = 40, 4, 30
    from paper_1704_03767_b200.pairindex import JobSpace
    tt = JobSpace(m, q).total_tiles
    cells = int(lib.tb_tile_cells(m, q, 0, tt))
    compact = np.zeros((cells, 2), np.uint32)
    n1 = np.zeros(m, np.uint64)
    out = np.zeros(cells * 48 + 16, np.uint8)
    off = (-out.ctypes.data) % 16
    assert lib.tb_expand_records(compact.ctypes.data, n1.ctypes.data, m, n, q, 0, tt, 0, out.ctypes.data + off, 4) == 0
    ctx = mp.get_context("fork")
    p = ctx.Process(target=_expand_child, args=(m, q, n, tt, cells))
    p.start()
    p.join(60)
    assert p.exitcode == 0


def _expand_child(m, q, n, tt, cells):
    from paper_1704_03767_b200 import _lib
    lib = _lib.load()
    compact = np.zeros((cells, 2), np.uint32)
    n1 = np.zeros(m, np.uint64)
    out = np.zeros(cells * 48 + 16, np.uint8)
    off = (-out.ctypes.data) % 16
    rc = lib.tb_expand_records(compact.ctypes.data, n1.ctypes.data, m, n, q, 0, tt, 0, out.ctypes.data + off, 4)
    raise SystemExit(0 if rc == 0 else 1)


@pytest.mark.parametrize("m,q,naive", [(37, 8, 0), (101, 4, 0), (64, 8, 1), (257, 3, 0)])
def test_expand_records_num_host(m, q, naive):
    """tb_expand_records_num: 48-byte records from a 4-byte numerator stream, n3 from the tied rows' table
    (zero for any pair with an untied variable), for any tile sub-range and thread count."""
    from paper_1704_03767_b200 import _lib
    from paper_1704_03767_b200.engine import CELL_DTYPE
    from paper_1704_03767_b200.pairindex import JobSpace

    rng = np.random.default_rng(m * 7 + q)
    n = 60
    n0 = n * (n - 1) // 2
    space = JobSpace(m, q)
    tied = np.sort(rng.choice(m, m // 5, replace=False))
    n1 = np.zeros(m, np.uint64)
    n1[tied] = rng.integers(1, 50, tied.size)
    tidx = np.full(m, -1, np.int32)
    tidx[tied] = np.arange(tied.size, dtype=np.int32)
    nt = tied.size
    n3t = rng.integers(0, 9, nt * (nt + 1) // 2).astype(np.int64)
    lib = _lib.load()
    tt = space.total_tiles
    for lo, hi in ((0, tt), (tt // 4, tt // 4 + max(1, tt // 3)), (tt - 1, tt)):
        ii, jj = space.cells_in_tile_order(lo, hi)
        a, b = tidx[ii].astype(np.int64), tidx[jj].astype(np.int64)
        both = (a >= 0) & (b >= 0)
        n3 = np.where(both, n3t[np.where(both, a * (2 * nt - a + 1) // 2 + b - a, 0)], 0)
        nd = rng.integers(0, 300, ii.size)
        num = (n0 - n1[ii].astype(np.int64) - n1[jj].astype(np.int64) + n3 - 2 * nd).astype(np.int32)
        exp = np.zeros(ii.size, CELL_DTYPE)
        exp["i"], exp["j"], exp["numerator"] = ii, jj, num
        if not naive:
            exp["n_d"], exp["n1"], exp["n2"], exp["n3"] = nd, n1[ii], n1[jj], n3
        for nthreads in (1, 5):
            buf = np.zeros(ii.size * 48 + 16, np.uint8)
            off = (-buf.ctypes.data) % 16
            out = buf[off:off + ii.size * 48]
            rc = lib.tb_expand_records_num(num.ctypes.data, n1.ctypes.data, tidx.ctypes.data, n3t.ctypes.data, nt,
                                           m, n, q, lo, hi - lo, naive, out.ctypes.data, nthreads)
            assert rc == 0, lib.tb_last_error()
            assert out.tobytes() == exp.tobytes(), (lo, hi, nthreads)
