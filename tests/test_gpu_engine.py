"""The drop-in engine (compute_all_pairs) on the device vs the reference's byte streams.

Golden streams are the reference BinaryWriter output of
taucorr.compute_all_pairs(synth_dataset(...), "sorted", tile_size=q)
(oracle/gen_golden.py:gen_engine); identical bytes prove record order,
counts, the n_d sentinel and shard concatenation.
"""

from __future__ import annotations

import hashlib
import io
import logging

import numpy as np
import pytest

from conftest import gold_path, load_json

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def _stream(ds, kernel, q, **kw):
    import paper_1704_03767_b200 as tb
    s = io.BytesIO()
    tb.compute_all_pairs(ds, kernel, tile_size=q, sink=tb.BinaryWriter(s, ds.n), **kw)
    return s.getvalue()


@pytest.mark.parametrize("kernel", ["sorted", "vectorized", "gemm", "merge", "auto"])
def test_streams_match_reference(kernel):
    import paper_1704_03767_b200 as tb
    gold = load_json("engine_streams.json")
    for (m, n, tie, seed) in [(64, 48, 0.3, 512), (13, 10, 0.2, 1), (512, 48, 0.3, 512)]:
        ds = tb.synth_dataset(m, n, tie_fraction=tie, seed=seed)
        assert hashlib.sha256(ds.ranks.tobytes()).hexdigest() == gold[f"synth_m{m}_n{n}_t{tie}_s{seed}_sha256"]
        for q in (1, 3, 4, 8):
            if m == 512 and q == 1 and kernel != "sorted":
                continue
            blob = _stream(ds, kernel, q)
            assert hashlib.sha256(blob).hexdigest() == gold[f"m{m}_n{n}_t{tie}_s{seed}_q{q}"], (kernel, m, q)
    with open(gold_path("stream_m64_n48_t0.3_s512_q4.bin"), "rb") as fh:
        ref = fh.read()
    assert _stream(tb.synth_dataset(64, 48, 0.3, 512), kernel, 4, pass_tiles=7) == ref


def test_shards_concatenate_and_invariance():
    import paper_1704_03767_b200 as tb
    ds = tb.synth_dataset(512, 48, tie_fraction=0.3, seed=512)
    full = _stream(ds, "sorted", 4)
    parts = b"".join(_stream(ds, "sorted", 4, shard=(i, 4), workers=2) for i in range(4))
    assert parts == full
    for workers in (1, 4):
        for pass_tiles in (7, 4096):
            for overlap in (True, False):
                assert _stream(ds, "sorted", 4, workers=workers, pass_tiles=pass_tiles, overlap=overlap) == full


def test_naive_semantics_and_fallback(caplog):
    import paper_1704_03767_b200 as tb
    ds = tb.synth_dataset(17, 30, tie_fraction=0.3, seed=5)
    chunks = []
    tb.compute_all_pairs(ds, "naive", tile_size=4, sink=lambda r: chunks.append(r.copy()))
    nv = np.concatenate(chunks)
    chunks = []
    tb.compute_all_pairs(ds, "sorted", tile_size=4, sink=lambda r: chunks.append(r.copy()))
    so = np.concatenate(chunks)
    assert np.array_equal(nv["numerator"], so["numerator"])
    assert (nv["n_d"] == 0).all() and (nv["n1"] == 0).all() and (nv["n3"] == 0).all()
    ranks = np.array([[0, 40000, 2, 3], [3, 2, 1, 0]], dtype=np.int32)
    ds2 = tb.Dataset(labels=["a", "b"], ranks=ranks)
    with caplog.at_level(logging.WARNING, logger="taucorr"):
        summary = tb.compute_all_pairs(ds2, "vectorized", tile_size=2)
    assert summary.kernel == "sorted" and summary.requested_kernel == "vectorized"
    assert any("falling back" in r.message for r in caplog.records)


def test_tsv_matches_reference():
    import paper_1704_03767_b200 as tb
    gold = load_json("engine_streams.json")
    ds = tb.synth_dataset(6, 9, tie_fraction=0.4, seed=12)
    s = io.StringIO()
    tb.compute_all_pairs(ds, "sorted", tile_size=2, sink=tb.TsvWriter(s, ds.labels, ds.n))
    assert s.getvalue() == gold["tsv_m6_n9_t0.4_s12_q2"]


def test_sink_failure_propagates():
    import paper_1704_03767_b200 as tb
    ds = tb.synth_dataset(12, 8, seed=10)

    def broken(_):
        raise OSError("disk full")

    with pytest.raises(OSError, match="disk full"):
        tb.compute_all_pairs(ds, "sorted", tile_size=2, pass_tiles=2, sink=broken)


@pytest.mark.parametrize("kernel", ["sorted", "gemm"])
def test_devices_split_matches_reference_stream(kernel):
    """compute_all_pairs(devices=[...]) splits the job range across GPUs (here the same GPU listed
    twice / three times) and still produces the reference byte stream, also per shard."""
    import paper_1704_03767_b200 as tb
    gold = load_json("engine_streams.json")
    ds = tb.synth_dataset(512, 48, tie_fraction=0.3, seed=512)
    for devs in ([0, 0], [0, 0, 0]):
        blob = _stream(ds, kernel, 4, devices=devs, pass_tiles=97)
        assert hashlib.sha256(blob).hexdigest() == gold["m512_n48_t0.3_s512_q4"], (kernel, devs)
    full = _stream(ds, kernel, 4)
    parts = b"".join(_stream(ds, kernel, 4, shard=(i, 3), devices=[0, 0]) for i in range(3))
    assert parts == full
    with pytest.raises(tb.ConfigError):
        tb.compute_all_pairs(ds, kernel, device=0, devices=[0])
