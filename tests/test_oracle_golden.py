"""Pin the CPU oracle (oracle/) against the reference's own golden vectors."""

import math

import numpy as np

from conftest import load_json, load_npz, split_pairs


def test_kats(oracle):
    k = load_json("kats.json")
    t = k["tied_example"]
    nd, n1, n2, n3 = oracle.sorted_counts(t["u"], t["v"])
    assert (nd, n1, n2, n3) == (t["n_d"], t["n1"], t["n2"], t["n3"])
    num = oracle.numerator_from_counts(3, nd, n1, n2, n3)
    assert num == t["numerator"] == 1
    ta, tb = oracle.derive_taus([num], [n1], [n2], 3)
    assert tb[0] == t["tau_b"] == 0.5
    r = k["reversal4"]
    c = oracle.sorted_counts(r["u"], r["v"])
    assert c[0] == r["n_d"] == 6
    assert oracle.numerator_from_counts(4, *c) == r["numerator"] == -6
    th = k["third"]
    assert oracle.naive_numerator(th["u"], th["v"]) == th["numerator"] == 1
    c = k["constant"]
    cc = oracle.sorted_counts(c["u"], c["v"])
    ta, tb = oracle.derive_taus([oracle.numerator_from_counts(4, *cc)], [cc[1]], [cc[2]], 4)
    assert math.isnan(tb[0]) and not c["defined_b"]
    for vals, expected in k["rank_transform"]:
        assert oracle.rank_transform(np.array(vals)).tolist() == expected


def test_corpus_vs_reference(oracle):
    z = load_npz("corpus.npz")
    counts = z["counts"]
    brute = z["brute"]
    for u, v, k in split_pairs(z):
        c = oracle.sorted_counts(u, v)
        assert c == tuple(counts[k, :4]), k
        p = oracle.packed_counts(u, v)
        assert p == c
        b = oracle.pair_scan(u, v)
        assert (b["nc"], b["n_d"], b["n1"], b["n2"], b["n3"]) == tuple(brute[k])
        num = oracle.numerator_from_counts(len(u), *c)
        assert num == counts[k, 4]
        if c[1] == 0 and c[2] == 0:
            assert oracle.naive_numerator(u, v) == num
    # bit-exact tau against the reference finalize
    n = z["n"]
    ta = np.empty(len(n))
    tb = np.empty(len(n))
    for k in range(len(n)):
        a, b = oracle.derive_taus([counts[k, 4]], [counts[k, 1]], [counts[k, 2]], int(n[k]))
        ta[k], tb[k] = a[0], b[0]
    np.testing.assert_array_equal(ta, z["tau_a"])
    np.testing.assert_array_equal(tb, z["tau_b"])


def test_boundary_vs_reference(oracle):
    z = load_npz("boundary.npz")
    for u, v, k in split_pairs(z):
        c = oracle.sorted_counts(u, v)
        assert c == tuple(z["counts"][k, :4])
        assert oracle.packed_counts(u, v) == c


def test_bijection_vs_reference(oracle):
    z = load_npz("bijection.npz")
    for key in z.files:
        if not key.endswith("_j"):
            continue
        m = int(key[1:-2])
        yx = z[key[:-2] + "_yx"]
        for j, (y, x) in zip(z[key].tolist()[:300], yx.tolist()[:300]):
            assert oracle.job_coord(j, m) == (y, x)
            assert oracle.row_prefix(y, m) + x - y == j


def test_config1_full_vs_reference(oracle):
    """Config 1 (256x200) every cell, threaded oracle vs reference engine records."""
    from paper_1704_03767_b200 import workloads

    z = load_npz("config1.npz")
    x = workloads.generate(1)
    import hashlib
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["x_sha256"])
    ranks = oracle.rank_matrix(x)
    assert hashlib.sha256(ranks.tobytes()).hexdigest() == str(z["ranks_sha256"])
    num, counts = oracle.all_pairs(ranks, z["pi"], z["pj"], oracle.KERNEL_PACKED, threads=4)
    np.testing.assert_array_equal(num, z["numerator"])
    np.testing.assert_array_equal(counts, z["counts"])
    ta, tb = oracle.derive_taus(num, counts[:, 1], counts[:, 2], int(z["n"]))
    np.testing.assert_array_equal(ta, z["tau_a"])
    np.testing.assert_array_equal(tb, z["tau_b"])


def test_config_samples_vs_reference(oracle):
    """Configs 2, 3 sampled pairs (configs 4/5 generation is too heavy for the CPU suite)."""
    import hashlib
    from paper_1704_03767_b200 import workloads

    for k in (2, 3):
        z = load_npz(f"config{k}.npz")
        x = workloads.generate(k)
        assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["x_sha256"])
        pi, pj = z["pi"][:400], z["pj"][:400]
        rows = np.unique(np.concatenate([pi, pj]))
        ranks = np.zeros(x.shape, np.int32)
        for r in rows:
            ranks[r] = oracle.rank_transform(x[r])
        num, counts = oracle.all_pairs(ranks, pi, pj, oracle.KERNEL_SORTED, threads=4)
        np.testing.assert_array_equal(counts, z["counts"][:400])
        np.testing.assert_array_equal(num, z["numerator"][:400])
