"""Pin the CPU oracle against the reference's own outputs (tests/golden/).

The fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  Everything here is CPU-only.
"""
import hashlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle
from paper_2410_01231_b200 import synth


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CASES = ["unif", "unif_self", "lattice", "dups", "gauss_d33", "m1"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("strategy", ["rng", "alpha"])
def test_oracle_prune_matches_reference_cases(golden_cases, name, strategy):
    g = golden_cases
    data = g[f"{name}_data"]
    M = int(g[f"{name}_M"])
    alpha = float(g[f"{name}_alpha"]) if strategy == "alpha" else 60.0
    a = oracle.prune_all(data, g[f"{name}_off"], g[f"{name}_counts"], g[f"{name}_ids"],
                         g[f"{name}_dists"], M, strategy, alpha)
    b = oracle.add_reverse_and_prune(data, a[0], a[1], a[2], M, strategy, alpha)
    for ph, res in (("a", a), ("b", b)):
        p = f"{name}_{strategy}_{ph}_"
        np.testing.assert_array_equal(res[0], g[p + "ids"])
        np.testing.assert_array_equal(res[1], g[p + "dists"])
        np.testing.assert_array_equal(res[2], g[p + "counts"])
        assert res[3] == int(g[p + "de"]) and res[4] == int(g[p + "ae"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_slack_one_is_the_reference_rng_rule(golden_cases, name):
    """The "slack" extension (no reference equivalent) anchors to the
    reference at s = 1: it must give the reference's own "rng" outputs on
    every edge case (ties, duplicates, self entries, empty rows); s > 1 keeps
    a superset-leaning degree (more edges survive)."""
    g = golden_cases
    data = g[f"{name}_data"]
    M = int(g[f"{name}_M"])
    a = oracle.prune_all(data, g[f"{name}_off"], g[f"{name}_counts"], g[f"{name}_ids"],
                         g[f"{name}_dists"], M, "slack", 1.0)
    b = oracle.add_reverse_and_prune(data, a[0], a[1], a[2], M, "slack", 1.0)
    for ph, res in (("a", a), ("b", b)):
        p = f"{name}_rng_{ph}_"
        np.testing.assert_array_equal(res[0], g[p + "ids"])
        np.testing.assert_array_equal(res[2], g[p + "counts"])
        assert res[3] == int(g[p + "de"])
    a2 = oracle.prune_all(data, g[f"{name}_off"], g[f"{name}_counts"], g[f"{name}_ids"],
                          g[f"{name}_dists"], M, "slack", 1.5)
    assert a2[2].sum() >= a[2].sum()


@pytest.mark.parametrize("name", CASES)
def test_oracle_pool_matches_reference_cases(golden_cases, name):
    g = golden_cases
    data = g[f"{name}_data"]
    truth = g[f"{name}_truth"]
    ids, _ = oracle.knn_pool_ids(data, truth.shape[1], True)
    np.testing.assert_array_equal(ids, truth)
    np.testing.assert_array_equal(oracle.ground_truth_table(data, truth.shape[1], True), truth)


def test_oracle_triangle(golden_cases):
    g = golden_cases
    pts = g["tri_data"]
    assert oracle.squared_l2(pts[1], pts[0]) == float(g["tri_d01"])
    assert oracle.squared_l2(pts[2], pts[0]) == float(g["tri_d02"])
    ids = np.array([1, 2], np.int32)
    d = np.array([g["tri_d01"], g["tri_d02"]], np.float32)
    off = np.array([0, 2, 2, 2], np.int64)
    cnt = np.array([2, 0, 0], np.int32)
    for strategy, alpha, want in (("alpha", 120.0, [1]), ("alpha", 150.0, [1, 2]),
                                  ("rng", 60.0, [1])):
        r = oracle.prune_all(pts, off, cnt, ids, d, 2, strategy, alpha)
        assert r[0][0, :r[2][0]].tolist() == want


CONFIGS = {
    "cfg1_2k": lambda: synth.cfg1(2_000),
    "cfg1_full": lambda: synth.cfg1(10_000),
    "cfg2_4k": lambda: synth.cfg2(4_000),
    "cfg3_2k": lambda: synth.cfg3(2_000),
    "cfg4_2k": lambda: synth.cfg4(2_000),
}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_oracle_composition_matches_reference(name):
    g = load_golden(name)
    data = CONFIGS[name]()
    assert sha(data) == str(g["data_digest"]), "synthetic recipe drifted"
    K, R = int(g["meta_K"]), int(g["meta_R"])
    truth, _ = oracle.knn_pool_ids(data, K, True)
    assert sha(truth) == str(g["truth__sha256"])
    ids, dists = oracle.list_dists_sorted(data, truth)
    assert sha(ids) == str(g["pool_ids__sha256"])
    assert sha(dists) == str(g["pool_dists__sha256"])
    for tag, strategy, alpha in (("rng", "rng", 60.0), ("a66", "alpha", 66.0)):
        a, b = oracle.refine_ab(data, ids, dists, R, strategy, alpha)
        for ph, res in (("a", a), ("b", b)):
            p = f"{tag}_{ph}_"
            assert sha(res[0]) == str(g[p + "ids__sha256"]), p
            assert sha(res[1]) == str(g[p + "dists__sha256"]), p
            assert sha(res[2]) == str(g[p + "counts__sha256"]), p
            assert res[3] == int(g[p + "de"]) and res[4] == int(g[p + "ae"]), p


def _search_golden():
    import numpy as np
    from pathlib import Path
    return np.load(Path(__file__).resolve().parent / "golden" / "search.npz", allow_pickle=False)


def test_oracle_search_and_connect_match_reference():
    """Beam search (search_batch, kann_search) and phase C (entry_point +
    _connect via finish_refine) of the oracle restatement equal the reference's
    outputs (tests/golden/search.npz, made by make_golden.py search)."""
    import numpy as np
    g = _search_golden()
    for name in g["names"]:
        data = g[f"{name}_data"]
        M = int(g[f"{name}_R"])
        adj, cnt, ep, over = oracle.finish_connect(data, g[f"{name}_b_ids"],
                                                   g[f"{name}_b_counts"], M)
        assert ep == int(g[f"{name}_c_ep"]), name
        np.testing.assert_array_equal(adj, g[f"{name}_c_adj"], err_msg=name)
        np.testing.assert_array_equal(cnt, g[f"{name}_c_counts"], err_msg=name)
        np.testing.assert_array_equal(over, g[f"{name}_c_over"], err_msg=name)
        q = g[f"{name}_queries"]
        for tag, k, L in (("k10L40", 10, 40), ("k1L16", 1, 16)):
            ids, d, dc = oracle.search_batch(data, adj, cnt, q, k, L, ep)
            np.testing.assert_array_equal(ids, g[f"{name}_{tag}_ids"], err_msg=name)
            np.testing.assert_array_equal(d, g[f"{name}_{tag}_dists"], err_msg=name)
            np.testing.assert_array_equal(dc, g[f"{name}_{tag}_dcount"], err_msg=name)
        ki, kd, _ = oracle.search_batch(data, adj, cnt, q[0], 5, 24, data.shape[0] // 2)
        m = len(g[f"{name}_kann_ids"])
        np.testing.assert_array_equal(ki[0, :m], g[f"{name}_kann_ids"])
        np.testing.assert_array_equal(kd[0, :m], g[f"{name}_kann_dists"])


def test_oracle_row_subset_reprune_equals_full():
    """add_reverse_and_prune(rows=...) (the seeded-row check used at full
    config sizes) returns exactly the full re-prune's rows for those rows, and
    phase A on a masked CSR exactly the full phase A's."""
    data = synth.cfg1(3000)
    ids, dists = oracle.knn_pools(data, 32)
    n = data.shape[0]
    off = np.arange(n + 1, dtype=np.int64) * 32
    cnt = np.full(n, 32, np.int32)
    a = oracle.prune_all(data, off, cnt, ids.ravel(), dists.ravel(), 16, "alpha", 66.0)
    sel = np.sort(np.random.default_rng(5).choice(n, 300, replace=False))
    masked = np.zeros(n, np.int32)
    masked[sel] = 32
    a_sel = oracle.prune_all(data, off, masked, ids.ravel(), dists.ravel(), 16, "alpha", 66.0)
    for k in range(3):
        np.testing.assert_array_equal(a_sel[k][sel], a[k][sel])
    full = oracle.add_reverse_and_prune(data, a[0], a[1], a[2], 16, "alpha", 66.0)
    part = oracle.add_reverse_and_prune(data, a[0], a[1], a[2], 16, "alpha", 66.0, rows=sel)
    for k in range(3):
        np.testing.assert_array_equal(part[k][sel], full[k][sel])
    assert part[3] < full[3] and (part[2][np.setdiff1d(np.arange(n), sel)] == 0).all()
