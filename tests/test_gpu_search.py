"""GPU parity for the beam search and phase C: the
CUDA path against the reference's own outputs (tests/golden/search.npz) and
the pinned oracle restatement at larger sizes.  Exact: ids, fp32 distances,
distance counts, entry points, appended edges and widened widths."""
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle
from paper_2410_01231_b200 import (Dataset, ProximityGraph, PruneParams, entry_point,
                                   finish_refine, kann_search, knn_pools, prune_all, refine,
                                   search_batch, synth)

pytestmark = pytest.mark.gpu

G = np.load(Path(__file__).resolve().parent / "golden" / "search.npz", allow_pickle=False)
NAMES = [str(x) for x in G["names"]]


@pytest.mark.parametrize("name", NAMES)
def test_search_batch_and_kann_search_match_reference(name):
    data = G[f"{name}_data"]
    ds = Dataset.from_array(data)
    g = ProximityGraph(adj=G[f"{name}_c_adj"], counts=G[f"{name}_c_counts"],
                       M=int(G[f"{name}_R"]), ep=int(G[f"{name}_c_ep"]))
    q = G[f"{name}_queries"]
    for tag, k, L in (("k10L40", 10, 40), ("k1L16", 1, 16)):
        ids, d, dc = search_batch(ds, g, q, k, L)
        np.testing.assert_array_equal(ids, G[f"{name}_{tag}_ids"])
        np.testing.assert_array_equal(d, G[f"{name}_{tag}_dists"])
        np.testing.assert_array_equal(dc, G[f"{name}_{tag}_dcount"])
    ki, kd = kann_search(ds, g, q[0], 5, 24, ep=ds.n // 2)
    np.testing.assert_array_equal(ki, G[f"{name}_kann_ids"])
    np.testing.assert_array_equal(kd, G[f"{name}_kann_dists"])


@pytest.mark.parametrize("name", NAMES)
def test_entry_point_and_connect_match_reference(name):
    data = G[f"{name}_data"]
    ds = Dataset.from_array(data)
    M = int(G[f"{name}_R"])
    interim = ProximityGraph(adj=G[f"{name}_b_ids"], counts=G[f"{name}_b_counts"], M=M, ep=0)
    assert entry_point(ds, interim, k=1, L=max(M + 1, 32), seed=0) == int(G[f"{name}_ep"])
    # phase C from the phase-B graph (finish_refine's tail), via the public call
    K = int(G[f"{name}_K"])
    strategy, alpha = str(G[f"{name}_strategy"]), float(G[f"{name}_alpha"])
    ids, dists = knn_pools(ds, K)
    off = np.arange(ds.n + 1, dtype=np.int64) * K
    cnt = np.full(ds.n, K, np.int32)
    params = PruneParams(M=M, alpha=alpha, strategy=strategy)
    a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), params)
    gr = finish_refine(ds, a[0], a[1], a[2], params, connect=True, ep=None, seed=0)
    assert gr.ep == int(G[f"{name}_c_ep"])
    np.testing.assert_array_equal(gr.adj, G[f"{name}_c_adj"])
    np.testing.assert_array_equal(gr.counts, G[f"{name}_c_counts"])
    np.testing.assert_array_equal(gr.over_cap, G[f"{name}_c_over"])
    gr.validate()
    # refine end to end gives the same graph
    g2 = refine(ds, off, cnt, ids.ravel(), dists.ravel(), params, connect=True, ep=None)
    np.testing.assert_array_equal(g2.adj, gr.adj)


def test_search_errors_follow_reference():
    data = G["cfg1_2k_data"]
    ds = Dataset.from_array(data)
    g = ProximityGraph(adj=G["cfg1_2k_c_adj"], counts=G["cfg1_2k_c_counts"], M=24,
                       ep=int(G["cfg1_2k_c_ep"]))
    with pytest.raises(ValueError, match="k must not exceed"):
        kann_search(ds, g, data[0], 20, 10)
    with pytest.raises(ValueError, match="entry point"):
        kann_search(ds, g, data[0], 1, 10, ep=ds.n)
    with pytest.raises(ValueError, match="query must have shape"):
        kann_search(ds, g, data[0, :5], 1, 10)
    with pytest.raises(ValueError, match="queries must be"):
        search_batch(ds, g, data[0], 1, 10)


def test_phase_c_and_search_at_scale_against_oracle():
    """cfg2 100k and a split two-half set (exact-integer path): phase C and a
    2,000-query batch search equal the oracle restatement bit-for-bit."""
    rng = np.random.default_rng(5)
    # two halves 128 apart per dimension: phase B leaves them disconnected
    half = np.floor(synth.cfg2(20_000) / 2.0)
    split = np.vstack([half, half + 128.0]).astype(np.float32)
    for data, K, R in ((synth.cfg2(100_000), 32, 16), (split, 16, 8)):
        ds = Dataset.from_array(data)
        ids, dists = knn_pools(ds, K)
        off = np.arange(ds.n + 1, dtype=np.int64) * K
        cnt = np.full(ds.n, K, np.int32)
        params = PruneParams(M=R)
        a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), params)
        from paper_2410_01231_b200 import add_reverse_and_prune
        b = add_reverse_and_prune(ds, a[0], a[1], a[2], params)
        gr = finish_refine(ds, a[0], a[1], a[2], params, connect=True, ep=None, seed=3)
        o_adj, o_cnt, o_ep, o_over = oracle.finish_connect(data, b[0], b[2], R, seed=3)
        assert gr.ep == o_ep
        np.testing.assert_array_equal(gr.adj, o_adj)
        np.testing.assert_array_equal(gr.counts, o_cnt)
        np.testing.assert_array_equal(gr.over_cap, o_over)
        q = data[rng.choice(ds.n, 2000, replace=False)] + rng.normal(0, 2, (2000, 128)).astype(
            np.float32)
        s_ids, s_d, s_dc = search_batch(ds, gr, q, 10, 64)
        o_ids, o_d, o_dc = oracle.search_batch(data, o_adj, o_cnt, q, 10, 64, o_ep)
        np.testing.assert_array_equal(s_ids, o_ids)
        np.testing.assert_array_equal(s_d, o_d)
        np.testing.assert_array_equal(s_dc, o_dc)


@pytest.mark.parametrize("n,d", [(100_000, 33), (20_000, 960)])
def test_centroid_equals_numpy_mean_bit_for_bit(n, d):
    """core.centroid (core.py:153-155): numpy's float64 mean over axis 0 (rows
    added in order), cast to fp32 -- on heavy-tailed float data, where a
    different summation order would change the last ulp."""
    import torch
    from paper_2410_01231_b200 import kernels
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((n, d)) * rng.uniform(0.1, 1000, (n, 1))).astype(np.float32)
    got = kernels.centroid(torch.from_numpy(x).cuda()).cpu().numpy()
    want = x.mean(axis=0, dtype=np.float64).astype(np.float32)
    np.testing.assert_array_equal(got, want)
