"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
outputs and the pinned CPU oracle.  Integer / index work must be bit-exact;
list distances must equal the reference's fp32 squared_l2 bit-for-bit (the
north star's 1e-5 relative tolerance is checked too, as the weaker bound)."""
import hashlib

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import oracle
from paper_2410_01231_b200 import (Dataset, PruneParams, add_reverse_and_prune, alpha_prune,
                                   ground_truth_table, knn_pools, prune_all, refine,
                                   rng_prune, synth)
from paper_2410_01231_b200 import kernels

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5  # north_star: pairwise distances within 1e-5 relative


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CASES = ["unif", "unif_self", "lattice", "dups", "gauss_d33", "m1"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("strategy", ["rng", "alpha"])
def test_prune_phases_match_reference_cases(golden_cases, name, strategy):
    g = golden_cases
    ds = Dataset.from_array(g[f"{name}_data"])
    M = int(g[f"{name}_M"])
    alpha = float(g[f"{name}_alpha"]) if strategy == "alpha" else 60.0
    params = PruneParams(M=M, alpha=alpha, strategy=strategy)
    a = prune_all(ds, g[f"{name}_off"], g[f"{name}_counts"], g[f"{name}_ids"],
                  g[f"{name}_dists"], params)
    b = add_reverse_and_prune(ds, a[0], a[1], a[2], params)
    for ph, res in (("a", a), ("b", b)):
        p = f"{name}_{strategy}_{ph}_"
        np.testing.assert_array_equal(res[0], g[p + "ids"])
        np.testing.assert_array_equal(res[1], g[p + "dists"])
        np.testing.assert_array_equal(res[2], g[p + "counts"])
        assert res[3] == int(g[p + "de"]) and res[4] == int(g[p + "ae"])


@pytest.mark.parametrize("name", CASES)
def test_ground_truth_table_matches_reference_cases(golden_cases, name):
    g = golden_cases
    ds = Dataset.from_array(g[f"{name}_data"])
    truth = g[f"{name}_truth"]
    np.testing.assert_array_equal(ground_truth_table(ds, None, k=truth.shape[1],
                                                     exclude_self=True), truth)


def test_hand_triangle_and_single_row_api(golden_cases):
    g = golden_cases
    pts = g["tri_data"]
    ds = Dataset.from_array(pts)
    ids = np.array([1, 2], np.int32)
    d = np.array([g["tri_d01"], g["tri_d02"]], np.float32)
    assert alpha_prune(ds, 0, ids, d, 2, 120.0)[0].tolist() == [1]
    assert alpha_prune(ds, 0, ids, d, 2, 150.0)[0].tolist() == [1, 2]
    assert rng_prune(ds, 0, ids, d, 2)[0].tolist() == [1]
    with pytest.raises(ValueError, match="ascending"):
        rng_prune(ds, 0, ids[::-1].copy(), d[::-1].copy(), 2)
    # coincident points (test_prune.py:123-146)
    pts = np.array([[0, 0], [0, 0], [1, 0], [0, 1]], np.float32)
    ds = Dataset.from_array(pts)
    assert rng_prune(ds, 0, np.array([1, 2, 3], np.int32),
                     np.array([0, 1, 1], np.float32), 3)[0].tolist() == [1]
    pts = np.array([[0, 0], [1, 0], [1, 0]], np.float32)
    ds = Dataset.from_array(pts)
    assert alpha_prune(ds, 0, np.array([1, 2], np.int32), np.array([1, 1], np.float32),
                       2, 179.0)[0].tolist() == [1]


def test_reverse_phase_adds_missing_backlink():
    pts = np.array([[0.0], [1.0], [2.1]], np.float32)
    ds = Dataset.from_array(pts)
    ids = np.full((3, 2), -1, np.int32)
    dists = np.full((3, 2), np.inf, np.float32)
    counts = np.zeros(3, np.int32)
    ids[1, 0], dists[1, 0], counts[1] = 0, 1.0, 1
    ids[2, 0], dists[2, 0], counts[2] = 1, oracle.squared_l2(pts[2], pts[1]), 1
    b_ids, _, b_counts, _, _ = add_reverse_and_prune(ds, ids, dists, counts,
                                                     PruneParams(M=2, strategy="rng"))
    assert 1 in b_ids[0, : b_counts[0]]
    assert 2 in b_ids[1, : b_counts[1]]


CONFIGS = {
    "cfg1_2k": lambda: synth.cfg1(2_000),
    "cfg1_full": lambda: synth.cfg1(10_000),
    "cfg2_4k": lambda: synth.cfg2(4_000),
    "cfg3_2k": lambda: synth.cfg3(2_000),
    "cfg4_2k": lambda: synth.cfg4(2_000),
}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_hot_path_matches_reference_configs(name):
    """pool -> phase A -> phase B against the reference's own outputs, exact."""
    g = load_golden(name)
    data = CONFIGS[name]()
    assert sha(data) == str(g["data_digest"])
    K, R = int(g["meta_K"]), int(g["meta_R"])
    ds = Dataset.from_array(data)
    ids, dists, gt = knn_pools(ds, K, want_gt=True)
    assert sha(gt) == str(g["truth__sha256"])
    assert sha(ids) == str(g["pool_ids__sha256"])
    assert sha(dists) == str(g["pool_dists__sha256"])
    n = ds.n
    off = np.arange(n + 1, dtype=np.int64) * K
    cnt = np.full(n, K, np.int32)
    for tag, params in (("rng", PruneParams(M=R)),
                        ("a66", PruneParams(M=R, alpha=66.0, strategy="alpha"))):
        a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), params)
        b = add_reverse_and_prune(ds, a[0], a[1], a[2], params)
        for ph, res in (("a", a), ("b", b)):
            p = f"{tag}_{ph}_"
            assert sha(res[0]) == str(g[p + "ids__sha256"]), p
            assert sha(res[1]) == str(g[p + "dists__sha256"]), p
            assert sha(res[2]) == str(g[p + "counts__sha256"]), p
            assert res[3] == int(g[p + "de"]) and res[4] == int(g[p + "ae"]), p
        graph = refine(ds, off, cnt, ids.ravel(), dists.ravel(), params, connect=False, ep=0)
        graph.validate()
        assert sha(graph.adj) == str(g[f"{tag}_b_ids__sha256"])


def _edge_agreement(a_ids, a_cnt, b_ids, b_cnt):
    n = a_ids.shape[0]
    ea = {(u, int(v)) for u in range(n) for v in a_ids[u, :a_cnt[u]]}
    eb = {(u, int(v)) for u in range(n) for v in b_ids[u, :b_cnt[u]]}
    return len(ea & eb) / max(1, len(ea | eb))


@pytest.mark.parametrize("gen,n,K,R", [(synth.cfg2, 20_000, 128, 32),
                                       (synth.cfg1, 10_000, 64, 24),
                                       (synth.cfg3, 6_000, 128, 32)])
def test_larger_prefixes_against_oracle(gen, n, K, R):
    """Bigger seeded prefixes: the CUDA path vs the oracle, exact."""
    data = gen(n)
    ds = Dataset.from_array(data)
    ids, dists = knn_pools(ds, K)
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(n, 300, replace=False))
    o_ids, o_d = oracle.knn_pools(data, K, rows)
    np.testing.assert_array_equal(ids[rows], o_ids)
    np.testing.assert_array_equal(dists[rows], o_d)
    for strategy, alpha in (("rng", 60.0), ("alpha", 66.0)):
        params = PruneParams(M=R, alpha=alpha, strategy=strategy)
        off = np.arange(n + 1, dtype=np.int64) * K
        cnt = np.full(n, K, np.int32)
        a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), params)
        b = add_reverse_and_prune(ds, a[0], a[1], a[2], params)
        oa, ob = oracle.refine_ab(data, ids, dists, R, strategy, alpha)
        for res, ores in ((a, oa), (b, ob)):
            np.testing.assert_array_equal(res[0], ores[0])
            np.testing.assert_array_equal(res[1], ores[1])
            np.testing.assert_array_equal(res[2], ores[2])
            assert res[3] == ores[3] and res[4] == ores[4]


def test_float_fallback_rows_with_duplicates():
    """Many exact duplicates at the pool boundary defeat the fp32 margin proof:
    those rows go through the exact float64 rescan and must still match."""
    rng = np.random.default_rng(3)
    base = rng.standard_normal((20, 16)).astype(np.float32)
    data = np.repeat(base, 100, axis=0)  # 2000 points, 100 exact copies each
    data[::7] += 1e-3 * rng.standard_normal((len(data[::7]), 16)).astype(np.float32)
    ds = Dataset.from_array(data)
    K = 48
    r = kernels.knn_pools(ds.device_data(), K, None, True, 2, True)
    fb = kernels.fallback_rows(r.ws)
    assert fb > 0
    o_ids, o_d = oracle.knn_pools(data, K)
    np.testing.assert_array_equal(r.pool_ids.cpu().numpy(), o_ids)
    np.testing.assert_array_equal(r.pool_dists.cpu().numpy(), o_d)
    gt, _ = oracle.knn_pool_ids(data, K)
    np.testing.assert_array_equal(r.gt_ids.cpu().numpy(), gt)


def test_hub_node_long_reverse_list():
    """A hub chosen by every point: its merged list is far longer than the
    per-warp shared-memory sort, exercising the long-slice path."""
    rng = np.random.default_rng(8)
    pts = rng.standard_normal((3000, 64))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    data = np.vstack([np.zeros((1, 64)), pts]).astype(np.float32)
    ds = Dataset.from_array(data)
    K, R = 16, 8
    ids, dists = knn_pools(ds, K)
    assert (ids[1:, 0] == 0).mean() > 0.9
    params = PruneParams(M=R)
    off = np.arange(ds.n + 1, dtype=np.int64) * K
    cnt = np.full(ds.n, K, np.int32)
    a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), params)
    b = add_reverse_and_prune(ds, a[0], a[1], a[2], params)
    oa, ob = oracle.refine_ab(data, ids, dists, R)
    for res, ores in ((a, oa), (b, ob)):
        for i in range(3):
            np.testing.assert_array_equal(res[i], ores[i])
        assert res[3] == ores[3] and res[4] == ores[4]


def test_queries_table_and_errors():
    data = synth.cfg1(3000)
    ds = Dataset.from_array(data)
    q = synth.gen_synthetic(50, 32, "gaussian", seed=77)
    table = ground_truth_table(ds, q, k=7)
    assert table.shape == (50, 7)
    for i in range(50):
        d64 = ((data.astype(np.float64) - q[i].astype(np.float64)) ** 2).sum(1)
        order = np.lexsort((np.arange(len(d64)), d64))[:7]
        assert table[i].tolist() == order.tolist()
    with pytest.raises(ValueError):
        ground_truth_table(ds, q[:, :5], k=3)
    with pytest.raises(ValueError):
        ground_truth_table(ds, q, k=3, exclude_self=True)


def test_distance_tolerance_statement():
    """The north-star tolerance (1e-5 relative) holds trivially: list
    distances are bit-identical to the reference's fp32 squared_l2."""
    data = synth.cfg3(1500)
    ds = Dataset.from_array(data)
    ids, dists = knn_pools(ds, 64)
    for u in range(0, 1500, 97):
        for j in range(0, 64, 9):
            ref = oracle.squared_l2(data[ids[u, j]], data[u])
            assert dists[u, j] == ref
            assert abs(dists[u, j] - ref) <= REL_TOL * ref


def test_device_resident_api_keeps_tensors_on_gpu():
    data = torch.from_numpy(synth.cfg2(3000)).cuda()
    ds = Dataset(data)
    assert ds.is_u8()
    ids, dists = knn_pools(ds, 32)
    assert ids.is_cuda and dists.is_cuda
    off = torch.arange(0, 3001 * 32, 32, dtype=torch.int64, device="cuda")
    cnt = torch.full((3000,), 32, dtype=torch.int32, device="cuda")
    a = prune_all(ds, off, cnt, ids.reshape(-1), dists.reshape(-1), PruneParams(M=16))
    assert a[0].is_cuda and int(a[3]) > 0


def test_builder_host_outputs_equal_device_outputs():
    """RngBuilder.build(host_out=...): the final kernel writes adjacency and
    degrees straight into pinned host memory; identical to the device build."""
    from paper_2410_01231_b200.index import RngBuilder, pool_mode
    X = torch.from_numpy(synth.cfg2(20000)).cuda()
    b = RngBuilder(20000, 128, 64, PruneParams(M=24), pool_mode(X))
    dev = b.build(X)
    ids, cnt = dev.ids.cpu(), dev.counts.cpu()
    h_ids = torch.full((20000, 24), 7, dtype=torch.int32).pin_memory()
    h_cnt = torch.zeros(20000, dtype=torch.int32).pin_memory()
    b.build(X, host_out=(h_ids, h_cnt))
    torch.cuda.synchronize()
    assert torch.equal(h_ids, ids) and torch.equal(h_cnt, cnt)
    with pytest.raises(ValueError):
        b.build(X, host_out=(torch.zeros((20000, 24), dtype=torch.int32), h_cnt))


@pytest.mark.parametrize("strategy,alpha", [("rng", 60.0), ("alpha", 66.0)])
def test_exact_integer_selection_equals_fp32_path(strategy, alpha):
    """Integer-valued [0,255] data: the u8 dp4a selection path (pgk_prune_rows_ex
    with data_u8) gives the same rows and counters as the fp32 sequential path."""
    data = synth.cfg2(8000)
    ds = Dataset.from_array(data)
    K, R = 64, 24
    ids, dists = knn_pools(ds, K)
    X = ds.device_data()
    u8 = kernels.make_u8(X)
    params = PruneParams(M=R, alpha=alpha, strategy=strategy)
    off = np.arange(ds.n + 1, dtype=np.int64) * K
    cnt = np.full(ds.n, K, np.int32)
    args = (X, off, cnt, ids.ravel(), dists.ravel(), params.strategy_code, params.cos_alpha, R)
    a32 = kernels.prune_batch(*args)
    a8 = kernels.prune_batch(*args, u8=u8)
    for x, y in zip(a32, a8):
        assert torch.equal(x, y)
    b32 = kernels.add_reverse_and_prune(X, a32[0], a32[1], a32[2], params.strategy_code,
                                        params.cos_alpha, R)
    b8 = kernels.add_reverse_and_prune(X, a8[0], a8[1], a8[2], params.strategy_code,
                                       params.cos_alpha, R, u8=u8)
    for x, y in zip(b32, b8):
        assert torch.equal(x, y)


def test_row_order_does_not_change_results():
    """The selection kernels' optional processing order (pgk_knn_order) is a
    performance hint only."""
    data = synth.cfg2(6000)
    ds = Dataset.from_array(data)
    K, R = 48, 16
    r = kernels.knn_pools(ds.device_data(), K, None, True, 1, False)
    order = kernels.knn_order(r.ws, ds.n, ds.d, K, 1)
    assert sorted(order.cpu().tolist()) == list(range(ds.n))
    X = ds.device_data()
    u8 = kernels.make_u8(X)
    params = PruneParams(M=R, alpha=66.0, strategy="alpha")
    off = np.arange(ds.n + 1, dtype=np.int64) * K
    cnt = np.full(ds.n, K, np.int32)
    args = (X, off, cnt, r.pool_ids.reshape(-1), r.pool_dists.reshape(-1), 1, params.cos_alpha, R)
    a0 = kernels.prune_batch(*args, u8=u8)
    a1 = kernels.prune_batch(*args, u8=u8, order=order)
    for x, y in zip(a0, a1):
        assert torch.equal(x, y)
    b0 = kernels.add_reverse_and_prune(X, a0[0], a0[1], a0[2], 1, params.cos_alpha, R, u8=u8)
    b1 = kernels.add_reverse_and_prune(X, a0[0], a0[1], a0[2], 1, params.cos_alpha, R, u8=u8,
                                       order=order)
    for x, y in zip(b0, b1):
        assert torch.equal(x, y)


def test_gram_selection_hub_rows_and_fallback():
    """Exact-integer data with a hub: rows of <= 128 candidates go through the
    tensor-core Gram kernel, the hub's long merged list through the per-warp
    kernel; both must match the oracle (and the fp32 path)."""
    rng = np.random.default_rng(21)
    center = np.full((1, 64), 128.0)
    pts = center + 30.0 * rng.choice([-1.0, 1.0], size=(2500, 64))
    data = np.vstack([center, pts]).astype(np.float32)
    ds = Dataset.from_array(data)
    assert ds.is_u8()
    K, R = 24, 12
    ids, dists = knn_pools(ds, K)
    for strategy, alpha in (("rng", 60.0), ("alpha", 70.0)):
        params = PruneParams(M=R, alpha=alpha, strategy=strategy)
        off = np.arange(ds.n + 1, dtype=np.int64) * K
        cnt = np.full(ds.n, K, np.int32)
        a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), params)
        b = add_reverse_and_prune(ds, a[0], a[1], a[2], params)
        oa, ob = oracle.refine_ab(data, ids, dists, R, strategy, alpha)
        for res, ores in ((a, oa), (b, ob)):
            for i in range(3):
                np.testing.assert_array_equal(res[i], ores[i])
            assert res[3] == ores[3] and res[4] == ores[4]
    # the hub's reverse list is long (in-degree > 128)
    assert (a[0][1:, 0] == 0).mean() > 0.9


def test_tensor_core_cxc_gram_selection_path():
    """The batched per-point C x C Gram kernel (tcgen05 kind::i8 + bitmask scan,
    the default for exact-integer rows) and the per-warp lazy kernel
    (PGK_GRAM=0) give the same phase A / B rows and counters, each in a fresh
    process (the default path itself is checked against the oracle above)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2410_01231_b200 import Dataset, PruneParams, knn_pools, prune_all, add_reverse_and_prune, synth
rng = np.random.default_rng(21)
center = np.full((1, 64), 128.0)
hub = np.vstack([center, center + 30.0 * rng.choice([-1.0, 1.0], size=(1500, 64))])
out = {}
for name, data in (("cfg2", synth.cfg2(6000)), ("hub", hub.astype(np.float32))):
    ds = Dataset.from_array(data)
    K = 64 if name == "cfg2" else 24
    ids, dists = knn_pools(ds, K)
    off = np.arange(ds.n + 1, dtype=np.int64) * K
    cnt = np.full(ds.n, K, np.int32)
    for st, al in (("rng", 60.0), ("alpha", 66.0)):
        p = PruneParams(M=20, alpha=al, strategy=st)
        a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), p)
        b = add_reverse_and_prune(ds, a[0], a[1], a[2], p)
        for ph, r in (("a", a), ("b", b)):
            out[f"{name}_{st}_{ph}_ids"] = r[0]; out[f"{name}_{st}_{ph}_cnt"] = r[2]
            out[f"{name}_{st}_{ph}_ev"] = np.array([r[3], r[4]])
np.savez(sys.argv[1], **out)
''' % str(root)
    res = {}
    for tag, env in (("gram", {"PGK_GRAM": "1"}), ("warp", {"PGK_GRAM": "0"})):
        path = f"/tmp/pgk_gram_{tag}.npz"
        subprocess.check_call([sys.executable, "-c", code, path],
                              env=dict(os.environ, **env), timeout=600)
        res[tag] = dict(np.load(path))
    assert res["gram"].keys() == res["warp"].keys()
    for k in res["gram"]:
        np.testing.assert_array_equal(res["gram"][k], res["warp"][k], err_msg=k)


def test_float_tile_pruning_equals_full_scan():
    """The pruned F32 pool (tile bounds + approximate survivors + float64
    rerank) returns exactly the brute-force result (PGK_DISABLE_PRUNE=1), pools
    and both phases, on float configs where pruning applies, each in a fresh
    process."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2410_01231_b200 import Dataset, PruneParams, knn_pools, prune_all, add_reverse_and_prune, synth
out = {}
for name, data, K, R in (("cfg1", synth.cfg1(10000), 64, 24), ("cfg3", synth.cfg3(30000), 128, 32),
                         ("cfg4", synth.cfg4(12000), 256, 64)):
    ds = Dataset.from_array(data)
    ids, dists = knn_pools(ds, K)
    off = np.arange(ds.n + 1, dtype=np.int64) * K
    cnt = np.full(ds.n, K, np.int32)
    p = PruneParams(M=R)
    a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), p)
    b = add_reverse_and_prune(ds, a[0], a[1], a[2], p)
    out[name + "_ids"], out[name + "_d"] = ids, dists
    out[name + "_b"], out[name + "_bc"] = b[0], b[2]
np.savez(sys.argv[1], **out)
''' % str(root)
    res = {}
    # pruned = the default: tensor-core passes (pool_tc_f32.cu) where d >= 64;
    # tc_pass2 = SIMT pass 1 + tensor-core pass 2; simt = both passes SIMT
    for tag, env in (("pruned", {}), ("tc_pass2", {"PGK_F32_TC": "1"}),
                     ("simt", {"PGK_F32_TC": "0"}), ("full", {"PGK_DISABLE_PRUNE": "1"})):
        path = f"/tmp/pgk_f32prune_{tag}.npz"
        subprocess.check_call([sys.executable, "-c", code, path],
                              env=dict(os.environ, **env), timeout=900)
        res[tag] = dict(np.load(path))
    for tag in ("pruned", "tc_pass2", "simt"):
        for k in res["full"]:
            np.testing.assert_array_equal(res[tag][k], res["full"][k], err_msg=f"{tag}:{k}")


@pytest.mark.parametrize("cfg,rows", [(3, 300), (4, 150)])
def test_full_scale_float_pools_on_seeded_rows(cfg, rows):
    """Config 3 (1M x 960) and config 4 (2M x 768) at full size: the pools of
    seeded rows equal the oracle's exact k-NN (float64, id ties) with fp32
    list distances (prefixes + seeded rows at full N)."""
    c = synth.CONFIGS[cfg]
    data = c["gen"](c["n"], c["n"])
    ds = Dataset.from_array(data)
    ids, dists = knn_pools(ds, c["K"])
    sel = np.sort(np.random.default_rng(100 + cfg).choice(ds.n, rows, replace=False))
    o_ids, o_d = oracle.knn_pools(data, c["K"], rows=sel)
    np.testing.assert_array_equal(ids[sel], o_ids)
    np.testing.assert_array_equal(dists[sel], o_d)


@pytest.mark.parametrize("gen,n,K,R", [(synth.cfg1, 3000, 64, 24), (synth.cfg2, 6000, 64, 24),
                                       (synth.cfg4, 3000, 128, 32)])
def test_slack_strategy_against_oracle(gen, n, K, R):
    """The "slack" extension (BASELINE config 4's alpha=1.2; no reference
    equivalent, parity pinned to the oracle restatement): phases A and B,
    counters included, on float, exact-integer and unit-norm data; slack 1.0
    reproduces "rng" exactly."""
    data = gen(n)
    ds = Dataset.from_array(data)
    ids, dists = knn_pools(ds, K)
    off = np.arange(ds.n + 1, dtype=np.int64) * K
    cnt = np.full(ds.n, K, np.int32)
    for s in (1.0, 1.2):
        p = PruneParams(M=R, alpha=s, strategy="slack")
        a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), p)
        b = add_reverse_and_prune(ds, a[0], a[1], a[2], p)
        oa = oracle.prune_all(data, off, cnt, ids.ravel(), dists.ravel(), R, "slack", s)
        ob = oracle.add_reverse_and_prune(data, oa[0], oa[1], oa[2], R, "slack", s)
        for res, ref in ((a, oa), (b, ob)):
            np.testing.assert_array_equal(res[0], ref[0])
            np.testing.assert_array_equal(res[2], ref[2])
            assert res[3] == ref[3] and res[4] == 0
        if s == 1.0:
            r = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), PruneParams(M=R))
            np.testing.assert_array_equal(a[0], r[0])
            assert a[3] == r[3]


@pytest.mark.parametrize("n,chunks,integer", [(20000, 8, True), (12345, 5, True), (9000, 3, False)])
def test_build_host_pipeline_equals_device_build(n, chunks, integer):
    """RngBuilder.build_host (chunked copy, per-chunk u8 rows, device-side
    exact-integer check, per-chunk tile-center assignment) equals the device
    build; data that are not exact-integer fall back to the float path."""
    from paper_2410_01231_b200 import _lib
    from paper_2410_01231_b200.index import RngBuilder, pool_mode
    data = synth.cfg2(n)
    if not integer:
        data = data + np.float32(0.25)  # same shape, no longer integer-valued
    X = torch.from_numpy(data).cuda()
    ref = RngBuilder(n, 128, 64, PruneParams(M=24), pool_mode(X)).build(X)
    ids, cnt = ref.ids.cpu(), ref.counts.cpu()
    b = RngBuilder(n, 128, 64, PruneParams(M=24), _lib.POOL_U8)
    host = torch.from_numpy(data).pin_memory()
    h_ids = torch.full((n, 24), 7, dtype=torch.int32).pin_memory()
    h_cnt = torch.zeros(n, dtype=torch.int32).pin_memory()
    for _ in range(2):  # the second call reuses the pipeline's buffers
        b.build_host(host, host_out=(h_ids, h_cnt), chunks=chunks)
        torch.cuda.synchronize()
        assert torch.equal(h_ids, ids) and torch.equal(h_cnt, cnt)


@pytest.mark.parametrize("n,d,integer", [(20000, 128, True), (20000, 128, False), (3000, 32, False)])
def test_numpy_api_build_rng_index(n, d, integer):
    """index.build_rng_index (numpy in, ProximityGraph out; the caller's array
    page-locked in place for the chunked pipeline, builder cached per shape)
    equals the oracle's phases A+B on the oracle's pools, twice in a row."""
    from paper_2410_01231_b200.index import build_rng_index
    data = synth.cfg2(n) if d == 128 else synth.cfg1(n)
    if not integer and d == 128:
        data = data + np.float32(0.25)
    o_ids, o_d = oracle.knn_pools(data, 64)
    _, ob = oracle.refine_ab(data, o_ids, o_d, 24, "rng", 60.0)
    for _ in range(2):
        g = build_rng_index(data, 64, 24)
        np.testing.assert_array_equal(g.counts, ob[2])
        np.testing.assert_array_equal(g.adj, ob[0])


@pytest.mark.parametrize("strategy,alpha", [("rng", 60.0), ("alpha", 66.0)])
def test_reverse_pass_union_sizes_through_pair_single_and_hub_paths(strategy, alpha):
    """Phase B on exact-integer rows whose unions span 0..~400 candidates: the
    paired Gram kernel (<= 64), the single-point Gram kernel (65..128) and the
    per-warp hub kernel (> 128), against the oracle (rows, counters)."""
    rng = np.random.default_rng(21)
    n, M = 4000, 32
    data = synth.cfg2(n)
    ds = Dataset.from_array(data)
    # phase-A-like rows: per-row degree 0..M, targets Zipf-skewed (hubs)
    counts = rng.integers(0, M + 1, n).astype(np.int32)
    ids = np.full((n, M), -1, np.int32)
    dists = np.full((n, M), np.inf, np.float32)
    for u in range(n):
        c = counts[u]
        cand = np.unique(np.minimum(rng.zipf(1.6, 3 * M) - 1, n - 1))
        cand = cand[cand != u][:c]
        counts[u] = len(cand)
        d = ((data[cand].astype(np.float64) - data[u]) ** 2).sum(1).astype(np.float32)
        o = np.lexsort((cand, d))
        ids[u, :len(cand)] = cand[o]
        dists[u, :len(cand)] = d[o]
    params = PruneParams(M=M, alpha=alpha, strategy=strategy)
    got = add_reverse_and_prune(ds, ids, dists, counts, params)
    want = oracle.add_reverse_and_prune(data, ids, dists, counts, M, strategy, alpha)
    for i in range(3):
        np.testing.assert_array_equal(got[i], want[i])
    assert got[3] == want[3] and got[4] == want[4]


@pytest.mark.parametrize("strategy,alpha", [("rng", 60.0), ("alpha", 66.0)])
def test_full_scale_cfg2_build_through_the_bench_path(strategy, alpha):
    """Config 2 at its full size (1M x 128, K=128, R=32, rng) through the bench's
    RngBuilder: the pools of 300 seeded rows equal the oracle's exact k-NN;
    every pool row is sorted by (dist, id), self-free, duplicate-free and its
    fp32 distances equal a direct recomputation; phases A and B over ALL 1M
    rows equal the oracle's (ids, dists, degrees, dist_evals) when fed the
    GPU's pools (full-N phases A+B beside seeded pool rows);
    the alpha case covers the angle counters too."""
    from paper_2410_01231_b200.index import RngBuilder, pool_mode
    c = synth.CONFIGS[2]
    n, K, R = c["n"], c["K"], c["R"]
    data = c["gen"](n, n)
    X = torch.from_numpy(data).cuda()
    b = RngBuilder(n, data.shape[1], K, PruneParams(M=R, alpha=alpha, strategy=strategy),
                   pool_mode(X))
    out = b.build(X)
    torch.cuda.synchronize()
    p_ids, p_d = (t.cpu().numpy() for t in b.pool_out[:2])
    # pool properties on every row (direct-difference fp32 sums of integers
    # below 2^24 are exact, so the recomputation is the reference's value)
    for r0 in range(0, n, 8192):
        r1 = min(n, r0 + 8192)
        ii = b.pool_out[0][r0:r1].long()
        dd = ((X[ii] - X[r0:r1, None, :]) ** 2).sum(-1)
        assert torch.equal(dd, b.pool_out[1][r0:r1]), r0
    rows = np.arange(n)[:, None]
    assert (p_ids != rows).all() and (p_ids >= 0).all()
    key_sorted = (p_d[:, 1:] > p_d[:, :-1]) | ((p_d[:, 1:] == p_d[:, :-1]) & (p_ids[:, 1:] > p_ids[:, :-1]))
    assert key_sorted.all()
    sel = np.sort(np.random.default_rng(202).choice(n, 300, replace=False))
    o_ids, o_d = oracle.knn_pools(data, K, rows=sel)
    np.testing.assert_array_equal(p_ids[sel], o_ids)
    np.testing.assert_array_equal(p_d[sel], o_d)
    # phases A and B over all rows against the oracle on the same pools
    off = np.arange(n + 1, dtype=np.int64) * K
    cnt = np.full(n, K, np.int32)
    oa = oracle.prune_all(data, off, cnt, p_ids.ravel(), p_d.ravel(), R, strategy, alpha)
    np.testing.assert_array_equal(b.a_out[0].cpu().numpy(), oa[0])
    np.testing.assert_array_equal(b.a_out[1].cpu().numpy(), oa[1])
    np.testing.assert_array_equal(out.a_counts.cpu().numpy(), oa[2])
    ob = oracle.add_reverse_and_prune(data, oa[0], oa[1], oa[2], R, strategy, alpha)
    np.testing.assert_array_equal(out.ids.cpu().numpy(), ob[0])
    np.testing.assert_array_equal(out.dists.cpu().numpy(), ob[1])
    np.testing.assert_array_equal(out.counts.cpu().numpy(), ob[2])
    de = out.dist_evals.cpu().numpy()
    assert int(de[0]) == oa[3] and int(de[1]) == ob[3]
    ae = out.angle_evals.cpu().numpy()
    assert int(ae[0]) == oa[4] and int(ae[1]) == ob[4]
    assert strategy == "alpha" or oa[4] == ob[4] == 0


@pytest.mark.parametrize("cfg,strategy,alpha,nrows", [(3, "rng", 60.0, 2000),
                                                       (4, "slack", 1.2, 1000)])
def test_full_scale_float_build_on_seeded_rows(cfg, strategy, alpha, nrows):
    """Configs 3 (1M x 960, rng) and 4 (2M x 768, K=256, R=64, BASELINE's
    alpha=1.2 as the slack rule) at full size through RngBuilder: phase A of
    seeded rows and the phase-B re-prune of seeded rows (fed the GPU's
    phase-A rows of ALL points, so the reverse edges are complete) equal the
    oracle's rows and per-row counters bit for bit; the pools of the first
    100 seeded rows equal the oracle's exact k-NN."""
    from paper_2410_01231_b200.index import RngBuilder, pool_mode
    c = synth.CONFIGS[cfg]
    n, K, R = c["n"], c["K"], c["R"]
    data = c["gen"](n, n)
    X = torch.from_numpy(data).cuda()
    b = RngBuilder(n, data.shape[1], K, PruneParams(M=R, alpha=alpha, strategy=strategy),
                   pool_mode(X))
    out = b.build(X)
    torch.cuda.synchronize()
    del X
    p_ids, p_d = (t.cpu().numpy() for t in b.pool_out[:2])
    sel = np.sort(np.random.default_rng(300 + cfg).choice(n, nrows, replace=False))
    o_ids, o_d = oracle.knn_pools(data, K, rows=sel[:100])
    np.testing.assert_array_equal(p_ids[sel[:100]], o_ids)
    np.testing.assert_array_equal(p_d[sel[:100]], o_d)
    off = np.arange(n + 1, dtype=np.int64) * K
    cnt = np.zeros(n, np.int32)
    cnt[sel] = K
    oa = oracle.prune_all(data, off, cnt, p_ids.ravel(), p_d.ravel(), R, strategy, alpha)
    a_ids, a_d, a_cnt, a_de = (t.cpu().numpy() for t in b.a_out[:4])
    np.testing.assert_array_equal(a_ids[sel], oa[0][sel])
    np.testing.assert_array_equal(a_d[sel], oa[1][sel])
    np.testing.assert_array_equal(a_cnt[sel], oa[2][sel])
    assert int(a_de[sel].sum()) == oa[3]
    ob = oracle.add_reverse_and_prune(data, a_ids, a_d, a_cnt, R, strategy, alpha, rows=sel)
    np.testing.assert_array_equal(out.ids.cpu().numpy()[sel], ob[0][sel])
    np.testing.assert_array_equal(out.dists.cpu().numpy()[sel], ob[1][sel])
    np.testing.assert_array_equal(out.counts.cpu().numpy()[sel], ob[2][sel])
    assert int(b.b_out[3].cpu().numpy()[sel].sum()) == ob[3]


def test_build_host_stream_equals_device_builds():
    """RngBuilder.build_host_stream (double-buffered: dataset i+1 copied while
    dataset i builds) gives every dataset the device build's adjacency; a
    dataset that is not exact-integer goes through the float path."""
    from paper_2410_01231_b200 import _lib
    from paper_2410_01231_b200.index import RngBuilder, pool_mode
    n = 20000
    sets = [synth.cfg2(n), synth.cfg2(n, n_full=2 * n), synth.cfg2(n) + np.float32(0.25)]
    b = RngBuilder(n, 128, 64, PruneParams(M=24), _lib.POOL_U8)
    hosts = [torch.from_numpy(x).pin_memory() for x in sets]
    outs = [(torch.zeros((n, 24), dtype=torch.int32).pin_memory(),
             torch.zeros(n, dtype=torch.int32).pin_memory()) for _ in sets]
    b.build_host_stream(hosts, outs)
    for x, (h_ids, h_cnt) in zip(sets, outs):
        X = torch.from_numpy(x).cuda()
        ref = RngBuilder(n, 128, 64, PruneParams(M=24), pool_mode(X)).build(X)
        assert torch.equal(h_ids, ref.ids.cpu()) and torch.equal(h_cnt, ref.counts.cpu())


def _lattice_float(n, d, seed):
    """Integer-valued float data above the exact-integer range (values up to
    1000): distance ties and exact duplicates everywhere, so many pair tests
    sit exactly on their threshold."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 4, size=(n, d)).astype(np.float32) * 250.0
    base[n // 2:] = base[: n - n // 2]          # every row has an exact duplicate
    base[: n // 8, 0] += 1.0                    # ... some of them one step apart
    return np.ascontiguousarray(base)


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "lattice"])
def test_gram_f32_selection_against_oracle(name):
    """The tensor-core float selection (prune_gram_f32.cu: bf16 hi/lo Gram on
    rows centred on the point, proven pair classification, float64 / exact
    fp32 chains for undecided pairs) equals the oracle's phases A and B, ids,
    dists, degrees, dist_evals and angle_evals, for rng, the alpha rule (66 and
    95 degrees) and the slack rule; the lattice
    data put most pair tests exactly on their threshold (zero distances,
    F == dv ties), which forces the exact-chain path."""
    if name == "cfg3":
        data, K, R = synth.cfg3(5000), 128, 32
    elif name == "cfg4":
        data, K, R = synth.cfg4(4000), 120, 32
    else:
        data, K, R = _lattice_float(3000, 128, 5), 96, 24
    ds = Dataset.from_array(data)
    ids, dists = knn_pools(ds, K)
    o_ids, o_dists = oracle.knn_pools(data, K)
    np.testing.assert_array_equal(ids, o_ids)
    off = np.arange(ds.n + 1, dtype=np.int64) * K
    cnt = np.full(ds.n, K, np.int32)
    for strategy, s in (("rng", 60.0), ("slack", 1.2), ("alpha", 66.0), ("alpha", 95.0)):
        p = PruneParams(M=R, alpha=s, strategy=strategy)
        a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), p)
        b = add_reverse_and_prune(ds, a[0], a[1], a[2], p)
        oa = oracle.prune_all(data, off, cnt, ids.ravel(), dists.ravel(), R, strategy, s)
        ob = oracle.add_reverse_and_prune(data, oa[0], oa[1], oa[2], R, strategy, s)
        for res, ref in ((a, oa), (b, ob)):
            for i in range(3):
                np.testing.assert_array_equal(res[i], ref[i], err_msg=f"{name} {strategy} [{i}]")
            assert res[3] == ref[3] and res[4] == ref[4], (name, strategy, s)


def test_gram_f32_equals_prune_kernel_on_larger_prefixes():
    """PGK_GRAM_F32=0 (per-warp prune_kernel) and the default tensor-core
    selection give identical phases A and B, counters included, on 60k-row
    prefixes of configs 3 and 4 (fresh processes: the switch is read once)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    for cfg, k in ((3, 0), (4, 128)):
        out = subprocess.run([sys.executable, str(root / "tools" / "gram_f32_check.py"), "--config",
                              str(cfg), "--n", "60000", "--k", str(k), "--reps", "1"],
                             capture_output=True, text=True, timeout=1200, check=True).stdout
        cmp_line = [json.loads(l) for l in out.splitlines() if l.startswith('{"compare"')]
        assert cmp_line and all(v == 0 for v in cmp_line[0]["differing_entries"].values()), out


@pytest.mark.parametrize("R", [1, 4, 24, 33])
@pytest.mark.parametrize("strategy,alpha", [("rng", 60.0), ("slack", 1.3)])
def test_fused_merge_prune_kernel_edge_shapes(R, strategy, alpha):
    """Phase B's in-warp merge + prune of short unions (merge_prune_kernel:
    register merge, 32 x 32 Gram by mma.sync, masks / greedy / lazy counters in
    one warp) against the oracle over the shapes that steer it: M = 1 and 4
    (the scan stops at the M-th kept neighbour well inside the row), M = 24
    (unions straddling the 32-candidate limit, so rows split between this
    kernel and the tcgen05 pair kernel), phase-A rows wider than a warp
    (R = 33: own parts of 33 entries leave the two-part merge), on a tie-heavy
    integer lattice (duplicate distances, zero distances) and on clustered
    data; and against the unfused path (PGK_REV_FUSED is read once per
    process, so that comparison is the oracle's)."""
    rng = np.random.default_rng(7)
    lattice = rng.integers(0, 4, size=(3000, 16)).astype(np.float32)  # many ties / duplicates
    for data, K in ((synth.cfg2(5000), 48), (lattice, 40)):
        ds = Dataset.from_array(data)
        ids, dists = knn_pools(ds, K)
        off = np.arange(ds.n + 1, dtype=np.int64) * K
        cnt = np.full(ds.n, K, np.int32)
        p = PruneParams(M=R, alpha=alpha, strategy=strategy)
        a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), p)
        b = add_reverse_and_prune(ds, a[0], a[1], a[2], p)
        oa = oracle.prune_all(data, off, cnt, ids.ravel(), dists.ravel(), R, strategy, alpha)
        ob = oracle.add_reverse_and_prune(data, oa[0], oa[1], oa[2], R, strategy, alpha)
        for res, ref in ((a, oa), (b, ob)):
            np.testing.assert_array_equal(res[0], ref[0])
            np.testing.assert_array_equal(res[1], ref[1])
            np.testing.assert_array_equal(res[2], ref[2])
            assert res[3] == ref[3] and res[4] == ref[4]


def test_build_host_falls_back_when_tiles_are_not_supported():
    """RngBuilder.build_host on shapes the tile-pruned pipeline does not take
    (pgk_tiles_supported false: K > 256 here, PGK_DISABLE_PRUNE=1 in a
    subprocess -- the switch is read once per process) copies, then builds:
    same rows as the device build instead of a ValueError."""
    import os
    import subprocess
    import sys
    from paper_2410_01231_b200 import _lib
    from paper_2410_01231_b200.index import RngBuilder
    n, K, R = 6000, 300, 24
    assert not _lib.lib().pgk_tiles_supported(n, 128, K)
    data = synth.cfg2(n)
    X = torch.from_numpy(data).cuda()
    ref = RngBuilder(n, 128, K, PruneParams(M=R), _lib.POOL_U8).build(X)
    b = RngBuilder(n, 128, K, PruneParams(M=R), _lib.POOL_U8)
    h_ids = torch.full((n, R), 7, dtype=torch.int32).pin_memory()
    h_cnt = torch.zeros(n, dtype=torch.int32).pin_memory()
    b.build_host(torch.from_numpy(data).pin_memory(), host_out=(h_ids, h_cnt))
    torch.cuda.synchronize()
    assert torch.equal(h_ids, ref.ids.cpu()) and torch.equal(h_cnt, ref.counts.cpu())
    code = (
        "import torch, numpy as np\n"
        "from paper_2410_01231_b200 import _lib, synth, PruneParams\n"
        "from paper_2410_01231_b200.index import RngBuilder\n"
        "n, K, R = 6000, 64, 24\n"
        "assert not _lib.lib().pgk_tiles_supported(n, 128, K)\n"
        "data = synth.cfg2(n)\n"
        "ref = RngBuilder(n, 128, K, PruneParams(M=R), _lib.POOL_U8).build(torch.from_numpy(data).cuda())\n"
        "h = (torch.zeros((n, R), dtype=torch.int32).pin_memory(), torch.zeros(n, dtype=torch.int32).pin_memory())\n"
        "RngBuilder(n, 128, K, PruneParams(M=R), _lib.POOL_U8).build_host(torch.from_numpy(data).pin_memory(), host_out=h)\n"
        "torch.cuda.synchronize()\n"
        "assert torch.equal(h[0], ref.ids.cpu()) and torch.equal(h[1], ref.counts.cpu())\n"
        "print('ok')\n")
    env = dict(os.environ, PGK_DISABLE_PRUNE="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
