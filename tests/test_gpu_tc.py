"""GPU: the tcgen05 (kind::i8) exact pool kernel against the SIMT kernel and
the oracle (integer-valued data in [0,255], d <= 128)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle
from paper_2410_01231_b200 import Dataset, knn_pools, synth, kernels

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("n,K", [(200, 10), (1000, 64), (5000, 128), (20000, 128), (3001, 256)])
def test_tc_pool_matches_oracle(n, K):
    data = synth.cfg2(n)
    ds = Dataset.from_array(data)
    assert ds.is_u8()
    ids, dists, gt = knn_pools(ds, K, want_gt=True)
    rows = np.unique(np.concatenate([np.arange(min(n, 64)), np.arange(n - 64, n),
                                     np.random.default_rng(n).choice(n, 200)]))
    o_ids, o_d = oracle.knn_pools(data, K, rows)
    np.testing.assert_array_equal(ids[rows], o_ids)
    np.testing.assert_array_equal(dists[rows], o_d)
    np.testing.assert_array_equal(gt[rows], o_ids)  # exact integers: both orders coincide


def test_tc_pool_small_d_and_ties():
    """d = 3 integer lattice with massive exact ties (id tie-break)."""
    g = np.stack(np.meshgrid(np.arange(20), np.arange(20), np.arange(3)), -1)
    data = g.reshape(-1, 3).astype(np.float32)
    ds = Dataset.from_array(data)
    ids, dists = knn_pools(ds, 30)
    o_ids, o_d = oracle.knn_pools(data, 30)
    np.testing.assert_array_equal(ids, o_ids)
    np.testing.assert_array_equal(dists, o_d)


def test_tc_matches_simt_path():
    """Same pools from the SIMT U8 kernel (PGK_DISABLE_TC=1, fresh process)."""
    n, K = 12000, 128
    data = synth.cfg2(n)
    ids, dists = knn_pools(Dataset.from_array(data), K)
    code = ("import sys, numpy as np; sys.path.insert(0, %r);"
            "from paper_2410_01231_b200 import Dataset, knn_pools, synth;"
            "i, d = knn_pools(Dataset.from_array(synth.cfg2(%d)), %d);"
            "np.save('/tmp/pgk_simt_ids.npy', i); np.save('/tmp/pgk_simt_d.npy', d)"
            % (str(ROOT), n, K))
    env = dict(os.environ, PGK_DISABLE_TC="1")
    subprocess.check_call([sys.executable, "-c", code], env=env, timeout=600)
    np.testing.assert_array_equal(ids, np.load("/tmp/pgk_simt_ids.npy"))
    np.testing.assert_array_equal(dists, np.load("/tmp/pgk_simt_d.npy"))


def test_tc_queries_table():
    data = synth.cfg2(4000)
    q = synth.cfg2(4100)[4000:]
    from paper_2410_01231_b200 import ground_truth_table
    table = ground_truth_table(Dataset.from_array(data), q, k=16)
    for i in range(0, 100, 7):
        d64 = ((data.astype(np.float64) - q[i].astype(np.float64)) ** 2).sum(1)
        assert table[i].tolist() == np.lexsort((np.arange(4000), d64))[:16].tolist()


def _pools_subprocess(gen_code, K, env_extra):
    code = ("import sys, numpy as np; sys.path.insert(0, %r);"
            "from paper_2410_01231_b200 import Dataset, knn_pools, synth;"
            "data = %s; i, d = knn_pools(Dataset.from_array(data), %d);"
            "np.save('/tmp/pgk_sub_ids.npy', i); np.save('/tmp/pgk_sub_d.npy', d)"
            % (str(ROOT), gen_code, K))
    env = dict(os.environ, **env_extra)
    subprocess.check_call([sys.executable, "-c", code], env=env, timeout=600)
    return np.load("/tmp/pgk_sub_ids.npy"), np.load("/tmp/pgk_sub_d.npy")


@pytest.mark.parametrize("gen_code,K", [
    ("synth.cfg2(30000)", 128),
    ("np.random.default_rng(3).integers(0, 256, (9000, 128)).astype(np.float32)", 64),
    ("np.repeat(np.random.default_rng(4).integers(0, 256, (300, 96)), 20, axis=0)"
     ".astype(np.float32)", 32),
    # small K: pass-1 lists of a single tile (one-tile blocks stress the
    # A-tile / block-index barrier of the dynamic schedule)
    ("synth.cfg2(100000)", 16),
    ("synth.cfg2(100000)", 32),
])
def test_tile_pruned_pool_equals_full_scan(gen_code, K):
    """Exact tile pruning (default) vs the full tcgen05 scan (PGK_DISABLE_PRUNE=1):
    clustered, uniform (little to prune) and duplicate-heavy data."""
    data = eval(gen_code, {"np": np, "synth": synth})
    ids, dists = knn_pools(Dataset.from_array(data), K)
    f_ids, f_d = _pools_subprocess(gen_code, K, {"PGK_DISABLE_PRUNE": "1"})
    np.testing.assert_array_equal(ids, f_ids)
    np.testing.assert_array_equal(dists, f_d)
    rows = np.random.default_rng(1).choice(len(data), 150, replace=False)
    o_ids, o_d = oracle.knn_pools(data, K, rows)
    np.testing.assert_array_equal(ids[rows], o_ids)


@pytest.mark.parametrize("n,d,K", [(30000, 128, 128), (12000, 100, 64)])
def test_pool_from_callers_u8_rows_equals_fp32_input(n, d, K):
    """pgk_knn_pools_u8 (the caller's make_u8 rows and norms feed the center
    assignment and the tile gather) equals pgk_knn_pools on the fp32 rows."""
    import torch
    from paper_2410_01231_b200 import _lib, kernels
    rng = np.random.default_rng(7)
    data = synth.cfg2(n) if d == 128 else rng.integers(0, 256, (n, d)).astype(np.float32)
    X = torch.from_numpy(data).cuda()
    a = kernels.knn_pools(X, K, mode=_lib.POOL_U8, want_gt=False)
    b = kernels.knn_pools(X, K, mode=_lib.POOL_U8, want_gt=False, u8=kernels.make_u8(X))
    assert torch.equal(a.pool_ids, b.pool_ids) and torch.equal(a.pool_dists, b.pool_dists)


@pytest.mark.parametrize("n,nq", [(5000, 700), (20000, 0)])
def test_nearest_neighbour_k1_path(n, nq):
    """K = 1 (the epilogue's nearest-neighbour path, which also assigns points
    to tile centers): query tables and the self pool equal the oracle's exact
    (float64 dist, id) nearest neighbour, ties on duplicates included."""
    from paper_2410_01231_b200 import ground_truth_table
    rng = np.random.default_rng(17)
    data = synth.cfg2(n)
    data[rng.choice(n, 200, replace=False)] = data[rng.choice(n, 200, replace=False)]  # dups
    ds = Dataset.from_array(data)
    if nq:
        q = synth.cfg2(n + nq)[n:]
        got = ground_truth_table(ds, q, k=1)
        for i in range(0, nq, 13):
            d64 = ((data.astype(np.float64) - q[i].astype(np.float64)) ** 2).sum(1)
            assert got[i, 0] == np.lexsort((np.arange(n), d64))[0]
    else:
        ids, dists = knn_pools(ds, 1)
        rows = rng.choice(n, 300, replace=False)
        o_ids, o_d = oracle.knn_pools(data, 1, rows)
        np.testing.assert_array_equal(ids[rows], o_ids)
        np.testing.assert_array_equal(dists[rows], o_d)
