"""Full-size parity checks shared by tests/test_gpu_fullscale.py (asserts) and
tools/parity_report.py (writes the numbers to profiles/).  GPU + oracle; the
oracle is the checker only (TEST INFRASTRUCTURE).

* pool exactness at the benchmarked sizes: the tile-pruned pools equal the
  brute-force kernels (PGK_POOL_NO_PRUNE: every pair scanned) on EVERY row,
  and the oracle's float64 exact k-NN (oracle.py:31-65 restated) on 2,000
  seeded rows;
* north_star's graph figures at a config-2 prefix: edge agreement of the
  GPU graph with the oracle-built graph (phases A, B and C) and recall@10 of
  the reference's greedy search (search.py:81-94) on both graphs, with
  mean_recall (oracle.py:68-84) against the exact float64 top-10.
"""
from __future__ import annotations

import time

import numpy as np
import torch

from oracle import oracle
from paper_2410_01231_b200 import (Dataset, PruneParams, _lib, kernels, pool, prune, search,
                                   synth)


def _equal_rows(a_ids, a_d, b_ids, b_d) -> int:
    same = (a_ids == b_ids).all(1) & (a_d == b_d).all(1)
    return int(same.sum().item())


def pool_exactness(cfg: int, oracle_rows: int = 2000, seed: int = 7, n: int = 0) -> dict:
    """Pruned pools vs the brute-force pools on all rows, and vs the oracle on
    `oracle_rows` seeded rows, at config `cfg`'s full size (or n rows of the
    config's recipe drawn as an n-row array: the scale test)."""
    c = synth.CONFIGS[cfg]
    K = c["K"]
    n = n or c["n"]
    data = c["gen"](n, n)
    X = torch.from_numpy(data).cuda()
    mode = _lib.POOL_U8 if kernels.detect_u8(X) else _lib.POOL_F32
    t0 = time.perf_counter()
    a = kernels.knn_pools(X, K, mode=mode, want_gt=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pruned_work = kernels.knn_work(a.ws, n, n, data.shape[1], K, mode)
    del a.ws
    b = kernels.knn_pools(X, K, mode=mode | _lib.POOL_NO_PRUNE, want_gt=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del b.ws
    eq = _equal_rows(a.pool_ids, a.pool_dists, b.pool_ids, b.pool_dists)
    sel = np.sort(np.random.default_rng(seed + cfg).choice(n, oracle_rows, replace=False))
    t3 = time.perf_counter()
    o_ids, o_d = oracle.knn_pools(data, K, rows=sel)
    t4 = time.perf_counter()
    p_ids = a.pool_ids[torch.from_numpy(sel).cuda()].cpu().numpy()
    p_d = a.pool_dists[torch.from_numpy(sel).cuda()].cpu().numpy()
    o_eq = int(((p_ids == o_ids).all(1) & (p_d == o_d).all(1)).sum())
    return {"config": cfg, "n": n, "K": K, "mode": "u8" if mode == _lib.POOL_U8 else "f32",
            "rows_equal_bruteforce": eq, "rows": n,
            "oracle_rows": int(oracle_rows), "oracle_rows_equal": o_eq,
            "pruned_path_ran": bool(pruned_work[3]),
            "seconds": {"pruned": t1 - t0, "bruteforce": t2 - t1, "oracle_rows": t4 - t3}}


def exact_topk(data: np.ndarray, queries: np.ndarray, k: int, chunk: int = 1000) -> np.ndarray:
    """Exact (float64 dist, id) top-k of each query (oracle.py:31-65 with
    queries; integer-valued data make every float64 sum exact)."""
    x = data.astype(np.float64)
    xn = (x * x).sum(1)
    out = np.empty((queries.shape[0], k), np.int32)
    for lo in range(0, queries.shape[0], chunk):
        q = queries[lo:lo + chunk].astype(np.float64)
        d2 = xn[None, :] - 2.0 * (q @ x.T) + (q * q).sum(1)[:, None]
        np.maximum(d2, 0.0, out=d2)
        out[lo:lo + chunk] = np.argsort(d2, axis=1, kind="stable")[:, :k]
    return out


def _edges(adj: np.ndarray, counts: np.ndarray) -> np.ndarray:
    n = adj.shape[0]
    live = np.arange(adj.shape[1])[None, :] < counts[:, None]
    u = np.broadcast_to(np.arange(n, dtype=np.int64)[:, None], adj.shape)[live]
    return u * n + adj[live].astype(np.int64)


def graph_recall(n: int = 50_000, n_queries: int = 10_000, Ls=(10, 20, 50, 100),
                 strategy: str = "rng", alpha: float = 60.0) -> dict:
    """Config-2 prefix of n rows: GPU graph (pools, phases A, B, C through the
    package's reference-named API) vs the oracle-built graph; edge agreement
    and recall@10 of the greedy search on both."""
    c = synth.CONFIGS[2]
    K, R = c["K"], c["R"]
    data = synth.cfg2(n)
    ds = Dataset.from_array(data)
    params = PruneParams(M=R, alpha=alpha, strategy=strategy)
    t0 = time.perf_counter()
    ids, dists = pool.knn_pools(ds, K)
    off = np.arange(n + 1, dtype=np.int64) * K
    cnt = np.full(n, K, np.int32)
    g = prune.refine(ds, off, cnt, ids.ravel(), dists.ravel(), params, connect=True)
    t1 = time.perf_counter()
    o_ids, o_d = oracle.knn_pools(data, K)
    _, ob = oracle.refine_ab(data, o_ids, o_d, R, strategy, alpha)
    o_adj, o_cnt, o_ep, o_over = oracle.finish_connect(data, ob[0], ob[2], R, ep=None, seed=0)
    t2 = time.perf_counter()
    e_gpu, e_orc = _edges(g.adj, g.counts), _edges(o_adj, o_cnt)
    common = np.intersect1d(e_gpu, e_orc).size
    q = synth.cfg2_queries(n_queries)
    truth = exact_topk(data, q, 10)
    og = prune.ProximityGraph(adj=o_adj, counts=o_cnt, M=R, ep=o_ep, over_cap=o_over)
    rows = []
    for L in Ls:
        g_ids, _, g_dc = search.search_batch(ds, g, q, 10, L)
        x_ids, _, x_dc = search.search_batch(ds, og, q, 10, L)   # GPU search, oracle graph
        r_ids, _, r_dc = oracle.search_batch(data, o_adj, o_cnt, q, 10, L, o_ep)
        rows.append({"L": L, "recall_at_10_gpu_graph": pool.mean_recall(g_ids, truth, 10),
                     "recall_at_10_oracle_graph": pool.mean_recall(r_ids, truth, 10),
                     "gpu_search_equals_oracle_search": bool(np.array_equal(x_ids, r_ids)
                                                             and np.array_equal(x_dc, r_dc)),
                     "dist_evals_per_query_gpu_graph": float(g_dc.mean())})
    return {"config": 2, "n": n, "K": K, "R": R, "strategy": strategy, "alpha": alpha,
            "queries": n_queries, "query_recipe": "synth.cfg2_queries (seed-1 centres, "
                                                  "default_rng(1001) assignment + noise)",
            "edges_gpu": int(e_gpu.size), "edges_oracle": int(e_orc.size),
            "edge_agreement": common / max(e_orc.size, 1),
            "graphs_identical": bool(np.array_equal(g.counts, o_cnt)
                                     and g.ep == o_ep and e_gpu.size == common == e_orc.size),
            "ep_gpu": int(g.ep), "ep_oracle": int(o_ep), "search": rows,
            "seconds": {"gpu_build_with_phase_c": t1 - t0, "oracle_build": t2 - t1}}
