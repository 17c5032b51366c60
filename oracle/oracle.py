"""CPU oracle for the RNG index-construction hot path -- TEST INFRASTRUCTURE.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this module, and only as the checker / the
timed CPU baseline.  The product package never imports it.

Two layers:

* ``pgk_oracle.c`` (built to ``oracle/liboracle.so``): plain-C restatement of
  the reference's numba kernels (_kernels.py:17-42, 298-324, 364-427, 530-588)
  and a float64 direct-difference exact-kNN pool.  OpenMP over points.
* numpy orchestration restating prune.py:109-151 (phase A / phase B) and
  oracle.py:31-65 (``ground_truth_table``, float64 BLAS norm expansion plus a
  stable argsort, exactly as the reference computes it).

Pinned against tests/golden/*.npz, which hold outputs of the reference itself
(tests/golden/make_golden.py); see tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "pgk_oracle.c"
LIB = HERE / "liboracle.so"

EMPTY = -1
_STRATEGIES = ("rng", "alpha", "slack")


def _param(strategy: str, alpha: float) -> float:
    """The rule's float64 kernel parameter: cos(alpha) (prune.py:54-56), or
    s^2 for the "slack" extension (no reference equivalent)."""
    return float(alpha) * float(alpha) if strategy == "slack" else cos_alpha(alpha)


def build(force: bool = False) -> Path:
    """Compile the C restatement (gcc, OpenMP, no FMA contraction)."""
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        tmp = LIB.with_suffix(".so.tmp")
        subprocess.check_call([
            "gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
            "-fPIC", "-shared", "-std=c99", str(SRC), "-o", str(tmp), "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.orc_squared_l2.restype = ctypes.c_float
        L.orc_squared_l2.argtypes = [P, P, I64]
        L.orc_cos_angle_from_sq.restype = D
        L.orc_cos_angle_from_sq.argtypes = [ctypes.c_float] * 3
        L.orc_prune_batch.restype = None
        L.orc_prune_batch.argtypes = [P, I64, I64, P, P, P, P, I32, D, I64, I64,
                                      P, P, P, P, P]
        L.orc_sort_pairs.argtypes = [P, P, I64]
        L.orc_scatter_reverse.argtypes = [P, P, P, I64, I64, P, P, P]
        L.orc_merge_with_reverse.argtypes = [P, P, P, I64, I64, P, P, P, P, P, P, P]
        L.orc_knn_pool.argtypes = [P, I64, I64, I64, I32, P, I64, P, P]
        L.orc_list_dists_sorted.argtypes = [P, I64, P, I64, I64, P, P]
        L.orc_search_many.restype = None
        L.orc_search_many.argtypes = [P, I64, I64, P, I64, P, P, I64, I64, I64, I32, I32, P,
                                      P, P]
        L.orc_mark_reachable.restype = None
        L.orc_mark_reachable.argtypes = [P, I64, P, I64, I32, P]
        L.orc_num_threads.restype = I32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def cos_alpha(alpha_deg: float) -> float:
    """PruneParams.cos_alpha (prune.py:54-56)."""
    return math.cos(math.radians(alpha_deg))


def squared_l2(a, b) -> float:
    a, b = _f32(a), _f32(b)
    return float(lib().orc_squared_l2(_p(a), _p(b), a.shape[0]))


def prune_all(data, cand_off, cand_counts, cand_ids, cand_dists, M: int,
              strategy: str = "rng", alpha: float = 60.0, cap=None):
    """prune.py:109-126 -> (ids (n, width), dists, counts, dist_evals, angle_evals)."""
    data = _f32(data)
    n, d = data.shape
    width = M if cap is None else cap
    cand_off = np.ascontiguousarray(cand_off, np.int64)
    cand_counts = np.ascontiguousarray(cand_counts, np.int32)
    cand_ids = np.ascontiguousarray(cand_ids, np.int32)
    cand_dists = np.ascontiguousarray(cand_dists, np.float32)
    out_ids = np.full((n, width), EMPTY, np.int32)
    out_dists = np.full((n, width), np.inf, np.float32)
    out_counts = np.zeros(n, np.int32)
    de = np.zeros(n, np.int64)
    ae = np.zeros(n, np.int64)
    lib().orc_prune_batch(_p(data), n, d, _p(cand_off), _p(cand_counts), _p(cand_ids),
                          _p(cand_dists), _STRATEGIES.index(strategy), _param(strategy, alpha),
                          M, width, _p(out_ids), _p(out_dists), _p(out_counts),
                          _p(de), _p(ae))
    return out_ids, out_dists, out_counts, int(de.sum()), int(ae.sum())


def add_reverse_and_prune(data, ids, dists, counts, M: int, strategy: str = "rng",
                          alpha: float = 60.0, rows=None):
    """prune.py:129-151 (phase B).  rows: re-prune only these rows (the merged
    lists still take reverse edges from every row; other rows come back empty)
    -- the per-row independence of the re-prune, used for seeded-row checks
    at sizes where the full CPU re-prune is too slow."""
    data = _f32(data)
    n = data.shape[0]
    ids = np.ascontiguousarray(ids, np.int32)
    dists = np.ascontiguousarray(dists, np.float32)
    counts = np.ascontiguousarray(counts, np.int32)
    width = ids.shape[1]
    live = np.arange(width)[None, :] < counts[:, None]
    flat = ids[live]  # row-major == np.concatenate of live prefixes
    rev_counts = np.bincount(flat, minlength=n).astype(np.int64)
    rev_off = np.zeros(n + 1, np.int64)
    np.cumsum(rev_counts, out=rev_off[1:])
    rev_ids = np.empty(int(rev_off[-1]), np.int32)
    rev_dists = np.empty(int(rev_off[-1]), np.float32)
    lib().orc_scatter_reverse(_p(ids), _p(dists), _p(counts), n, width, _p(rev_off),
                              _p(rev_ids), _p(rev_dists))
    mrg_cap = counts.astype(np.int64) + rev_counts
    mrg_off = np.zeros(n + 1, np.int64)
    np.cumsum(mrg_cap, out=mrg_off[1:])
    mrg_ids = np.empty(int(mrg_off[-1]), np.int32)
    mrg_dists = np.empty(int(mrg_off[-1]), np.float32)
    mrg_counts = np.zeros(n, np.int32)
    lib().orc_merge_with_reverse(_p(ids), _p(dists), _p(counts), n, width, _p(rev_off),
                                 _p(rev_ids), _p(rev_dists), _p(mrg_off), _p(mrg_ids),
                                 _p(mrg_dists), _p(mrg_counts))
    if rows is not None:
        keep = np.zeros(n, bool)
        keep[np.asarray(rows)] = True
        mrg_counts[~keep] = 0
    return prune_all(data, mrg_off, mrg_counts, mrg_ids, mrg_dists, M, strategy, alpha)


def knn_pool_ids(data, k: int, exclude_self: bool = True, rows=None):
    """Exact k-NN ids in (float64 dist, id) order (oracle.py:31-65 semantics,
    direct-difference float64).  ``rows`` restricts the query rows."""
    data = _f32(data)
    n, d = data.shape
    if rows is None:
        nr, rp = n, None
    else:
        rows = np.ascontiguousarray(rows, np.int64)
        nr, rp = rows.shape[0], _p(rows)
    out = np.empty((nr, k), np.int32)
    d64 = np.empty((nr, k), np.float64)
    lib().orc_knn_pool(_p(data), n, d, k, int(exclude_self), rp, nr, _p(out), _p(d64))
    return out, d64


def list_dists_sorted(data, ids, rows=None):
    """fp32 ``squared_l2(data[v], data[u])`` for an id table, rows re-sorted by
    (fp32 dist, id) (test_nsg.py:16-24 + sort_pairs)."""
    data = _f32(data)
    ids = np.array(ids, dtype=np.int32, copy=True, order="C")
    nr, k = ids.shape
    if rows is None:
        rp = None
    else:
        rows = np.ascontiguousarray(rows, np.int64)
        rp = _p(rows)
    dists = np.empty((nr, k), np.float32)
    lib().orc_list_dists_sorted(_p(data), data.shape[1], rp, nr, k, _p(ids), _p(dists))
    return ids, dists


def knn_pools(data, k: int, rows=None):
    """The hot path's candidate pools: exact k-NN (self excluded), fp32 list
    distances, rows ascending by (fp32 dist, id)."""
    ids, _ = knn_pool_ids(data, k, True, rows)
    return list_dists_sorted(data, ids, rows)


def ground_truth_table(data, k: int = 10, exclude_self: bool = False,
                       chunk: int = 256) -> np.ndarray:
    """oracle.py:31-65 restated with numpy (queries=None): float64 norm
    expansion through BLAS, clamp at 0, diagonal +inf, stable argsort."""
    if k < 1:
        raise ValueError("k must be >= 1")
    base = np.asarray(data, dtype=np.float64)
    n = base.shape[0]
    base_sq = np.einsum("ij,ij->i", base, base)
    out = np.empty((n, k), np.int32)
    for lo in range(0, n, chunk):
        hi = min(lo + chunk, n)
        block = base[lo:hi]
        d2 = base_sq[None, :] - 2.0 * (block @ base.T)
        d2 += np.einsum("ij,ij->i", block, block)[:, None]
        np.maximum(d2, 0.0, out=d2)
        if exclude_self:
            d2[np.arange(hi - lo), np.arange(lo, hi)] = np.inf
        order = np.argsort(d2, axis=1, kind="stable")
        out[lo:hi] = order[:, :k]
    return out


def refine_ab(data, pool_ids, pool_dists, M: int, strategy: str = "rng",
              alpha: float = 60.0):
    """Phases A and B on (n, K) pools (prune.py:232-249 with connect=False)."""
    n, K = pool_ids.shape
    off = np.arange(n + 1, dtype=np.int64) * K
    cnt = np.full(n, K, np.int32)
    a = prune_all(data, off, cnt, pool_ids.ravel(), pool_dists.ravel(), M, strategy, alpha)
    b = add_reverse_and_prune(data, a[0], a[1], a[2], M, strategy, alpha)
    return a, b


# ---------------------------------------------------------------------------
# Beam search and phase C (search.py:43-94, prune.py:154-229) -- restated on
# the C search core above; pinned by tests/golden/search.npz.
# ---------------------------------------------------------------------------

def search_batch(data, adj, counts, queries, k: int, L: int, ep: int, exclude: int = -1):
    """search.py:81-94 / _kernels.search_many: (ids, dists, dist_counts)."""
    data = _f32(data)
    adj = np.ascontiguousarray(adj, np.int32)
    counts = np.ascontiguousarray(counts, np.int32)
    q = _f32(np.atleast_2d(queries))
    nq = q.shape[0]
    ids = np.full((nq, k), EMPTY, np.int32)
    dists = np.full((nq, k), np.inf, np.float32)
    dc = np.zeros(nq, np.int64)
    lib().orc_search_many(_p(data), data.shape[0], data.shape[1], _p(adj), adj.shape[1],
                          _p(counts), _p(q), nq, k, L, int(ep), int(exclude), _p(ids),
                          _p(dists), _p(dc))
    return ids, dists, dc


def centroid(data) -> np.ndarray:
    """core.py:153-155: float64 mean, returned float32."""
    return np.asarray(data, np.float32).mean(axis=0, dtype=np.float64).astype(np.float32)


def entry_point(data, adj, counts, k: int, L: int, seed: int = 0) -> int:
    """prune.py:154-162: beam search for the centroid from a seeded random node."""
    n = np.asarray(data).shape[0]
    rn = int(np.random.default_rng(seed).integers(0, n))
    ids, _, _ = search_batch(data, adj, counts, centroid(data), k, L, rn)
    return int(ids[0, 0])


def mark_reachable(adj, counts, start: int, seen=None) -> np.ndarray:
    adj = np.ascontiguousarray(adj, np.int32)
    counts = np.ascontiguousarray(counts, np.int32)
    n = adj.shape[0]
    seen = np.zeros(n, np.uint8) if seen is None else np.ascontiguousarray(seen, np.uint8)
    lib().orc_mark_reachable(_p(adj), adj.shape[1], _p(counts), n, int(start), _p(seen))
    return seen


def connect(data, adj, counts, M: int, ep: int, connect_L: int):
    """prune.py:165-199 (_connect): one edge per unreachable component head
    (the first unreached id), from its nearest reachable node found by a
    beam search from ep; widening by one column when that node's row is
    full.  Returns (adj, counts, appended)."""
    adj = np.array(adj, np.int32, copy=True)
    counts = np.array(counts, np.int32, copy=True)
    n = adj.shape[0]
    seen = mark_reachable(adj, counts, ep)
    appended = 0
    while not seen.all():
        v = int(np.flatnonzero(seen == 0)[0])
        ids, _, _ = search_batch(data, adj, counts, np.asarray(data)[v], 1, connect_L, ep)
        r = int(ids[0, 0])
        if counts[r] == adj.shape[1]:
            adj = np.hstack([adj, np.full((n, 1), EMPTY, np.int32)])
        adj[r, counts[r]] = v
        counts[r] += 1
        appended += 1
        seen = mark_reachable(adj, counts, v, seen)
    return adj, counts, appended


def finish_connect(data, b_ids, b_counts, M: int, ep=None, seed: int = 0, connect_L=None):
    """The phase-C tail of prune.py:202-229 (finish_refine) on a phase-B graph:
    (adj, counts, ep, over_cap)."""
    L = max(M + 1, 32) if connect_L is None else connect_L
    if ep is None:
        ep = entry_point(data, b_ids, b_counts, 1, L, seed)
    adj, counts, _ = connect(data, b_ids, b_counts, M, ep, L)
    return adj, counts, int(ep), np.flatnonzero(counts > M).astype(np.int32)
