"""Exact k-NN candidate pools -- drop-in for the reference's
``pgann.oracle`` (``ground_truth_table`` / ``exact_knn`` / recall helpers,
oracle.py:17-84) plus ``knn_pools``, the hot path's pool step: exact k-NN
(self excluded), fp32 ``squared_l2`` list distances, rows ascending by
(fp32 dist, id) -- the composition the reference's tests feed to
``prune_all`` (test_nsg.py:16-24, test_prune.py:35-41).

All distance work runs in libpgk.so (``pgk_knn_pools``): exact integer
arithmetic for [0,255]-integer data, otherwise an fp32 pass + float64 rerank
with a proven boundary (see csrc/pool_simt.cu).
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _lib, kernels
from .core import Dataset


def _mode(ds: Dataset, queries) -> int:
    if not ds.is_u8():
        return _lib.POOL_F32
    if queries is not None and not kernels.detect_u8(queries):
        return _lib.POOL_F32
    return _lib.POOL_U8


def knn_pools(ds: Dataset, k: int, want_gt: bool = False):
    """(ids (n, k) int32, dists (n, k) float32[, gt_ids]) -- exact k-NN of every
    point, self excluded, ascending (fp32 dist, id).  numpy for a numpy
    dataset, device tensors for a device dataset."""
    if k < 1:
        raise ValueError("k must be >= 1")
    r = kernels.knn_pools(ds.device_data(), k, None, True, _mode(ds, None), want_gt)
    if isinstance(ds.data, torch.Tensor):
        return (r.pool_ids, r.pool_dists, r.gt_ids) if want_gt else (r.pool_ids, r.pool_dists)
    out = (r.pool_ids.cpu().numpy(), r.pool_dists.cpu().numpy())
    return out + (r.gt_ids.cpu().numpy(),) if want_gt else out


def ground_truth_table(ds: Dataset, queries: Optional[np.ndarray] = None, k: int = 10,
                       exclude_self: bool = False, chunk: int = 256) -> np.ndarray:
    """Exact kNN ids for each query row; queries=None means every node
    (oracle.py:31-65).  ``chunk`` is accepted for signature compatibility (the
    GPU kernel tiles on its own; results do not depend on it)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    q = None
    if queries is not None:
        q = np.asarray(queries, dtype=np.float32) if not isinstance(queries, torch.Tensor) \
            else queries
        if q.ndim != 2 or q.shape[1] != ds.d:
            raise ValueError("queries must be (nq, d)")
        if exclude_self:
            raise ValueError("exclude_self requires queries=None")
    r = kernels.knn_pools(ds.device_data(), k, q, exclude_self, _mode(ds, q), True)
    return r.gt_ids.cpu().numpy()


def exact_knn(ds: Dataset, q: np.ndarray, k: int,
              exclude_id: Optional[int] = None) -> tuple[np.ndarray, np.ndarray]:
    """The k nearest ids and squared distances to q, ascending (dist, id)
    (oracle.py:17-28).  Distances are float64 like the reference's."""
    if k < 1:
        raise ValueError("k must be >= 1")
    q = np.asarray(q, dtype=np.float32).reshape(1, -1)
    kk = min(ds.n, k + (1 if exclude_id is not None else 0))
    ids = ground_truth_table(ds, q, k=kk)[0]
    if exclude_id is not None:
        ids = ids[ids != exclude_id]
    ids = ids[:k].astype(np.int32)
    X = ds.device_data()
    sel = X[torch.as_tensor(ids, dtype=torch.int64, device=X.device)].double()
    qd = torch.as_tensor(q[0], device=X.device).double()
    d2 = ((sel - qd) ** 2).sum(dim=1).cpu().numpy()
    return ids, d2


def recall_at_k(approx_ids, exact_ids, k: int) -> float:
    """|approx[:k] & exact[:k]| / k (oracle.py:68-74)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    a = set(int(x) for x in np.asarray(approx_ids).ravel()[:k])
    e = set(int(x) for x in np.asarray(exact_ids).ravel()[:k])
    return len(a & e) / k


def mean_recall(approx_table, exact_table, k: int) -> float:
    """Mean recall_at_k across rows (oracle.py:77-84)."""
    if approx_table.shape[0] != exact_table.shape[0]:
        raise ValueError("tables must have matching row counts")
    total = 0.0
    for i in range(approx_table.shape[0]):
        total += recall_at_k(approx_table[i], exact_table[i], k)
    return total / approx_table.shape[0]
