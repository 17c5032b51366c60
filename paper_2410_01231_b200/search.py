"""Beam search over a proximity graph, mirroring the reference's
``search.py`` (search.py:25-94): ``kann_search`` (one query) and
``search_batch`` (many), same arguments, results, distance counts and
errors.  The search runs in libpgk.so (search.cu: warp per query, exact
pool / visited-set semantics of _kernels._search_core)."""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import kernels
from .core import Dataset
from .graph import ProximityGraph


def _graph_tensors(g: ProximityGraph):
    adj = g.adj if isinstance(g.adj, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(g.adj, np.int32))
    counts = g.counts if isinstance(g.counts, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(g.counts, np.int32))
    return adj, counts


def _check_args(ds: Dataset, g: ProximityGraph, q, k: int, L: int,
                ep: Optional[int]) -> int:
    """search.py:25-40."""
    if g.n != ds.n:
        raise ValueError("graph and dataset sizes differ")
    if k < 1:
        raise ValueError("k must be >= 1")
    if k > L:
        raise ValueError("k must not exceed the pool width L")
    if tuple(q.shape[-1:]) != (ds.d,):
        raise ValueError(f"query must have shape ({ds.d},)")
    if ep is None:
        ep = g.ep
    if not (0 <= ep < g.n):
        raise ValueError("entry point out of range")
    return int(ep)


def kann_search(ds: Dataset, g: ProximityGraph, q, k: int, L: int,
                ep: Optional[int] = None):
    """Beam search: expand the first unexpanded pool entry until the first L
    entries are all expanded; returns up to k (ids, dists) ascending (dist, id)."""
    qa = q if isinstance(q, torch.Tensor) else np.ascontiguousarray(q, np.float32)
    if tuple(qa.shape) != (ds.d,):
        raise ValueError(f"query must have shape ({ds.d},)")
    ep = _check_args(ds, g, qa, k, L, ep)
    adj, counts = _graph_tensors(g)
    ids, dists, _, _ = kernels.beam_search(ds.device_data(), adj, counts, qa, k, L, ep)
    ids, dists = ids[0].cpu().numpy(), dists[0].cpu().numpy()
    m = int((ids >= 0).sum())
    return ids[:m], dists[:m]


def search_batch(ds: Dataset, g: ProximityGraph, queries, k: int, L: int,
                 ep: Optional[int] = None):
    """Multi-query search -> (ids (nq, k) -1 padded, dists +inf padded,
    dist_counts (nq,) int64) (search.py:81-94)."""
    if queries.ndim != 2 or queries.shape[1] != ds.d:
        raise ValueError("queries must be (nq, d)")
    ep = _check_args(ds, g, queries[0], k, L, ep)
    adj, counts = _graph_tensors(g)
    ids, dists, dc, _ = kernels.beam_search(ds.device_data(), adj, counts, queries, k, L, ep)
    return ids.cpu().numpy(), dists.cpu().numpy(), dc.cpu().numpy()


__all__ = ["kann_search", "search_batch"]
