"""Layered small-world index, layer-global construction (FastHNSW),
mirroring the reference's ``hnsw.py`` (hnsw.py:21-56, 133-192) and the
layered graph types of ``graph.py`` (graph.py:102-200): every node's top
layer is drawn up front, and each layer's graph is built over its whole
member set -- a complete digraph when the layer fits within M, otherwise
the iterative NSG build (nsg.build_fastnsg, on the GPU) restricted to the
members with k = L = ef.  ``layered_search`` is the reference's greedy
descent + bottom-layer beam search (search.py:97-130)."""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import kernels
from .core import Dataset
from .graph import EMPTY, ProximityGraph
from .nsg import FastNsgStats, build_fastnsg


def complete_graph(n: int, ep: int = 0) -> ProximityGraph:
    """Complete digraph; every node links to every other node ascending."""
    width = max(n - 1, 1)
    grid = np.broadcast_to(np.arange(n, dtype=np.int32), (n, n))
    keep = ~np.eye(n, dtype=bool)
    adj = np.empty((n, width), np.int32)
    if n > 1:
        adj[:, : n - 1] = grid[keep].reshape(n, n - 1)
    counts = np.full(n, n - 1, dtype=np.int32)
    return ProximityGraph(adj=adj, counts=counts, M=width, ep=ep)


@dataclass
class LayerGraph:
    """One layer: a local-id graph plus the (ascending) global member ids."""
    members: np.ndarray
    graph: ProximityGraph

    def local_of(self, global_id: int) -> int:
        pos = int(np.searchsorted(self.members, global_id))
        if pos >= len(self.members) or self.members[pos] != global_id:
            raise KeyError(f"node {global_id} not a member of this layer")
        return pos


@dataclass
class LayeredGraph:
    """Nested layers; layers[0] covers every node."""
    layers: list
    levels: np.ndarray
    ep: int
    m_factor: float

    @property
    def n(self) -> int:
        return len(self.layers[0].members)

    @property
    def max_level(self) -> int:
        return len(self.layers) - 1


@dataclass(frozen=True)
class LayerAssignment:
    """Per-node highest layer, drawn from a geometric-like decay."""
    levels: np.ndarray
    m_factor: float

    @property
    def m_l(self) -> int:
        return int(self.levels.max())

    def members(self, i: int) -> np.ndarray:
        return np.flatnonzero(self.levels >= i).astype(np.int32)


def assign_layers(n: int, m_factor: float, seed: int = 0) -> LayerAssignment:
    """l(u) = floor(-ln(U) * m_factor), U uniform on (0, 1] (hnsw.py:40-50):
    the same generator calls as the reference, so the same levels."""
    if m_factor <= 0:
        raise ValueError("m_factor must be > 0")
    if n < 1:
        raise ValueError("n must be >= 1")
    u = 1.0 - np.random.default_rng(seed).random(n)
    return LayerAssignment(levels=np.floor(-np.log(u) * m_factor).astype(np.int32),
                           m_factor=float(m_factor))


def _default_m_factor(M: int) -> float:
    if M < 2:
        raise ValueError("m_factor must be given explicitly when M < 2")
    return 1.0 / math.log(M)


@dataclass
class FastHnswStats:
    levels: Optional[np.ndarray] = None
    layer_sizes: list = field(default_factory=list)
    layer_stats: list = field(default_factory=list)


def build_fasthnsw(ds: Dataset, k0: int, ef: int, M: int, alpha: float = 66.0,
                   m_factor: Optional[float] = None, seed: int = 0, max_iters: int = 2,
                   connect_layers: bool = True, use_cache: bool = True,
                   stats: Optional[FastHnswStats] = None) -> LayeredGraph:
    """Layer-global construction (hnsw.py:141-192), top layer first."""
    if ef < 1:
        raise ValueError("ef must be >= 1")
    if M < 1:
        raise ValueError("M must be >= 1")
    if m_factor is None:
        m_factor = _default_m_factor(M)
    assign = assign_layers(ds.n, m_factor, seed)
    levels, m_l = assign.levels, assign.m_l
    top = assign.members(m_l)
    rng = np.random.default_rng(seed)
    ep = int(top[rng.integers(0, len(top))])
    if stats is not None:
        stats.levels = levels.copy()
    X = ds.device_data()
    layers = [None] * (m_l + 1)
    for i in range(m_l, -1, -1):
        members = assign.members(i)
        n_i = len(members)
        if stats is not None:
            stats.layer_sizes.insert(0, n_i)
        if n_i <= M or n_i <= 2:
            g = complete_graph(n_i, ep=int(np.searchsorted(members, ep)))
            if stats is not None:
                stats.layer_stats.insert(0, None)
        else:
            rows = torch.from_numpy(members.astype(np.int64)).to(X.device)
            sub = Dataset(X.index_select(0, rows).contiguous())
            sub_stats = FastNsgStats() if stats is not None else None
            g = build_fastnsg(sub, k0=min(k0, n_i - 1), k=min(ef, n_i - 1), L=min(ef, n_i - 1),
                              M=M, alpha=alpha, max_iters=max_iters, seed=seed + i + 1,
                              use_cache=use_cache, connect=connect_layers, stats=sub_stats)
            if stats is not None:
                stats.layer_stats.insert(0, sub_stats)
        layers[i] = LayerGraph(members=members, graph=g)
    return LayeredGraph(layers=layers, levels=levels, ep=ep, m_factor=m_factor)


def layered_search(ds: Dataset, lg: LayeredGraph, q, k: int, L: int):
    """Greedy descent through the upper layers (beam width 1), then a full
    beam search on the bottom layer (search.py:97-130)."""
    ids, dists, _ = layered_search_counted(ds, lg, q, k, L)
    return ids, dists


def layered_search_counted(ds: Dataset, lg: LayeredGraph, q, k: int, L: int):
    q = np.ascontiguousarray(q, dtype=np.float32)
    if q.shape != (ds.d,):
        raise ValueError(f"query must have shape ({ds.d},)")
    if k < 1 or k > L:
        raise ValueError("need 1 <= k <= L")
    X = ds.device_data()
    w = lg.ep
    n_dist = 0
    for li in range(lg.max_level, 0, -1):
        layer = lg.layers[li]
        rows = torch.from_numpy(layer.members.astype(np.int64)).to(X.device)
        sub = X.index_select(0, rows).contiguous()
        ids, _, dc, _ = kernels.beam_search(sub, layer.graph.adj, layer.graph.counts, q, 1, 1,
                                            layer.local_of(w))
        n_dist += int(dc[0].item())
        w = int(layer.members[int(ids[0, 0].item())])
    bottom = lg.layers[0]
    ids, dists, dc, _ = kernels.beam_search(X, bottom.graph.adj, bottom.graph.counts, q, k, L, w)
    ids, dists = ids[0].cpu().numpy(), dists[0].cpu().numpy()
    m = int((ids >= 0).sum())
    return ids[:m], dists[:m], n_dist + int(dc[0].item())


def layered_search_batch(ds: Dataset, lg: LayeredGraph, queries, k: int, L: int):
    """layered_search for every row of ``queries`` at once: per layer ONE
    beam-search launch over all queries, each from its own entry node (the
    queries are independent, so every row equals its sequential search,
    search.py:97-130).  Returns (ids (nq, k) -1 padded, dists (nq, k) +inf
    padded, dist_counts (nq,)) as numpy arrays."""
    Q = np.ascontiguousarray(queries, dtype=np.float32)
    if Q.ndim != 2 or Q.shape[1] != ds.d:
        raise ValueError(f"queries must have shape (nq, {ds.d})")
    if k < 1 or k > L:
        raise ValueError("need 1 <= k <= L")
    X = ds.device_data()
    nq = Q.shape[0]
    Qd = torch.from_numpy(Q).to(X.device)
    w = torch.full((nq,), lg.ep, dtype=torch.int64, device=X.device)
    n_dist = torch.zeros(nq, dtype=torch.int64, device=X.device)
    for li in range(lg.max_level, 0, -1):
        layer = lg.layers[li]
        mem = torch.from_numpy(layer.members.astype(np.int64)).to(X.device)
        sub = X.index_select(0, mem).contiguous()
        local = torch.searchsorted(mem, w).to(torch.int32)
        ids, _, dc, _ = kernels.beam_search(sub, layer.graph.adj, layer.graph.counts, Qd, 1, 1,
                                            eps=local)
        n_dist += dc
        w = mem[ids[:, 0].long()]
    bottom = lg.layers[0]
    ids, dists, dc, _ = kernels.beam_search(X, bottom.graph.adj, bottom.graph.counts, Qd, k, L,
                                            eps=w.to(torch.int32))
    return ids.cpu().numpy(), dists.cpu().numpy(), (n_dist + dc).cpu().numpy()


__all__ = ["complete_graph", "LayerGraph", "LayeredGraph", "LayerAssignment", "assign_layers",
           "FastHnswStats", "build_fasthnsw", "layered_search", "layered_search_counted", "layered_search_batch"]
