"""Graph container, mirroring the reference's ``graph.ProximityGraph``
(graph.py:20-99): fixed-width (n, width) int32 adjacency with -1 padding,
out-degree counts, degree cap M, entry point, over-cap tags."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

EMPTY = -1


@dataclass
class ProximityGraph:
    adj: np.ndarray            # (n, width) int32, -1 padded
    counts: np.ndarray         # (n,) int32 out-degrees
    M: int
    ep: int
    over_cap: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int32))

    @property
    def n(self) -> int:
        return self.adj.shape[0]

    def neighbors(self, u: int) -> np.ndarray:
        return self.adj[u, : self.counts[u]]

    def mean_degree(self) -> float:
        return float(self.counts.mean())

    def to_csr(self):
        """(offsets int64 (n+1), neighbour ids int32) (graph.py:63-71)."""
        counts = np.asarray(self.counts, np.int64)
        offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        live = np.arange(self.adj.shape[1])[None, :] < counts[:, None]
        return offsets, np.asarray(self.adj, np.int32)[live]

    @classmethod
    def from_csr(cls, offsets, nbrs, M: int, ep: int, over_cap=None) -> "ProximityGraph":
        """Row-padded adjacency of width max(max degree, 1) (graph.py:73-85)."""
        offsets = np.asarray(offsets, np.int64)
        counts = np.diff(offsets).astype(np.int32)
        n = counts.shape[0]
        width = max(int(counts.max()) if n else 0, 1)
        adj = np.full((n, width), EMPTY, dtype=np.int32)
        rows = np.repeat(np.arange(n), counts)
        cols = np.arange(int(offsets[-1])) - np.repeat(offsets[:-1], counts)
        adj[rows, cols] = np.asarray(nbrs, np.int32)
        over = np.empty(0, np.int32) if over_cap is None else np.asarray(over_cap, np.int32)
        return cls(adj=adj, counts=counts, M=M, ep=ep, over_cap=over)

    def validate(self) -> None:
        """Structural checks (graph.py:41-61), vectorised; ValueError on violation."""
        n = self.n
        if self.counts.shape != (n,):
            raise ValueError("counts shape mismatch")
        if not (0 <= self.ep < n):
            raise ValueError("entry point out of range")
        c = self.counts.astype(np.int64)
        if np.any(c > self.adj.shape[1]):
            raise ValueError(f"count exceeds row width at node {int(np.argmax(c > self.adj.shape[1]))}")
        over = np.zeros(n, bool)
        over[np.asarray(self.over_cap, np.int64)] = True
        bad = (c > self.M) & ~over
        if np.any(bad):
            u = int(np.argmax(bad))
            raise ValueError(f"degree {int(c[u])} > M={self.M} at untagged node {u}")
        live = np.arange(self.adj.shape[1])[None, :] < c[:, None]
        a = np.where(live, self.adj, 0)
        if np.any(live & ((self.adj < 0) | (self.adj >= n))):
            u = int(np.argmax(np.any(live & ((self.adj < 0) | (self.adj >= n)), axis=1)))
            raise ValueError(f"neighbor id out of range at node {u}")
        if np.any(live & (a == np.arange(n)[:, None])):
            u = int(np.argmax(np.any(live & (a == np.arange(n)[:, None]), axis=1)))
            raise ValueError(f"self-loop at node {u}")
        s = np.sort(np.where(live, self.adj, np.iinfo(np.int32).max), axis=1)
        dup = (s[:, 1:] == s[:, :-1]) & (s[:, 1:] != np.iinfo(np.int32).max)
        if np.any(dup):
            raise ValueError(f"duplicate neighbor at node {int(np.argmax(np.any(dup, axis=1)))}")

    def to_csr(self) -> tuple[np.ndarray, np.ndarray]:
        counts = self.counts.astype(np.int64)
        offsets = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(counts, out=offsets[1:])
        live = np.arange(self.adj.shape[1])[None, :] < counts[:, None]
        return offsets, self.adj[live].astype(np.int32)
