"""Vector files and index persistence, format-compatible with the
reference's ``dataset_io.py``: GPU-built graphs round-trip
through the reference's own loader and vice versa.

* ``.fvecs`` / ``.ivecs`` / ``.bvecs``: per record a little-endian int32
  dimension, then the payload (float32 / int32 / uint8); every record must
  carry the same dimension (dataset_io.py:32-84).
* ``PGIX`` flat index (dataset_io.py:113-190): magic, u32 version 1, u8 kind 0,
  u32 M, u64 n, u64 ep, u32 #over-cap + int32 ids, u64 CSR offsets (n+1),
  int32 neighbour ids.  Vectors are never stored.  Loading validates the
  structure and raises ``CorruptIndexError`` (a ValueError) like the
  reference.
* ``PGIX`` layered index (kind 1, dataset_io.py:174-245): the FastHNSW
  hierarchy (``hnsw.LayeredGraph``), per layer its ascending member ids and a
  flat body; the loader checks nesting, coverage and the entry point.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .core import Dataset
from .graph import ProximityGraph

MAGIC = b"PGIX"
VERSION = 1
KIND_FLAT, KIND_LAYERED = 0, 1
_ITEM = {".fvecs": np.dtype("<f4"), ".ivecs": np.dtype("<i4"), ".bvecs": np.dtype(np.uint8)}


class CorruptIndexError(ValueError):
    """An index file failed structural validation."""


def _kind_of(path: Path) -> np.dtype:
    item = _ITEM.get(path.suffix.lower())
    if item is None:
        raise ValueError(f"{path}: unknown vector extension {path.suffix.lower()!r}")
    return item


def load_vecs(path) -> np.ndarray:
    """A .fvecs / .ivecs / .bvecs file as a 2-d array of its natural dtype."""
    path = Path(path)
    item = _kind_of(path)
    blob = np.fromfile(path, dtype=np.uint8)
    if blob.size == 0:
        raise ValueError(f"{path}: empty vector file")
    if blob.size < 4:
        raise ValueError(f"{path}: truncated vector file")
    dim = int(np.frombuffer(blob[:4].tobytes(), "<i4")[0])
    if dim <= 0:
        raise ValueError(f"{path}: bad leading dimension {dim}")
    rec = 4 + dim * item.itemsize
    if blob.size % rec:
        raise ValueError(f"{path}: file size not a multiple of the record size")
    table = blob.reshape(-1, rec)
    if not np.all(np.ascontiguousarray(table[:, :4]).view("<i4").ravel() == dim):
        raise ValueError(f"{path}: inconsistent record dimensions")
    return np.ascontiguousarray(table[:, 4:]).view(item).reshape(table.shape[0], dim)


def save_vecs(path, arr) -> None:
    """Write a 2-d array in the vecs flavour named by the extension."""
    path = Path(path)
    item = _kind_of(path)
    arr = np.asarray(arr)
    if arr.ndim != 2:
        raise ValueError("array must be 2-d")
    n, d = arr.shape
    out = np.empty((n, 4 + d * item.itemsize), np.uint8)
    out[:, :4] = np.full((n, 1), d, "<i4").view(np.uint8)
    out[:, 4:] = np.ascontiguousarray(arr, dtype=item).view(np.uint8).reshape(n, -1)
    out.tofile(path)


def load_dataset(path) -> Dataset:
    """A vecs file as a Dataset (ints / bytes widened to float32)."""
    return Dataset.from_array(load_vecs(path).astype(np.float32))


def _as_host(a) -> np.ndarray:
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def _flat_body(g: ProximityGraph) -> list:
    """u64 n, u64 ep, u32 #over-cap + int32 ids, u64 offsets, int32 neighbours
    (dataset_io.py:114-120)."""
    host = ProximityGraph(adj=_as_host(g.adj), counts=_as_host(g.counts), M=g.M, ep=g.ep,
                          over_cap=_as_host(g.over_cap))
    offsets, nbrs = host.to_csr()
    over = np.asarray(host.over_cap, "<i4")
    return [struct.pack("<QQI", host.n, int(g.ep), over.size), over.tobytes(),
            offsets.astype("<u8").tobytes(), nbrs.astype("<i4").tobytes()]


def save_index(path, g) -> None:
    """Write a PGIX index: flat (ProximityGraph) or layered (hnsw.LayeredGraph:
    u32 bottom M, u64 n, u64 ep, f64 m_factor, u32 #layers, then per layer
    u64 #members + int32 members, u32 M and a flat body; dataset_io.py:174-195)."""
    from .hnsw import LayeredGraph
    if isinstance(g, ProximityGraph):
        parts = [MAGIC, struct.pack("<IBI", VERSION, KIND_FLAT, int(g.M))] + _flat_body(g)
    elif isinstance(g, LayeredGraph):
        parts = [MAGIC, struct.pack("<IBI", VERSION, KIND_LAYERED, int(g.layers[0].graph.M)),
                 struct.pack("<QQdI", g.n, int(g.ep), float(g.m_factor), len(g.layers))]
        for layer in g.layers:
            mem = np.asarray(_as_host(layer.members), "<i4")
            parts += [struct.pack("<Q", mem.size), mem.tobytes(),
                      struct.pack("<I", int(layer.graph.M))] + _flat_body(layer.graph)
    else:
        raise TypeError(f"cannot serialize {type(g).__name__}")
    Path(path).write_bytes(b"".join(parts))


class _Cursor:
    """Bounds-checked little-endian reads over one file's bytes."""

    def __init__(self, path: Path):
        self.path = path
        self.buf = memoryview(path.read_bytes())
        self.pos = 0

    def take(self, nbytes: int) -> memoryview:
        if self.pos + nbytes > len(self.buf):
            raise CorruptIndexError(f"{self.path}: truncated index file")
        out = self.buf[self.pos:self.pos + nbytes]
        self.pos += nbytes
        return out

    def fields(self, fmt: str):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))

    def array(self, dtype: str, count: int) -> np.ndarray:
        dt = np.dtype(dtype)
        return np.frombuffer(self.take(dt.itemsize * count), dt).copy()

    def end(self) -> None:
        if self.pos != len(self.buf):
            raise CorruptIndexError(f"{self.path}: trailing bytes in index file")


def _read_flat(c: _Cursor, M: int) -> ProximityGraph:
    """A flat body with the reference's checks (dataset_io.py:142-167)."""
    path = c.path
    n, ep = c.fields("<QQ")
    if n < 1:
        raise CorruptIndexError(f"{path}: empty graph")
    if ep >= n:
        raise CorruptIndexError(f"{path}: entry point {ep} out of range")
    (n_over,) = c.fields("<I")
    over = c.array("<i4", n_over)
    offsets = c.array("<u8", n + 1).astype(np.int64)
    if offsets[0] != 0 or np.any(np.diff(offsets) < 0):
        raise CorruptIndexError(f"{path}: bad CSR offsets")
    nbrs = c.array("<i4", int(offsets[-1]))
    if nbrs.size and (nbrs.min() < 0 or nbrs.max() >= n):
        raise CorruptIndexError(f"{path}: neighbor id out of range")
    deg = np.diff(offsets)
    untagged = np.setdiff1d(np.flatnonzero(deg > M), over)
    if untagged.size:
        u = int(untagged[0])
        raise CorruptIndexError(f"{path}: node {u} degree {deg[u]} exceeds M={M}")
    return ProximityGraph.from_csr(offsets, nbrs, M=int(M), ep=int(ep), over_cap=over)


def _read_layered(c: _Cursor):
    """The layered body (dataset_io.py:213-245): nested, ascending member
    lists, the bottom layer = every node, the entry point in the top layer;
    levels are rebuilt from the nesting."""
    from .hnsw import LayeredGraph, LayerGraph
    path = c.path
    c.fields("<I")  # bottom layer's M, repeated in its own body
    n_total, ep, m_factor, n_layers = c.fields("<QQdI")
    if n_layers < 1:
        raise CorruptIndexError(f"{path}: layered index without layers")
    layers = []
    for li in range(n_layers):
        (n_members,) = c.fields("<Q")
        members = c.array("<i4", n_members)
        if np.any(np.diff(members) <= 0):
            raise CorruptIndexError(f"{path}: layer {li} members not ascending")
        (layer_m,) = c.fields("<I")
        g = _read_flat(c, layer_m)
        if g.n != n_members:
            raise CorruptIndexError(f"{path}: layer {li} graph size mismatch")
        layers.append(LayerGraph(members=members, graph=g))
    c.end()
    if len(layers[0].members) != n_total:
        raise CorruptIndexError(f"{path}: bottom layer must cover all nodes")
    if not np.array_equal(layers[0].members, np.arange(n_total, dtype=np.int32)):
        raise CorruptIndexError(f"{path}: bottom layer must contain every node")
    levels = np.zeros(n_total, dtype=np.int32)
    for li in range(1, n_layers):
        mem = layers[li].members
        if not np.all(np.isin(mem, layers[li - 1].members)):
            raise CorruptIndexError(f"{path}: layer {li} not nested")
        levels[mem] = li
    if ep >= n_total or levels[ep] != n_layers - 1:
        raise CorruptIndexError(f"{path}: entry point not in the top layer")
    return LayeredGraph(layers=layers, levels=levels, ep=int(ep), m_factor=float(m_factor))


def load_index(path):
    """Read a PGIX index (flat -> ProximityGraph, layered -> LayeredGraph) with
    the reference's structural checks (dataset_io.py:198-245)."""
    c = _Cursor(Path(path))
    if bytes(c.take(4)) != MAGIC:
        raise CorruptIndexError(f"{c.path}: not an index file (bad magic)")
    version, kind = c.fields("<IB")
    if version != VERSION:
        raise CorruptIndexError(f"{c.path}: unsupported version {version}")
    if kind == KIND_LAYERED:
        return _read_layered(c)
    if kind != KIND_FLAT:
        raise CorruptIndexError(f"{c.path}: unknown index kind {kind}")
    (M,) = c.fields("<I")
    g = _read_flat(c, M)
    c.end()
    return g


__all__ = ["CorruptIndexError", "load_vecs", "save_vecs", "load_dataset", "save_index",
           "load_index"]
