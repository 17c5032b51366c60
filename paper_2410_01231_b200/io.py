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
  reference.  The layered kind (FastHNSW, f3) is recognised and refused.
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


def save_index(path, g: ProximityGraph) -> None:
    """Write a flat PGIX index (CSR adjacency, M, entry point, over-cap tags)."""
    if not isinstance(g, ProximityGraph):
        raise TypeError(f"cannot serialize {type(g).__name__}")
    host = ProximityGraph(adj=_as_host(g.adj), counts=_as_host(g.counts), M=g.M, ep=g.ep,
                          over_cap=_as_host(g.over_cap))
    offsets, nbrs = host.to_csr()
    over = np.asarray(host.over_cap, "<i4")
    parts = [MAGIC, struct.pack("<IBI", VERSION, KIND_FLAT, int(g.M)),
             struct.pack("<QQI", host.n, int(g.ep), over.size), over.tobytes(),
             offsets.astype("<u8").tobytes(), nbrs.astype("<i4").tobytes()]
    Path(path).write_bytes(b"".join(parts))


def load_index(path) -> ProximityGraph:
    """Read a flat PGIX index with the reference's structural checks."""
    path = Path(path)
    buf = memoryview(path.read_bytes())
    pos = 0

    def take(nbytes: int) -> memoryview:
        nonlocal pos
        if pos + nbytes > len(buf):
            raise CorruptIndexError(f"{path}: truncated index file")
        out = buf[pos:pos + nbytes]
        pos += nbytes
        return out

    def fields(fmt: str):
        return struct.unpack(fmt, take(struct.calcsize(fmt)))

    def array(dtype: str, count: int) -> np.ndarray:
        dt = np.dtype(dtype)
        return np.frombuffer(take(dt.itemsize * count), dt).copy()

    if bytes(take(4)) != MAGIC:
        raise CorruptIndexError(f"{path}: not an index file (bad magic)")
    version, kind = fields("<IB")
    if version != VERSION:
        raise CorruptIndexError(f"{path}: unsupported version {version}")
    if kind == KIND_LAYERED:
        raise NotImplementedError(f"{path}: layered (FastHNSW) indexes are not part of this "
                                  "build")
    if kind != KIND_FLAT:
        raise CorruptIndexError(f"{path}: unknown index kind {kind}")
    (M,) = fields("<I")
    n, ep = fields("<QQ")
    if n < 1:
        raise CorruptIndexError(f"{path}: empty graph")
    if ep >= n:
        raise CorruptIndexError(f"{path}: entry point {ep} out of range")
    (n_over,) = fields("<I")
    over = array("<i4", n_over)
    offsets = array("<u8", n + 1).astype(np.int64)
    if offsets[0] != 0 or np.any(np.diff(offsets) < 0):
        raise CorruptIndexError(f"{path}: bad CSR offsets")
    nbrs = array("<i4", int(offsets[-1]))
    if nbrs.size and (nbrs.min() < 0 or nbrs.max() >= n):
        raise CorruptIndexError(f"{path}: neighbor id out of range")
    if pos != len(buf):
        raise CorruptIndexError(f"{path}: trailing bytes in index file")
    deg = np.diff(offsets)
    untagged = np.setdiff1d(np.flatnonzero(deg > M), over)
    if untagged.size:
        u = int(untagged[0])
        raise CorruptIndexError(f"{path}: node {u} degree {deg[u]} exceeds M={M}")
    return ProximityGraph.from_csr(offsets, nbrs, M=int(M), ep=int(ep), over_cap=over)


__all__ = ["CorruptIndexError", "load_vecs", "save_vecs", "load_dataset", "save_index",
           "load_index"]
