"""Device-level wrappers over the C ABI: torch CUDA tensors in, torch CUDA
tensors out, everything enqueued on the current stream with no host sync.

These are the building blocks of the reference-signature API (prune.py,
pool.py) and of the bench's device-resident timed region.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check, ptr

_F32, _I32, _I64 = torch.float32, torch.int32, torch.int64


def _dev(t, dtype) -> torch.Tensor:
    dev = _lib.device()
    if isinstance(t, torch.Tensor):
        t = t.to(device=dev, dtype=dtype)
    else:
        t = torch.as_tensor(t, dtype=dtype).to(dev)
    return t.contiguous()


def make_u8(X: torch.Tensor):
    """Exact-integer copy of an integer-valued [0,255] dataset (d <= 128):
    (rows of 128 bytes, int32 squared norms) -- pgk_make_u8."""
    X = _dev(X, _F32)
    n, d = X.shape
    xu8 = torch.empty((n, 128), dtype=torch.uint8, device=X.device)
    norms = torch.empty(n, dtype=_I32, device=X.device)
    check(_lib.lib().pgk_make_u8(ptr(X), n, d, ptr(xu8), ptr(norms), _lib.stream_handle()))
    return xu8, norms


def prune_batch(X: torch.Tensor, cand_off, cand_counts, cand_ids, cand_dists,
                strategy: int, cos_alpha: float, M: int, width: int | None = None,
                row_node=None, out=None, u8=None, order=None, ws=None):
    """Phase-A scan (pgk_prune_rows_ex).  ``u8`` = make_u8(X) selects the
    exact-integer distance path.  Returns device tensors (ids (rows, width),
    dists, counts, dist_evals (rows,), angle_evals (rows,))."""
    X = _dev(X, _F32)
    n, d = X.shape
    cand_off = _dev(cand_off, _I64)
    cand_counts = _dev(cand_counts, _I32)
    cand_ids = _dev(cand_ids, _I32)
    cand_dists = _dev(cand_dists, _F32)
    rows = cand_counts.shape[0]
    width = M if width is None else width
    dev = X.device
    if out is None:
        out = (torch.empty((rows, width), dtype=_I32, device=dev),
               torch.empty((rows, width), dtype=_F32, device=dev),
               torch.empty(rows, dtype=_I32, device=dev),
               torch.empty(rows, dtype=_I64, device=dev),
               torch.empty(rows, dtype=_I64, device=dev))
    ids, dists, counts, de, ae = out
    rn = None if row_node is None else _dev(row_node, _I32)
    xu8, norms = (None, None) if u8 is None else u8
    if ws is None:  # row lists of the tensor-core selection kernels (u8 and fp32)
        ws = _lib.workspace(prune_workspace_bytes(rows))
    check(_lib.lib().pgk_prune_rows_ex(
        ptr(X), ptr(xu8), ptr(norms), n, d, rows, ptr(rn), ptr(order), ptr(cand_off),
        ptr(cand_counts),
        ptr(cand_ids), ptr(cand_dists), int(strategy), float(cos_alpha), int(M), int(width),
        ptr(ids), ptr(dists), ptr(counts), ptr(de), ptr(ae), ptr(ws),
        0 if ws is None else ws.numel(), _lib.stream_handle()))
    return ids, dists, counts, de, ae


def prune_workspace_bytes(n_rows: int) -> int:
    b = ctypes.c_size_t(0)
    check(_lib.lib().pgk_prune_workspace(int(n_rows), ctypes.byref(b)))
    return int(b.value)


def reverse_workspace_bytes(n: int, a_width: int) -> int:
    b = ctypes.c_size_t(0)
    check(_lib.lib().pgk_reverse_workspace(int(n), int(a_width), ctypes.byref(b)))
    return int(b.value)


def add_reverse_and_prune(X: torch.Tensor, a_ids, a_dists, a_counts, strategy: int,
                          cos_alpha: float, M: int, width: int | None = None, ws=None,
                          out=None, u8=None, order=None):
    """Phase B (pgk_add_reverse_and_prune_ex); device tensors in and out."""
    X = _dev(X, _F32)
    n, d = X.shape
    a_ids = _dev(a_ids, _I32)
    a_dists = _dev(a_dists, _F32)
    a_counts = _dev(a_counts, _I32)
    a_width = a_ids.shape[1]
    width = M if width is None else width
    dev = X.device
    if ws is None:
        ws = _lib.workspace(reverse_workspace_bytes(n, a_width))
    if out is None:
        out = (torch.empty((n, width), dtype=_I32, device=dev),
               torch.empty((n, width), dtype=_F32, device=dev),
               torch.empty(n, dtype=_I32, device=dev),
               torch.empty(n, dtype=_I64, device=dev),
               torch.empty(n, dtype=_I64, device=dev))
    ids, dists, counts, de, ae = out
    xu8, norms = (None, None) if u8 is None else u8
    check(_lib.lib().pgk_add_reverse_and_prune_ex(
        ptr(X), ptr(xu8), ptr(norms), ptr(order), n, d, ptr(a_ids), ptr(a_dists), ptr(a_counts), a_width,
        int(strategy),
        float(cos_alpha), int(M), int(width), ptr(ids), ptr(dists), ptr(counts), ptr(de),
        ptr(ae), ptr(ws), ws.numel(), _lib.stream_handle()))
    return ids, dists, counts, de, ae


def knn_workspace_bytes(n: int, nq: int, d: int, k: int, mode: int) -> int:
    b = ctypes.c_size_t(0)
    check(_lib.lib().pgk_knn_workspace(int(n), int(nq), int(d), int(k), int(mode),
                                       ctypes.byref(b)))
    return int(b.value)


def detect_u8(X: torch.Tensor) -> bool:
    """True when every value is an integer in [0, 255] (and d <= 258): the
    exact integer pool path applies.  One blocking 4-byte read."""
    X = _dev(X, _F32)
    ws = _lib.workspace(256)
    flag = ctypes.c_int(0)
    check(_lib.lib().pgk_detect_u8(ptr(X), X.shape[0], X.shape[1], ctypes.byref(flag),
                                   ptr(ws), ws.numel(), _lib.stream_handle()))
    return bool(flag.value)


@dataclass
class PoolResult:
    pool_ids: torch.Tensor    # (nq, k) int32, rows ascending by (fp32 dist, id)
    pool_dists: torch.Tensor  # (nq, k) float32 squared_l2 list distances
    gt_ids: torch.Tensor | None  # (nq, k) int32 in (float64 dist, id) order
    ws: torch.Tensor


def knn_pools(X: torch.Tensor, k: int, queries=None, exclude_self: bool = True,
              mode: int = _lib.POOL_AUTO, want_gt: bool = True, ws=None,
              out=None, u8=None, assigned: bool = False) -> PoolResult:
    """Exact k-NN pools (pgk_knn_pools); device tensors, no sync (unless
    mode == AUTO, which reads one flag).  u8: optional (rows, norms) from
    make_u8 for the exact-integer self pool (pgk_knn_pools_u8): the pool
    then reuses them instead of converting X again."""
    X = _dev(X, _F32)
    n, d = X.shape
    Q = None if queries is None else _dev(queries, _F32)
    nq = n if Q is None else Q.shape[0]
    dev = X.device
    if ws is None:
        ws = _lib.workspace(knn_workspace_bytes(n, nq, d, k, mode))
    if out is None:
        out = (torch.empty((nq, k), dtype=_I32, device=dev),
               torch.empty((nq, k), dtype=_F32, device=dev),
               torch.empty((nq, k), dtype=_I32, device=dev) if want_gt else None)
    pool_ids, pool_dists, gt = out
    if u8 is not None and Q is None and exclude_self and mode == _lib.POOL_U8:
        xu8, norms = u8
        check(_lib.lib().pgk_knn_pools_u8(
            ptr(X), ptr(xu8), ptr(norms), n, d, int(k), int(bool(assigned)), ptr(gt),
            ptr(pool_ids), ptr(pool_dists), ptr(ws), ws.numel(), _lib.stream_handle()))
        return PoolResult(pool_ids, pool_dists, gt, ws)
    check(_lib.lib().pgk_knn_pools(
        ptr(X), n, d, ptr(Q), nq, int(k), int(bool(exclude_self)), int(mode), ptr(gt),
        ptr(pool_ids), ptr(pool_dists), ptr(ws), ws.numel(), _lib.stream_handle()))
    return PoolResult(pool_ids, pool_dists, gt, ws)


def knn_work(ws: torch.Tensor, n: int, nq: int, d: int, k: int, mode: int):
    """(pass-2, pass-1, assignment) 128x128 tile pairs executed by the last
    pruned pool call on ``ws`` and whether the pruned path ran (blocking)."""
    out = (ctypes.c_uint64 * 4)()
    check(_lib.lib().pgk_knn_work(ptr(ws), int(n), int(nq), int(d), int(k), int(mode), out,
                                  _lib.stream_handle()))
    return int(out[0]), int(out[1]), int(out[2]), bool(out[3])


def knn_order(ws: torch.Tensor, n: int, d: int, k: int, mode: int, out=None):
    """Locality processing order for the selection passes (pgk_knn_order)."""
    if out is None:
        out = torch.empty(n, dtype=_I32, device=ws.device)
    check(_lib.lib().pgk_knn_order(ptr(ws), int(n), int(d), int(k), int(mode), ptr(out),
                                   _lib.stream_handle()))
    return out


def fallback_rows(ws: torch.Tensor) -> int:
    """Rows of the last knn_pools call on ``ws`` that needed the exact
    float64 rescan (blocking)."""
    v = ctypes.c_int(0)
    check(_lib.lib().pgk_knn_fallback_rows(ptr(ws), ctypes.byref(v), _lib.stream_handle()))
    return int(v.value)


# ---------------------------------------------------------------------------
# beam search / phase C (search.cu)
# ---------------------------------------------------------------------------

def beam_search(X: torch.Tensor, adj: torch.Tensor, counts: torch.Tensor, queries, k: int,
                L: int, ep: int = 0, exclude: int = -1, eps=None, exp_cap: int = 0):
    """Beam search per query row (search.cu); returns device tensors
    (ids (nq, k), dists (nq, k), dist_counts (nq,), n_expanded (nq,)) and,
    with exp_cap > 0, the first exp_cap expanded nodes of each query (nq,
    exp_cap) as a fifth element."""
    dev = _lib.device()
    n, d = X.shape
    adj = _dev(adj, torch.int32)
    counts = _dev(counts, torch.int32)
    Q = _dev(queries, torch.float32).reshape(-1, d).contiguous()
    nq = Q.shape[0]
    eps_t = None if eps is None else _dev(eps, torch.int32)
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    dc = torch.empty(nq, dtype=torch.int64, device=dev)
    nexp = torch.empty(nq, dtype=torch.int64, device=dev)
    exps = torch.empty((nq, exp_cap), dtype=torch.int32, device=dev) if exp_cap > 0 else None
    worst = torch.empty((nq, exp_cap), dtype=torch.int64, device=dev) if exp_cap > 0 else None
    sz = ctypes.c_size_t(0)
    _lib.check(_lib.lib().pgk_search_workspace(n, nq, ctypes.byref(sz)))
    ws = _lib.workspace(sz.value)
    _lib.check(_lib.lib().pgk_beam_search_ex(
        _lib.ptr(X), n, d, _lib.ptr(adj), adj.shape[1], _lib.ptr(counts), _lib.ptr(Q), nq, k,
        L, _lib.ptr(eps_t), int(ep), int(exclude), _lib.ptr(ids), _lib.ptr(dists),
        _lib.ptr(dc), _lib.ptr(nexp), _lib.ptr(exps), _lib.ptr(worst), int(exp_cap),
        _lib.ptr(ws), ws.numel(), _lib.stream_handle()))
    if exp_cap > 0:
        return ids, dists, dc, nexp, exps, worst
    return ids, dists, dc, nexp


def pair_dists(X: torch.Tensor, a, b) -> torch.Tensor:
    """squared_l2(X[a[i]], X[b[i]]) per pair (fp32, reference order)."""
    a = _dev(a, torch.int32).contiguous()
    b = _dev(b, torch.int32).contiguous()
    out = torch.empty(a.numel(), dtype=torch.float32, device=X.device)
    _lib.check(_lib.lib().pgk_pair_dists(_lib.ptr(X), X.shape[1], _lib.ptr(a), _lib.ptr(b),
                                         a.numel(), _lib.ptr(out), _lib.stream_handle()))
    return out


def component_heads(adj: torch.Tensor, counts: torch.Tensor, seen: torch.Tensor,
                    ws: torch.Tensor) -> torch.Tensor:
    """Phase C's component heads in order (device int32), marking `seen`."""
    n = adj.shape[0]
    heads = torch.empty(n, dtype=torch.int32, device=adj.device)
    m = ctypes.c_int32(0)
    _lib.check(_lib.lib().pgk_component_heads(
        _lib.ptr(adj), adj.shape[1], _lib.ptr(counts), n, _lib.ptr(seen), _lib.ptr(heads),
        ctypes.byref(m), _lib.ptr(ws), ws.numel(), _lib.stream_handle()))
    return heads[: m.value]


def reach_workspace(n: int) -> torch.Tensor:
    sz = ctypes.c_size_t(0)
    _lib.check(_lib.lib().pgk_reach_workspace(n, ctypes.byref(sz)))
    return _lib.workspace(sz.value)


def mark_reachable(adj: torch.Tensor, counts: torch.Tensor, start: int, seen: torch.Tensor,
                   ws: torch.Tensor) -> None:
    """Extend the bitmap `seen` (int32 words viewed as uint32) from `start`."""
    _lib.check(_lib.lib().pgk_mark_reachable(
        _lib.ptr(adj), adj.shape[1], _lib.ptr(counts), adj.shape[0], int(start),
        _lib.ptr(seen), _lib.ptr(ws), ws.numel(), _lib.stream_handle()))


def first_unseen(seen: torch.Tensor, n: int, ws: torch.Tensor) -> int:
    out = ctypes.c_int32(0)
    _lib.check(_lib.lib().pgk_first_unseen(_lib.ptr(seen), n, ctypes.byref(out), _lib.ptr(ws),
                                           _lib.stream_handle()))
    return int(out.value)


def centroid(X: torch.Tensor) -> torch.Tensor:
    """float64 column means of the device dataset, as float32 (d,)."""
    n, d = X.shape
    sz = ctypes.c_size_t(0)
    _lib.check(_lib.lib().pgk_centroid_workspace(n, d, ctypes.byref(sz)))
    ws = _lib.workspace(sz.value)
    out = torch.empty(d, dtype=torch.float32, device=X.device)
    _lib.check(_lib.lib().pgk_centroid(_lib.ptr(X), n, d, _lib.ptr(out), _lib.ptr(ws),
                                       ws.numel(), _lib.stream_handle()))
    return out


# ---------------------------------------------------------------------------
# NN-Descent / FastNSG bookkeeping (nnd.cu)
# ---------------------------------------------------------------------------

def knng_init(X: torch.Tensor, draws: torch.Tensor, k0: int):
    """Rows from the first k0 distinct draws, sorted by (dist, id); returns
    (ids, dists, shortfall) device tensors."""
    dev = X.device
    n, d = X.shape
    draws = _dev(draws, torch.int64).contiguous()
    ids = torch.empty((n, k0), dtype=torch.int32, device=dev)
    dists = torch.empty((n, k0), dtype=torch.float32, device=dev)
    short = torch.empty(n, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().pgk_knng_init(_lib.ptr(X), n, d, _lib.ptr(draws), draws.shape[1], k0,
                                        _lib.ptr(ids), _lib.ptr(dists), _lib.ptr(short),
                                        _lib.stream_handle()))
    return ids, dists, short


def knng_sort_rows(X: torch.Tensor, rows, ids: torch.Tensor, dists: torch.Tensor) -> None:
    """Distances + (dist, id) sort of the listed rows' current ids (in place)."""
    rows = _dev(rows, torch.int32).contiguous()
    _lib.check(_lib.lib().pgk_knng_sort_rows(_lib.ptr(X), X.shape[1], _lib.ptr(rows),
                                             rows.numel(), ids.shape[1], _lib.ptr(ids),
                                             _lib.ptr(dists), _lib.stream_handle()))


def knng_round(X: torch.Tensor, ids, dists, flags, cap_new: int, cap_old: int):
    """One NN-Descent round -> (ids, dists, flags, upd (n,), evals (n,))."""
    n, d = X.shape
    k0 = ids.shape[1]
    o_ids, o_d, o_f = torch.empty_like(ids), torch.empty_like(dists), torch.empty_like(flags)
    upd = torch.empty(n, dtype=torch.int64, device=X.device)
    ev = torch.empty(n, dtype=torch.int64, device=X.device)
    sz = ctypes.c_size_t(0)
    _lib.check(_lib.lib().pgk_knng_round_workspace(n, k0, cap_new + cap_old, ctypes.byref(sz)))
    ws = _lib.workspace(sz.value)
    _lib.check(_lib.lib().pgk_knng_round(
        _lib.ptr(X), n, d, k0, _lib.ptr(ids), _lib.ptr(dists), _lib.ptr(flags), cap_new, cap_old,
        _lib.ptr(o_ids), _lib.ptr(o_d), _lib.ptr(o_f), _lib.ptr(upd), _lib.ptr(ev),
        _lib.ptr(ws), ws.numel(), _lib.stream_handle()))
    return o_ids, o_d, o_f, upd, ev


def mark_fresh(cand: torch.Tensor, ccnt: torch.Tensor, prev: torch.Tensor,
               pcnt: torch.Tensor) -> torch.Tensor:
    n, cw = cand.shape
    fresh = torch.empty((n, cw), dtype=torch.uint8, device=cand.device)
    _lib.check(_lib.lib().pgk_mark_fresh(_lib.ptr(cand), cw, _lib.ptr(ccnt), _lib.ptr(prev),
                                         prev.shape[1], _lib.ptr(pcnt), n, _lib.ptr(fresh),
                                         _lib.stream_handle()))
    return fresh
