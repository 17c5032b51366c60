"""ctypes binding of libpgk.so (include/pgk.h).

There is deliberately no CPU fallback: if the library is missing or no CUDA
device is present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

PKG = Path(__file__).resolve().parent
# PGK_LIB_PATH: an alternative in-tree build of the same library (kernel
# variants compared by tools/build_variant.py); default the package's own
LIB_PATH = Path(os.environ.get("PGK_LIB_PATH", PKG / "libpgk.so"))

OK, ERR_INVALID, ERR_CUDA, ERR_NOMEM, ERR_UNSUPPORTED = 0, 1, 2, 3, 4
POOL_AUTO, POOL_U8, POOL_F32 = 0, 1, 2
POOL_NO_PRUNE = 0x10  # OR into a mode: brute-force kernels, no tile pruning

_lib = None


def lib():
    """Load libpgk.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python -m paper_2410_01231_b200.build_ext)")
        L = ctypes.CDLL(str(LIB_PATH))
        P, I64, I, D, SZ = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                            ctypes.c_double, ctypes.c_size_t)
        L.pgk_version.restype = ctypes.c_char_p
        L.pgk_last_error.restype = ctypes.c_char_p
        L.pgk_launch_count.restype = I64
        L.pgk_device_check.argtypes = [P]
        L.pgk_prune_batch.argtypes = [P, I64, I64, P, P, P, P, I, D, I64, I64,
                                      P, P, P, P, P, P]
        L.pgk_prune_rows.argtypes = [P, I64, I64, I64, P, P, P, P, P, I, D, I64, I64,
                                     P, P, P, P, P, P]
        L.pgk_prune_rows_ex.argtypes = [P, P, P, I64, I64, I64, P, P, P, P, P, P, I, D, I64,
                                        I64, P, P, P, P, P, P, SZ, P]
        L.pgk_prune_workspace.argtypes = [I64, P]
        L.pgk_make_u8.argtypes = [P, I64, I64, P, P, P]
        L.pgk_add_reverse_and_prune_ex.argtypes = [P, P, P, P, I64, I64, P, P, P, I64, I, D,
                                                   I64, I64, P, P, P, P, P, P, SZ, P]
        L.pgk_knn_order.argtypes = [P, I64, I64, I64, I, P, P]
        L.pgk_reverse_workspace.argtypes = [I64, I64, P]
        L.pgk_add_reverse_and_prune.argtypes = [P, I64, I64, P, P, P, I64, I, D, I64, I64,
                                                P, P, P, P, P, P, SZ, P]
        L.pgk_detect_u8.argtypes = [P, I64, I64, P, P, SZ, P]
        L.pgk_knn_workspace.argtypes = [I64, I64, I64, I64, I, P]
        L.pgk_knn_pools.argtypes = [P, I64, I64, P, I64, I64, I, I, P, P, P, P, SZ, P]
        L.pgk_knn_pools_u8.argtypes = [P, P, P, I64, I64, I64, I, P, P, P, P, SZ, P]
        L.pgk_tiles_center_stride.restype = I64
        L.pgk_tiles_supported.argtypes = [I64, I64, I64]
        L.pgk_tiles_u8_prepare.argtypes = [P, SZ, I64, I64, I64, P, P]
        L.pgk_tiles_u8_assign.argtypes = [P, SZ, I64, I64, I64, P, P, I64, I64, P]
        L.pgk_detect_u8_async.argtypes = [P, I64, I64, P, P]
        L.pgk_copy_rows_h2d.argtypes = [P, P, I64, I64, I64, P]
        L.pgk_knn_fallback_rows.argtypes = [P, P, P]
        L.pgk_knn_work.argtypes = [P, I64, I64, I64, I64, I, P, P]
        I32 = ctypes.c_int32
        L.pgk_search_workspace.argtypes = [I64, I64, P]
        L.pgk_beam_search.argtypes = [P, I64, I64, P, I64, P, P, I64, I64, I64, P, I32, I32,
                                      P, P, P, P, P, SZ, P]
        L.pgk_beam_search_ex.argtypes = [P, I64, I64, P, I64, P, P, I64, I64, I64, P, I32, I32,
                                         P, P, P, P, P, P, I64, P, SZ, P]
        L.pgk_pair_dists.argtypes = [P, I64, P, P, I64, P, P]
        L.pgk_component_heads.argtypes = [P, I64, P, I64, P, P, P, P, SZ, P]
        L.pgk_reach_workspace.argtypes = [I64, P]
        L.pgk_mark_reachable.argtypes = [P, I64, P, I64, I32, P, P, SZ, P]
        L.pgk_first_unseen.argtypes = [P, I64, P, P, P]
        L.pgk_centroid_workspace.argtypes = [I64, I64, P]
        L.pgk_centroid.argtypes = [P, I64, I64, P, P, SZ, P]
        L.pgk_knng_init.argtypes = [P, I64, I64, P, I64, I64, P, P, P, P]
        L.pgk_knng_sort_rows.argtypes = [P, I64, P, I64, I64, P, P, P]
        L.pgk_knng_round_workspace.argtypes = [I64, I64, I64, P]
        L.pgk_knng_round.argtypes = [P, I64, I64, I64, P, P, P, I64, I64, P, P, P, P, P, P, SZ,
                                     P]
        L.pgk_mark_fresh.argtypes = [P, I64, P, P, I64, P, I64, P, P]
        for f in ("pgk_device_check", "pgk_prune_batch", "pgk_prune_rows", "pgk_prune_rows_ex",
                  "pgk_prune_workspace",
                  "pgk_make_u8", "pgk_add_reverse_and_prune_ex", "pgk_reverse_workspace",
                  "pgk_add_reverse_and_prune", "pgk_detect_u8", "pgk_knn_workspace",
                  "pgk_knn_pools", "pgk_knn_pools_u8", "pgk_knn_fallback_rows", "pgk_knn_work",
                  "pgk_knn_order", "pgk_search_workspace", "pgk_tiles_u8_prepare",
                  "pgk_tiles_u8_assign", "pgk_detect_u8_async", "pgk_copy_rows_h2d", "pgk_beam_search", "pgk_reach_workspace",
                  "pgk_beam_search_ex", "pgk_component_heads", "pgk_pair_dists",
                  "pgk_mark_reachable", "pgk_first_unseen", "pgk_centroid_workspace",
                  "pgk_centroid", "pgk_knng_init", "pgk_knng_sort_rows",
                  "pgk_knng_round_workspace", "pgk_knng_round", "pgk_mark_fresh"):
            getattr(L, f).restype = I
        _lib = L
    return _lib


EXPORTS = ("pgk_version", "pgk_last_error", "pgk_device_check", "pgk_prune_batch",
           "pgk_prune_rows", "pgk_prune_rows_ex", "pgk_prune_workspace", "pgk_make_u8", "pgk_add_reverse_and_prune_ex",
           "pgk_reverse_workspace", "pgk_add_reverse_and_prune", "pgk_detect_u8",
           "pgk_knn_workspace", "pgk_knn_pools", "pgk_knn_pools_u8", "pgk_knn_fallback_rows",
           "pgk_tiles_center_stride", "pgk_tiles_supported", "pgk_tiles_u8_prepare", "pgk_tiles_u8_assign",
           "pgk_detect_u8_async", "pgk_copy_rows_h2d",
           "pgk_knn_work",
           "pgk_knn_order", "pgk_search_workspace", "pgk_beam_search", "pgk_reach_workspace",
           "pgk_mark_reachable", "pgk_first_unseen", "pgk_centroid_workspace", "pgk_centroid",
           "pgk_beam_search_ex", "pgk_component_heads", "pgk_pair_dists", "pgk_knng_init", "pgk_knng_sort_rows", "pgk_knng_round_workspace", "pgk_knng_round",
           "pgk_mark_fresh", "pgk_launch_count")


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().pgk_last_error().decode(errors="replace")
    if rc == ERR_INVALID:
        raise ValueError(msg)
    if rc == ERR_NOMEM:
        raise MemoryError(msg)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


_device_ok = False


def device() -> torch.device:
    """The CUDA device the kernels run on (raises without a B200)."""
    global _device_ok
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2410_01231_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    if not _device_ok:
        sms = ctypes.c_int(0)
        check(lib().pgk_device_check(ctypes.byref(sms)))
        _device_ok = True
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def launch_count() -> int:
    return int(lib().pgk_launch_count())


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device())
