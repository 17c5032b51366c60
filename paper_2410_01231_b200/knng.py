"""Approximate kNN graph by NN-Descent, mirroring the reference's
``knng.py`` (knng.py:1-125): bulk-synchronous rounds over a frozen
snapshot, fresh/old flags for the incremental join, early stop on the
accepted-update count.  Rows, flags and update counts equal the
reference's; the random draws come from the same numpy generator calls.
The kernels are in nnd.cu (init rows, capped reverse lists, join sets,
join round)."""

from __future__ import annotations

import math

import numpy as np
import torch

from . import kernels
from .core import Dataset


class KnngState:
    """k0-NN lists: each row ascending (dist, id), exactly k0 wide.  The rows
    live on the device; ``ids`` / ``dists`` / ``flags`` give numpy copies."""

    def __init__(self, ids: torch.Tensor, dists: torch.Tensor, flags: torch.Tensor,
                 iterations: int = 0, last_updates: int = -1):
        self.d_ids, self.d_dists, self.d_flags = ids, dists, flags
        self.iterations = iterations
        self.last_updates = last_updates

    @property
    def ids(self) -> np.ndarray:
        return self.d_ids.cpu().numpy()

    @property
    def dists(self) -> np.ndarray:
        return self.d_dists.cpu().numpy()

    @property
    def flags(self) -> np.ndarray:
        return self.d_flags.cpu().numpy().astype(bool)

    @property
    def n(self) -> int:
        return int(self.d_ids.shape[0])

    @property
    def k0(self) -> int:
        return int(self.d_ids.shape[1])


def knng_init_random(ds: Dataset, k0: int, seed: int = 0) -> KnngState:
    """k0 distinct random non-self neighbours per node, sorted by (dist, id)
    (knng.py:40-61)."""
    n = ds.n
    if not (1 <= k0 < n):
        raise ValueError("need 1 <= k0 < n")
    X = ds.device_data()
    dev = X.device
    if k0 == n - 1:
        base = torch.arange(n, dtype=torch.int32, device=dev)
        full = base.repeat(n, 1)
        keep = full != base[:, None]
        ids = full[keep].reshape(n, n - 1).contiguous()
        dists = torch.empty((n, k0), dtype=torch.float32, device=dev)
        kernels.knng_sort_rows(X, base, ids, dists)
    else:
        rng = np.random.default_rng(seed)
        pad = max(16, k0 // 2)
        draws = rng.integers(0, n - 1, size=(n, k0 + pad)).astype(np.int64)
        ids, dists, short = kernels.knng_init(X, torch.from_numpy(draws), k0)
        bad = np.flatnonzero(short.cpu().numpy())
        if bad.size:
            # rare: an exact sample without replacement, seeded per row
            fix = np.empty((bad.size, k0), np.int32)
            for t, u in enumerate(bad):
                row_rng = np.random.default_rng([seed, 977, int(u)])
                pick = row_rng.permutation(n - 1)[:k0].astype(np.int64)
                pick[pick >= u] += 1
                fix[t] = pick
            rows = torch.from_numpy(bad.astype(np.int32)).to(dev)
            ids[rows.long()] = torch.from_numpy(fix).to(dev)
            kernels.knng_sort_rows(X, rows, ids, dists)
    flags = torch.ones((n, k0), dtype=torch.uint8, device=dev)
    return KnngState(ids, dists, flags, iterations=0)


def knng_descent_iterate(ds: Dataset, state: KnngState, rho: float = 1.0) -> KnngState:
    """One NN-Descent round; returns a new state (knng.py:64-101)."""
    if not (0.0 < rho <= 1.0):
        raise ValueError("rho must be in (0, 1]")
    cap = max(1, int(math.ceil(rho * state.k0)))
    ids, dists, flags, upd, _ = kernels.knng_round(ds.device_data(), state.d_ids, state.d_dists,
                                                   state.d_flags, cap, cap)
    return KnngState(ids, dists, flags, iterations=state.iterations + 1,
                     last_updates=int(upd.sum().item()))


def build_knng(ds: Dataset, k0: int, iters: int, seed: int = 0, rho: float = 1.0,
               min_update_frac: float = 0.001) -> KnngState:
    """Random init plus up to `iters` rounds, stopping once a round's accepted
    updates fall below min_update_frac * n * k0 (knng.py:104-115)."""
    state = knng_init_random(ds, k0, seed)
    threshold = min_update_frac * ds.n * k0
    for _ in range(iters):
        state = knng_descent_iterate(ds, state, rho=rho)
        if state.last_updates < threshold:
            break
    return state


__all__ = ["KnngState", "knng_init_random", "knng_descent_iterate", "build_knng"]
