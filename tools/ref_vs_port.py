"""Time the reference's own CPU build (pgann: numpy-BLAS ground_truth_table +
numba kernels) beside the oracle port (numpy-BLAS restatement + C/OpenMP
restatement of the numba kernels) on the same seeded prefix, same thread
count, and check that both produce the same graph.

Build container only (imports the read-only reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src:. \
        python tools/ref_vs_port.py --cfg 2 --n 16337 --threads 8

Writes one JSON line to stdout (committed as profiles/r02_ref_vs_port.json):
the stage times of each arm and whether the phase-B graphs are identical.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--n", type=int, default=16337)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    os.environ.setdefault("NUMBA_NUM_THREADS", str(a.threads))
    os.environ.setdefault("OMP_NUM_THREADS", str(a.threads))
    import numpy as np
    from numba import njit, prange

    from pgann import _kernels
    from pgann.core import Dataset
    from pgann.oracle import ground_truth_table
    from pgann.prune import PruneParams, add_reverse_and_prune, prune_all

    from oracle import oracle
    from paper_2410_01231_b200 import synth

    @njit(parallel=True, cache=True)
    def list_dists(data, ids):
        n, k = ids.shape
        out = np.empty((n, k), np.float32)
        for u in prange(n):
            for j in range(k):
                out[u, j] = _kernels.squared_l2(data[ids[u, j]], data[u])
        return out

    @njit(cache=True)
    def resort(ids, dists):
        for u in range(ids.shape[0]):
            _kernels.sort_pairs(ids[u], dists[u], ids.shape[1])

    c = synth.CONFIGS[a.cfg]
    K, R = c["K"], c["R"]
    data = c["gen"](a.n) if a.cfg == 1 else c["gen"](a.n, c["n"])
    n = data.shape[0]

    def reference(x):
        t = {}
        t0 = time.perf_counter()
        ds = Dataset.from_array(x)
        truth = ground_truth_table(ds, None, k=K, exclude_self=True)
        t["pool"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        ids = truth.astype(np.int32).copy()
        dists = list_dists(ds.data, ids)
        resort(ids, dists)
        t["list_dists"] = time.perf_counter() - t1
        t2 = time.perf_counter()
        m = x.shape[0]
        off = np.arange(m + 1, dtype=np.int64) * K
        cnt = np.full(m, K, np.int32)
        p = PruneParams(M=R, strategy="rng")
        A = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), p)
        t["phase_A"] = time.perf_counter() - t2
        t3 = time.perf_counter()
        B = add_reverse_and_prune(ds, A[0], A[1], A[2], p)
        t["phase_B"] = time.perf_counter() - t3
        t["total"] = time.perf_counter() - t0
        return t, B

    def port(x):
        t = {}
        t0 = time.perf_counter()
        truth = oracle.ground_truth_table(x, K, exclude_self=True)
        t["pool"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        ids, dists = oracle.list_dists_sorted(x, truth)
        t["list_dists"] = time.perf_counter() - t1
        t2 = time.perf_counter()
        _, B = oracle.refine_ab(x, ids, dists, R, "rng", 60.0)
        t["phases_AB"] = time.perf_counter() - t2
        t["total"] = time.perf_counter() - t0
        return t, B

    warm = data[:500]  # numba JIT + caches, untimed
    reference(warm)
    port(warm)
    tr, Br = reference(data)
    tp, Bp = port(data)
    same = all(np.array_equal(Br[i], Bp[i]) for i in range(3)) and Br[3] == Bp[3]
    print(json.dumps({
        "what": "reference pgann (numba) vs the oracle port, same seeded prefix, same threads",
        "config": a.cfg, "n": n, "K": K, "R": R, "strategy": "rng", "threads": a.threads,
        "host": f"build container, {os.cpu_count()} cores",
        "reference_s": tr, "port_s": tp,
        "reference_points_per_s": n / tr["total"], "port_points_per_s": n / tp["total"],
        "port_over_reference": tr["total"] / tp["total"],
        "phase_B_graphs_identical": bool(same),
    }))


if __name__ == "__main__":
    main()
