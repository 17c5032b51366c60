"""Config 5: FastHNSW build of 200k x 128 (config-2 recipe,
seed 4; ef=200, one M=32 for every layer -- the reference has a single M,
SURVEY A.1), timed on the GPU, plus recall@10 of the layered search over
10,000 seeded queries against the exact neighbours.  Prints one JSON line.

    python tools/bench_cfg5.py [--n N] [--queries Q] [--L L]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_01231_b200 import Dataset, ground_truth_table, hnsw, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--queries", type=int, default=10_000)
    ap.add_argument("--ef", type=int, default=200)
    ap.add_argument("--M", type=int, default=32)
    ap.add_argument("--k0", type=int, default=32)
    ap.add_argument("--L", type=int, default=100)
    a = ap.parse_args()
    base, q = synth.cfg5(a.n, a.queries)
    ds = Dataset.from_array(base)
    ds.device_data()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = hnsw.FastHnswStats()
    lg = hnsw.build_fasthnsw(ds, k0=a.k0, ef=a.ef, M=a.M, seed=4, stats=st)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    gt = ground_truth_table(ds, q, k=10)
    t1 = time.perf_counter()
    ids, _, _ = hnsw.layered_search_batch(ds, lg, q, 10, a.L)
    search_s = time.perf_counter() - t1
    hits = sum(len(set(ids[i][ids[i] >= 0].tolist()) & set(gt[i].tolist()))
               for i in range(a.queries))
    print(json.dumps({
        "workload": f"cfg5 FastHNSW build N={a.n} d=128 (cfg2 recipe, seed 4), k0={a.k0}, "
                    f"ef={a.ef}, M={a.M} (all layers), max_iters=2, alpha=66",
        "build_s": build_s, "points_per_s": a.n / build_s,
        "layers": [len(layer.members) for layer in lg.layers],
        "recall_at_10": hits / (10 * a.queries), "search_L": a.L, "queries": a.queries,
        "search_s_batched": search_s,
        "reference_cpu_s": 336.2, "reference_recall_at_10_L100": 0.95167,
        "reference_note": "tests/golden/cfg5.npz: the reference's own build (numba, 8 threads, "
                          "build container) and layered search; SURVEY 6.2 measured 250.3 s",
    }))


if __name__ == "__main__":
    main()
