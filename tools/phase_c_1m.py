"""Phase C (connectivity repair, prune.py:165-199) on the config-2 1M phase-B
graph: time it and report recall@10 of the search before and after.

    python tools/phase_c_1m.py [--n N]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_01231_b200 import Dataset, ProximityGraph, pool, prune, search, synth  # noqa: E402
from paper_2410_01231_b200.index import RngBuilder, pool_mode  # noqa: E402
from paper_2410_01231_b200.prune import PruneParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    a = ap.parse_args()
    data = synth.cfg2(a.n)
    X = torch.from_numpy(data).cuda()
    R, K = 32, 128
    b = RngBuilder(a.n, 128, K, PruneParams(M=R), pool_mode(X))
    out = b.build(X)
    torch.cuda.synchronize()
    ds = Dataset.from_array(data)
    ds._dev = X
    g = ProximityGraph(adj=out.ids, counts=out.counts, M=R, ep=0)
    L = max(R + 1, 32)
    t0 = time.perf_counter()
    ep = prune.entry_point(ds, g, k=1, L=L)
    t1 = time.perf_counter()
    adj, counts, appended = prune._connect(ds, out.ids, out.counts, R, ep, L)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    gc = ProximityGraph(adj=adj, counts=counts, M=R, ep=ep)
    q = synth.cfg2_queries(10_000)
    truth = pool.ground_truth_table(ds, q, k=10)
    rec = {}
    for L2 in (20, 50, 100, 200):
        i0, _, _ = search.search_batch(ds, g, q, 10, L2, ep=ep)
        i1, _, _ = search.search_batch(ds, gc, q, 10, L2, ep=ep)
        rec[f"L{L2}"] = {"phase_b": pool.mean_recall(i0, truth, 10),
                         "phase_c": pool.mean_recall(i1, truth, 10)}
    print(json.dumps({"n": a.n, "entry_point_s": t1 - t0, "phase_c_s": t2 - t1,
                      "repair_edges": int(appended), "ep": int(ep), "recall_at_10": rec}))


if __name__ == "__main__":
    main()
