"""Full-size parity figures on the GPU box -> one JSON object (committed as
profiles/r02_parity.json): pruned pools vs brute force on every row and vs
the oracle on 2,000 seeded rows (configs 2, 3, 4), and the config-2 prefix
graph comparison (edge agreement, recall@10 on the GPU vs the oracle graph).

    python tools/parity_report.py [--configs 2,3,4] [--n 50000] > gpurun_out/parity.json
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from _fullscale import graph_recall, pool_exactness  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4")
    ap.add_argument("--n", type=int, default=50_000)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--scale-n", type=int, default=0, help="also config 2's recipe at this size")
    a = ap.parse_args()
    out = {"pools": [], "graphs": []}
    for cfg in [int(x) for x in a.configs.split(",") if x]:
        r = pool_exactness(cfg)
        print(json.dumps(r), file=sys.stderr, flush=True)
        out["pools"].append(r)
    if a.scale_n:
        r = pool_exactness(2, oracle_rows=300, n=a.scale_n)
        print(json.dumps(r), file=sys.stderr, flush=True)
        out["pools"].append(r)
    if not a.no_graph:
        for strategy, alpha in (("rng", 60.0), ("alpha", 66.0)):
            r = graph_recall(a.n, 10_000, strategy=strategy, alpha=alpha)
            print(json.dumps(r), file=sys.stderr, flush=True)
            out["graphs"].append(r)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
