"""Float selection: the tensor-core Gram kernel (prune_gram_f32.cu, default)
against the per-warp prune_kernel (PGK_GRAM_F32=0) on a config prefix, each in
a fresh process: phases A and B must be identical (ids, dists, counts and the
dist_evals counters); times per phase are printed.

    python tools/gram_f32_check.py --config 3 --n 100000
"""
import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def child(a):
    import numpy as np
    import torch
    from paper_2410_01231_b200 import kernels, synth, _lib
    from paper_2410_01231_b200.index import RngBuilder
    from paper_2410_01231_b200.prune import PruneParams
    c = synth.CONFIGS[a.config]
    data = c["gen"](a.n) if a.config == 1 else c["gen"](a.n, c["n"])
    X = torch.from_numpy(data).cuda()
    n, d = X.shape
    strat = a.strategy
    p = PruneParams(M=c["R"], strategy=strat, alpha=a.alpha) if strat != "rng" else PruneParams(M=c["R"])
    b = RngBuilder(n, d, a.k or c["K"], p, _lib.POOL_F32)
    ids, dd = b.pools(X)
    order = b.order()
    torch.cuda.synchronize()
    res = {}
    for rep in range(a.reps):
        t0 = time.perf_counter()
        ra = kernels.prune_batch(X, b.cand_off, b.cand_counts, ids, dd, p.strategy_code, p.kernel_param,
                                 p.M, p.M, out=b.a_out, order=order, ws=b.prune_ws)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rb = kernels.add_reverse_and_prune(X, b.a_out[0], b.a_out[1], b.a_out[2], p.strategy_code,
                                           p.kernel_param, p.M, p.M, ws=b.rev_ws, out=b.b_out,
                                           order=order)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        res = {"A_ms": round(1e3 * (t1 - t0), 2), "B_ms": round(1e3 * (t2 - t1), 2)}
    out = {}
    for tag, r in (("a", ra), ("b", rb)):
        for i, name in enumerate(("ids", "dists", "counts", "de", "ae")):
            out[f"{tag}_{name}"] = r[i].cpu().numpy()
    np.savez(a.out, **out)
    res.update(mode=os.environ.get("PGK_GRAM_F32", "default"), n=n, d=d,
               mean_deg_A=float(ra[2].float().mean()), de_A=int(ra[3].sum()))
    print(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--strategy", default="rng")
    ap.add_argument("--alpha", type=float, default=1.2)
    ap.add_argument("--modes", default="0,1")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    if a.out:
        child(a)
        return
    import numpy as np
    res = {}
    for m in a.modes.split(","):
        path = f"/tmp/gramf32_{a.config}_{m}.npz"
        env = dict(os.environ, PGK_GRAM_F32=m)
        subprocess.check_call([sys.executable, __file__, "--config", str(a.config), "--n", str(a.n),
                               "--k", str(a.k), "--reps", str(a.reps), "--strategy", a.strategy,
                               "--alpha", str(a.alpha), "--out", path], env=env, timeout=3000)
        res[m] = dict(np.load(path))
    base = a.modes.split(",")[0]
    for m in a.modes.split(",")[1:]:
        diff = {k: int((res[m][k] != res[base][k]).sum()) for k in res[base]}
        print(json.dumps({"compare": f"{m} vs {base}", "differing_entries": diff}))


if __name__ == "__main__":
    main()
