"""Float pools: tensor-core passes (PGK_F32_TC=2 / 1) against the SIMT passes
(PGK_F32_TC=0) on a config prefix, each in a fresh process (the switch is read
once per process): pool ids / dists must be identical, times and the number
of rows that needed the exact rescan are printed.

    python tools/f32_tc_check.py --config 3 --n 100000
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
    c = synth.CONFIGS[a.config]
    data = c["gen"](a.n) if a.config == 1 else c["gen"](a.n, c["n"])
    K = a.k or c["K"]
    X = torch.from_numpy(data).cuda()
    n, d = X.shape
    ws = _lib.workspace(kernels.knn_workspace_bytes(n, n, d, K, _lib.POOL_F32))
    times = []
    for rep in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = kernels.knn_pools(X, K, mode=_lib.POOL_F32, ws=ws)
        torch.cuda.synchronize()
        times.append(1e3 * (time.perf_counter() - t0))
    fb = kernels.fallback_rows(ws)
    if a.kernels:
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            kernels.knn_pools(X, K, mode=_lib.POOL_F32, ws=ws)
            torch.cuda.synchronize()
        agg = {}
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                k = e.name[:70]
                agg[k] = (agg.get(k, (0, 0))[0] + e.device_time / 1e3, agg.get(k, (0, 0))[1] + 1)
        for k, (ms, cnt) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:14]:
            print(f"  {ms:9.3f} ms  x{cnt:<4d} {k}")
    np.savez(a.out, ids=r.pool_ids.cpu().numpy(), dists=r.pool_dists.cpu().numpy())
    print(json.dumps({"mode": os.environ.get("PGK_F32_TC", "default"), "n": n, "d": d, "K": K,
                      "ms": [round(t, 2) for t in times], "fallback_rows": fb}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--modes", default="0,1,2")
    ap.add_argument("--out", default="")
    ap.add_argument("--kernels", action="store_true")
    a = ap.parse_args()
    if a.out:
        child(a)
        return
    import numpy as np
    res = {}
    for m in a.modes.split(","):
        path = f"/tmp/f32tc_{a.config}_{m}.npz"
        env = dict(os.environ, PGK_F32_TC=m)
        subprocess.check_call([sys.executable, __file__, "--config", str(a.config), "--n", str(a.n),
                               "--k", str(a.k), "--reps", str(a.reps), "--out", path] +
                              (["--kernels"] if a.kernels else []), env=env,
                              timeout=3000)
        res[m] = dict(np.load(path))
    base = a.modes.split(",")[0]
    for m in a.modes.split(",")[1:]:
        same_ids = bool((res[m]["ids"] == res[base]["ids"]).all())
        same_d = bool((res[m]["dists"] == res[base]["dists"]).all())
        bad = int((res[m]["ids"] != res[base]["ids"]).any(axis=1).sum())
        print(json.dumps({"compare": f"{m} vs {base}", "ids_equal": same_ids,
                          "dists_equal": same_d, "rows_differing": bad}))


if __name__ == "__main__":
    main()
