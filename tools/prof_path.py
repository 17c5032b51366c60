"""Run one hot-path stage on a config prefix (profiling driver for ncu).

    python tools/prof_path.py --stage pool|prune|all --config 2 --n 131072
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2410_01231_b200 import kernels, synth  # noqa: E402
from paper_2410_01231_b200.index import RngBuilder, pool_mode  # noqa: E402
from paper_2410_01231_b200.prune import PruneParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", default="all")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--kernels", action="store_true",
                    help="per-kernel device time of the last rep (CUPTI trace)")
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    data = c["gen"](a.n) if a.config == 1 else c["gen"](a.n, c["n"])
    X = torch.from_numpy(data).cuda()
    b = RngBuilder(a.n, data.shape[1], c["K"], PruneParams(M=c["R"]), pool_mode(X))
    ids, d = b.pools(X)
    torch.cuda.synchronize()
    p = b.params
    prof = None
    for rep in range(a.reps):
        if a.kernels and rep == a.reps - 1:
            prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA])
            prof.__enter__()
        t0 = time.perf_counter()
        u8 = b.u8_rows(X)
        if a.stage in ("pool", "all"):
            ids, d = b.pools(X, u8)
        order = b.order()
        if a.stage in ("prune", "all"):
            r = kernels.prune_batch(X, b.cand_off, b.cand_counts, ids, d, p.strategy_code,
                                    p.cos_alpha, p.M, p.M, out=b.a_out, u8=u8, order=order,
                                    ws=b.prune_ws)
        if a.stage in ("reverse", "all"):
            kernels.add_reverse_and_prune(X, b.a_out[0], b.a_out[1], b.a_out[2],
                                          p.strategy_code, p.cos_alpha, p.M, p.M, ws=b.rev_ws,
                                          out=b.b_out, u8=u8, order=order)
        torch.cuda.synchronize()
        print(f"{a.stage} n={a.n}: {1e3 * (time.perf_counter() - t0):.2f} ms")
    if prof is not None:
        prof.__exit__(None, None, None)
        seq = [(e.name, e.device_time) for e in prof.events()
               if e.device_type == torch.autograd.DeviceType.CUDA]
        for name, us in seq:
            print(f"  {us / 1e3:8.3f} ms  {name[:90]}")


if __name__ == "__main__":
    main()
