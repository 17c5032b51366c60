"""GPU timeline of one host-data build (RngBuilder.build_host) on config 2:
copies and kernels with start offsets, to check what the chunked copy hides.

    python tools/prof_e2e.py [--n N] [--chunks C]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2410_01231_b200 import _lib, synth  # noqa: E402
from paper_2410_01231_b200.index import RngBuilder  # noqa: E402
from paper_2410_01231_b200.prune import PruneParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1000000)
    ap.add_argument("--chunks", type=int, default=8)
    a = ap.parse_args()
    data = synth.cfg2(a.n)
    host = torch.from_numpy(data).pin_memory()
    b = RngBuilder(a.n, 128, 128, PruneParams(M=32), _lib.POOL_U8)
    ids = torch.empty((a.n, 32), dtype=torch.int32).pin_memory()
    cnt = torch.empty(a.n, dtype=torch.int32).pin_memory()
    for _ in range(3):
        b.build_host(host, (ids, cnt), a.chunks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        e0.record()
        b.build_host(host, (ids, cnt), a.chunks)
        e1.record()
        torch.cuda.synchronize()
    print(f"build_host: {e0.elapsed_time(e1):.2f} ms")
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    t0 = min(e.time_range.start for e in evs)
    for e in sorted(evs, key=lambda e: e.time_range.start):
        dur = (e.time_range.end - e.time_range.start) / 1e3
        if dur > 0.05:
            print(f"  +{(e.time_range.start - t0) / 1e3:8.3f} ms  {dur:7.3f} ms  {e.name[:70]}")


if __name__ == "__main__":
    main()
