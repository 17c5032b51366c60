"""e2e (host data in, adjacency out) time of RngBuilder.build_host at config 2
for several copy-chunk counts (CUDA events, L2 flushed between runs)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2410_01231_b200 import _lib, synth
from paper_2410_01231_b200.index import RngBuilder
from paper_2410_01231_b200.prune import PruneParams

n = 1000000
host = torch.from_numpy(synth.cfg2(n)).pin_memory()
b = RngBuilder(n, 128, 128, PruneParams(M=32), _lib.POOL_U8)
ids = torch.empty((n, 32), dtype=torch.int32).pin_memory()
cnt = torch.empty(n, dtype=torch.int32).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for chunks in (2, 4, 8, 16, 32):
    for _ in range(3):
        b.build_host(host, host_out=(ids, cnt), chunks=chunks)
    ts = []
    for _ in range(8):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        b.build_host(host, host_out=(ids, cnt), chunks=chunks)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"chunks {chunks:3d}: median {ts[len(ts) // 2]:.2f} ms  min {ts[0]:.2f} ms")
