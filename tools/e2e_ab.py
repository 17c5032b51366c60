import sys, time
sys.path.insert(0, ".")
import torch
from paper_2410_01231_b200 import _lib, synth
from paper_2410_01231_b200.index import RngBuilder, pool_mode
from paper_2410_01231_b200.prune import PruneParams
n = 1000000
data = synth.cfg2(n)
host = torch.from_numpy(data).pin_memory()
b = RngBuilder(n, 128, 128, PruneParams(M=32), _lib.POOL_U8)
ids = torch.empty((n, 32), dtype=torch.int32).pin_memory()
cnt = torch.empty(n, dtype=torch.int32).pin_memory()
Xe = torch.empty((n, 128), dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def old():
    Xe.copy_(host, non_blocking=True)
    assert pool_mode(Xe) == _lib.POOL_U8
    b.build(Xe, host_out=(ids, cnt))
def new():
    b.build_host(host, host_out=(ids, cnt))
for name, f in (("old", old), ("new", new), ("old", old), ("new", new)):
    for _ in range(3): f()
    torch.cuda.synchronize()
    ts = []
    for s in range(10):
        flush.fill_(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(name, "median %.2f ms min %.2f" % (ts[5], ts[0]), "->", "%.2fM pts/s" % (n / ts[5] / 1e3))
