import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2410_01231_b200 import synth, PruneParams
from paper_2410_01231_b200.index import RngBuilder, pool_mode
data = synth.cfg2(1_000_000)
X = torch.from_numpy(data).cuda()
b = RngBuilder(1_000_000, 128, 128, PruneParams(M=32), pool_mode(X))
out = b.build(X); torch.cuda.synchronize()
ids = b.a_out[0].cpu().numpy(); cnt = b.a_out[2].cpu().numpy()
n = ids.shape[0]
live = np.arange(32)[None, :] < cnt[:, None]
src = np.repeat(np.arange(n), cnt); dst = ids[live]
rev = np.bincount(dst, minlength=n)
# reciprocal: edge u->v where v->u also exists
key = src.astype(np.int64) * n + dst
rkey = dst.astype(np.int64) * n + src
recip = np.isin(rkey, key)
dup = np.bincount(src[recip], minlength=n)
union = cnt + rev - dup
for t in (16, 24, 32, 40, 48, 64, 96, 128):
    print(t, float((union <= t).mean()))
print("mean", union.mean())
