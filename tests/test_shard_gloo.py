"""Multi-process (gloo, world_size 2, CPU) test of the sharded path's only
collective: the phase-B reverse-edge exchange (paper_2410_01231_b200/shard.py)
must deliver to every rank exactly the reverse lists the single-process
scatter (prune.py:134-141) builds for its rows."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_01231_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _phase_a(n, width, seed):
    rng = np.random.default_rng(seed)
    ids = np.full((n, width), -1, np.int32)
    dists = np.full((n, width), np.inf, np.float32)
    counts = rng.integers(0, width + 1, size=n).astype(np.int32)
    for u in range(n):
        nb = rng.choice(np.delete(np.arange(n), u), size=counts[u], replace=False)
        ids[u, :counts[u]] = nb
        dists[u, :counts[u]] = np.sort(rng.random(counts[u]).astype(np.float32))
    return ids, dists, counts


def _worker(rank, world, port, n, width, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids, dists, counts = _phase_a(n, width, seed)
    lo, hi = shard.row_range(n, world, rank)
    dst, src, dd = shard.exchange_reverse(torch.from_numpy(ids[lo:hi]),
                                          torch.from_numpy(dists[lo:hi]),
                                          torch.from_numpy(counts[lo:hi]), lo, n)
    got = {}
    for v, u, x in zip(dst.tolist(), src.tolist(), dd.tolist()):
        got.setdefault(v, []).append((u, x))
    q.put((rank, lo, hi, got))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,width", [(257, 6), (40, 3)])
def test_reverse_exchange_world2(n, width):
    world, seed = 2, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, width, seed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids, dists, counts = _phase_a(n, width, seed)
    want = shard.reverse_lists_reference(ids, counts, n)
    seen = set()
    for rank, lo, hi, got in results:
        for v in range(lo, hi):
            pairs = sorted(got.get(v, []))
            assert [u for u, _ in pairs] == want[v]
            for u, x in pairs:  # the owner's stored distance travels with the edge
                j = int(np.nonzero(ids[u, :counts[u]] == v)[0][0])
                assert x == float(dists[u, j])
            seen.add(v)
        assert all(lo <= v < hi for v in got)
    assert seen == set(range(n))


def test_row_range_and_owner():
    for n in (1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            rr = [shard.row_range(n, world, r) for r in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == n
            assert all(rr[i][1] == rr[i + 1][0] for i in range(world - 1))
            owners = shard.owner_of(torch.arange(n), n, world).tolist()
            for r, (lo, hi) in enumerate(rr):
                assert all(owners[i] == r for i in range(lo, hi))
