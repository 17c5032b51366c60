"""Row sharding of the hot path across ranks (one process per GPU).

The path shards by point: pools and phase A are independent per row, so each
rank owns a contiguous row range [lo, hi) and needs no collective for them.
Phase B has exactly one exchange: the reverse edge (v <- u, dist) of every
phase-A edge u -> v must reach the rank that owns v.  ``exchange_reverse``
does that with a single ``all_to_all_single`` of packed (int32 dst, int32
src, fp32 dist) triples, 12 bytes per edge (NCCL over NVLink for CUDA tensors, gloo for CPU tensors), after
which every rank holds, for each of its own rows, the same reverse list the
single-process scatter (prune.add_reverse_and_prune, prune.py:134-141)
would have built -- up to order, which the phase-B (dist, id) sort removes.

This module is host-side plumbing; the kernels are unchanged.  ``bench.py``
runs independent replicas (DESIGN.md section e); the sharded exchange is
exercised by tests/test_shard_gloo.py with world_size 2 on CPU.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def row_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row range of ``rank``."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def owner_of(ids: torch.Tensor, n: int, world: int) -> torch.Tensor:
    """Rank owning each row id under ``row_range``."""
    base, extra = divmod(n, world)
    big = extra * (base + 1)
    ids = ids.to(torch.int64)
    if base == 0:
        return ids.clone()
    return torch.where(ids < big, ids // (base + 1), extra + (ids - big) // base)


def exchange_reverse(a_ids: torch.Tensor, a_dists: torch.Tensor, a_counts: torch.Tensor,
                     lo: int, n: int, group=None):
    """Send every local phase-A edge u -> v (u in [lo, lo+rows)) as the
    reverse edge (dst=v, src=u, dist) to v's owner.

    Returns (dst, src, dist) tensors of the reverse edges this rank owns
    (dst in its row range), in arbitrary order."""
    world = dist.get_world_size(group)
    rows, width = a_ids.shape
    live = torch.arange(width, device=a_ids.device)[None, :] < a_counts[:, None].to(torch.int64)
    src = (torch.arange(rows, device=a_ids.device, dtype=torch.int64)[:, None] + lo) \
        .expand(rows, width)[live]
    dst = a_ids[live].to(torch.int32)
    dd = a_dists[live].contiguous().view(torch.int32)  # fp32 bits
    own = owner_of(dst, n, world)
    order = torch.argsort(own, stable=True)
    # 12 bytes per edge: (int32 dst, int32 src, fp32 dist bits) rows
    packed = torch.stack([dst[order], src[order].to(torch.int32), dd[order]], dim=1).contiguous()
    send_counts = torch.bincount(own, minlength=world)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    out = torch.empty((int(recv_counts.sum()), 3), dtype=torch.int32, device=a_ids.device)
    dist.all_to_all_single(out, packed, [int(x) for x in recv_counts.tolist()],
                           [int(x) for x in send_counts.tolist()], group=group)
    return out[:, 0].to(torch.int64), out[:, 1].to(torch.int64), out[:, 2].view(torch.float32)


def reverse_lists_reference(a_ids, a_counts, n: int):
    """Single-process reverse lists (prune.py:134-141 semantics) as
    {v: sorted list of owners u}, for checking."""
    rev = {v: [] for v in range(n)}
    for u in range(a_ids.shape[0]):
        for j in range(int(a_counts[u])):
            rev[int(a_ids[u, j])].append(u)
    return {v: sorted(us) for v, us in rev.items()}
