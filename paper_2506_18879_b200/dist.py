"""Context sharding across GPUs: host-side plan and exchange.

Each rank holds a contiguous range of every stream's tokens (boundaries on
128-token tiles so packed records stay 32-B aligned), attends with
cvq_cache_attention_partial -> (m, l, o) per row, and the partials of all
ranks are all-gathered (NCCL over NVLink on GPUs; any torch.distributed
backend works) and merged with the LSE combine kernel (cvq_lse_combine).
"""
from __future__ import annotations

TILE = 128


def shard_plan(n_tokens: int, world: int, align: int = TILE):
    """[(lo, hi)] per rank: contiguous, aligned, covering [0, n_tokens)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    per = -(-n_tokens // world)
    per = -(-per // align) * align
    out = []
    for r in range(world):
        lo = min(n_tokens, r * per)
        hi = min(n_tokens, (r + 1) * per)
        out.append((lo, hi))
    return out


def gather_partials(m, l, o, group=None):
    """All-gather this rank's (m [rows], l [rows], o [rows, d]) partials.

    Returns (M [world, rows], Lh [world, rows], O [world, rows, d]) in rank
    order -- the part-major layout cvq_lse_combine consumes.  An empty shard
    contributes l = 0, which the combine skips.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rows, d = o.shape
    M = torch.empty((world, rows), dtype=m.dtype, device=m.device)
    Lh = torch.empty((world, rows), dtype=l.dtype, device=l.device)
    O = torch.empty((world, rows, d), dtype=o.dtype, device=o.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(M, m.contiguous(), group=group)
        dist.all_gather_into_tensor(Lh, l.contiguous(), group=group)
        dist.all_gather_into_tensor(O.view(world, rows * d), o.contiguous().view(-1), group=group)
    else:  # gloo has no all_gather_into_tensor: list form into views of the same buffers
        dist.all_gather(list(M.unbind(0)), m.contiguous(), group=group)
        dist.all_gather(list(Lh.unbind(0)), l.contiguous(), group=group)
        dist.all_gather(list(O.unbind(0)), o.contiguous(), group=group)
    return M, Lh, O
