"""Context sharding across GPUs: host-side plan and exchange.

Each rank holds a contiguous range of every stream's tokens (boundaries on
128-token tiles so packed records stay 32-B aligned), attends with
ranks are all-gathered (NCCL over NVLink on GPUs; any torch.distributed
backend works) and merged with the LSE combine kernel (cvq_lse_combine).
"""
from __future__ import annotations

TILE = 128


def shard_plan(n_tokens: int, world: int, align: int = TILE):
    """[(lo, hi)] per rank: contiguous, aligned, covering [0, n_tokens) --
    the library's host-side plan (cvq_shard_plan, mgpu.cu), the same one the
    C-ABI shard group and bench.py use."""
    import ctypes as C

    from paper_2506_18879_b200 import commvq as G
    if world < 1:
        raise ValueError("world must be >= 1")
    b = (C.c_uint64 * (2 * world))()
    G._check(G._lib.cvq_shard_plan(C.c_uint64(n_tokens), C.c_uint32(world), C.c_uint32(align), b))
    return [(int(b[2 * r]), int(b[2 * r + 1])) for r in range(world)]


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
    else:  # gloo: host tensors, list form into views of the same buffers
        hm, hl, ho = (x.contiguous().cpu() for x in (m, l, o))
        HM, HL, HO = (torch.empty(t.shape, dtype=t.dtype) for t in (M, Lh, O))
        dist.all_gather(list(HM.unbind(0)), hm, group=group)
        dist.all_gather(list(HL.unbind(0)), hl, group=group)
        dist.all_gather(list(HO.unbind(0)), ho, group=group)
        M.copy_(HM)
        Lh.copy_(HL)
        O.copy_(HO)
    return M, Lh, O


def packed_views(buf, rows, d):
    """(m, l, o) views into one packed block buf [rows*(d+2)]."""
    return buf[:rows], buf[rows:2 * rows], buf[2 * rows:].view(rows, d)


def gather_packed(buf, group=None):
    """All-gather this rank's packed block [rows*(d+2)] -> [world][rows*(d+2)]
    in rank order (one collective), the input of cvq_lse_combine_packed."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world, buf.numel()), dtype=buf.dtype, device=buf.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, buf.contiguous(), group=group)
    else:  # gloo: host tensors
        hb = buf.contiguous().cpu()
        HO = torch.empty((world, hb.numel()), dtype=hb.dtype)
        dist.all_gather(list(HO.unbind(0)), hb, group=group)
        out.copy_(HO)
    return out


class PeerMerge:
    """Context-shard merge over NVLink peer memory: no collective on the data
    path.  Each rank's cvq_cache_attention_partial writes its packed
    [m | l | o] block into a symmetric-memory buffer (torch symmetric memory,
    mapped on every peer); a device-side barrier publishes the blocks; each
    rank's combine kernel then reads all peers' blocks itself
    (cvq_lse_combine_ptrs).  Double-buffered by step parity: a rank writes
    step k+2's block only after the barrier of step k+1, which every peer
    passes only after finishing its combine of step k (stream order)."""

    def __init__(self, rows, d, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        grp = group or dist.group.WORLD
        self.rows, self.d = rows, d
        self.block = rows * (d + 2)
        self.buf = symm.empty(2 * self.block, dtype=torch.float32, device="cuda")
        self.buf.zero_()
        self.hdl = symm.rendezvous(self.buf, grp.group_name)
        self.world = self.hdl.world_size
        self.ptrs = self.hdl.buffer_ptrs_dev  # device array of the peers' buffer addresses
        self.step = 0

    def views(self):
        """(m, l, o) of this step's local block."""
        slot = self.step & 1
        return packed_views(self.buf[slot * self.block:(slot + 1) * self.block], self.rows, self.d)

    def merge(self, out, G, ctx):
        """Publish this step's block and merge all ranks' blocks into out.

        The symmetric-memory barrier runs on torch's current stream; the
        combine must run after it and before the next step's writes, so ctx
        must be bound to that same stream: it is required and
        checked, not defaulted."""
        import torch
        if ctx is None or ctx.stream_ptr != torch.cuda.current_stream().cuda_stream:
            raise ValueError("PeerMerge.merge: ctx must wrap torch's current stream "
                             "(Context(device, torch.cuda.current_stream().cuda_stream))")
        slot = self.step & 1
        self.hdl.barrier(channel=0)
        G.lse_combine_ptrs(self.ptrs, slot * self.block, self.world, self.rows, self.d, out, ctx)
        self.step += 1
