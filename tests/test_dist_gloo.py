"""World-size-2 gloo test of the context-sharded decode on CPU.

Each rank takes its shard of every stream (paper_2506_18879_b200.dist
.shard_plan), forms split-K partials (m, l, o) from the oracle's scores of
its tokens into one packed block [m | l | o], exchanges the blocks with
dist.gather_packed (the single collective bench.py makes over NCCL; the
three-tensor gather_partials must agree), and the LSE merge of the gathered
partials must equal the
oracle's unsharded fused_attention.  The merge restated here in numpy is the
algebra of k_combine (attn.cu); the kernel itself is covered on the GPU.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_18879_b200.dist import TILE, shard_plan


def test_shard_plan_covers_and_aligns():
    for n in (1, 127, 128, 1000, 131072, 1048576):
        for w in (1, 2, 4, 8):
            plan = shard_plan(n, w)
            assert plan[0][0] == 0 and plan[-1][1] == n
            for (lo, hi), (lo2, _) in zip(plan, plan[1:]):
                assert hi == lo2 and (lo % TILE == 0 or lo == n)
            assert all(hi >= lo for lo, hi in plan)


def lse_merge(M, Lh, O):
    """k_combine (attn.cu): sum_p o_p l_p e^{m_p - M} / sum_p l_p e^{m_p - M}."""
    live = Lh > 0
    Mx = np.where(live, M, -np.inf).max(0)
    wts = np.where(live, Lh * np.exp(M - Mx), 0.0)
    return (wts[..., None] * O).sum(0) / wts.sum(0)[..., None]


def _worker(rank, world, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import KQ, Oracle
        from paper_2506_18879_b200.dist import gather_packed, gather_partials, packed_views
        from tests import fixtures as fx

        P = Oracle("port")
        kq = KQ(16, 8, 16, 3)
        nc, n, streams, gq = 16, 1000, 3, 2
        rows = []
        for s in range(streams):
            rng = P.rng(100 + s)
            atoms = rng.normal(2 * kq.n_atoms, 0.5)
            a, b = fx.random_key_codes(kq, n, rng=rng)
            bits = fx.random_value_codes(nc, n, rng=rng)
            vrows = rng.normal(nc * 16).reshape(nc, 16)
            for h in range(gq):
                q = rng.normal(16)
                rows.append((atoms, a, b, bits, vrows, q))
        lo, hi = shard_plan(n, world)[rank]
        t = n - 1
        pk = torch.zeros(len(rows) * (16 + 2))
        mt, lt, ot = packed_views(pk, len(rows), 16)
        m, l, o = mt.numpy(), lt.numpy(), ot.numpy()  # views: writes land in pk
        for i, (atoms, a, b, bits, vrows, q) in enumerate(rows):
            sc = P.fused_scores(kq, atoms, a, b, bits, vrows, q, t)[lo:hi]
            if hi > lo:
                m[i] = sc.max()
                p = np.exp(sc - m[i])
                l[i] = p.sum()
                o[i] = ((p @ bits[lo:hi]) @ vrows) / l[i]
        parts = gather_packed(pk).numpy().astype(np.float64)  # [world][rows*(d+2)]
        R = len(rows)
        M, Lh, O = parts[:, :R], parts[:, R:2 * R], parts[:, 2 * R:].reshape(world, R, 16)
        M3, L3, O3 = gather_partials(mt, lt, ot)
        assert np.array_equal(M3.numpy(), M.astype(np.float32))
        assert np.array_equal(O3.numpy(), O.astype(np.float32))
        out = lse_merge(M, Lh, O)
        if rank == 0:
            worst = 0.0
            for i, (atoms, a, b, bits, vrows, q) in enumerate(rows):
                want, _, _ = P.fused_attention(kq, atoms, a, b, bits, vrows, q, t)
                worst = max(worst, fx.rel_err(out[i], want))
            np.save(os.path.join(result_dir, "worst.npy"), np.array([worst]))
        # decode steps (cvq_mgpu_decode_step): the new tokens go to the LAST
        # shard only and every rank attends at the new global end; after k
        # steps the merge equals the unsharded attention over n + k tokens
        k_new = 3
        n2 = n + k_new
        lo2, hi2 = (lo, hi + k_new) if rank == world - 1 else (lo, hi)
        pk2 = torch.zeros(len(rows) * (16 + 2))
        mt2, lt2, ot2 = packed_views(pk2, len(rows), 16)
        m2, l2, o2 = mt2.numpy(), lt2.numpy(), ot2.numpy()
        ext = []
        for s in range(streams):  # the first n tokens are the same draws
            rng = P.rng(100 + s)
            atoms = rng.normal(2 * kq.n_atoms, 0.5)
            a, b = fx.random_key_codes(kq, n2, rng=P.rng(900 + s))
            bits = fx.random_value_codes(nc, n2, rng=P.rng(950 + s))
            vrows = P.rng(990 + s).normal(nc * 16).reshape(nc, 16)
            for h in range(gq):
                ext.append((atoms, a, b, bits, vrows, P.rng(10 * s + h).normal(16)))
        for i, (atoms, a, b, bits, vrows, q) in enumerate(ext):
            sc = P.fused_scores(kq, atoms, a, b, bits, vrows, q, n2 - 1)[lo2:hi2]
            if hi2 > lo2:
                m2[i] = sc.max()
                p = np.exp(sc - m2[i])
                l2[i] = p.sum()
                o2[i] = ((p @ bits[lo2:hi2]) @ vrows) / l2[i]
        parts2 = gather_packed(pk2).numpy().astype(np.float64)
        R2 = len(ext)
        out2 = lse_merge(parts2[:, :R2], parts2[:, R2:2 * R2],
                         parts2[:, 2 * R2:].reshape(world, R2, 16))
        if rank == 0:
            worst2 = 0.0
            for i, (atoms, a, b, bits, vrows, q) in enumerate(ext):
                want, _, _ = P.fused_attention(kq, atoms, a, b, bits, vrows, q, n2 - 1)
                worst2 = max(worst2, fx.rel_err(out2[i], want))
            np.save(os.path.join(result_dir, "worst_decode.npy"), np.array([worst2]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_decode_merges_to_unsharded(tmp_path, world):
    port = 29500 + (os.getpid() % 1000)
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    worst = float(np.load(tmp_path / "worst.npy")[0])
    assert worst <= 1e-5, worst
    worst_decode = float(np.load(tmp_path / "worst_decode.npy")[0])
    assert worst_decode <= 1e-5, worst_decode
