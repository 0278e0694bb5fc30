#!/usr/bin/env python
"""CommVQ decode-attention benchmark (BASELINE.json metric).

Workload (BASELINE.json configs[2], "C3"): full 32-layer LLaMA-3.1-8B KV
shape, batch 2, 128K context, 1-bit CommVQ (per KV head: d=128, g=64, L=64,
R=11, N_c=128), 8 KV heads x 4 GQA query heads.  One step = one decode step
of attention for every (seq, layer, q head) over the packed cache resident in
HBM.  metric = KV-tokens/s (one KV-token = one cached token of one
(seq, layer): all 8 KV heads, 32 q heads), whole job over all ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU (torchrun): the context is sharded contiguously across ranks
(cvq_shard_plan; position offsets kept global); each step runs the C-ABI
shard group (cvq_mgpu_attention: partial on the local shard, one NCCL
all-gather of the packed (m, l, o) blocks, LSE combine -- all inside
libcvq_b200) -- strong scaling of the fixed C3 job.  e2e at
N > 1 is cvq_mgpu_decode_step with host buffers (the last shard appends).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n_layers, n_seqs, n_kv, q_per_kv, N, d, g, L, R, n_codes)
    "c3": (32, 2, 8, 4, 131072, 128, 64, 64, 11, 128),
    "c1": (1, 1, 8, 4, 8192, 128, 64, 64, 11, 128),
    "c2": (1, 1, 8, 4, 32768, 128, 64, 64, 21, 256),
    "c5": (1, 1, 8, 4, 1048576, 128, 64, 64, 21, 256),
}
BYTES_PER_KVHT = {11: 32.5, 21: 63.5}
TENSOR_NOMINAL_TFLOPS = 2250.0  # B200 dense fp16/bf16, /opt/skills/guides/B200_PROFILING.md


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, dev):
        self.dev, self.samples, self.proc = dev, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_reference(cfg, n_calls, threads, seed=7):
    """Times the reference's fused_attention (oracle/_ref, compiled from the
    reference sources) on this host: n_calls independent q-head calls at the
    workload's context length over `threads` std::threads."""
    import ctypes as C

    from oracle.oracle import REF_SO, PORT_SO  # noqa: F401
    layers, B, H, Gq, N, d, g, L, R, nc = cfg
    if os.path.exists(REF_SO):
        lib, kind = C.CDLL(REF_SO), "reference"
    else:
        raise RuntimeError("oracle/_ref/libcvq_ref.so missing")
    f = lib.cvqr_bench_fused
    f.argtypes = [C.c_size_t] * 10 + [C.c_uint64, C.c_void_p, C.c_void_p]
    secs, cs = C.c_double(), C.c_double()
    n_streams = max(1, min(H, n_calls // Gq))
    rc = f(d, g, L, R, nc, N, n_streams, Gq, n_calls, threads, seed, C.byref(secs), C.byref(cs))
    if rc != 0:
        raise RuntimeError("reference bench failed")
    qhead_tokens = n_calls * N
    # one KV-token covers all q heads of one (seq, layer): 32 q-head calls
    kv_tokens_per_s = qhead_tokens / secs.value / (H * Gq)
    return kv_tokens_per_s, secs.value, kind


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    layers, B, H, Gq, N, d, g, L, R, nc = cfg
    threads = os.cpu_count() or 1
    vals = []
    for it in range(args.warmup + args.steps):
        v, secs, kind = cpu_reference(cfg, threads, threads, seed=11 + it)
        if it >= args.warmup:
            vals.append((v, secs))
    value = float(np.median([v for v, _ in vals]))
    ms = float(np.median([s for _, s in vals])) * 1e3
    line = {
        "metric": "CommVQ decode-attention KV-tokens/s @128K ctx", "value": value,
        "unit": "KV-tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (random codebooks/codes, commvq::Rng)",
        "impl": "reference",
        "config": {"workload": args.config, "n_layers": layers, "n_seqs": B, "n_kv_heads": H,
                   "q_per_kv": Gq, "context": N, "key": [d, g, L, R], "n_codes": nc,
                   "sample": f"{threads} q-head fused_attention calls per step at N={N}"},
        "cpu_baseline": {"value": value, "unit": "KV-tokens/s", "cores": threads, "kind": kind,
                         "sample": f"{threads} q-head fused_attention calls per step at N={N}"},
        "e2e": {"value": value, "unit": "KV-tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)  # ~0.75 s timed: several clock samples
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--mgpu-world1", action="store_true",
                    help="run the cvq_mgpu shard group (NCCL, world 1) as at N > 1 (test)")
    ap.add_argument("--no-naive", action="store_true",
                    help="skip timing the decode-then-attend baseline on the same cache")
    ap.add_argument("--merge", default="nccl", choices=["nccl", "peer"],
                    help="N>1 shard merge: the C-ABI shard group (one NCCL all-gather of packed "
                         "partials + combine inside libcvq_b200), or peer (experimental): "
                         "symmetric-memory blocks read by the combine kernel over NVLink")
    ap.add_argument("--keys", default="tc", choices=["fp32", "fp16", "tc"],
                    help="score kernel: tc = tcgen05 one-hot MMA (fp16 codebook), fp16 / fp32 = "
                         "CUDA-core gather with that codebook precision; fp32 accumulation always")
    ap.add_argument("--tc-variant", default="sparse", choices=["sparse", "dense", "pair"],
                    help="tcgen05 score kernel: 2:4-sparse (default), dense one-hot, or CTA-pair")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # --dist-backend gloo lets several ranks share one GPU (host-staged
    # exchange) to exercise the sharded path where only one GPU is available
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    from paper_2506_18879_b200 import commvq as G

    layers, B, H, Gq, N, d, g, L, R, nc = cfg
    kq = G.KeyQuantConfig(d, g, L, R)
    S, rows = B * layers * H, B * layers * H * Gq
    # contiguous context shards, boundaries at multiples of 128 tokens
    from paper_2506_18879_b200.dist import shard_plan
    lo, hi = shard_plan(N, world)[rank]
    n_local = hi - lo
    extra = 2 * (args.steps + args.warmup) + 16  # room for the e2e decode steps' appends
    # a real (non-default) stream shared by torch and libcvq, so the CUDA
    # events below see the library's kernels
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = G.Context(local, stream.cuda_stream)
    cache = G.QuantizedKVCache(kq, nc, n_seqs=B, n_layers=layers, n_kv_heads=H, q_per_kv=Gq,
                               capacity=n_local + extra, hidden=2 * nc, position_offset=lo, ctx=ctx,
                               keys=args.keys)
    if args.tc_variant != "sparse":
        cache.set_variant({"dense": "tc_dense", "pair": "tc_pair"}[args.tc_variant])
    rs = np.random.default_rng(1234)
    for layer in range(layers):
        for h in range(H):
            cache.set_key_codebook(layer, h, 0.3 * rs.standard_normal(2 * kq.n_atoms))
            cache.set_value_quantizer(
                layer, h, rs.standard_normal((nc, d)) / 16,
                0.1 * rs.standard_normal((d, 2 * nc)), np.zeros(2 * nc),
                0.1 * rs.standard_normal((2 * nc, nc)), np.zeros(nc))
    # synthetic packed codes straight into the HBM pools (any bit pattern is
    # a valid code stream: fields are log2(L) bits); tails stay zero.
    kp, ks, vp, vs = cache.pools()
    kwords = (n_local * kq.bits_per_token + 63) // 64
    vwords = (n_local * nc + 63) // 64
    gen = torch.Generator(device="cuda").manual_seed(99 + rank)
    for ptr, stride, nw, bits_total in ((kp, ks, kwords, n_local * kq.bits_per_token),
                                        (vp, vs, vwords, n_local * nc)):
        pool = _pool_tensor(ptr, S * stride).view(S, stride)
        for s in range(S):
            pool[s, :nw] = torch.randint(-2**63, 2**63 - 1, (nw,), dtype=torch.int64,
                                         device="cuda", generator=gen)
            tail = bits_total % 64
            if tail:
                pool[s, nw - 1] &= (1 << tail) - 1
    cache.set_length(n_local)
    torch.cuda.synchronize()
    # the query is the same on every rank (broadcast); only the context shards differ
    qgen = torch.Generator(device="cuda").manual_seed(7)
    q = torch.randn(B, layers, H * Gq, d, device="cuda", generator=qgen)
    out = torch.empty_like(q)
    t_q = N - 1  # global query position (last cached token)
    peer = group = None
    merge_note = None
    if world > 1 and args.merge == "peer":
        # experimental: symmetric-memory blocks read by the combine over NVLink
        from paper_2506_18879_b200.dist import PeerMerge
        peer = PeerMerge(rows, d)
    elif (world > 1 and args.dist_backend == "nccl") or args.mgpu_world1:
        # the C-ABI shard group (mgpu.cu): partial -> one ncclAllGather of the
        # packed [m | l | o] blocks -> LSE combine, inside libcvq_b200
        import torch.distributed as dist
        try:
            uid = [G.ShardGroup.unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(uid, src=0)
            group = G.ShardGroup(cache, rank, world, uid[0])
            merge_note = "cvq_mgpu (in-library ncclAllGather + LSE combine)"
        except Exception as ex:  # keep the run measurable: torch.distributed gather
            group = None
            merge_note = "torch.distributed all-gather (cvq_mgpu init failed: %s)" % str(ex)[:120]
    # gloo (several ranks sharing one GPU, host-staged exchange): the same
    # packed blocks gathered through torch.distributed
    from paper_2506_18879_b200.dist import gather_packed, packed_views
    pk = torch.empty(rows * (d + 2), device="cuda")
    m_p, l_p, o_p = packed_views(pk, rows, d)

    def step():
        if world == 1 and group is None:
            cache.attention(q, t_q, out)
        elif peer is not None:
            m_v, l_v, o_v = peer.views()
            cache.attention_partial(q, m_v, l_v, o_v, t_q)
            peer.merge(out, G, ctx)
        elif group is not None:
            group.attention(q, t_q, out)
        else:
            cache.attention_partial(q, m_p, l_p, o_p, t_q)
            G.lse_combine_packed(gather_packed(pk), rows, d, out, ctx)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    if group is not None:
        # the in-library exchange against the torch.distributed one on the
        # first step; on any disagreement all ranks fall back together
        import torch.distributed as dist
        group.attention(q, t_q, out)
        ref_out = torch.empty_like(out)
        cache.attention_partial(q, m_p, l_p, o_p, t_q)
        G.lse_combine_packed(gather_packed(pk) if world > 1 else pk.view(1, -1), rows, d, ref_out, ctx)
        torch.cuda.synchronize()
        bad = torch.tensor([0.0 if torch.isfinite(out).all() and
                            float((out - ref_out).abs().max()) <= 1e-4 * float(ref_out.abs().max())
                            else 1.0], device="cuda")
        if world > 1:
            dist.all_reduce(bad)
        if float(bad) > 0:
            group = None
            merge_note = "torch.distributed all-gather (cvq_mgpu result disagreed on step 0)"
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    launches0 = G.launch_count()
    _lib_profile(ctx, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms_total = e0.elapsed_time(e1)
    main_ms, main_n = _lib_profile_read(ctx)
    _lib_profile(ctx, False)
    launches = G.launch_count() - launches0
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms_total], device="cuda" if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms = ms_total / args.steps
    kv_tokens = B * layers * N
    value = kv_tokens / (ms / 1e3)

    # ---- roofline of the dominant kernel (live CUDA-event timing) ----
    # the north-star roofline is HBM on compressed-cache bytes
    # (32.5 B / 63.5 B per KV-head-token) against MEASURED_PEAKS; the binding
    # resource of this algorithm is the tensor pipe (one-hot MMA), reported
    # alongside against 2 x the measured bf16 burst (2:4 sparse doubles the
    # dense rate) at the clock the run saw.
    hbm, tflops, src = peaks()
    kvht_per_launch = S * n_local
    bytes_per_launch = kvht_per_launch * BYTES_PER_KVHT[R]
    avg_main_ms = main_ms / max(main_n, 1)
    achieved = bytes_per_launch / (avg_main_ms / 1e3) / 1e9
    traffic = traffic_step = traffic_src = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(f"{args.config}/{args.keys}" +
                                   ("" if args.tc_variant == "sparse" else "_" + args.tc_variant))
        if tr and world == 1:
            traffic = tr["dram_bytes_per_launch"]
            traffic_step = tr.get("dram_bytes_per_step")
            traffic_src = tr.get("source")
    except Exception:
        pass
    clk_sum = clk.summary()
    kname = {"tc": {"sparse": "k_sp_score (2:4-sparse one-hot tcgen05 MMA)",
                    "dense": "k_tc_score (dense one-hot tcgen05 MMA)",
                    "pair": "k_sp_score CTA-pair"}[args.tc_variant],
             "fp16": "k_fast_score_h (CUDA cores, fp16 codebook)",
             "fp32": "k_fast_score (CUDA cores, fp32 codebook)"}[args.keys]
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "traffic_step": traffic_step,
            "traffic_note": "dram__bytes_read+write per launch of the score kernel and per whole "
                            "step (all kernels) from one ncu capture (%s)" % traffic_src,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (%s)" % src, "kernel": kname,
            "kernel_ms": avg_main_ms, "kernel_share_of_step": avg_main_ms / ms,
            "algorithmic_bytes_per_launch": bytes_per_launch,
            "bytes_per_kv_head_token": BYTES_PER_KVHT[R],
            "kv_head_tokens_per_s_kernel": kvht_per_launch / (avg_main_ms / 1e3),
            "step_hbm_achieved_gbs": bytes_per_launch / (ms / 1e3) / 1e9,
            "step_frac": bytes_per_launch / (ms / 1e3) / 1e9 / hbm}
    if args.keys == "tc":
        # one-hot MMA: per KV-head-token 2 * 128 reals * (2 sides * 64 levels) * R
        # = 4*R*L*d logical flops, executed on the tensor pipe
        flops = kvht_per_launch * 4.0 * R * L * d
        ach_tf = flops / (avg_main_ms / 1e3) / 1e12
        sparse = R in (11, 21) and args.tc_variant != "dense"
        peak_tf = tflops * (2 if sparse else 1)
        roof["tensor"] = {
            "achieved": ach_tf, "peak": peak_tf, "unit": "TFLOP/s", "frac": ach_tf / peak_tf,
            "peak_source": "%s x MEASURED_PEAKS bf16_tflops burst (%.1f, cuBLAS dense)%s" % (
                "2" if sparse else "1", tflops,
                "; 2:4-sparse tcgen05 runs at twice the dense rate" if sparse else ""),
            "sm_mhz_median": clk_sum.get("sm_mhz"),
            "frac_vs_nominal": ach_tf / (TENSOR_NOMINAL_TFLOPS * (2 if sparse else 1)),
            "algorithmic_flops_per_launch": flops}

    # ---- the decode-then-attend baseline on the same cache (Table 4) ----
    naive = None
    if world == 1 and not args.no_naive:
        try:
            nout = torch.empty_like(q)
            cache.attention_naive(q, t_q, nout)  # warm (scratch)
            torch.cuda.synchronize()
            ne0, ne1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ne0.record(stream)
            for _ in range(3):
                cache.attention_naive(q, t_q, nout)
            ne1.record(stream)
            torch.cuda.synchronize()
            naive_ms = ne0.elapsed_time(ne1) / 3
            naive = {"ms_per_step": naive_ms, "value": kv_tokens / (naive_ms / 1e3),
                     "unit": "KV-tokens/s", "naive_over_fused": naive_ms / ms,
                     "rel_diff_vs_fused": float(((nout - out).norm() / out.norm()).item()),
                     "path": "cvq_cache_attention_naive: dense fp16 dequantisation of every key "
                             "(RoPE) and value (tensor-core bits x C_V) + flash-decoding",
                     "paper_table4": "naive/optimized 6.0x @8K, 8.4x @32K, 9.6x @128K "
                                     "(PAPER.md:464-466, other hardware)"}
        except Exception as ex:  # e.g. scratch too large for the device
            naive = {"unavailable": str(ex)[:200]}

    # ---- e2e through the C-ABI with host buffers (decode_step) ----
    e2e = None
    if not args.no_e2e and group is not None:
        # every rank passes its pinned host buffers; the last rank appends
        kh = torch.from_numpy(np.random.default_rng(5).standard_normal((B, layers, H, d))
                              .astype(np.float32)).pin_memory()
        vh = torch.from_numpy(np.random.default_rng(6).standard_normal((B, layers, H, d))
                              .astype(np.float32)).pin_memory()
        qh = torch.from_numpy(np.random.default_rng(7).standard_normal((B, layers, H * Gq, d))
                              .astype(np.float32)).pin_memory()
        oh = torch.empty_like(qh).pin_memory()
        n_e2e = min(args.steps, 8)
        group.decode_step(kh, vh, qh, oh)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            group.decode_step(kh, vh, qh, oh)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / n_e2e
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        n_now = group.size()
        e2e = {"value": B * layers * n_now / (e2e_ms / 1e3), "unit": "KV-tokens/s",
               "h2d_bytes_per_step": int(kh.numel() * 4 * 2 + qh.numel() * 4),
               "d2h_bytes_per_step": int(oh.numel() * 4), "ms_per_step": e2e_ms,
               "path": "cvq_mgpu_decode_step (last shard appends k,v; partial + NCCL all-gather "
                       "+ combine) with pinned host buffers on every rank, max over ranks"}
    if not args.no_e2e and world == 1 and group is None:
        kh = np.random.default_rng(5).standard_normal((B, layers, H, d)).astype(np.float32)
        vh = np.random.default_rng(6).standard_normal((B, layers, H, d)).astype(np.float32)
        qh = np.random.default_rng(7).standard_normal((B, layers, H * Gq, d)).astype(np.float32)
        oh = np.zeros_like(qh)
        k_pin = torch.from_numpy(kh).pin_memory()
        v_pin = torch.from_numpy(vh).pin_memory()
        q_pin = torch.from_numpy(qh).pin_memory()
        o_pin = torch.from_numpy(oh).pin_memory()
        n_e2e = min(args.steps, 8)
        cache.decode_step(k_pin, v_pin, q_pin, o_pin)  # warm (allocations)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            cache.decode_step(k_pin, v_pin, q_pin, o_pin)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / n_e2e
        # breakdown: the append alone (encode + pack of one token per stream)
        kd, vd = k_pin.cuda(), v_pin.cuda()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for _ in range(2):
            cache.append(kd, vd)
        torch.cuda.synchronize()
        append_ms = (time.perf_counter() - t1) * 1e3 / 2
        n_now = cache.size()
        e2e = {"value": B * layers * n_now / (e2e_ms / 1e3), "unit": "KV-tokens/s",
               "h2d_bytes_per_step": int(kh.nbytes + vh.nbytes + qh.nbytes),
               "d2h_bytes_per_step": int(oh.nbytes), "ms_per_step": e2e_ms,
               "append_ms": append_ms,
               "path": "cvq_cache_decode_step (append k,v + attention) with pinned host buffers"}

    # ---- prefill encode throughput (BASELINE configs[3], "C4"), sampled ----
    prefill = None
    if not args.no_prefill and world == 1:
        del cache
        torch.cuda.empty_cache()
        # one sequence, every (layer, kv head) stream; >= 16K tokens so the
        # projection to C4 (128K x 32 layers x 8 heads) rests on a real run
        n_pre, S_pre = 16384 + 128, layers * H
        pc = G.QuantizedKVCache(kq, nc, n_seqs=1, n_layers=layers, n_kv_heads=H, q_per_kv=Gq,
                                capacity=2 * n_pre, hidden=2 * nc, ctx=ctx, keys=args.keys)
        rs2 = np.random.default_rng(77)
        for layer in range(layers):
            for h in range(H):
                pc.set_key_codebook(layer, h, 0.3 * rs2.standard_normal(2 * kq.n_atoms))
                pc.set_value_quantizer(
                    layer, h, rs2.standard_normal((nc, d)) / 16,
                    0.1 * rs2.standard_normal((d, 2 * nc)), np.zeros(2 * nc),
                    0.1 * rs2.standard_normal((2 * nc, nc)), np.zeros(nc))
        Kp = 0.5 * torch.randn(1, layers, H, n_pre, d, device="cuda", generator=gen)
        Vp = torch.randn(1, layers, H, n_pre, d, device="cuda", generator=gen)
        pc.prefill(Kp[:, :, :, :128].contiguous(), Vp[:, :, :, :128].contiguous())  # warm
        Kt, Vt = Kp[:, :, :, 128:].contiguous(), Vp[:, :, :, 128:].contiguous()  # inputs, untimed
        torch.cuda.synchronize()
        pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pe0.record(stream)
        pc.prefill(Kt, Vt)
        pe1.record(stream)
        torch.cuda.synchronize()
        p_ms = pe0.elapsed_time(pe1)
        th = S_pre * (n_pre - 128) / (p_ms / 1e3)  # token-heads/s
        prefill = {"token_heads_per_s": th, "kv_tokens_per_s": th / H, "unit": "KV-tokens/s",
                   "sample": f"{n_pre - 128} tokens x {S_pre} streams, fp32 K/V on device "
                             "(one prefill call, 16 chunks back to back: sustained clocks)",
                   "c4_projected_s": 131072 * 32 * 8 / th,  # configs[3]: 128K x 32 layers x 8 heads
                   "encoders": "bit-exact fp64 key search + value MLP, device packing"}
        del pc, Kt, Vt

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            n_calls = 4 * threads  # ~0.5 s per call per core at 128K: ~2 s wall
            v, secs, kind = cpu_reference(cfg, n_calls, threads)
            cpu = {"value": v, "unit": "KV-tokens/s", "cores": threads, "kind": kind,
                   "sample": f"{n_calls} q-head fused_attention calls at N={N} "
                             f"({secs:.1f} s wall)"}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "KV-tokens/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {
            "metric": "CommVQ decode-attention KV-tokens/s @128K ctx", "value": value,
            "unit": "KV-tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": ("f16 one-hot x f16 codebook MMA, f32 accumulate (fp64-reduced phases; int codes)"
                      if args.keys == "tc" else
                      "f32 accumulate, %s key codebook (fp64-reduced phases; int codes)" % args.keys),
            "data": "synthetic (random codebooks, random packed codes, random q)",
            "config": {"workload": args.config, "n_layers": layers, "n_seqs": B,
                       "n_kv_heads": H, "q_per_kv": Gq, "context": N, "key": [d, g, L, R],
                       "n_codes": nc, "parallelism": f"context-shard x{world}",
                       "merge": args.merge if world > 1 else None,
                       "exchange": merge_note,
                       "l2": "inputs (packed cache) larger than L2"},
            "kv_head_tokens_per_s": value * H, "roofline": roof, "clocks": clk_sum,
            "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu, "prefill": prefill,
            "naive": naive,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


class _CudaArray:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False),
                                         "version": 3}


def _pool_tensor(ptr, n_words):
    """int64 view of a libcvq device pool (no copy)."""
    import torch
    return torch.as_tensor(_CudaArray(ptr, n_words), device="cuda")


def _lib_profile(ctx, on):
    from paper_2506_18879_b200 import commvq as G
    G._check(G._lib.cvq_context_profile(ctx.h, G._i(1 if on else 0)))


def _lib_profile_read(ctx):
    import ctypes as C

    from paper_2506_18879_b200 import commvq as G
    ms, n = C.c_double(), C.c_uint64()
    G._check(G._lib.cvq_context_profile_read(ctx.h, C.byref(ms), C.byref(n)))
    return ms.value, n.value


if __name__ == "__main__":
    main()
