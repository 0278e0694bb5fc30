"""Decode-then-attend vs the fused path on B200 (Table 4:
optimized 0.4 / 1.1 / 3.8 ms vs naive 2.4 / 9.2 / 36.6 ms per layer-token at
8K / 32K / 128K).  Shape: 1 layer, batch 1, 8 KV x 4 q heads, 1-bit, random
codes; both paths over the same cache, CUDA events, 10 timed steps.

python tools/naive_vs_fused.py > profiles/r02_naive_vs_fused.json
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2506_18879_b200 import commvq as G  # noqa: E402


def timed(fn, steps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    stream = torch.cuda.current_stream()
    ctx = G.Context(0, stream.cuda_stream)
    kq = G.KeyQuantConfig(128, 64, 64, 11)
    H, Gq, nc = 8, 4, 128
    rs = np.random.default_rng(1)
    for n in (8192, 32768, 131072):
        c = G.QuantizedKVCache(kq, nc, n_kv_heads=H, q_per_kv=Gq, capacity=n, ctx=ctx, keys="tc")
        for h in range(H):
            c.set_key_codebook(0, h, 0.3 * rs.standard_normal(2 * kq.n_atoms))
            c.set_value_quantizer(0, h, rs.standard_normal((nc, 128)) / 16)
        kp, ks, vp, vs = c.pools()
        for ptr, stride in ((kp, ks), (vp, vs)):
            pool = bench._pool_tensor(ptr, H * stride).view(H, stride)
            pool.copy_(torch.randint(-2**62, 2**62, pool.shape, dtype=torch.int64, device="cuda"))
        c.set_length(n)
        q = torch.randn(1, 1, H * Gq, 128, device="cuda")
        out_f, out_n = torch.empty_like(q), torch.empty_like(q)
        tf = timed(lambda: c.attention(q, n - 1, out_f))
        tn = timed(lambda: c.attention_naive(q, n - 1, out_n))
        torch.cuda.synchronize()
        rel = float(((out_f - out_n).norm() / out_f.norm()).item())
        print(json.dumps({"context": n, "layers": 1, "batch": 1, "kv_heads": H, "q_heads": H * Gq,
                          "bits": 1, "fused_ms": tf, "naive_ms": tn, "naive_over_fused": tn / tf,
                          "rel_diff": rel,
                          "paper_table4_ratio": {8192: 6.0, 32768: 8.4, 131072: 9.6}[n]}), flush=True)
        del c


if __name__ == "__main__":
    main()
