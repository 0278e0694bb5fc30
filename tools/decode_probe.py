"""Where the time of one decode step goes at a small config (C1 / C2):
append (encode + pack), attention, and the full host-buffer decode_step,
each timed with CUDA events over 50 repetitions.  Run under ncu with
--metrics gpu__time_duration.sum for the per-kernel split.

python tools/decode_probe.py [c1|c2|c3]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2506_18879_b200 import commvq as G  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    layers, B, H, Gq, N, d, g, L, R, nc = bench.CONFIGS[name]
    kq = G.KeyQuantConfig(d, g, L, R)
    S = B * layers * H
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = G.Context(0, stream.cuda_stream)
    cache = G.QuantizedKVCache(kq, nc, n_seqs=B, n_layers=layers, n_kv_heads=H, q_per_kv=Gq,
                               capacity=N + 4 * reps + 64, hidden=2 * nc, ctx=ctx, keys="tc")
    rs = np.random.default_rng(1)
    for layer in range(layers):
        for h in range(H):
            cache.set_key_codebook(layer, h, 0.3 * rs.standard_normal(2 * kq.n_atoms))
            cache.set_value_quantizer(layer, h, rs.standard_normal((nc, d)) / 16,
                                      0.1 * rs.standard_normal((d, 2 * nc)), np.zeros(2 * nc),
                                      0.1 * rs.standard_normal((2 * nc, nc)), np.zeros(nc))
    kp, ks, vp, vs = cache.pools()
    gen = torch.Generator(device="cuda").manual_seed(3)
    for ptr, stride in ((kp, ks), (vp, vs)):
        pool = bench._pool_tensor(ptr, S * stride).view(S, stride)
        pool.copy_(torch.randint(-2**62, 2**62, pool.shape, dtype=torch.int64, device="cuda",
                                 generator=gen))
    cache.set_length(N)
    k = torch.randn(B, layers, H, d, device="cuda", generator=gen)
    v = torch.randn(B, layers, H, d, device="cuda", generator=gen)
    q = torch.randn(B, layers, H * Gq, d, device="cuda", generator=gen)
    out = torch.empty_like(q)
    kh, vh, qh = (x.cpu().pin_memory() for x in (k, v, q))
    oh = torch.empty_like(qh).pin_memory()

    def timed(fn, n):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(n):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3, (time.perf_counter() - t0) / n * 1e6

    res = {}
    res["append (device k,v)"] = timed(lambda: cache.append(k, v), reps)
    res["attention (device q)"] = timed(lambda: cache.attention(q, None, out), reps)
    res["decode_step (device)"] = timed(lambda: cache.decode_step(k, v, q, out), reps)
    res["decode_step (pinned host)"] = timed(lambda: cache.decode_step(kh, vh, qh, oh), reps)
    cache.synchronize()
    for k_, (dev_us, wall_us) in res.items():
        print(f"{name} {k_:28s} device {dev_us:8.1f} us/step   wall {wall_us:8.1f} us/step")


if __name__ == "__main__":
    main()
