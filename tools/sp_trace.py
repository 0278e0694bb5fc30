"""clock64 trace of the sparse score kernel (build with CVQ_NVCC_EXTRA=-DSP_TRACE).

Runs the C3 attention step a few times and prints, for CTA 0 over 4 tiles,
when the MMA warp waited for A stages / D buffers, when the producers waited
for and published stages, and when the epilogue warps waited for / released
D (attn_sp.cu, SP_TRACE layout).  python tools/sp_trace.py [c3|c5|c2]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2506_18879_b200 import commvq as G  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    layers, B, H, Gq, N, d, g, L, R, nc = bench.CONFIGS[name]
    kq = G.KeyQuantConfig(d, g, L, R)
    S = B * layers * H
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = G.Context(0, stream.cuda_stream)
    cache = G.QuantizedKVCache(kq, nc, n_seqs=B, n_layers=layers, n_kv_heads=H, q_per_kv=Gq,
                               capacity=N, hidden=0, ctx=ctx, keys="tc")
    rs = np.random.default_rng(1)
    for layer in range(layers):
        for h in range(H):
            cache.set_key_codebook(layer, h, 0.3 * rs.standard_normal(2 * kq.n_atoms))
            cache.set_value_quantizer(layer, h, rs.standard_normal((nc, d)) / 16)
    kp, ks, vp, vs = cache.pools()
    gen = torch.Generator(device="cuda").manual_seed(3)
    for ptr, stride in ((kp, ks), (vp, vs)):
        pool = bench._pool_tensor(ptr, S * stride).view(S, stride)
        pool.copy_(torch.randint(-2**62, 2**62, pool.shape, dtype=torch.int64, device="cuda",
                                 generator=gen))
    cache.set_length(N)
    q = torch.randn(B, layers, H * Gq, d, device="cuda", generator=gen)
    out = torch.empty_like(q)
    for _ in range(3):
        cache.attention(q, N - 1, out)
    torch.cuda.synchronize()
    buf = (C.c_longlong * 8192)()
    rc = G._lib.cvq_debug_sp_trace(buf, 8192)
    assert rc == 0, rc
    t = np.frombuffer(buf, dtype=np.int64).copy()
    z = t[144 + 0] - 4000  # a reference point before tile 0's end
    if len(sys.argv) > 2:  # absolute: relative to the kernel's first trace point
        z = min(v for v in t if v > 0)
    rel = lambda v: int(v - z) if v else -1  # noqa: E731
    for k in range(4):
        print(f"--- tile {k}: MMA dempty wait {rel(t[128 + k])} -> {rel(t[136 + k])}, dfull commit {rel(t[144 + k])}")
        for r in range(11):
            prod = []
            for qq in range(4):
                b = 256 + qq * 64 + k * 16 + r
                prod.append(f"{rel(t[b]):6d}>{rel(t[b + 256]):6d}>{rel(t[b + 512]):6d}")
            mw = f"{rel(t[k * 16 + r]):6d}>{rel(t[64 + k * 16 + r]):6d}>{rel(t[192 + k * 16 + r]):6d}"
            print(f"  r{r:2d} mma afull {mw} | prod q wait>got>arrive " + " ".join(prod))
        ep = []
        for w in range(16):
            b = 1024 + w * 16
            ep.append((rel(t[b + k]), rel(t[b + 4 + k]), rel(t[b + 8 + k]), rel(t[b + 12 + k])))
        ep = np.array(ep)
        print("  epilogue dfull wait begin min/max %d/%d, got min/max %d/%d, release max %d, end max %d"
              % (ep[:, 0].min(), ep[:, 0].max(), ep[:, 1].min(), ep[:, 1].max(), ep[:, 2].max(),
                 ep[:, 3].max()))
        for w in range(16):
            print("    epi w%2d: wait %6d got %6d rel %6d end %6d" % (w, *ep[w]))


if __name__ == "__main__":
    main()
