"""Small parity-config run of the attention kernels for compute-sanitizer
(memcheck / racecheck / synccheck): the 2:4-sparse tcgen05 score kernel
(1-bit and 2-bit presets), the dense tcgen05 kernel, the fp16 CUDA-core
kernel, k_fast_value / k_combine_project, plus an append (encoders, pack).
Each output is checked against the oracle (1e-3), so a sanitizer run also
proves the instrumented kernels computed the right thing.

compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import KQ, Oracle  # noqa: E402
from paper_2506_18879_b200 import commvq as G  # noqa: E402
from tests import fixtures as fx  # noqa: E402

P = Oracle("port")


def run(R, keys, variant, n=700, H=2, Gq=4):
    kq = KQ(128, 64, 64, R)
    nc = 128 if R == 11 else 256
    rng = P.rng(R * 7 + n)
    c = G.QuantizedKVCache(kq, nc, n_kv_heads=H, q_per_kv=Gq, capacity=n, keys=keys)
    if variant:
        c.set_variant(variant)
    streams = []
    for h in range(H):
        atoms = rng.normal(2 * kq.n_atoms, 0.3)
        vrows = rng.normal(nc * 128, 1 / 16).reshape(nc, 128)
        a, b = fx.random_key_codes(kq, n, rng=rng)
        bits = fx.random_value_codes(nc, n, rng=rng)
        c.set_key_codebook(0, h, atoms)
        c.set_value_quantizer(0, h, vrows)
        c.import_stream(0, 0, h, P.pack_key_codes(kq, a, b), P.pack_value_codes(bits), n)
        streams.append((atoms, vrows, a, b, bits))
    q = rng.normal(H * Gq * 128).reshape(1, 1, H * Gq, 128).astype(np.float32)
    out = c.attention(q, n - 1)
    worst = 0.0
    for h in range(H):
        atoms, vrows, a, b, bits = streams[h]
        want, _, _ = P.fused_attention(kq, atoms, a, b, bits, vrows,
                                       q[0, 0, h * Gq].astype(np.float64), n - 1)
        worst = max(worst, fx.rel_err(out[0, 0, h * Gq], want))
    print(f"R={R} keys={keys} variant={variant or 'default'}: worst rel err {worst:.2e}", flush=True)
    assert worst <= 1e-3


def append_roundtrip():
    f = fx.CacheFixture()
    c = G.QuantizedKVCache(f.kq, 8, capacity=4, hidden=16)
    c.set_key_codebook(0, 0, f.atoms)
    c.set_value_quantizer(0, 0, f.vrows, f.w1, f.b1, f.w2, f.b2)
    K, V = P.gen_synth(20, 8, 8, 1), P.gen_synth(20, 8, 8, 2)
    c.prefill(K[None, None, None, :12], V[None, None, None, :12])
    for i in range(12, 20):
        c.append(K[None, None, None, i], V[None, None, None, i])
    kw, vw = c.export_stream(0, 0, 0)
    a, b = P.encode_keys(f.kq, f.atoms, K)
    assert (kw == P.pack_key_codes(f.kq, a, b)).all()
    print("append/prefill + growth: words exact", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "sp"):
        run(11, "tc", None)
        run(21, "tc", None, n=300)
    if which in ("all", "dense"):
        run(11, "tc", "tc_dense")
    if which in ("all", "fast"):
        run(11, "fp16", None)
    if which in ("all", "append"):
        append_roundtrip()
    print("sanitize probe ok")
