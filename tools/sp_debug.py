"""Debug: per-token softmax weights of the sparse vs dense tcgen05 score
kernels (value rows = identity, token p's value code = bit p, so the
attention output IS the softmax over the 128 tokens)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import KQ, Oracle  # noqa: E402
from paper_2506_18879_b200 import commvq as G  # noqa: E402
from tests import fixtures as fx  # noqa: E402

P = Oracle()
kq = KQ(128, 64, 64, 11)
n, nc = 128, 128
Gq = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rng = P.rng(5)
c = G.QuantizedKVCache(kq, nc, n_kv_heads=1, q_per_kv=Gq, capacity=n, keys="tc")
atoms = rng.normal(2 * kq.n_atoms, 0.3)
c.set_key_codebook(0, 0, atoms)
c.set_value_quantizer(0, 0, np.eye(nc, 128))
a, b = fx.random_key_codes(kq, n, rng=rng)
mode = sys.argv[2] if len(sys.argv) > 2 else ""
if mode == "same":  # every token the same codes
    a = np.tile(a[:11], n)
    b = np.tile(b[:11], n)
elif mode == "sweep":  # token p: every code (a and b, all rounds) = p % 64
    a = np.repeat(np.arange(n) % 64, 11).astype(a.dtype)
    b = a.copy()
elif mode == "half":  # token p: every code = p // 2
    a = np.repeat(np.arange(n) // 2, 11).astype(a.dtype)
    b = a.copy()
elif mode == "rot":  # field (r, side) of token p = (p + 7 r + 3 side) % 64
    r = np.tile(np.arange(11), n)
    pp = np.repeat(np.arange(n), 11)
    a = ((pp + 7 * r) % 64).astype(a.dtype)
    b = ((pp + 7 * r + 3) % 64).astype(a.dtype)
elif mode == "ra":  # random a, b = 0
    b = np.zeros_like(a)
elif mode == "rb":
    a = np.zeros_like(b)
elif mode == "rtok":  # random code per token, same for all fields
    x = np.random.default_rng(1).integers(0, 64, n)
    a = np.repeat(x, 11).astype(a.dtype)
    b = a.copy()
elif mode == "rtok2":  # random per token, a and b differ
    x = np.random.default_rng(1).integers(0, 64, n)
    y = np.random.default_rng(2).integers(0, 64, n)
    a = np.repeat(x, 11).astype(a.dtype)
    b = np.repeat(y, 11).astype(a.dtype)
elif mode == "sweepa":  # only side a varies
    a = np.repeat(np.arange(n) % 64, 11).astype(a.dtype)
    b = np.zeros_like(a)
elif mode == "sweepb":
    b = np.repeat(np.arange(n) % 64, 11).astype(a.dtype)
    a = np.zeros_like(b)
bits = np.eye(n, nc, dtype=np.uint8)
c.import_stream(0, 0, 0, P.pack_key_codes(kq, a, b), P.pack_value_codes(bits), n)
q = rng.normal(Gq * 128).reshape(1, 1, Gq, 128).astype(np.float32)
t = n - 1
out_sp = c.attention(q, t)[0, 0]
c.set_variant("tc_dense")
out_d = c.attention(q, t)[0, 0]
np.set_printoptions(precision=3, suppress=True, linewidth=200)
for h in range(Gq):
    ls, ld = np.log(np.maximum(out_sp[h], 1e-30)), np.log(np.maximum(out_d[h], 1e-30))
    d = ls - ld
    print("head", h, "max |dlog| =", np.abs(d - d.mean()).max())
    print((d - d.mean()).reshape(4, 32))
    want, _, _ = P.fused_attention(kq, atoms, a, b, bits, np.eye(nc, 128),
                                   q[0, 0, h].astype(np.float64), t)
    lw = np.log(np.maximum(want[:n], 1e-300))
    es, ed = ls - lw, ld - lw
    print("vs oracle: sparse max", np.abs(es - es.mean()).max(), "dense max", np.abs(ed - ed.mean()).max())
    print("sparse err by token:")
    print((es - es.mean()).reshape(4, 32))
