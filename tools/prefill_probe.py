"""Prefill (C4-shaped) probe: one prefill of n tokens x 256 streams."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_18879_b200 import commvq as G  # noqa: E402

n, L_, H = 1024, 32, 8
kq = G.KeyQuantConfig(128, 64, 64, 11)
pc = G.QuantizedKVCache(kq, 128, n_seqs=1, n_layers=L_, n_kv_heads=H, q_per_kv=4, capacity=n,
                        hidden=256)
rs = np.random.default_rng(77)
for layer in range(L_):
    for h in range(H):
        pc.set_key_codebook(layer, h, 0.3 * rs.standard_normal(2 * kq.n_atoms))
        pc.set_value_quantizer(layer, h, rs.standard_normal((128, 128)) / 16,
                               0.1 * rs.standard_normal((128, 256)), np.zeros(256),
                               0.1 * rs.standard_normal((256, 128)), np.zeros(128))
gen = torch.Generator(device="cuda").manual_seed(5)
K = 0.5 * torch.randn(1, L_, H, n, 128, device="cuda", generator=gen)
V = torch.randn(1, L_, H, n, 128, device="cuda", generator=gen)
torch.cuda.synchronize()
t = time.perf_counter()
pc.prefill(K, V)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print("prefill", n, "tokens x", L_ * H, "streams:", dt, "s ->", n * L_ * H / dt, "token-heads/s")
