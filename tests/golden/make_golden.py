"""Generates tests/golden/*.npz from the UNMODIFIED reference library.

Run here (where /root/reference exists and oracle/_ref/libcvq_ref.so is
built): `python tests/golden/make_golden.py`.  The fixtures are small and
committed; they travel to the GPU box, where the reference tree does not
exist, and pin both the C restatement and the CUDA path to the reference's
own outputs.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import KQ, Oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def attention_cases(R):
    """fused_attention / naive outputs on seeded instances (test_attn.cpp
    fixture generators), including the 1-bit and 2-bit head presets."""
    shapes = [  # d, g, L, R, n, n_codes, t_extra, atom_scale
        (2, 1, 2, 1, 2, 2, 0, 1.0),
        (8, 2, 4, 1, 1, 8, 0, 1.0), (8, 2, 4, 3, 64, 8, 0, 1.0), (8, 4, 2, 2, 64, 16, 5, 1.0),
        (16, 4, 8, 2, 256, 8, 0, 1.0), (16, 8, 4, 1, 256, 16, 0, 1.0), (8, 2, 4, 2, 1024, 8, 0, 1.0),
        (64, 16, 64, 3, 300, 32, 0, 1.0), (128, 64, 64, 11, 700, 128, 0, 0.3),
        (128, 64, 64, 21, 333, 256, 0, 0.3), (128, 64, 64, 11, 129, 128, 1_000_000, 0.3),
        (16, 8, 2048, 2, 65, 32, 0, 1.0),
    ]
    cases = {}
    for ci, (d, g, L, Rr, n, nc, te, sc) in enumerate(shapes):
        kq = KQ(d, g, L, Rr)
        rng = R.rng(5000 + ci)
        atoms = rng.normal(2 * kq.n_atoms, sc)
        m = n * kq.rounds * kq.groups
        a = rng.index(m, L)
        b = rng.index(m, L)
        bits = rng.bits(n * nc).reshape(n, nc)
        vrows = rng.normal(nc * d, 1.0 / 16 if sc < 1 else 1.0).reshape(nc, d)
        q = rng.normal(d)
        t = n - 1 + te
        out, pred, meas = R.fused_attention(kq, atoms, a, b, bits, vrows, q, t)
        nout, npred, nmeas = R.naive_attention(kq, atoms, a, b, bits, vrows, q, t)
        cases[f"attn{ci}"] = dict(
            kq=np.array([d, g, L, Rr]), atoms=atoms, a=a, b=b, bits=bits, vrows=vrows, q=q,
            t=np.array(t), out=out, flops=np.array([pred, meas]), naive_out=nout,
            naive_flops=np.array([npred, nmeas]),
            key_words=R.pack_key_codes(kq, a, b), value_words=R.pack_value_codes(bits))
    return cases


def encode_cases(R):
    shapes = [  # d, g, L, R, n, rank
        (8, 2, 4, 2, 40, 8), (12, 3, 4, 2, 64, 12), (16, 4, 16, 3, 48, 16),
        (128, 64, 64, 11, 48, 32), (128, 64, 64, 21, 24, 32), (128, 16, 16, 4, 32, 32),
    ]
    cases = {}
    for ci, (d, g, L, Rr, n, rank) in enumerate(shapes):
        kq = KQ(d, g, L, Rr)
        rng = R.rng(7000 + ci)
        atoms = rng.normal(2 * kq.n_atoms, 0.3 if d == 128 else 1.0)
        keys = R.gen_synth(n, d, rank, 7100 + ci)
        if ci == 1:  # near-ties: midpoints between two centers of round 0
            xy = atoms.reshape(Rr, d // 2, L, 2)
            for i in range(n):
                a1, b1, a2, b2 = (rng.index(4, L)).tolist()
                for grp in range(kq.groups):
                    for s in range(g):
                        j = grp * g + s
                        c1 = (xy[0, j, a1, 0] - xy[0, j, b1, 1], xy[0, j, a1, 1] + xy[0, j, b1, 0])
                        c2 = (xy[0, j, a2, 0] - xy[0, j, b2, 1], xy[0, j, a2, 1] + xy[0, j, b2, 0])
                        keys[i, 2 * j] = 0.5 * (c1[0] + c2[0])
                        keys[i, 2 * j + 1] = 0.5 * (c1[1] + c2[1])
        a, b = R.encode_keys(kq, atoms, keys)
        hidden, nc = 2 * d, d
        w1 = rng.normal(d * hidden, 0.1).reshape(d, hidden)
        b1 = rng.normal(hidden, 0.05)
        w2 = rng.normal(hidden * nc, 0.1).reshape(hidden, nc)
        b2 = rng.normal(nc, 0.05)
        vals = R.gen_synth(n, d, rank, 7200 + ci)
        bits, logits = R.encoder_forward_infer(w1, b1, w2, b2, vals)
        cases[f"enc{ci}"] = dict(
            kq=np.array([d, g, L, Rr]), atoms=atoms, keys=keys, a=a, b=b,
            key_words=R.pack_key_codes(kq, a, b), w1=w1, b1=b1, w2=w2, b2=b2, vals=vals,
            bits=bits, logits=logits, value_words=R.pack_value_codes(bits))
    return cases


def main():
    R = Oracle("ref")
    for name, cases in (("attention", attention_cases(R)), ("encode", encode_cases(R))):
        flat = {}
        for cname, arrs in cases.items():
            for k, v in arrs.items():
                flat[f"{cname}/{k}"] = v
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **flat)
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
