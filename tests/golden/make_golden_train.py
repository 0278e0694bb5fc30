"""Generates tests/golden/train.npz: train_key_codebook results of the
UNMODIFIED reference library (oracle/_ref) on small seeded calibration sets
(gen_synth, ctf.cpp:97-144).  Run here: `python tests/golden/make_golden_train.py`.
The GPU trainer (train.cu) is pinned to these fixtures on the GPU box."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import KQ, Oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# name: (d, g, L, R, n, rank, seed, soft_iters, hard_iters_max, factorized)
CASES = {
    "g1_L8": (8, 4, 8, 2, 256, 4, 11, 6, 25, False),
    "g2_L4": (8, 2, 4, 2, 96, 3, 12, 5, 25, False),
    "fact_L16": (16, 8, 16, 1, 600, 6, 13, 4, 20, True),
    "head_L64": (128, 64, 64, 1, 4352, 32, 14, 2, 4, False),
}


def main():
    R = Oracle("reference")
    arrays = {}
    for name, (d, g, L, Rr, n, rank, seed, si, hi, fact) in CASES.items():
        kq = KQ(d, g, L, Rr)
        calib = R.gen_synth(n, d, rank, seed)
        atoms, traces, mse = R.train_key_codebook(kq, calib, soft_iters=si, hard_iters_max=hi,
                                                  seed=seed, factorized=fact)
        arrays[f"{name}/cfg"] = np.array([d, g, L, Rr, n, rank, seed, si, hi, int(fact)], np.int64)
        arrays[f"{name}/calib"] = calib
        arrays[f"{name}/atoms"] = atoms
        arrays[f"{name}/mse"] = mse
        flat = [np.asarray(t) for row in traces for t in row]
        arrays[f"{name}/trace_len"] = np.array([len(t) for t in flat], np.int64)
        arrays[f"{name}/trace"] = np.concatenate(flat) if flat else np.zeros(0)
        print(name, "mse", mse, "trace lens", [len(t) for t in flat])
    np.savez_compressed(os.path.join(OUT, "train.npz"), **arrays)


if __name__ == "__main__":
    main()
