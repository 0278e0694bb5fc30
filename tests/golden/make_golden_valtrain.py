"""Generates tests/golden/valtrain.npz: train_value_quantizer results of the
UNMODIFIED reference library (oracle/_ref) on small seeded calibration sets.
Run here: `python tests/golden/make_golden_valtrain.py`."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# name: (n, d, n_codes, steps, batch, step_size, hidden, seed, ckpt_every, freeze, init_cb, rank)
CASES = {
    "small": (96, 8, 8, 300, 16, 1e-2, 0, 5, 50, False, False, 3),
    "freeze_init": (64, 8, 16, 200, 8, 5e-3, 24, 6, 40, True, True, 4),
    "diverge": (64, 8, 8, 400, 16, 5.0, 0, 7, 25, False, False, 3),
    "head": (512, 128, 128, 60, 64, 1e-3, 0, 8, 20, False, False, 32),
}


def main():
    R = Oracle("reference")
    arrays = {}
    for name, (n, d, nc, steps, batch, lr, hidden, seed, ck, fr, init, rank) in CASES.items():
        calib = R.gen_synth(n, d, rank, seed)
        icb = None
        if init:
            icb = np.random.default_rng(seed).standard_normal((nc, d)) * 0.1
            arrays[f"{name}/init_cb"] = icb
        r = R.train_value_quantizer(calib, nc, steps=steps, batch=batch, step_size=lr,
                                    hidden=hidden, seed=seed, checkpoint_every=ck, freeze=fr,
                                    init_codebook=icb)
        arrays[f"{name}/cfg"] = np.array([n, d, nc, steps, batch, hidden, seed, ck, int(fr),
                                          int(init), rank], np.int64)
        arrays[f"{name}/lr"] = np.array([lr])
        arrays[f"{name}/calib"] = calib
        for k in ("w1", "b1", "w2", "b2", "codebook", "loss_curve"):
            arrays[f"{name}/{k}"] = r[k]
        arrays[f"{name}/status"] = np.array([int(r["diverged"]), r["steps_run"]], np.int64)
        print(name, "diverged", r["diverged"], "steps_run", r["steps_run"], "curve",
              len(r["loss_curve"]), "last loss", r["loss_curve"][-1])
    np.savez_compressed(os.path.join(OUT, "valtrain.npz"), **arrays)


if __name__ == "__main__":
    main()
