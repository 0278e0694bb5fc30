"""Key-codebook training throughput (train.cu) vs the reference on the host.

GPU: train_key_codebook on the 1-bit head preset geometry (d=128, g=64,
L=64), one round, n calibration rows from gen_synth (ctf.cpp:97-144),
EmConfig defaults (30 soft iterations, up to 100 hard).  Reference:
oracle/_ref's train_key_codebook on a bounded sample (fewer rows and
iterations, single-threaded as the reference is), reported per
point-iteration.  Prints one JSON line."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def synth(n, d, rank, seed):
    rng = np.random.default_rng(seed)  # low-rank + noise, gen_synth-like spread
    base = rng.standard_normal((n, rank)) @ rng.standard_normal((rank, d)) / np.sqrt(rank)
    return base + 0.1 * rng.standard_normal((n, d))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--cpu-n", type=int, default=4352)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    from paper_2506_18879_b200 import commvq as G
    import torch
    kq = G.KeyQuantConfig(128, 64, 64, args.rounds)
    calib = synth(args.n, 128, 32, 3)
    em = G.EmConfig()
    G.train_key_codebook(calib[:4096], G.KeyQuantConfig(128, 64, 64, 1),
                         G.EmConfig(soft_iters=1, hard_iters_max=1))  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    atoms, rep = G.train_key_codebook(calib, kq, em)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    hard_iters = sum(len(t) for row in rep["hard_objective"] for t in row)
    pit = args.n * args.rounds * em.soft_iters + args.n * hard_iters
    line = {"metric": "key-codebook EM point-iterations/s (d=128, g=64, L=64)",
            "gpu": {"n": args.n, "rounds": args.rounds, "soft_iters": em.soft_iters,
                    "hard_estep_calls": hard_iters, "seconds": gpu_s,
                    "point_iterations_per_s": pit / gpu_s,
                    "mse": [float(x) for x in rep["reconstruction_mse"]]}}
    if not args.no_cpu:
        from oracle.oracle import KQ, Oracle, have_ref
        if have_ref():
            R = Oracle("reference")
            c = calib[:args.cpu_n]
            t1 = time.perf_counter()
            _, traces, _ = R.train_key_codebook(KQ(128, 64, 64, 1), c, soft_iters=2, hard_iters_max=2)
            cpu_s = time.perf_counter() - t1
            chard = sum(len(t) for row in traces for t in row)
            cpit = args.cpu_n * 2 + args.cpu_n * chard
            line["cpu_reference"] = {"n": args.cpu_n, "soft_iters": 2, "hard_estep_calls": chard,
                                     "seconds": cpu_s, "cores": 1,
                                     "point_iterations_per_s": cpit / cpu_s}
            line["speedup"] = (pit / gpu_s) / (cpit / cpu_s)
    print(json.dumps(line))
    # ---- value quantizer (valquant.cpp:172-383): default ValTrainConfig,
    # d = 128, n_codes = 128 (1-bit), H = 256
    vcal = synth(args.n, 128, 32, 4)
    vcfg = G.ValTrainConfig()
    G.train_value_quantizer(vcal[:1024], 128, G.ValTrainConfig(steps=5))  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = G.train_value_quantizer(vcal, 128, vcfg)
    torch.cuda.synchronize()
    vg = time.perf_counter() - t0
    vline = {"metric": "value-quantizer SGD steps/s (d=128, n_codes=128, batch=256)",
             "gpu": {"steps": r["steps_run"], "seconds": vg, "steps_per_s": r["steps_run"] / vg,
                     "final_loss": float(r["loss_curve"][-1])}}
    if not args.no_cpu:
        from oracle.oracle import Oracle, have_ref
        if have_ref():
            t1 = time.perf_counter()
            Oracle("reference").train_value_quantizer(vcal, 128, steps=20)
            vc = time.perf_counter() - t1
            vline["cpu_reference"] = {"steps": 20, "seconds": vc, "cores": 1,
                                      "steps_per_s": 20 / vc}
            vline["speedup"] = (r["steps_run"] / vg) / (20 / vc)
    print(json.dumps(vline))


if __name__ == "__main__":
    main()
