"""Value-quantizer training on the GPU (train_value.cu)
against the compiled reference's train_value_quantizer (valquant.cpp:172-383).

Fixtures: tests/golden/valtrain.npz from make_golden_valtrain.py (oracle/_ref).
The random stream is the reference's own and every reduction runs in the
reference order; the device exp/log differ from libm in the last bits only,
so weights, codebook and loss curve are compared at 1e-9 relative and the
status (diverged, steps_run, curve length) exactly."""
import os

import numpy as np
import pytest

from oracle.oracle import Oracle, have_ref

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "valtrain.npz")
CASES = ["small", "freeze_init", "diverge", "head"]
KEYS = ("w1", "b1", "w2", "b2", "codebook")


def _load(name):
    z = np.load(GOLD)
    n, d, nc, steps, batch, hidden, seed, ck, fr, init, rank = (int(x) for x in z[f"{name}/cfg"])
    c = dict(n=n, d=d, nc=nc, steps=steps, batch=batch, hidden=hidden, seed=seed, ck=ck,
             freeze=bool(fr), lr=float(z[f"{name}/lr"][0]), calib=z[f"{name}/calib"],
             init=z[f"{name}/init_cb"] if init else None,
             diverged=bool(z[f"{name}/status"][0]), steps_run=int(z[f"{name}/status"][1]))
    for k in KEYS + ("loss_curve",):
        c[k] = z[f"{name}/{k}"]
    return c


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", CASES[:3])
def test_golden_valtrain_fixture_matches_reference(name):
    c = _load(name)
    r = Oracle("reference").train_value_quantizer(
        c["calib"], c["nc"], steps=c["steps"], batch=c["batch"], step_size=c["lr"],
        hidden=c["hidden"], seed=c["seed"], checkpoint_every=c["ck"], freeze=c["freeze"],
        init_codebook=c["init"])
    for k in KEYS + ("loss_curve",):
        assert np.array_equal(r[k], c[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_valtrain_matches_reference(name):
    from paper_2506_18879_b200 import commvq as G
    c = _load(name)
    cfg = G.ValTrainConfig(steps=c["steps"], batch=c["batch"], step_size=c["lr"],
                           hidden=c["hidden"], seed=c["seed"], checkpoint_every=c["ck"],
                           freeze_codebook=c["freeze"])
    r = G.train_value_quantizer(c["calib"], c["nc"], cfg, init_codebook=c["init"])
    assert r["diverged"] == c["diverged"]
    assert r["steps_run"] == c["steps_run"]
    assert len(r["loss_curve"]) == len(c["loss_curve"])
    worst = 0.0
    for k in KEYS:
        scale = max(np.max(np.abs(c[k])), 1e-300)
        worst = max(worst, np.max(np.abs(r[k] - c[k])) / scale)
    lc = np.max(np.abs(r["loss_curve"] - c["loss_curve"]) / np.abs(c["loss_curve"]))
    print(name, "params rel err", worst, "loss rel err", lc)
    assert worst <= 1e-9
    assert lc <= 1e-9


@pytest.mark.gpu
def test_gpu_valtrain_errors():
    """valquant.cpp:175-200 preconditions."""
    from paper_2506_18879_b200 import commvq as G
    x = np.ones((8, 4))
    with pytest.raises(ValueError):
        G.train_value_quantizer(x, 0)
    with pytest.raises(ValueError):  # fewer rows than batch
        G.train_value_quantizer(x, 4, G.ValTrainConfig(batch=16))
    with pytest.raises(ValueError):
        G.train_value_quantizer(x, 4, G.ValTrainConfig(batch=4, gumbel_t_start=0.1,
                                                       gumbel_t_end=1.0))
    bad = x.copy()
    bad[1, 1] = np.inf
    with pytest.raises(ValueError):
        G.train_value_quantizer(bad, 4, G.ValTrainConfig(batch=4))
