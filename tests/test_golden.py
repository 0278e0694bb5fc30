"""The reference's own outputs (committed fixtures) pin the C restatement
here and the CUDA path on the GPU box."""
import numpy as np
import pytest

from oracle.oracle import Oracle
from tests import golden_io
from tests.fixtures import rel_err

ATT = golden_io.load("attention")
ENC = golden_io.load("encode")


@pytest.mark.parametrize("name", sorted(ATT))
def test_port_matches_golden_attention(name):
    c = ATT[name]
    P = Oracle("port")
    out, pred, meas = P.fused_attention(c["kq"], c["atoms"], c["a"], c["b"], c["bits"], c["vrows"],
                                        c["q"], int(c["t"]))
    assert (out == c["out"]).all() and [pred, meas] == c["flops"].tolist()
    nout, npred, nmeas = P.naive_attention(c["kq"], c["atoms"], c["a"], c["b"], c["bits"],
                                           c["vrows"], c["q"], int(c["t"]))
    assert (nout == c["naive_out"]).all() and [npred, nmeas] == c["naive_flops"].tolist()
    assert (P.pack_key_codes(c["kq"], c["a"], c["b"]) == c["key_words"]).all()
    assert (P.pack_value_codes(c["bits"]) == c["value_words"]).all()


@pytest.mark.parametrize("name", sorted(ENC))
def test_port_matches_golden_encode(name):
    c = ENC[name]
    P = Oracle("port")
    a, b = P.encode_keys(c["kq"], c["atoms"], c["keys"])
    assert (a == c["a"]).all() and (b == c["b"]).all()
    bits, logits = P.encoder_forward_infer(c["w1"], c["b1"], c["w2"], c["b2"], c["vals"])
    assert (bits == c["bits"]).all() and (logits == c["logits"]).all()


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(ATT))
def test_gpu_matches_golden_attention(name):
    from paper_2506_18879_b200 import commvq as G
    c = ATT[name]
    out, rep = G.fused_attention(c["kq"], c["atoms"], c["a"], c["b"], c["bits"], c["vrows"],
                                 c["q"], int(c["t"]))
    assert rel_err(out, c["out"]) <= 1e-4
    assert [rep.predicted_mults, rep.measured_mults] == c["flops"].tolist()
    nout, nrep = G.naive_attention(c["kq"], c["atoms"], c["a"], c["b"], c["bits"], c["vrows"],
                                   c["q"], int(c["t"]))
    assert rel_err(nout, c["naive_out"]) <= 1e-4
    assert [nrep.predicted_mults, nrep.measured_mults] == c["naive_flops"].tolist()
    assert (G.pack_key_codes(c["kq"], c["a"], c["b"]) == c["key_words"]).all()
    assert (G.pack_value_codes(c["bits"]) == c["value_words"]).all()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(ENC))
def test_gpu_matches_golden_encode(name):
    from paper_2506_18879_b200 import commvq as G
    c = ENC[name]
    a, b = G.encode_keys(c["kq"], c["atoms"], c["keys"])
    assert (a == c["a"]).all() and (b == c["b"]).all()
    assert (G.pack_key_codes(c["kq"], a, b) == c["key_words"]).all()
    bits, logits = G.encoder_forward_infer(c["w1"], c["b1"], c["w2"], c["b2"], c["vals"])
    assert (bits == c["bits"]).all() and (logits == c["logits"]).all()
    assert (G.pack_value_codes(bits) == c["value_words"]).all()
