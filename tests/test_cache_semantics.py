"""Device-resident cache semantics the reference's QuantizedKVCache has
(cache.hpp:62-113, cache.cpp:188-373) and round 1 lacked:

* no fixed capacity: appends / prefill / imports past the initial
  reservation grow the pools (the reference's vectors grow,
  cache.cpp:256-285), with words identical to the reference packing;
* an append whose value encoder yields non-finite logits throws
  TrainingError and leaves the cache unchanged (valquant.cpp:86-87) -- here
  the error is deferred to the next synchronising call (appends never wait
  for the device) but the observable state is the same;
* the tcgen05 fp16-operand guard: a key codebook whose atoms make the fp16
  operand too coarse demotes the cache to the fp32 kernels (key_mode()).
"""
import numpy as np
import pytest

from oracle.oracle import KQ, Oracle
from tests import fixtures as fx

pytestmark = pytest.mark.gpu

P = Oracle("port")


@pytest.fixture(scope="module")
def G():
    from paper_2506_18879_b200 import commvq
    return commvq


def _cache(G, f, capacity, keys="fp32"):
    c = G.QuantizedKVCache(f.kq, 8, capacity=capacity, hidden=16, keys=keys)
    c.set_key_codebook(0, 0, f.atoms)
    c.set_value_quantizer(0, 0, f.vrows, f.w1, f.b1, f.w2, f.b2)
    return c


def test_appends_grow_past_initial_capacity(G):
    """test_cache.cpp:155-180 (prefill == appends, word-exact) with the
    device cache created for 16 tokens and filled with 700 (prefill 300, then
    400 single appends): words equal the oracle cache's; capacity grew."""
    f = fx.CacheFixture()
    K = P.gen_synth(700, 8, 8, 3)
    V = P.gen_synth(700, 8, 8, 4)
    c = _cache(G, f, 16)
    c.prefill(K[None, None, None, :300], V[None, None, None, :300])
    for i in range(300, 700):
        c.append(K[None, None, None, i], V[None, None, None, i])
    assert c.size() == 700 and c.capacity_tokens() >= 700
    kw, vw = c.export_stream(0, 0, 0)
    a, b = P.encode_keys(f.kq, f.atoms, K)
    bits, _ = P.encoder_forward_infer(f.w1, f.b1, f.w2, f.b2, V)
    assert (kw == P.pack_key_codes(f.kq, a, b)).all() and (vw == P.pack_value_codes(bits)).all()
    q = P.rng(9).normal(8)
    out = c.attention(q.reshape(1, 1, 1, 8).astype(np.float32), 699)
    want, _, _ = P.fused_attention(f.kq, f.atoms, a, b, bits, f.vrows, q, 699)
    assert fx.rel_err(out.reshape(-1), want) <= 1e-5


def test_import_and_set_length_grow(G):
    kq = KQ(128, 64, 64, 11)
    c = G.QuantizedKVCache(kq, 128, capacity=128, keys="tc")
    rng = P.rng(3)
    atoms = rng.normal(2 * kq.n_atoms, 0.3)
    vrows = rng.normal(128 * 128, 1 / 16).reshape(128, 128)
    c.set_key_codebook(0, 0, atoms)
    c.set_value_quantizer(0, 0, vrows)
    n = 5000
    a, b = fx.random_key_codes(kq, n, rng=rng)
    bits = fx.random_value_codes(128, n, rng=rng)
    c.import_stream(0, 0, 0, P.pack_key_codes(kq, a, b), P.pack_value_codes(bits), n)
    assert c.capacity_tokens() >= n
    q = rng.normal(128)
    out = c.attention(q.reshape(1, 1, 1, 128).astype(np.float32), n - 1)
    want, _, _ = P.fused_attention(kq, atoms, a, b, bits, vrows, q, n - 1)
    assert fx.rel_err(out.reshape(-1), want) <= 1e-3
    c.set_length(9000)
    assert c.size() == 9000 and c.capacity_tokens() >= 9000


def test_nonfinite_append_rolls_back(G):
    """A value row with an inf makes the logits non-finite: the append is
    dropped and TrainingError surfaces at the next synchronising call; the
    tokens before it are intact and later appends work again."""
    f = fx.CacheFixture()
    K = P.gen_synth(40, 8, 8, 5)
    V = P.gen_synth(40, 8, 8, 6)
    c = _cache(G, f, 64)
    c.prefill(K[None, None, None, :20], V[None, None, None, :20])
    bad = V[20].copy()
    bad[0] = np.inf
    c.append(K[None, None, None, 20], bad[None, None, None])  # returns at once
    c.append(K[None, None, None, 21], V[None, None, None, 21])  # skipped on the device
    with pytest.raises(G.TrainingError):
        c.synchronize()
    assert c.size() == 20
    for i in range(20, 40):
        c.append(K[None, None, None, i], V[None, None, None, i])
    assert c.size() == 40
    kw, vw = c.export_stream(0, 0, 0)
    a, b = P.encode_keys(f.kq, f.atoms, K)
    bits, _ = P.encoder_forward_infer(f.w1, f.b1, f.w2, f.b2, V)
    assert (kw == P.pack_key_codes(f.kq, a, b)).all() and (vw == P.pack_value_codes(bits)).all()
    # a failing prefill leaves the cache unchanged
    with pytest.raises(G.TrainingError):
        Vb = V[None, None, None, :10].copy()
        Vb[0, 0, 0, 7, 1] = np.nan
        c.prefill(K[None, None, None, :10], Vb)
    assert c.size() == 40


def test_decode_step_host_buffers_reports_encoder_error(G):
    f = fx.CacheFixture()
    K = P.gen_synth(10, 8, 8, 7)
    V = P.gen_synth(10, 8, 8, 8)
    c = _cache(G, f, 16)
    c.prefill(K[None, None, None, :9], V[None, None, None, :9])
    bad = V[9].copy()
    bad[3] = -np.inf
    q = np.ones((1, 1, 1, 8), np.float32)
    with pytest.raises(G.TrainingError):
        c.decode_step(K[None, None, None, 9], bad[None, None, None], q)
    assert c.size() == 9


@pytest.mark.parametrize("scale,want_mode", [(0.3, "tc"), (1.0, "tc"), (3.0, "fp32")])
def test_tc_fp16_guard(G, scale, want_mode):
    """sum_r max|U| <= 96 keeps the tcgen05 path (R = 11 at sigma 1.0: ~43);
    sigma 3.0 (~130) demotes to the fp32 kernels, which then meet 1e-4."""
    kq = KQ(128, 64, 64, 11)
    nc, n = 128, 3000
    rng = P.rng(int(scale * 100))
    atoms = rng.normal(2 * kq.n_atoms, scale)
    vrows = rng.normal(nc * 128, 1 / 16).reshape(nc, 128)
    c = G.QuantizedKVCache(kq, nc, capacity=n, keys="tc")
    c.set_key_codebook(0, 0, atoms)
    c.set_value_quantizer(0, 0, vrows)
    assert c.key_mode() == want_mode
    a, b = fx.random_key_codes(kq, n, rng=rng)
    bits = fx.random_value_codes(nc, n, rng=rng)
    c.import_stream(0, 0, 0, P.pack_key_codes(kq, a, b), P.pack_value_codes(bits), n)
    q = rng.normal(128)
    out = c.attention(q.reshape(1, 1, 1, 128).astype(np.float32), n - 1)
    want, _, _ = P.fused_attention(kq, atoms, a, b, bits, vrows, q, n - 1)
    assert fx.rel_err(out.reshape(-1), want) <= (1e-3 if want_mode == "tc" else 1e-4)


@pytest.mark.parametrize("shape", [(16, 4, 16, 3), (128, 64, 64, 11), (8, 2, 4, 2)])
def test_encode_keys_factorized_bit_exact(G, shape):
    """AssignSearch::factorized (keyquant.cpp:204-224, 724-730) on the
    device vs the oracle's factorized search, with constructed midpoints
    between two centers where brute force and factorized may disagree."""
    kq = KQ(*shape)
    rng = P.rng(sum(shape) + 5)
    atoms = rng.normal(2 * kq.n_atoms, 0.3 if kq.d == 128 else 1.0)
    keys = P.gen_synth(257, kq.d, min(kq.d, 32), 17)
    xy = atoms.reshape(kq.rounds, kq.subspaces, kq.n_levels, 2)
    for p in range(40):
        a1, b1, a2, b2 = rng.index(4, kq.n_levels).tolist()
        for j in range(kq.group_size):
            keys[p, 2 * j] = 0.5 * (xy[0, j, a1, 0] - xy[0, j, b1, 1] + xy[0, j, a2, 0] - xy[0, j, b2, 1])
            keys[p, 2 * j + 1] = 0.5 * (xy[0, j, a1, 1] + xy[0, j, b1, 0] + xy[0, j, a2, 1] + xy[0, j, b2, 0])
    for search in ("brute_force", "factorized"):
        ga, gb = G.encode_keys(kq, atoms, keys, search=search)
        oa, ob = P.encode_keys(kq, atoms, keys, factorized=(search == "factorized"))
        assert (ga == oa).all() and (gb == ob).all(), search


def test_single_stream_mirror_reuses_device_copies(G):
    """fused_attention called as a decode loop over growing, append-only
    arrays (the reference cache's key_codes_/value_codes_ vectors): every
    step equals the oracle; the device cache is reused (only the tail is
    uploaded) and an in-place change of earlier codes is detected."""
    kq = KQ(16, 4, 16, 3)
    nc, n_max = 16, 400
    rng = P.rng(77)
    atoms = rng.normal(2 * kq.n_atoms)
    vrows = rng.normal(nc * 16).reshape(nc, 16)
    a_all, b_all = fx.random_key_codes(kq, n_max, rng=rng)
    bits_all = fx.random_value_codes(nc, n_max, rng=rng)
    per = kq.rounds * kq.groups
    a = np.zeros(n_max * per, np.uint16)  # preallocated, filled in place
    b = np.zeros(n_max * per, np.uint16)
    bits = np.zeros((n_max, nc), np.uint8)
    for n in (1, 2, 50, 51, 200, 399, 400):
        a[:n * per], b[:n * per], bits[:n] = a_all[:n * per], b_all[:n * per], bits_all[:n]
        q = rng.normal(16)
        got, _ = G.fused_attention(kq, atoms, a[:n * per], b[:n * per], bits[:n], vrows, q, n - 1)
        want, _, _ = P.fused_attention(kq, atoms, a[:n * per], b[:n * per], bits[:n], vrows, q, n - 1)
        assert fx.rel_err(got, want) <= 1e-5, n
    a[0] = (a[0] + 1) % kq.n_levels  # rewrite an early code in place
    q = rng.normal(16)
    got, _ = G.fused_attention(kq, atoms, a, b, bits, vrows, q, n_max - 1)
    want, _, _ = P.fused_attention(kq, atoms, a, b, bits, vrows, q, n_max - 1)
    assert fx.rel_err(got, want) <= 1e-5


def test_single_level_codebook_cache(G):
    """n_levels = 1: zero-bit key fields.  Prefill, appends and attention
    run (round 1 launched a zero-width pack grid) and match the oracle."""
    kq = KQ(8, 2, 1, 2)
    f = fx.CacheFixture(kq=kq)
    c = G.QuantizedKVCache(kq, 8, capacity=4, hidden=16)
    c.set_key_codebook(0, 0, f.atoms)
    c.set_value_quantizer(0, 0, f.vrows, f.w1, f.b1, f.w2, f.b2)
    K, V = P.gen_synth(9, 8, 8, 41), P.gen_synth(9, 8, 8, 42)
    c.prefill(K[None, None, None, :5], V[None, None, None, :5])
    for i in range(5, 9):
        c.append(K[None, None, None, i], V[None, None, None, i])
    kw, vw = c.export_stream(0, 0, 0)
    a, b = P.encode_keys(kq, f.atoms, K)
    bits, _ = P.encoder_forward_infer(f.w1, f.b1, f.w2, f.b2, V)
    assert kw.size == 0 and (vw == P.pack_value_codes(bits)).all()
    q = P.rng(3).normal(8)
    out = c.attention(q.reshape(1, 1, 1, 8).astype(np.float32), 8)
    want, _, _ = P.fused_attention(kq, f.atoms, a, b, bits, f.vrows, q, 8)
    assert fx.rel_err(out.reshape(-1), want) <= 1e-5


def test_value_screen_presets_bit_exact(G):
    """The prefill value encoder screens with fp32 GEMMs and a rigorous error
    bound, re-computing undecided tokens exactly (k_encode_values_screen).
    Head-preset shapes (hidden 256, 128 codes): bits equal the reference's,
    including logits forced to exactly 0 (always undecided -> exact path) and
    a non-finite row (TrainingError, nothing appended)."""
    kq = KQ(128, 64, 64, 11)
    nc, hidden, n = 128, 256, 300
    rng = P.rng(2024)
    atoms = rng.normal(2 * kq.n_atoms, 0.3)
    vrows = rng.normal(nc * 128, 1 / 16).reshape(nc, 128)
    w1 = rng.normal(128 * hidden, 0.1).reshape(128, hidden)
    b1 = rng.normal(hidden, 0.05)
    w2 = rng.normal(hidden * nc, 0.1).reshape(hidden, nc)
    K = P.gen_synth(n, 128, 32, 3)
    V = P.gen_synth(n, 128, 32, 4)
    V[7, :5] = 0.0  # zero-skips
    _, l0 = P.encoder_forward_infer(w1, b1, w2, np.zeros(nc), V)
    b2 = rng.normal(nc, 0.05)
    b2[:12] = -l0[5, :12]  # token 5: twelve logits exactly 0 in the reference
    bits, lg = P.encoder_forward_infer(w1, b1, w2, b2, V)
    assert (lg[5, :12] == 0.0).all()
    c = G.QuantizedKVCache(kq, nc, capacity=n, hidden=hidden)
    c.set_key_codebook(0, 0, atoms)
    c.set_value_quantizer(0, 0, vrows, w1, b1, w2, b2)
    c.prefill(K[None, None, None], V[None, None, None])
    _, vw = c.export_stream(0, 0, 0)
    assert (vw == P.pack_value_codes(bits)).all()
    Vb = V.copy()
    Vb[40, 3] = np.inf
    c2 = G.QuantizedKVCache(kq, nc, capacity=n, hidden=hidden)
    c2.set_key_codebook(0, 0, atoms)
    c2.set_value_quantizer(0, 0, vrows, w1, b1, w2, b2)
    with pytest.raises(G.TrainingError):
        c2.prefill(K[None, None, None], Vb[None, None, None])
    assert c2.size() == 0


def test_preset_appends_bit_exact_with_near_ties(G):
    """Decode-step appends on the head preset run the fp32-screen small
    encoder (k_encode_keys_small32): codes of single-token appends equal the
    reference's, including keys constructed exactly midway between two
    centres (the screen is not decisive there: exact search)."""
    kq = KQ(128, 64, 64, 11)
    nc = 128
    rng = P.rng(77)
    atoms = rng.normal(2 * kq.n_atoms, 0.3)
    xy = atoms.reshape(11, 64, 64, 2)
    n = 24
    K = P.gen_synth(n, 128, 32, 8)
    for i in range(0, n, 3):  # every third key: a round-0 midpoint
        a1, b1, a2, b2 = rng.index(4, 64).tolist()
        for j in range(64):
            c1 = (xy[0, j, a1, 0] - xy[0, j, b1, 1], xy[0, j, a1, 1] + xy[0, j, b1, 0])
            c2 = (xy[0, j, a2, 0] - xy[0, j, b2, 1], xy[0, j, a2, 1] + xy[0, j, b2, 0])
            K[i, 2 * j] = 0.5 * (c1[0] + c2[0])
            K[i, 2 * j + 1] = 0.5 * (c1[1] + c2[1])
    V = P.gen_synth(n, 128, 32, 9)
    hidden = 256
    w1 = rng.normal(128 * hidden, 0.1).reshape(128, hidden)
    w2 = rng.normal(hidden * nc, 0.1).reshape(hidden, nc)
    b1, b2 = np.zeros(hidden), np.zeros(nc)
    vrows = rng.normal(nc * 128, 1 / 16).reshape(nc, 128)
    c = G.QuantizedKVCache(kq, nc, capacity=8, hidden=hidden)
    c.set_key_codebook(0, 0, atoms)
    c.set_value_quantizer(0, 0, vrows, w1, b1, w2, b2)
    for i in range(n):
        c.append(K[None, None, None, i], V[None, None, None, i])
    c.synchronize()
    kw, vw = c.export_stream(0, 0, 0)
    a, b = P.encode_keys(kq, atoms, K)
    bits, _ = P.encoder_forward_infer(w1, b1, w2, b2, V)
    assert (kw == P.pack_key_codes(kq, a, b)).all()
    assert (vw == P.pack_value_codes(bits)).all()


def test_two_group_preset_prefill_and_appends_bit_exact(G):
    """d = 256 with 64-subspace groups (two key groups per round): the fp32
    prefill encoder (k_encode_keys_t64) and the fp32 decode-step encoder
    (k_encode_keys_small32) both handle the second group's residual and
    slice offsets; words equal the reference packing."""
    kq = KQ(256, 64, 64, 3)
    nc, hidden = 128, 0
    rng = P.rng(555)
    atoms = rng.normal(2 * kq.n_atoms, 0.3)
    K = P.gen_synth(70, 256, 32, 12)
    V = P.gen_synth(70, 256, 32, 13)
    vrows = rng.normal(nc * 256, 1 / 16).reshape(nc, 256)
    w1 = rng.normal(256 * 128, 0.1).reshape(256, 128)
    w2 = rng.normal(128 * nc, 0.1).reshape(128, nc)
    b1, b2 = np.zeros(128), np.zeros(nc)
    c = G.QuantizedKVCache(kq, nc, capacity=80, hidden=128)
    c.set_key_codebook(0, 0, atoms)
    c.set_value_quantizer(0, 0, vrows, w1, b1, w2, b2)
    c.prefill(K[None, None, None, :60], V[None, None, None, :60])
    for i in range(60, 70):
        c.append(K[None, None, None, i], V[None, None, None, i])
    c.synchronize()
    kw, vw = c.export_stream(0, 0, 0)
    a, b = P.encode_keys(kq, atoms, K)
    bits, _ = P.encoder_forward_infer(w1, b1, w2, b2, V)
    assert (kw == P.pack_key_codes(kq, a, b)).all()
    assert (vw == P.pack_value_codes(bits)).all()
