"""Pins the CPU oracle before it is trusted as the GPU path's checker.

1. The reference's own known-answer tests, restated (test_attn.cpp,
   test_keyquant.cpp, test_valquant.cpp, test_cache.cpp, test_linalg.cpp),
   run against the C restatement and, when built, the compiled reference.
2. The C restatement is bit-identical to the compiled reference
   (oracle/_ref/libcvq_ref.so) on seeded instances of every hot-path function.
"""
import math

import numpy as np
import pytest

from oracle.oracle import KQ, Oracle, TrainingError, have_ref
from tests import fixtures as fx

BACKENDS = ["port"] + (["ref"] if have_ref() else [])


@pytest.fixture(params=BACKENDS)
def O(request):
    return Oracle(request.param)


def ref_or_skip():
    if not have_ref():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return Oracle("ref")


# ---------------------------------------------------------------- rng ----
def test_rng_streams_match_reference():
    R = ref_or_skip()
    P = Oracle("port")
    for seed in (0, 1, 42, 2**63 + 5):
        a, b = P.rng(seed), R.rng(seed)
        assert (a.u64(700) == b.u64(700)).all()  # crosses the 312-word twist
        assert (a.normal(333) == b.normal(333)).all()
        assert (a.index(500, 64) == b.index(500, 64)).all()
        assert (a.bits(100) == b.bits(100)).all()


# ------------------------------------------------------- attention KATs --
def test_fused_hand_expansion_two_tokens(O):
    """test_attn.cpp:165-217 -- d=2, one subspace/group/round, two levels."""
    kq = KQ(2, 1, 2, 1)
    atoms = np.array([0.7, -0.2, -0.4, 1.1])
    a = np.array([0, 1], np.uint16)
    b = np.array([1, 0], np.uint16)
    vrows = np.array([[1.5, -0.5], [0.25, 2.0]])
    bits = np.array([[1, 0], [1, 1]], np.uint8)
    q = np.array([0.3, -0.8])
    out, _, _ = O.fused_attention(kq, atoms, a, b, bits, vrows, q, 1)

    def center(a_, b_):
        xa, ya = (0.7, -0.2) if a_ == 0 else (-0.4, 1.1)
        xb, yb = (0.7, -0.2) if b_ == 0 else (-0.4, 1.1)
        return xa - yb, ya + xb

    def rot(v, pos):
        c, s = math.cos(pos), math.sin(pos)
        return v[0] * c - v[1] * s, v[0] * s + v[1] * c

    qr = rot((0.3, -0.8), 1)
    k0 = rot(center(0, 1), 0)
    k1 = rot(center(1, 0), 1)
    s0 = (qr[0] * k0[0] + qr[1] * k0[1]) / math.sqrt(2)
    s1 = (qr[0] * k1[0] + qr[1] * k1[1]) / math.sqrt(2)
    m = max(s0, s1)
    e0, e1 = math.exp(s0 - m), math.exp(s1 - m)
    w0, w1 = e0 / (e0 + e1), e1 / (e0 + e1)
    want = [w0 * 1.5 + w1 * 1.75, w0 * -0.5 + w1 * 1.5]
    assert out[0] == pytest.approx(want[0], rel=1e-12)
    assert out[1] == pytest.approx(want[1], rel=1e-12)


COMBOS = [  # test_attn.cpp:223-227: (d, g, L, R, n, n_codes)
    (8, 2, 4, 1, 1, 8), (8, 2, 4, 1, 2, 8), (8, 2, 4, 3, 64, 8), (8, 4, 2, 2, 64, 16),
    (16, 2, 4, 3, 64, 16), (16, 4, 8, 2, 256, 8), (16, 8, 4, 1, 256, 16), (8, 2, 4, 2, 1024, 8),
]


def test_fused_equals_naive_across_configs(O):
    """test_attn.cpp:219-244 (seeds 1000.., rel_err <= 1e-5)."""
    seed = 1000
    for d, g, L, R, n, nc in COMBOS:
        kq = KQ(d, g, L, R)
        atoms = fx.random_key_codebook(kq, seed); seed += 1
        a, b = fx.random_key_codes(kq, n, seed); seed += 1
        bits = fx.random_value_codes(nc, n, seed); seed += 1
        vrows = fx.random_value_codebook(nc, d, seed); seed += 1
        q = fx.random_vec(d, seed); seed += 1
        f, _, _ = O.fused_attention(kq, atoms, a, b, bits, vrows, q, n - 1)
        nv, _, _ = O.naive_attention(kq, atoms, a, b, bits, vrows, q, n - 1)
        assert fx.rel_err(f, nv) <= 1e-5


def test_query_position_must_cover_cache(O):
    """test_attn.cpp:246-263."""
    kq = KQ(8, 2, 4, 1)
    atoms = fx.random_key_codebook(kq, 21)
    a, b = fx.random_key_codes(kq, 4, 22)
    bits = fx.random_value_codes(8, 4, 23)
    vrows = fx.random_value_codebook(8, 8, 24)
    q = fx.random_vec(8, 25)
    with pytest.raises(ValueError):
        O.fused_attention(kq, atoms, a, b, bits, vrows, q, 2)
    with pytest.raises(ValueError):
        O.naive_attention(kq, atoms, a, b, bits, vrows, q, 2)
    with pytest.raises(ValueError):
        O.fused_attention(kq, atoms, a[:0], b[:0], bits[:0], vrows, q, 0)


def test_predicted_multiply_counts(O):
    """test_attn.cpp:265-286."""
    assert O.predicted_flops_naive(1, 1, 1) == 5
    assert O.predicted_flops_fused(1, 1, 1, 1, 1) == 5
    assert O.predicted_flops_naive(8192, 1024, 1024) == 17196654592
    assert O.predicted_flops_fused(8192, 1024, 1024, 11, 64) == (
        (11 * 1024 + 1024 + 1) * 8192 + 1024 * (1024 + 11 * 64))
    r1 = O.predicted_flops_naive(8192, 1024, 1024) / O.predicted_flops_fused(8192, 1024, 1024, 11, 64)
    r2 = O.predicted_flops_naive(131072, 1024, 1024) / O.predicted_flops_fused(131072, 1024, 1024, 11, 64)
    assert r1 > 100.0 and r2 > r1


def test_measured_multiplies_in_band(O):
    """test_attn.cpp:288-317."""
    kq = KQ(64, 8, 16, 3)
    n, nc = 1024, 64
    atoms = fx.random_key_codebook(kq, 31)
    a, b = fx.random_key_codes(kq, n, 32)
    bits = fx.random_value_codes(nc, n, 33)
    vrows = fx.random_value_codebook(nc, 64, 34)
    q = fx.random_vec(64, 35)
    _, pn, mn = O.naive_attention(kq, atoms, a, b, bits, vrows, q, n - 1)
    _, pf, mf = O.fused_attention(kq, atoms, a, b, bits, vrows, q, n - 1)
    assert pn == O.predicted_flops_naive(n, 64, nc)
    assert pf == O.predicted_flops_fused(n, 64, nc, 3, 16)
    assert 0.5 <= mn / pn <= 1.5 and 0.5 <= mf / pf <= 1.5
    assert mf < mn


def test_softmax_basics(O):
    """test_linalg.cpp:86-109."""
    assert np.allclose(O.softmax_row(np.zeros(4)), 0.25)
    sx = O.softmax_row(np.array([1.0, 2.0, 3.0]))
    sy = O.softmax_row(np.array([1001.0, 1002.0, 1003.0]))
    assert np.allclose(sx, sy, rtol=1e-12, atol=0)
    assert abs(sx.sum() - 1.0) <= 1e-15
    sb = O.softmax_row(np.array([1e300, 1e300]))
    assert sb[0] == pytest.approx(0.5) and np.isfinite(sb).all()
    with pytest.raises(ValueError):
        O.softmax_row(np.zeros(0))


# -------------------------------------------------------- encoder KATs --
def test_ties_break_to_smallest_pair(O):
    """test_keyquant.cpp:179-193: identical atoms -> every code (0, 0)."""
    kq = KQ(4, 2, 4, 1)
    atoms = np.tile([1.0, -0.5], kq.n_atoms)
    pts = fx.random_mat(16, 4, 77)
    for fact in (False, True):
        if O.kind == "ref" or not fact:
            a, b = O.encode_keys(kq, atoms, pts, factorized=fact)
            assert (a == 0).all() and (b == 0).all()


def test_brute_equals_factorized_equals_exhaustive(O):
    """test_keyquant.cpp:159-177 (exhaustive scan restated in numpy)."""
    kq = KQ(12, 3, 4, 1)
    atoms = fx.random_key_codebook(kq, 41)
    pts = fx.random_mat(64, 12, 42)
    a, b = O.encode_keys(kq, atoms, pts)
    af, bf = O.encode_keys(kq, atoms, pts, factorized=True)
    assert (a == af).all() and (b == bf).all()
    xy = atoms.reshape(kq.rounds, kq.subspaces, kq.n_levels, 2)
    for grp in range(kq.groups):
        subs = range(grp * kq.group_size, (grp + 1) * kq.group_size)
        for i in range(64):
            p = pts[i, grp * 2 * kq.group_size:(grp + 1) * 2 * kq.group_size]
            best, best_c = math.inf, 0
            for c in range(kq.n_levels ** 2):
                aa, bb = divmod(c, kq.n_levels)
                cen = []
                for s in subs:
                    cen += [xy[0, s, aa, 0] - xy[0, s, bb, 1], xy[0, s, aa, 1] + xy[0, s, bb, 0]]
                dist = sum((p[k] - cen[k]) ** 2 for k in range(len(cen)))
                if dist < best:
                    best, best_c = dist, c
            idx = i * kq.groups + grp
            assert (a[idx], b[idx]) == divmod(best_c, kq.n_levels)


def test_value_encoder_thresholds(O):
    """test_valquant.cpp:108-112: zero weights, b2={2,-3,0.5,-0.1} -> bits {1,0,1,0}."""
    w1, b1, w2 = np.zeros((4, 4)), np.zeros(4), np.zeros((4, 4))
    b2 = np.array([2.0, -3.0, 0.5, -0.1])
    bits, logits = O.encoder_forward_infer(w1, b1, w2, b2, np.array([[0.1, -0.2, 0.3, -0.4]]))
    assert bits[0].tolist() == [1, 0, 1, 0]
    assert (logits[0] == b2).all()
    with pytest.raises(TrainingError):
        O.encoder_forward_infer(w1, b1, w2, np.array([np.inf, 0, 0, 0]), np.ones((1, 4)))


# ----------------------------------------------------------- pack KATs --
def test_bit_order_little_endian(O):
    """test_cache.cpp:75-82 through the value packer: bits 1,0,1,0,1 -> 0b10101."""
    w = O.pack_value_codes(np.array([[1, 0, 1, 0, 1]], np.uint8))
    assert w.tolist() == [0b10101]


def test_key_packing_layout(O):
    """test_cache.cpp:94-112."""
    kq = KQ(8, 2, 4, 2)
    rng = O.rng(71)
    a = rng.index(9 * 4, 4)
    b = rng.index(9 * 4, 4)
    # reference draws all a then all b from one stream
    words = O.pack_key_codes(kq, a, b)
    assert words.size == (9 * kq.bits_per_token + 63) // 64
    a2, b2 = O.unpack_key_codes(kq, words, 9)
    assert (a2 == a).all() and (b2 == b).all()
    w0 = int(words[0])
    assert w0 & 3 == a[0] and (w0 >> 2) & 3 == b[0]
    assert (w0 >> 8) & 3 == a[kq.groups]  # token 0, round 1, group 0 at bit 8


def test_value_packing_order(O):
    """test_cache.cpp:114-124."""
    rng = O.rng(72)
    bits = rng.bits(17 * 8).reshape(17, 8)
    words = O.pack_value_codes(bits)
    assert words.size == (17 * 8 + 63) // 64
    assert (O.unpack_value_codes(8, words, 17) == bits).all()
    for k in range(8):
        assert (int(words[0]) >> k) & 1 == bits[0, k]


def test_payload_accounting_long_context():
    """test_cache.cpp:126-140 (1bit preset d=1024: 1056 bits/token, 34,078,720 B @128K)."""
    kq = KQ(1024, 64, 64, 11)
    assert kq.bits_per_token == 1056
    assert 131072 * (1056 + 1024) / 8 == 34078720.0
    assert KQ(128, 64, 64, 11).bits_per_token == 132
    assert KQ(128, 64, 64, 21).bits_per_token == 252


def test_unpack_rejects_bad_shapes(O):
    """cache.cpp:78-88 from_words validation."""
    kq = KQ(8, 2, 4, 1)
    with pytest.raises(ValueError):
        O.unpack_key_codes(kq, np.array([1, 2], np.uint64), 1)
    with pytest.raises(ValueError):
        O.unpack_value_codes(8, np.array([1 << 20], np.uint64), 1)


# ------------------------------------------- port == compiled reference --
@pytest.mark.parametrize("shape", [
    (8, 2, 4, 2, 33, 8), (64, 16, 64, 3, 257, 32), (128, 64, 64, 11, 300, 128),
    (128, 64, 64, 21, 130, 256), (128, 16, 64, 3, 64, 32), (128, 64, 2048, 21, 17, 32),
])
def test_port_matches_reference_attention(shape):
    R = ref_or_skip()
    P = Oracle("port")
    d, g, L, Rr, n, nc = shape
    kq = KQ(d, g, L, Rr)
    rng = P.rng(sum(shape))
    atoms = fx.random_key_codebook(kq, rng=rng, scale=0.3)
    a, b = fx.random_key_codes(kq, n, rng=rng)
    bits = fx.random_value_codes(nc, n, rng=rng)
    vrows = fx.random_value_codebook(nc, d, rng=rng)
    q = rng.normal(d)
    for t in (n - 1, n + 1000):
        for fn in ("fused_attention", "naive_attention"):
            o1 = getattr(P, fn)(kq, atoms, a, b, bits, vrows, q, t)
            o2 = getattr(R, fn)(kq, atoms, a, b, bits, vrows, q, t)
            assert (o1[0] == o2[0]).all() and o1[1:] == o2[1:], fn


@pytest.mark.parametrize("shape", [(8, 2, 4, 2, 40), (16, 4, 16, 3, 40), (128, 64, 64, 2, 24)])
def test_port_matches_reference_encoders(shape):
    R = ref_or_skip()
    P = Oracle("port")
    d, g, L, Rr, n = shape
    kq = KQ(d, g, L, Rr)
    atoms = fx.random_key_codebook(kq, 3 + d)
    keys = P.gen_synth(n, d, min(d, 32), 11)
    assert (keys == R.gen_synth(n, d, min(d, 32), 11)).all()
    pa = P.encode_keys(kq, atoms, keys)
    ra = R.encode_keys(kq, atoms, keys)
    assert (pa[0] == ra[0]).all() and (pa[1] == ra[1]).all()
    assert (P.pack_key_codes(kq, *pa) == R.pack_key_codes(kq, *ra)).all()
    assert (P.decode_keys(kq, atoms, *pa) == R.decode_keys(kq, atoms, *ra)).all()
    hidden, nc = 2 * d, d
    rng = P.rng(99)
    w1 = rng.normal(d * hidden, 0.1).reshape(d, hidden)
    b1 = np.zeros(hidden)
    w2 = rng.normal(hidden * nc, 0.1).reshape(hidden, nc)
    b2 = np.zeros(nc)
    pb, pl = P.encoder_forward_infer(w1, b1, w2, b2, keys)
    rb, rl = R.encoder_forward_infer(w1, b1, w2, b2, keys)
    assert (pb == rb).all() and (pl == rl).all()
    assert (P.pack_value_codes(pb) == R.pack_value_codes(rb)).all()
    rows = rng.normal(nc * d, 1 / 16).reshape(nc, d)
    assert (P.decode_values(rows, pb) == R.decode_values(rows, rb)).all()


def test_prefill_equals_appends_and_oracle_pack():
    """test_cache.cpp:155-180 on the compiled reference, and the oracle's
    encode+pack reproduces the reference cache's words exactly."""
    ref_or_skip()
    from oracle.oracle import RefCache
    P = Oracle("port")
    f = fx.CacheFixture()
    keys = fx.random_mat(24, 8, 81)
    vals = fx.random_mat(24, 8, 82)
    pre = RefCache(f.kq, f.atoms, f.vrows, f.w1, f.b1, f.w2, f.b2)
    pre.prefill(keys, vals)
    inc = RefCache(f.kq, f.atoms, f.vrows, f.w1, f.b1, f.w2, f.b2)
    for t in range(24):
        inc.append(keys[t], vals[t])
    assert (pre.key_words() == inc.key_words()).all()
    assert (pre.value_words() == inc.value_words()).all()
    a, b = P.encode_keys(f.kq, f.atoms, keys)
    assert (P.pack_key_codes(f.kq, a, b) == pre.key_words()).all()
    bits, _ = P.encoder_forward_infer(f.w1, f.b1, f.w2, f.b2, vals)
    assert (P.pack_value_codes(bits) == pre.value_words()).all()


def test_incremental_decode_matches_replay():
    """test_cache.cpp:182-229: decode_step == fused over the replayed prefix <= 1e-6."""
    ref_or_skip()
    from oracle.oracle import RefCache
    P = Oracle("port")
    f = fx.CacheFixture()
    steps = 16
    keys, vals, qs = fx.random_mat(steps, 8, 91), fx.random_mat(steps, 8, 92), fx.random_mat(steps, 8, 93)
    cache = RefCache(f.kq, f.atoms, f.vrows, f.w1, f.b1, f.w2, f.b2)
    a, b = P.encode_keys(f.kq, f.atoms, keys)
    bits, _ = P.encoder_forward_infer(f.w1, f.b1, f.w2, f.b2, vals)
    per = f.kq.rounds * f.kq.groups
    for t in range(steps):
        got = cache.decode_step(keys[t], vals[t], qs[t])
        want, _, _ = P.fused_attention(f.kq, f.atoms, a[:(t + 1) * per], b[:(t + 1) * per],
                                       bits[:t + 1], f.vrows, qs[t], t)
        assert fx.rel_err(got, want) <= 1e-6


def test_single_level_codebook_packs_nothing(O):
    """n_levels = 1 passes KeyQuantConfig::validate (is_pow2(1)) and gives
    zero-bit fields: the packed key stream is empty and unpacks to zeros
    (cache.cpp:90-135, BitBuffer appends of 0 bits); encode_keys picks the
    only center."""
    kq = KQ(8, 2, 1, 2)
    assert kq.bits_per_token == 0
    a = np.zeros(5 * kq.rounds * kq.groups, np.uint16)
    words = O.pack_key_codes(kq, a, a)
    assert words.size == 0
    a2, b2 = O.unpack_key_codes(kq, words, 5)
    assert (a2 == 0).all() and (b2 == 0).all()
    atoms = O.rng(5).normal(2 * kq.n_atoms)
    ea, eb = O.encode_keys(kq, atoms, O.rng(6).normal(5 * 8).reshape(5, 8))
    assert (ea == 0).all() and (eb == 0).all()
