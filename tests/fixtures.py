"""Seeded fixtures restated from the reference tests (all via commvq::Rng).

Each helper reproduces a reference fixture generator draw for draw, so the
same seed yields the same data as the reference test would build:

* random_key_codebook   test_attn.cpp:57-62  (atoms comm_mat(N, N))
* random_key_codes      test_attn.cpp:64-71  (a then b, rng.index(L))
* random_value_codes    test_attn.cpp:73-78  (next_u64() & 1)
* random_value_codebook test_attn.cpp:80-85  (N(0,1))
* random_mat/vec        oracles.hpp:124-136
* cache Fixture         test_cache.cpp:18-36
"""
import numpy as np

from oracle.oracle import KQ, Oracle

_O = None


def O():
    global _O
    if _O is None:
        _O = Oracle("port")
    return _O


def random_key_codebook(kq: KQ, seed=None, rng=None, scale=1.0):
    rng = rng or O().rng(seed)
    return rng.normal(2 * kq.n_atoms, scale)


def random_key_codes(kq: KQ, n, seed=None, rng=None):
    rng = rng or O().rng(seed)
    m = n * kq.rounds * kq.groups
    a = rng.index(m, kq.n_levels)
    b = rng.index(m, kq.n_levels)
    return a, b


def random_value_codes(n_codes, n, seed=None, rng=None):
    rng = rng or O().rng(seed)
    return rng.bits(n * n_codes).reshape(n, n_codes)


def random_value_codebook(n_codes, d, seed=None, rng=None, scale=1.0):
    rng = rng or O().rng(seed)
    return rng.normal(n_codes * d, scale).reshape(n_codes, d)


def random_mat(rows, cols, seed):
    return O().rng(seed).normal(rows * cols).reshape(rows, cols)


def random_vec(n, seed):
    return O().rng(seed).normal(n)


class CacheFixture:
    """test_cache.cpp:18-36 (d=8, g=2, L=4, R=2, N_c=8, hidden=16)."""

    def __init__(self, seed=51, kq=KQ(8, 2, 4, 2), n_codes=8, hidden=16):
        rng = O().rng(seed)
        self.kq = kq
        self.atoms = rng.normal(2 * kq.n_atoms)
        self.vrows = rng.normal(n_codes * kq.d, 0.5).reshape(n_codes, kq.d)
        self.w1 = rng.normal(kq.d * hidden, 0.4).reshape(kq.d, hidden)
        self.b1 = rng.normal(hidden, 0.1)
        self.w2 = rng.normal(hidden * n_codes, 0.4).reshape(hidden, n_codes)
        self.b2 = rng.normal(n_codes, 0.1)


def rel_err(a, b):
    """test_attn.cpp:87-94."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.sqrt(np.sum((a - b) ** 2) / max(np.sum(b * b), 1e-300)))
