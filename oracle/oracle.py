"""ctypes front-end for the CPU checkers.

TEST INFRASTRUCTURE ONLY.  Two interchangeable backends with one numpy API:

* ``Oracle("port")`` -- the C restatement ``oracle/_build/libcvq_oracle.so``
  (cvq_oracle.c, every function citing the reference file:line it follows);
* ``Oracle("ref")``  -- the unmodified reference library compiled from
  /root/reference sources into ``oracle/_ref/libcvq_ref.so`` (ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference arm may import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libcvq_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcvq_ref.so")

_sz = C.c_size_t
_u64 = C.c_uint64
_p = C.c_void_p
_d = C.c_double


class TrainingError(RuntimeError):
    """Mirror of commvq::TrainingError (error.hpp:11-15)."""


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


@dataclass(frozen=True)
class KQ:
    """KeyQuantConfig (keyquant.hpp:16-28)."""

    d: int
    group_size: int
    n_levels: int
    rounds: int

    @property
    def subspaces(self):
        return self.d // 2

    @property
    def groups(self):
        return self.subspaces // self.group_size

    @property
    def level_bits(self):
        b = 0
        while (1 << b) < self.n_levels:
            b += 1
        return b

    @property
    def bits_per_token(self):
        return self.rounds * self.groups * 2 * self.level_bits

    @property
    def n_atoms(self):
        return self.rounds * self.subspaces * self.n_levels


class _CKQ(C.Structure):
    _fields_ = [("d", _sz), ("group_size", _sz), ("n_levels", _sz), ("rounds", _sz)]


class _CAttnIn(C.Structure):
    _fields_ = [
        ("kq", C.POINTER(_CKQ)), ("n_codes", _sz), ("atoms_xy", _p), ("a", _p),
        ("b", _p), ("bits", _p), ("n_tokens", _sz), ("value_rows", _p), ("q", _p),
        ("t", _sz), ("rope_base", _d),
    ]


def words_for_bits(bits):
    return (bits + 63) // 64


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        L = self.lib
        pre = "cvqo_" if kind == "port" else "cvqr_"
        self.pre = pre
        getattr(L, pre + "last_error").restype = C.c_char_p
        getattr(L, pre + "rng_new").restype = _p
        getattr(L, pre + "rng_new").argtypes = [_u64]
        getattr(L, pre + "rng_free").argtypes = [_p]
        for nm, at in [
            ("rng_fill_normal", [_p, _p, _sz, _d]),
            ("rng_fill_index_u16", [_p, _p, _sz, _u64]),
            ("rng_fill_bit_u8", [_p, _p, _sz]),
            ("rng_fill_u64", [_p, _p, _sz]),
        ]:
            getattr(L, pre + nm).argtypes = at
            getattr(L, pre + nm).restype = None
        getattr(L, pre + "predicted_flops_fused").restype = _u64
        getattr(L, pre + "predicted_flops_fused").argtypes = [_sz] * 5
        getattr(L, pre + "predicted_flops_naive").restype = _u64
        getattr(L, pre + "predicted_flops_naive").argtypes = [_sz] * 3

    # ---- errors ----------------------------------------------------------
    def _check(self, rc):
        if rc == 0:
            return
        msg = getattr(self.lib, self.pre + "last_error")().decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 2:
            raise TrainingError(msg)
        if rc == 3:
            raise IndexError(msg)
        raise RuntimeError(msg)

    # ---- rng (rng.hpp:13-56) ------------------------------------------------
    def rng(self, seed):
        return _Rng(self, seed)

    # ---- attention ------------------------------------------------------
    def _attn_call(self, name, kq, atoms, a, b, bits, vrows, q, t, base):
        atoms = np.ascontiguousarray(atoms, np.float64)
        a = np.ascontiguousarray(a, np.uint16)
        b = np.ascontiguousarray(b, np.uint16)
        bits = np.ascontiguousarray(bits, np.uint8)
        vrows = np.ascontiguousarray(vrows, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        n_codes = vrows.shape[0]
        n = bits.shape[0] if bits.ndim == 2 else (bits.size // n_codes if n_codes else 0)
        out = np.zeros(kq.d, np.float64)
        pred, meas = _u64(0), _u64(0)
        if self.kind == "port":
            ckq = _CKQ(kq.d, kq.group_size, kq.n_levels, kq.rounds)
            cin = _CAttnIn(C.pointer(ckq), n_codes, _ptr(atoms), _ptr(a), _ptr(b), _ptr(bits),
                           n, _ptr(vrows), _ptr(q), t, base)
            f = getattr(self.lib, "cvqo_" + name)
            f.argtypes = [C.POINTER(_CAttnIn), _p, _p, _p]
            rc = f(C.byref(cin), _ptr(out), C.byref(pred), C.byref(meas))
        else:
            f = getattr(self.lib, "cvqr_" + name)
            f.argtypes = [_sz] * 5 + [_p] * 4 + [_sz, _p, _p, _sz, _d, _p, _p, _p]
            rc = f(kq.d, kq.group_size, kq.n_levels, kq.rounds, n_codes, _ptr(atoms), _ptr(a),
                   _ptr(b), _ptr(bits), n, _ptr(vrows), _ptr(q), t, base, _ptr(out),
                   C.byref(pred), C.byref(meas))
        self._check(rc)
        return out, pred.value, meas.value

    def fused_attention(self, kq, atoms, a, b, bits, vrows, q, t, base=10000.0):
        """attn.cpp:164-263 -> (out[d], predicted_mults, measured_mults)."""
        return self._attn_call("fused_attention", kq, atoms, a, b, bits, vrows, q, t, base)

    def naive_attention(self, kq, atoms, a, b, bits, vrows, q, t, base=10000.0):
        """attn.cpp:130-162."""
        return self._attn_call("naive_attention", kq, atoms, a, b, bits, vrows, q, t, base)

    def fused_scores(self, kq, atoms, a, b, bits, vrows, q, t, base=10000.0):
        """Pre-softmax scores of the fused pathway (attn.cpp:233); port only."""
        assert self.kind == "port"
        atoms = np.ascontiguousarray(atoms, np.float64)
        a = np.ascontiguousarray(a, np.uint16)
        b = np.ascontiguousarray(b, np.uint16)
        bits = np.ascontiguousarray(bits, np.uint8)
        vrows = np.ascontiguousarray(vrows, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        n_codes = vrows.shape[0]
        n = bits.size // n_codes
        ckq = _CKQ(kq.d, kq.group_size, kq.n_levels, kq.rounds)
        cin = _CAttnIn(C.pointer(ckq), n_codes, _ptr(atoms), _ptr(a), _ptr(b), _ptr(bits), n,
                       _ptr(vrows), _ptr(q), t, base)
        out = np.zeros(n, np.float64)
        f = self.lib.cvqo_fused_scores
        f.argtypes = [C.POINTER(_CAttnIn), _p]
        self._check(f(C.byref(cin), _ptr(out)))
        return out

    def reference_attention(self, q, K, V, t, base=10000.0):
        q = np.ascontiguousarray(q, np.float64)
        K = np.ascontiguousarray(K, np.float64)
        V = np.ascontiguousarray(V, np.float64)
        n, d = K.shape
        out = np.zeros(d)
        f = getattr(self.lib, self.pre + "reference_attention")
        f.argtypes = [_p, _p, _p, _sz, _sz, _d, _sz, _p]
        self._check(f(_ptr(q), _ptr(K), _ptr(V), n, d, base, t, _ptr(out)))
        return out

    def softmax_row(self, v):
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros_like(v)
        f = getattr(self.lib, self.pre + "softmax_row")
        f.argtypes = [_p, _sz, _p]
        self._check(f(_ptr(v), v.size, _ptr(out)))
        return out

    def predicted_flops_fused(self, n, d, n_codes, rounds, levels):
        return getattr(self.lib, self.pre + "predicted_flops_fused")(n, d, n_codes, rounds, levels)

    def predicted_flops_naive(self, n, d, n_codes):
        return getattr(self.lib, self.pre + "predicted_flops_naive")(n, d, n_codes)

    # ---- keyquant -------------------------------------------------------
    def encode_keys(self, kq, atoms, keys, factorized=False):
        """keyquant.cpp:705-739 -> (a, b) as uint16[n * R * groups]."""
        atoms = np.ascontiguousarray(atoms, np.float64)
        keys = np.ascontiguousarray(keys, np.float64)
        n = keys.shape[0]
        m = n * kq.rounds * kq.groups
        a = np.zeros(m, np.uint16)
        b = np.zeros(m, np.uint16)
        if self.kind == "port":
            ckq = _CKQ(kq.d, kq.group_size, kq.n_levels, kq.rounds)
            f = self.lib.cvqo_encode_keys_factorized if factorized else self.lib.cvqo_encode_keys
            f.argtypes = [C.POINTER(_CKQ), _p, _p, _sz, _p, _p]
            rc = f(C.byref(ckq), _ptr(atoms), _ptr(keys), n, _ptr(a), _ptr(b))
        else:
            f = self.lib.cvqr_encode_keys
            f.argtypes = [_sz] * 4 + [_p, _p, _sz, C.c_int, _p, _p]
            rc = f(kq.d, kq.group_size, kq.n_levels, kq.rounds, _ptr(atoms), _ptr(keys), n,
                   int(factorized), _ptr(a), _ptr(b))
        self._check(rc)
        return a, b

    def decode_keys(self, kq, atoms, a, b):
        atoms = np.ascontiguousarray(atoms, np.float64)
        a = np.ascontiguousarray(a, np.uint16)
        b = np.ascontiguousarray(b, np.uint16)
        n = a.size // (kq.rounds * kq.groups)
        out = np.zeros((n, kq.d))
        if self.kind == "port":
            ckq = _CKQ(kq.d, kq.group_size, kq.n_levels, kq.rounds)
            f = self.lib.cvqo_decode_keys
            f.argtypes = [C.POINTER(_CKQ), _p, _p, _p, _sz, _p]
            rc = f(C.byref(ckq), _ptr(atoms), _ptr(a), _ptr(b), n, _ptr(out))
        else:
            f = self.lib.cvqr_decode_keys
            f.argtypes = [_sz] * 4 + [_p, _p, _p, _sz, _p]
            rc = f(kq.d, kq.group_size, kq.n_levels, kq.rounds, _ptr(atoms), _ptr(a), _ptr(b),
                   n, _ptr(out))
        self._check(rc)
        return out

    # ---- valquant -------------------------------------------------------

    def decode_values(self, rows, bits):
        """valquant.cpp:115-128."""
        rows = np.ascontiguousarray(rows, np.float64)
        bits = np.ascontiguousarray(bits, np.uint8)
        n_codes, d = rows.shape
        n = bits.shape[0]
        out = np.zeros((n, d))
        name = "cvqo_decode_values" if self.kind == "port" else "cvqr_decode_values"
        f = getattr(self.lib, name)
        f.argtypes = [_sz, _sz, _p, _p, _sz, _p]
        self._check(f(n_codes, d, _ptr(rows), _ptr(bits), n, _ptr(out)))
        return out
    def encoder_forward_infer(self, w1, b1, w2, b2, values):
        """valquant.cpp:50-101 (infer mode), batched over rows of values."""
        w1 = np.ascontiguousarray(w1, np.float64)
        b1 = np.ascontiguousarray(b1, np.float64)
        w2 = np.ascontiguousarray(w2, np.float64)
        b2 = np.ascontiguousarray(b2, np.float64)
        values = np.ascontiguousarray(values, np.float64)
        d, hidden = w1.shape
        n_codes = w2.shape[1]
        n = values.shape[0]
        bits = np.zeros((n, n_codes), np.uint8)
        logits = np.zeros((n, n_codes))
        f = getattr(self.lib, self.pre + "encoder_forward_infer")
        f.argtypes = [_sz, _sz, _sz, _p, _p, _p, _p, _p, _sz, _p, _p]
        self._check(f(d, hidden, n_codes, _ptr(w1), _ptr(b1), _ptr(w2), _ptr(b2),
                      _ptr(values), n, _ptr(bits), _ptr(logits)))
        return bits, logits

    # ---- packing (cache.cpp:54-155) ---------------------------------------
    def pack_key_codes(self, kq, a, b):
        a = np.ascontiguousarray(a, np.uint16)
        b = np.ascontiguousarray(b, np.uint16)
        n = a.size // (kq.rounds * kq.groups)
        words = np.zeros(max(1, words_for_bits(n * kq.bits_per_token)), np.uint64)
        if self.kind == "port":
            ckq = _CKQ(kq.d, kq.group_size, kq.n_levels, kq.rounds)
            f = self.lib.cvqo_pack_key_codes
            f.argtypes = [C.POINTER(_CKQ), _p, _p, _sz, _p]
            self._check(f(C.byref(ckq), _ptr(a), _ptr(b), n, _ptr(words)))
            return words[: words_for_bits(n * kq.bits_per_token)]
        nw = _sz(0)
        f = self.lib.cvqr_pack_key_codes
        f.argtypes = [_sz] * 4 + [_p, _p, _sz, _p, _p]
        self._check(f(kq.d, kq.group_size, kq.n_levels, kq.rounds, _ptr(a), _ptr(b), n,
                      _ptr(words), C.byref(nw)))
        return words[: nw.value]

    def pack_value_codes(self, bits):
        bits = np.ascontiguousarray(bits, np.uint8)
        n, n_codes = bits.shape
        words = np.zeros(max(1, words_for_bits(n * n_codes)), np.uint64)
        if self.kind == "port":
            f = self.lib.cvqo_pack_value_codes
            f.argtypes = [_sz, _p, _sz, _p]
            self._check(f(n_codes, _ptr(bits), n, _ptr(words)))
            return words[: words_for_bits(n * n_codes)]
        nw = _sz(0)
        f = self.lib.cvqr_pack_value_codes
        f.argtypes = [_sz, _p, _sz, _p, _p]
        self._check(f(n_codes, _ptr(bits), n, _ptr(words), C.byref(nw)))
        return words[: nw.value]

    def unpack_key_codes(self, kq, words, n):
        words = np.ascontiguousarray(words, np.uint64)
        m = n * kq.rounds * kq.groups
        a = np.zeros(m, np.uint16)
        b = np.zeros(m, np.uint16)
        if self.kind == "port":
            ckq = _CKQ(kq.d, kq.group_size, kq.n_levels, kq.rounds)
            f = self.lib.cvqo_unpack_key_codes
            f.argtypes = [C.POINTER(_CKQ), _p, _sz, _sz, _p, _p]
            self._check(f(C.byref(ckq), _ptr(words), words.size, n, _ptr(a), _ptr(b)))
        else:
            f = self.lib.cvqr_unpack_key_codes
            f.argtypes = [_sz] * 4 + [_p, _sz, _sz, _p, _p]
            self._check(f(kq.d, kq.group_size, kq.n_levels, kq.rounds, _ptr(words), words.size,
                          n, _ptr(a), _ptr(b)))
        return a, b

    def unpack_value_codes(self, n_codes, words, n):
        words = np.ascontiguousarray(words, np.uint64)
        bits = np.zeros((n, n_codes), np.uint8)
        f = getattr(self.lib, self.pre + "unpack_value_codes")
        f.argtypes = [_sz, _p, _sz, _sz, _p]
        self._check(f(n_codes, _ptr(words), words.size, n, _ptr(bits)))
        return bits

    # ---- keyquant.cpp:641-703 (compiled reference only) -------------------
    def train_key_codebook(self, kq, calib, soft_iters=30, hard_iters_max=100, t0=0.0,
                           decay=0.9, tol=1e-6, ridge=-1.0, seed=1, factorized=False):
        """train_key_codebook -> (atoms [R*(d/2)*L*2], traces [R][groups], mse [R])."""
        assert self.kind == "reference", "training is pinned on the compiled reference"
        calib = np.ascontiguousarray(calib, np.float64)
        n = calib.shape[0]
        atoms = np.zeros(2 * kq.n_atoms)
        ng = kq.rounds * kq.groups
        cap = ng * (hard_iters_max + 2)
        obj = np.zeros(cap)
        olen = np.zeros(ng, np.uint64)
        mse = np.zeros(kq.rounds)
        f = self.lib.cvqr_train_key_codebook
        f.argtypes = [_sz] * 4 + [_p, _sz, _sz, _sz, _d, _d, _d, _d, _u64, C.c_int,
                                  _p, _p, _sz, _p, _p]
        self._check(f(kq.d, kq.group_size, kq.n_levels, kq.rounds, _ptr(calib), n, soft_iters,
                      hard_iters_max, t0, decay, tol, ridge, seed, int(factorized), _ptr(atoms),
                      _ptr(obj), cap, _ptr(olen), _ptr(mse)))
        traces, k = [], 0
        for r in range(kq.rounds):
            row = []
            for grp in range(kq.groups):
                ln = int(olen[r * kq.groups + grp])
                row.append(obj[k:k + ln].copy())
                k += ln
            traces.append(row)
        return atoms, traces, mse

    # ---- valquant.cpp:172-383 (compiled reference only) -------------------
    def train_value_quantizer(self, calib, n_codes, steps=10000, batch=256, step_size=1e-3,
                              t_start=1.0, t_end=0.1, hidden=0, seed=1, checkpoint_every=100,
                              freeze=False, init_codebook=None):
        assert self.kind == "reference", "training is pinned on the compiled reference"
        calib = np.ascontiguousarray(calib, np.float64)
        n, d = calib.shape
        H = hidden or 2 * n_codes
        out = {"w1": np.zeros((d, H)), "b1": np.zeros(H), "w2": np.zeros((H, n_codes)),
               "b2": np.zeros(n_codes), "codebook": np.zeros((n_codes, d))}
        curve = np.zeros(max(steps, 1))
        clen, sr = _sz(0), _sz(0)
        dv = C.c_int(0)
        init = None if init_codebook is None else np.ascontiguousarray(init_codebook, np.float64)
        f = self.lib.cvqr_train_value_quantizer
        f.argtypes = [_p, _sz, _sz, _sz, _sz, _sz, _d, _d, _d, _sz, _u64, _sz, C.c_int, _p,
                      _p, _p, _p, _p, _p, _p, C.POINTER(_sz), C.POINTER(C.c_int), C.POINTER(_sz)]
        self._check(f(_ptr(calib), n, d, n_codes, steps, batch, step_size, t_start, t_end, hidden,
                      seed, checkpoint_every, int(freeze), _ptr(init) if init is not None else None,
                      _ptr(out["w1"]), _ptr(out["b1"]), _ptr(out["w2"]), _ptr(out["b2"]),
                      _ptr(out["codebook"]), _ptr(curve), C.byref(clen), C.byref(dv),
                      C.byref(sr)))
        out["loss_curve"] = curve[:clen.value].copy()
        out["diverged"] = bool(dv.value)
        out["steps_run"] = int(sr.value)
        return out

    # ---- ctf.cpp:97-144 --------------------------------------------------
    def gen_synth(self, n, d, rank, seed):
        out = np.zeros((n, d))
        f = getattr(self.lib, self.pre + "gen_synth")
        f.argtypes = [_sz, _sz, _sz, _u64, _p]
        self._check(f(n, d, rank, seed, _ptr(out)))
        return out


class _Rng:
    """commvq::Rng (rng.hpp:13-56) driven through the chosen backend."""

    def __init__(self, o: Oracle, seed: int):
        self.o = o
        self.h = getattr(o.lib, o.pre + "rng_new")(seed)

    def __del__(self):
        try:
            getattr(self.o.lib, self.o.pre + "rng_free")(self.h)
        except Exception:
            pass

    def normal(self, n, scale=1.0):
        out = np.zeros(n)
        getattr(self.o.lib, self.o.pre + "rng_fill_normal")(self.h, _ptr(out), n, scale)
        return out

    def index(self, n, bound):
        out = np.zeros(n, np.uint16)
        getattr(self.o.lib, self.o.pre + "rng_fill_index_u16")(self.h, _ptr(out), n, bound)
        return out

    def bits(self, n):
        out = np.zeros(n, np.uint8)
        getattr(self.o.lib, self.o.pre + "rng_fill_bit_u8")(self.h, _ptr(out), n)
        return out

    def u64(self, n):
        out = np.zeros(n, np.uint64)
        getattr(self.o.lib, self.o.pre + "rng_fill_u64")(self.h, _ptr(out), n)
        return out


class RefCache:
    """commvq::QuantizedKVCache driven through oracle/_ref (cache.cpp:188-296)."""

    def __init__(self, kq, atoms, vrows, w1, b1, w2, b2):
        self.o = Oracle("ref")
        L = self.o.lib
        self.kq = kq
        self.keep = [np.ascontiguousarray(x, np.float64) for x in (atoms, vrows, w1, b1, w2, b2)]
        atoms, vrows, w1, b1, w2, b2 = self.keep
        L.cvqr_cache_new.restype = _p
        L.cvqr_cache_new.argtypes = [_sz] * 6 + [_p] * 6
        self.h = L.cvqr_cache_new(kq.d, kq.group_size, kq.n_levels, kq.rounds, vrows.shape[0],
                                  w1.shape[1], _ptr(atoms), _ptr(vrows), _ptr(w1), _ptr(b1),
                                  _ptr(w2), _ptr(b2))
        if not self.h:
            raise ValueError(L.cvqr_last_error().decode())
        L.cvqr_cache_free.argtypes = [_p]
        L.cvqr_cache_prefill.argtypes = [_p, _p, _p, _sz]
        L.cvqr_cache_append.argtypes = [_p, _p, _p]
        L.cvqr_cache_decode_step.argtypes = [_p, _p, _p, _p, _p]
        L.cvqr_cache_size.restype = _sz
        L.cvqr_cache_size.argtypes = [_p]
        L.cvqr_cache_key_words.restype = _sz
        L.cvqr_cache_key_words.argtypes = [_p, _p]
        L.cvqr_cache_value_words.restype = _sz
        L.cvqr_cache_value_words.argtypes = [_p, _p]

    def __del__(self):
        try:
            self.o.lib.cvqr_cache_free(self.h)
        except Exception:
            pass

    def prefill(self, K, V):
        K = np.ascontiguousarray(K, np.float64)
        V = np.ascontiguousarray(V, np.float64)
        self.o._check(self.o.lib.cvqr_cache_prefill(self.h, _ptr(K), _ptr(V), K.shape[0]))

    def append(self, k, v):
        k = np.ascontiguousarray(k, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        self.o._check(self.o.lib.cvqr_cache_append(self.h, _ptr(k), _ptr(v)))

    def decode_step(self, k, v, q):
        k = np.ascontiguousarray(k, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        out = np.zeros(self.kq.d)
        self.o._check(self.o.lib.cvqr_cache_decode_step(self.h, _ptr(k), _ptr(v), _ptr(q),
                                                         _ptr(out)))
        return out

    def size(self):
        return self.o.lib.cvqr_cache_size(self.h)

    def key_words(self):
        n = self.o.lib.cvqr_cache_key_words(self.h, None)
        out = np.zeros(n, np.uint64)
        self.o.lib.cvqr_cache_key_words(self.h, _ptr(out))
        return out

    def value_words(self):
        n = self.o.lib.cvqr_cache_value_words(self.h, None)
        out = np.zeros(n, np.uint64)
        self.o.lib.cvqr_cache_value_words(self.h, _ptr(out))
        return out


def have_ref():
    return os.path.exists(REF_SO)
