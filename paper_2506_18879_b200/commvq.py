"""ctypes mirror of the reference C++ API over the C-ABI (include/cvq.h).

Function names, argument meaning and error behaviour follow
commvq_core (/root/reference/proj/core/include/commvq/*.hpp), so the parity
tests read like the reference's own tests:

=====================================  =====================================
reference (C++)                        here
=====================================  =====================================
fused_attention(AttnInput, RopeTable)  fused_attention(...)      attn.hpp:62
naive_quantized_attention              naive_attention(...)      attn.hpp:56
encode_keys(Mat, KeyCodebook)          encode_keys(...)          keyquant.hpp:135
encoder_forward(Vec, Encoder, infer)   encoder_forward_infer()   valquant.hpp:62
pack/unpack_{key,value}_codes          same names                cache.hpp:36-41
QuantizedKVCache                       QuantizedKVCache (multi-stream, HBM)
predicted_flops_{fused,naive}          same names                attn.hpp:66-71
=====================================  =====================================

std::invalid_argument -> ValueError, commvq::TrainingError ->
TrainingError, std::out_of_range -> IndexError, commvq::IoError -> IoError,
device failures -> CudaError.  There is no CPU fallback: importing this
module fails loudly when libcvq_b200.so is missing, and every numeric call
runs on the B200.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libcvq_b200.so")

if not os.path.exists(SO_PATH):
    raise ImportError(
        f"{SO_PATH} is missing: build it with `python -m paper_2506_18879_b200.build` "
        "(there is no CPU fallback)")

_lib = C.CDLL(SO_PATH)
_p, _u32, _u64, _d, _i = C.c_void_p, C.c_uint32, C.c_uint64, C.c_double, C.c_int

CVQ_F32, CVQ_F64 = 0, 1
CVQ_DEVICE, CVQ_HOST = 0, 1


class TrainingError(RuntimeError):
    """commvq::TrainingError (error.hpp:11-15)."""


class IoError(RuntimeError):
    """commvq::IoError (error.hpp:17-20)."""


class CudaError(RuntimeError):
    """Device failure (no CPU fallback exists)."""


class NcclError(RuntimeError):
    """NCCL missing or a collective failed (shard groups)."""


_lib.cvq_last_error.restype = C.c_char_p
_lib.cvq_launch_count.restype = _u64
_lib.cvq_abi_version.restype = _i


def _check(rc):
    if rc == 0:
        return
    msg = _lib.cvq_last_error().decode()
    raise {1: ValueError, 2: TrainingError, 3: IndexError, 4: IoError,
           7: NcclError}.get(rc, CudaError)(msg)


def launch_count() -> int:
    """Kernel launches issued by libcvq_b200 in this process."""
    return int(_lib.cvq_launch_count())


class _KC(C.Structure):
    _fields_ = [("d", _u32), ("group_size", _u32), ("n_levels", _u32), ("rounds", _u32)]


class _Flops(C.Structure):
    _fields_ = [("predicted_mults", _u64), ("measured_mults", _u64)]


class _Desc(C.Structure):
    _fields_ = [("key", _KC), ("n_codes", _u32), ("hidden", _u32), ("n_seqs", _u32),
                ("n_layers", _u32), ("n_kv_heads", _u32), ("q_per_kv", _u32),
                ("capacity", _u64), ("position_offset", _u64), ("rope_base", _d),
                ("flags", _u32)]


CVQ_CACHE_KEYS_FP16 = 1
CVQ_CACHE_KEYS_TC = 2
# kernel variants (cvq.h CVQ_VARIANT_*), QuantizedKVCache.set_variant
VARIANTS = {"generic": 1, "tc_dense": 2, "tc_pair": 4, "fused": 8, "f32_weights": 16}


@dataclass(frozen=True)
class KeyQuantConfig:
    """keyquant.hpp:16-28."""

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
        return max(0, int(self.n_levels - 1).bit_length())

    @property
    def bits_per_token(self):
        return self.rounds * self.groups * 2 * self.level_bits

    @property
    def n_atoms(self):
        return self.rounds * self.subspaces * self.n_levels

    def _c(self):
        return _KC(self.d, self.group_size, self.n_levels, self.rounds)


@dataclass
class FlopReport:
    """attn.hpp:16-27."""

    pathway: str
    tokens: int
    d: int
    n_codes: int
    rounds: int
    n_levels: int
    predicted_mults: int
    measured_mults: int


def _kc(kq):
    if isinstance(kq, KeyQuantConfig):
        return kq
    return KeyQuantConfig(kq.d, kq.group_size, kq.n_levels, kq.rounds)


def _a(x, dt):
    return np.ascontiguousarray(x, dt)


def _ptr(x):
    return None if x is None else x.ctypes.data_as(_p)


class Context:
    """cvq_context: one device, one CUDA stream (cudaStream_t or None = a
    private stream).  Wrappers given CUDA torch tensors order the context's
    stream after torch's current stream on entry and torch's after the
    context's on return (no-op when they are the same stream)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = _p()
        _check(_lib.cvq_context_create(_i(device), _p(stream) if stream else None, C.byref(h)))
        self.h = h
        sp = _p()
        _check(_lib.cvq_context_stream(h, C.byref(sp)))
        self.stream_ptr = sp.value or 0

    def close(self):
        if getattr(self, "h", None):
            _lib.cvq_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(_lib.cvq_context_synchronize(self.h))


class _TorchOrder:
    """Stream ordering between torch's current stream and a context's stream
    around one library call on CUDA tensors (the library queues
    work on the context stream; torch writes inputs / reads outputs on its
    current stream)."""

    def __init__(self, ctx, *xs):
        self.ctx, self.xs, self.ext = ctx, xs, None

    def __enter__(self):
        if any(getattr(x, "is_cuda", False) for x in self.xs):
            import torch
            cur = torch.cuda.current_stream()
            if cur.cuda_stream != self.ctx.stream_ptr:
                self.cur = cur
                self.ext = torch.cuda.ExternalStream(self.ctx.stream_ptr)
                self.ext.wait_stream(cur)
        return self

    def __exit__(self, *exc):
        if self.ext is not None:
            self.cur.wait_stream(self.ext)
        return False


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# --------------------------------------------------------------- mirrors
def predicted_flops_fused(n, d, n_codes, rounds, n_levels):
    _lib.cvq_predicted_flops_fused.restype = _u64
    v = _lib.cvq_predicted_flops_fused(_u64(n), _u64(d), _u64(n_codes), _u64(rounds),
                                       _u64(n_levels))
    if v == 0:
        raise ValueError(_lib.cvq_last_error().decode())
    return int(v)


def predicted_flops_naive(n, d, n_codes):
    _lib.cvq_predicted_flops_naive.restype = _u64
    v = _lib.cvq_predicted_flops_naive(_u64(n), _u64(d), _u64(n_codes))
    if v == 0:
        raise ValueError(_lib.cvq_last_error().decode())
    return int(v)


def _attn(fn, kq, atoms, a, b, bits, vrows, q, t, base, ctx, want_scores=False):
    kq = _kc(kq)
    ctx = ctx or default_context()
    atoms = _a(atoms, np.float64)
    a = _a(a, np.uint16)
    b = _a(b, np.uint16)
    bits = _a(bits, np.uint8)
    vrows = _a(vrows, np.float64)
    q = _a(q, np.float64)
    n_codes = vrows.shape[0]
    n = bits.size // n_codes if n_codes else 0
    out = np.zeros(kq.d)
    fl = _Flops()
    kc = kq._c()
    scores = np.zeros(max(n, 1)) if want_scores else None
    if fn == "fused":
        rc = _lib.cvq_fused_attention(ctx.h, C.byref(kc), _u32(n_codes), _ptr(atoms), _ptr(a),
                                      _ptr(b), _u64(n), _ptr(bits), _ptr(vrows), _ptr(q),
                                      _u64(t), _d(base), _ptr(out), _ptr(scores), C.byref(fl))
    else:
        rc = _lib.cvq_naive_attention(ctx.h, C.byref(kc), _u32(n_codes), _ptr(atoms), _ptr(a),
                                      _ptr(b), _u64(n), _ptr(bits), _ptr(vrows), _ptr(q),
                                      _u64(t), _d(base), _ptr(out), C.byref(fl))
    _check(rc)
    rep = FlopReport(fn, n, kq.d, n_codes, kq.rounds, kq.n_levels, fl.predicted_mults,
                     fl.measured_mults)
    if want_scores:
        return out, rep, scores[:n]
    return out, rep


def fused_attention(kq, atoms, a, b, bits, vrows, q, t, base=10000.0, ctx=None,
                    return_scores=False):
    """attn.cpp:164-263 on the B200 -> (out[d], FlopReport[, scores])."""
    return _attn("fused", kq, atoms, a, b, bits, vrows, q, t, base, ctx, return_scores)


def naive_attention(kq, atoms, a, b, bits, vrows, q, t, base=10000.0, ctx=None):
    """attn.cpp:130-162 on the B200 -> (out[d], FlopReport)."""
    return _attn("naive", kq, atoms, a, b, bits, vrows, q, t, base, ctx)


def encode_keys(kq, atoms, keys, ctx=None, search="brute_force"):
    """keyquant.cpp:705-739 with the reference's AssignSearch ("brute_force"
    or "factorized", each bit-exact to the reference's own search) -> (a, b)
    uint16 in KeyCodes::idx order."""
    if search not in ("brute_force", "factorized"):
        raise ValueError("encode_keys: unknown search")
    kq = _kc(kq)
    ctx = ctx or default_context()
    atoms = _a(atoms, np.float64)
    keys = _a(keys, np.float64)
    if keys.ndim != 2 or keys.shape[1] != kq.d:
        raise ValueError("encode_keys: keys width != d")
    n = keys.shape[0]
    m = n * kq.rounds * kq.groups
    a = np.zeros(max(m, 1), np.uint16)
    b = np.zeros(max(m, 1), np.uint16)
    kc = kq._c()
    _check(_lib.cvq_encode_keys_search(ctx.h, C.byref(kc), _ptr(atoms), _ptr(keys), _u64(n),
                                       C.c_int32(1 if search == "factorized" else 0), _ptr(a),
                                       _ptr(b)))
    return a[:m], b[:m]


def decode_keys(kq, atoms, a, b, ctx=None):
    """keyquant.cpp:741-768: dense keys [n][d] from codes (bit-identical)."""
    kq = _kc(kq)
    ctx = ctx or default_context()
    atoms = _a(atoms, np.float64)
    a = _a(a, np.uint16).reshape(-1)
    b = _a(b, np.uint16).reshape(-1)
    per = kq.rounds * kq.groups
    if a.size != b.size or a.size % per:
        raise ValueError("decode_keys: codes do not match codebook")
    n = a.size // per
    out = np.zeros((max(n, 1), kq.d))
    kc = kq._c()
    _check(_lib.cvq_decode_keys(ctx.h, C.byref(kc), _ptr(atoms), _ptr(a), _ptr(b), _u64(n),
                                _ptr(out)))
    return out[:n]


def decode_values(rows, bits, ctx=None):
    """valquant.cpp:115-128: dense values [n][d] = sum of the codebook rows
    whose bit is set (bit-identical).  rows [n_codes][d], bits [n][n_codes]."""
    ctx = ctx or default_context()
    rows = _a(rows, np.float64)
    bits = _a(bits, np.uint8)
    if rows.ndim != 2 or bits.ndim != 2 or bits.shape[1] != rows.shape[0]:
        raise ValueError("decode_values: codes do not match codebook")
    n = bits.shape[0]
    out = np.zeros((max(n, 1), rows.shape[1]))
    _check(_lib.cvq_decode_values(ctx.h, _u32(rows.shape[0]), _u32(rows.shape[1]), _ptr(rows),
                                  _ptr(bits), _u64(n), _ptr(out)))
    return out[:n]


class _Em(C.Structure):
    _fields_ = [("soft_iters", _u64), ("hard_iters_max", _u64), ("t0", _d), ("decay", _d),
                ("tol", _d), ("ridge", _d), ("seed", _u64), ("search", C.c_int32)]


@dataclass
class EmConfig:
    """keyquant.hpp:71-80 (search: "brute_force" | "factorized")."""

    soft_iters: int = 30
    hard_iters_max: int = 100
    t0: float = 0.0
    decay: float = 0.9
    tol: float = 1e-6
    ridge: float = -1.0
    seed: int = 1
    search: str = "brute_force"

    def _c(self):
        if self.search not in ("brute_force", "factorized"):
            raise ValueError("EmConfig: unknown search")
        return _Em(self.soft_iters, self.hard_iters_max, self.t0, self.decay, self.tol,
                   self.ridge, self.seed, 1 if self.search == "factorized" else 0)


def train_key_codebook(calib, kq, em=None, ctx=None):
    """train_key_codebook (keyquant.cpp:641-703) on the B200.

    Returns (atoms [R*(d/2)*L*2] fp64 in CVQK order, report) where report has
    "hard_objective" [R][groups] -> list and "reconstruction_mse" [R]."""
    kq = _kc(kq)
    em = em or EmConfig()
    ctx = ctx or default_context()
    calib = _a(calib, np.float64)
    if calib.ndim != 2 or calib.shape[1] != kq.d:
        raise ValueError("train_key_codebook: calib width != d")
    n = calib.shape[0]
    atoms = np.zeros(2 * kq.n_atoms, np.float64)
    ng = kq.rounds * kq.groups
    cap = ng * (em.hard_iters_max + 2)
    obj = np.zeros(max(cap, 1), np.float64)
    olen = np.zeros(ng, np.uint64)
    mse = np.zeros(kq.rounds, np.float64)
    kc, ec = kq._c(), em._c()
    _check(_lib.cvq_train_key_codebook(ctx.h, C.byref(kc), _ptr(calib), _u64(n), C.byref(ec),
                                       _ptr(atoms), _ptr(obj), _u64(cap), _ptr(olen), _ptr(mse)))
    traces, k = [], 0
    for r in range(kq.rounds):
        row = []
        for grp in range(kq.groups):
            ln = int(olen[r * kq.groups + grp])
            row.append(obj[k:k + ln].copy())
            k += ln
        traces.append(row)
    return atoms, {"hard_objective": traces, "reconstruction_mse": mse}


class _ValCfg(C.Structure):
    _fields_ = [("steps", _u64), ("batch", _u64), ("step_size", _d), ("gumbel_t_start", _d),
                ("gumbel_t_end", _d), ("hidden", _u64), ("seed", _u64),
                ("checkpoint_every", _u64), ("freeze_codebook", C.c_int32)]


@dataclass
class ValTrainConfig:
    """valquant.hpp:76-86."""

    steps: int = 10000
    batch: int = 256
    step_size: float = 1e-3
    gumbel_t_start: float = 1.0
    gumbel_t_end: float = 0.1
    hidden: int = 0
    seed: int = 1
    checkpoint_every: int = 100
    freeze_codebook: bool = False

    def _c(self):
        return _ValCfg(self.steps, self.batch, self.step_size, self.gumbel_t_start,
                       self.gumbel_t_end, self.hidden, self.seed, self.checkpoint_every,
                       int(self.freeze_codebook))


def train_value_quantizer(calib, n_codes, cfg=None, init_codebook=None, ctx=None):
    """train_value_quantizer (valquant.cpp:172-383) on the B200 -> dict with
    w1 [d][H], b1, w2 [H][n_codes], b2, codebook [n_codes][d], loss_curve,
    diverged, steps_run (ValueTrainResult, valquant.hpp:88-94)."""
    cfg = cfg or ValTrainConfig()
    ctx = ctx or default_context()
    calib = _a(calib, np.float64)
    if calib.ndim != 2:
        raise ValueError("train_value_quantizer: calib must be 2-D")
    n, d = calib.shape
    H = cfg.hidden or 2 * n_codes
    out = {"w1": np.zeros((d, H)), "b1": np.zeros(H), "w2": np.zeros((H, n_codes)),
           "b2": np.zeros(n_codes), "codebook": np.zeros((n_codes, d))}
    curve = np.zeros(max(cfg.steps, 1))
    clen, sr = _u64(0), _u64(0)
    dv = C.c_int32(0)
    init = None if init_codebook is None else _a(init_codebook, np.float64)
    c = cfg._c()
    _check(_lib.cvq_train_value_quantizer(
        ctx.h, _ptr(calib) if n else None, _u64(n), _u32(d), _u32(n_codes), C.byref(c),
        _ptr(init) if init is not None else None, _ptr(out["w1"]), _ptr(out["b1"]),
        _ptr(out["w2"]), _ptr(out["b2"]), _ptr(out["codebook"]), _ptr(curve), C.byref(clen),
        C.byref(dv), C.byref(sr)))
    out["loss_curve"] = curve[:clen.value].copy()
    out["diverged"] = bool(dv.value)
    out["steps_run"] = int(sr.value)
    return out


def encoder_forward_infer(w1, b1, w2, b2, values, ctx=None):
    """valquant.cpp:50-101, infer mode, batched -> (bits[n][N_c], logits)."""
    ctx = ctx or default_context()
    w1, b1, w2, b2 = (_a(x, np.float64) for x in (w1, b1, w2, b2))
    values = _a(values, np.float64)
    d, hidden = w1.shape
    n_codes = w2.shape[1]
    if values.ndim != 2 or values.shape[1] != d:
        raise ValueError("encoder_forward: input size != d")
    n = values.shape[0]
    bits = np.zeros((max(n, 1), n_codes), np.uint8)
    logits = np.zeros((max(n, 1), n_codes))
    _check(_lib.cvq_encoder_forward_infer(ctx.h, _u32(d), _u32(hidden), _u32(n_codes), _ptr(w1),
                                          _ptr(b1), _ptr(w2), _ptr(b2), _ptr(values), _u64(n),
                                          _ptr(bits), _ptr(logits)))
    return bits[:n], logits[:n]


def _wfb(bits):
    return (bits + 63) // 64


def pack_key_codes(kq, a, b, ctx=None):
    """cache.cpp:90-106."""
    kq = _kc(kq)
    ctx = ctx or default_context()
    a = _a(a, np.uint16)
    b = _a(b, np.uint16)
    n = a.size // (kq.rounds * kq.groups)
    nw = _wfb(n * kq.bits_per_token)
    w = np.zeros(max(nw, 1), np.uint64)
    kc = kq._c()
    _check(_lib.cvq_pack_key_codes(ctx.h, C.byref(kc), _ptr(a), _ptr(b), _u64(n), _ptr(w)))
    return w[:nw]


def unpack_key_codes(kq, words, n, ctx=None):
    """cache.cpp:108-135."""
    kq = _kc(kq)
    ctx = ctx or default_context()
    words = _a(words, np.uint64)
    m = n * kq.rounds * kq.groups
    a = np.zeros(max(m, 1), np.uint16)
    b = np.zeros(max(m, 1), np.uint16)
    kc = kq._c()
    _check(_lib.cvq_unpack_key_codes(ctx.h, C.byref(kc), _ptr(words), _u64(words.size), _u64(n),
                                     _ptr(a), _ptr(b)))
    return a[:m], b[:m]


def pack_value_codes(bits, ctx=None):
    """cache.cpp:137-143; bits [n][n_codes]."""
    ctx = ctx or default_context()
    bits = _a(bits, np.uint8)
    n, n_codes = bits.shape
    nw = _wfb(n * n_codes)
    w = np.zeros(max(nw, 1), np.uint64)
    _check(_lib.cvq_pack_value_codes(ctx.h, _u32(n_codes), _ptr(bits), _u64(n), _ptr(w)))
    return w[:nw]


def unpack_value_codes(n_codes, words, n, ctx=None):
    """cache.cpp:145-155."""
    ctx = ctx or default_context()
    words = _a(words, np.uint64)
    bits = np.zeros((max(n, 1), n_codes), np.uint8)
    _check(_lib.cvq_unpack_value_codes(ctx.h, _u32(n_codes), _ptr(words), _u64(words.size),
                                       _u64(n), _ptr(bits)))
    return bits[:n]


# ------------------------------------------------ device-resident cache
def _buf(x, dtype=None):
    """(pointer, where, keepalive) for a numpy array (host) or torch tensor."""
    if isinstance(x, np.ndarray):
        x = np.ascontiguousarray(x, dtype) if dtype is not None else np.ascontiguousarray(x)
        return x.ctypes.data_as(_p), CVQ_HOST, x
    # torch tensor (duck-typed to avoid importing torch here)
    if not x.is_contiguous():
        raise ValueError("tensor must be contiguous")
    where = CVQ_DEVICE if x.is_cuda else CVQ_HOST
    return _p(x.data_ptr()), where, x


class QuantizedKVCache:
    """QuantizedKVCache (cache.hpp:63-113) for a whole model, resident in HBM.

    One code stream per (seq, layer, kv_head); codebooks per (layer, kv_head);
    each stream serves q_per_kv query heads.  Arrays are numpy (host) or torch
    (host or cuda) tensors.
    """

    def __init__(self, kq, n_codes, n_seqs=1, n_layers=1, n_kv_heads=1, q_per_kv=1,
                 capacity=1024, hidden=0, position_offset=0, rope_base=10000.0, ctx=None,
                 keys_fp16=False, keys="fp32"):
        """keys: on-chip key-codebook mode -- "fp32" (default), "fp16"
        (CVQ_CACHE_KEYS_FP16) or "tc" (tcgen05 one-hot MMA, CVQ_CACHE_KEYS_TC)."""
        self.kq = _kc(kq)
        self.ctx = ctx or default_context()
        self.n_codes, self.hidden = n_codes, hidden
        self.n_seqs, self.n_layers, self.n_kv_heads, self.q_per_kv = (n_seqs, n_layers,
                                                                      n_kv_heads, q_per_kv)
        self.capacity, self.position_offset = capacity, position_offset
        if keys_fp16:
            keys = "fp16"
        self.keys = keys
        flags = {"fp32": 0, "fp16": CVQ_CACHE_KEYS_FP16, "tc": CVQ_CACHE_KEYS_TC}[keys]
        d = _Desc(self.kq._c(), n_codes, hidden, n_seqs, n_layers, n_kv_heads, q_per_kv,
                  capacity, position_offset, rope_base, flags)
        h = _p()
        _check(_lib.cvq_cache_create(self.ctx.h, C.byref(d), C.byref(h)))
        self.h = h

    @property
    def n_streams(self):
        return self.n_seqs * self.n_layers * self.n_kv_heads

    @property
    def n_q_heads(self):
        return self.n_kv_heads * self.q_per_kv

    def close(self):
        if getattr(self, "h", None):
            _lib.cvq_cache_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self):
        n = _u64()
        _check(_lib.cvq_cache_length(self.h, C.byref(n)))
        return n.value

    def set_key_codebook(self, layer, head, atoms):
        atoms = _a(atoms, np.float64)
        if atoms.size != 2 * self.kq.n_atoms:
            raise ValueError("key codebook size mismatch")
        _check(_lib.cvq_cache_set_key_codebook(self.h, _u32(layer), _u32(head), _ptr(atoms)))

    def set_value_quantizer(self, layer, head, rows, w1=None, b1=None, w2=None, b2=None):
        rows = _a(rows, np.float64)
        ws = [None if x is None else _a(x, np.float64) for x in (w1, b1, w2, b2)]
        _check(_lib.cvq_cache_set_value_quantizer(self.h, _u32(layer), _u32(head),
                                                  *[_ptr(x) for x in ws], _ptr(rows)))

    def prefill(self, K, V):
        """K, V: [n_seqs][n_layers][n_kv_heads][n][d] float32/float64."""
        kp, where, kk = _buf(K)
        vp, _, vk = _buf(V)
        dt = CVQ_F64 if str(kk.dtype).endswith("float64") else CVQ_F32
        n = kk.shape[-2]
        with _TorchOrder(self.ctx, kk, vk):
            _check(_lib.cvq_cache_prefill(self.h, kp, vp, _u64(n), _i(dt), _i(where)))

    def append(self, k, v):
        """k, v: [n_seqs][n_layers][n_kv_heads][d] (cache.cpp:256-285).  Does
        not wait for the device: an encoder error surfaces at the next
        synchronising call (synchronize(), size(), host-buffer attention)."""
        kp, where, kk = _buf(k)
        vp, _, vk = _buf(v)
        dt = CVQ_F64 if str(kk.dtype).endswith("float64") else CVQ_F32
        with _TorchOrder(self.ctx, kk, vk):
            _check(_lib.cvq_cache_append(self.h, kp, vp, _i(dt), _i(where)))

    def synchronize(self):
        _check(_lib.cvq_cache_synchronize(self.h))

    def reserve(self, n):
        _check(_lib.cvq_cache_reserve(self.h, _u64(n)))

    def capacity_tokens(self):
        n = _u64()
        _check(_lib.cvq_cache_capacity(self.h, C.byref(n)))
        return n.value

    def set_variant(self, variant=0):
        """CVQ_VARIANT_* bits (or names: "generic", "tc_dense", "tc_pair",
        "fused") -- cross-check / experimental kernels; 0 = defaults."""
        if isinstance(variant, str):
            variant = [variant]
        if not isinstance(variant, int):
            variant = sum(VARIANTS[v] for v in variant)
        _check(_lib.cvq_cache_set_variant(self.h, _u32(variant)))

    def key_mode(self):
        """Effective key-codebook mode: "tc", "fp16" or "fp32" ("tc" caches
        whose codebook fails the fp16 guard report "fp32")."""
        f = _u32()
        _check(_lib.cvq_cache_key_mode(self.h, C.byref(f)))
        return "tc" if f.value & CVQ_CACHE_KEYS_TC else "fp16" if f.value & CVQ_CACHE_KEYS_FP16 else "fp32"

    def attention(self, q, t=None, out=None):
        """q: [n_seqs][n_layers][Hq][d] float32 -> out of the same shape."""
        if t is None:
            t = self.position_offset + self.size() - 1
        qp, where, qk = _buf(q, np.float32)
        if out is None:
            if where == CVQ_HOST:
                out = np.zeros(qk.shape, np.float32)
            else:
                out = qk.new_empty(qk.shape)
        op, _, ok = _buf(out)
        with _TorchOrder(self.ctx, qk, ok):
            _check(_lib.cvq_cache_attention(self.h, qp, _u64(t), op, _i(where)))
        return out

    def attention_naive(self, q, t=None, out=None):
        """Decode-then-attend (attn.cpp:130-162) over the same cache: dense
        fp16 dequantisation of every key / value, then dense attention."""
        if t is None:
            t = self.position_offset + self.size() - 1
        qp, where, qk = _buf(q, np.float32)
        if out is None:
            out = np.zeros(qk.shape, np.float32) if where == CVQ_HOST else qk.new_empty(qk.shape)
        op, _, ok = _buf(out)
        with _TorchOrder(self.ctx, qk, ok):
            _check(_lib.cvq_cache_attention_naive(self.h, qp, _u64(t), op, _i(where)))
        return out

    def attention_partial(self, q, m, l, o, t):
        """Device tensors: m, l [rows], o [rows][d] (split-K partial)."""
        with _TorchOrder(self.ctx, q, m, l, o):
            _check(_lib.cvq_cache_attention_partial(self.h, _p(q.data_ptr()), _u64(t),
                                                    _p(m.data_ptr()), _p(l.data_ptr()),
                                                    _p(o.data_ptr())))

    def decode_step(self, k, v, q, out=None):
        """cache.cpp:287-296: append (k, v) then attend q at the new last position."""
        kp, where, kk = _buf(k)
        vp, _, vk = _buf(v)
        dt = CVQ_F64 if str(kk.dtype).endswith("float64") else CVQ_F32
        qp, _, qk = _buf(q, np.float32)
        if out is None:
            out = np.zeros(qk.shape, np.float32) if where == CVQ_HOST else qk.new_empty(qk.shape)
        op, _, ok = _buf(out)
        with _TorchOrder(self.ctx, kk, vk, qk, ok):
            _check(_lib.cvq_cache_decode_step(self.h, kp, vp, _i(dt), qp, op, _i(where)))
        return out

    def import_stream(self, seq, layer, head, key_words, value_words, n_tokens):
        kw = _a(key_words, np.uint64)
        vw = _a(value_words, np.uint64)
        _check(_lib.cvq_cache_import_stream(self.h, _u32(seq), _u32(layer), _u32(head), _ptr(kw),
                                            _ptr(vw), _u64(n_tokens), _i(CVQ_HOST)))

    def export_stream(self, seq, layer, head):
        n = self.size()
        kw = np.zeros(max(1, _wfb(n * self.kq.bits_per_token)), np.uint64)
        vw = np.zeros(max(1, _wfb(n * self.n_codes)), np.uint64)
        _check(_lib.cvq_cache_export_stream(self.h, _u32(seq), _u32(layer), _u32(head), _ptr(kw),
                                            _ptr(vw), _i(CVQ_HOST)))
        return kw[:_wfb(n * self.kq.bits_per_token)], vw[:_wfb(n * self.n_codes)]

    def pools(self):
        """(key_ptr, key_stride_words, value_ptr, value_stride_words) device pointers."""
        kp, ks, vp, vs = C.POINTER(C.c_uint64)(), _u64(), C.POINTER(C.c_uint64)(), _u64()
        _check(_lib.cvq_cache_pools(self.h, C.byref(kp), C.byref(ks), C.byref(vp), C.byref(vs)))
        return (C.cast(kp, _p).value, ks.value, C.cast(vp, _p).value, vs.value)

    def set_length(self, n):
        _check(_lib.cvq_cache_set_length(self.h, _u64(n)))


class ShardGroup:
    """One rank of a context-sharded cache (cvq_mgpu, mgpu.cu):
    partial on the local shard -> one NCCL all-gather of the packed
    [m | l | o] blocks -> LSE combine, all inside the library.  Every rank
    builds its shard cache (position_offset = its first global token, from
    shard_plan) and calls these collectively.

    unique_id: 128 bytes from ShardGroup.unique_id() on one rank, broadcast
    by the caller (e.g. torch.distributed.broadcast_object_list)."""

    def __init__(self, shard, rank, world, unique_id):
        self.shard = shard
        uid = C.create_string_buffer(bytes(unique_id), 128)
        h = _p()
        _check(_lib.cvq_mgpu_init_rank(shard.h, uid, _i(rank), _i(world), C.byref(h)))
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_lib.cvq_mgpu_unique_id(buf))
        return buf.raw

    def close(self):
        if getattr(self, "h", None):
            _lib.cvq_mgpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self):
        n = _u64()
        _check(_lib.cvq_mgpu_length(self.h, C.byref(n)))
        return n.value

    def attention(self, q, t, out):
        qp, where, qk = _buf(q, np.float32)
        op, _, ok = _buf(out)
        with _TorchOrder(self.shard.ctx, qk, ok):
            _check(_lib.cvq_mgpu_attention(self.h, qp, _u64(t), op, _i(where)))
        return out

    def decode_step(self, k, v, q, out):
        """The last rank appends (k, v); every rank attends q at the new end."""
        kp, where, kk = _buf(k)
        vp, _, vk = _buf(v)
        dt = CVQ_F64 if str(kk.dtype).endswith("float64") else CVQ_F32
        qp, _, qk = _buf(q, np.float32)
        op, _, ok = _buf(out)
        with _TorchOrder(self.shard.ctx, kk, vk, qk, ok):
            _check(_lib.cvq_mgpu_decode_step(self.h, kp, vp, _i(dt), qp, op, _i(where)))
        return out


def lse_combine_packed(parts, rows, d, out, ctx=None):
    """Device tensor parts [P][rows*(d+2)] of packed [m | l | o] blocks ->
    out [rows][d] (cvq_lse_combine_packed)."""
    ctx = ctx or default_context()
    P = parts.shape[0]
    if parts.numel() != P * rows * (d + 2):
        raise ValueError("lse_combine_packed: parts must be [P][rows*(d+2)]")
    with _TorchOrder(ctx, parts, out):
        _check(_lib.cvq_lse_combine_packed(ctx.h, _p(parts.data_ptr()), _u32(P), _u64(rows),
                                           _u32(d), _p(out.data_ptr())))


def lse_combine_ptrs(ptrs_dev, offset, n_parts, rows, d, out, ctx=None):
    """ptrs_dev: device int64 tensor (or raw device address) of n_parts
    pointers to packed [m | l | o] blocks (peer buffers allowed); part p's
    block starts at ptrs[p] + offset floats -> out [rows][d]."""
    ctx = ctx or default_context()
    addr = ptrs_dev if isinstance(ptrs_dev, int) else ptrs_dev.data_ptr()
    with _TorchOrder(ctx, out):
        _check(_lib.cvq_lse_combine_ptrs(ctx.h, _p(addr), _u64(offset), _u32(n_parts), _u64(rows),
                                         _u32(d), _p(out.data_ptr())))


def lse_combine(m, l, o, out, ctx=None):
    """Device tensors m, l [P][rows], o [P][rows][d] -> out [rows][d]."""
    ctx = ctx or default_context()
    P, rows = m.shape
    d = o.shape[-1]
    with _TorchOrder(ctx, m, l, o, out):
        _check(_lib.cvq_lse_combine(ctx.h, _p(m.data_ptr()), _p(l.data_ptr()), _p(o.data_ptr()),
                                    _u32(P), _u64(rows), _u32(d), _p(out.data_ptr())))
