// capi.cu -- host side of the C-ABI (include/cvq.h): contexts, the
// device-resident multi-stream cache, the single-stream mirrors of the
// reference API, argument validation mirroring the reference exceptions.
// Every numeric entry point launches sm_100a kernels; there is no CPU
// fallback.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/cvq.h"
#include <cuda_fp16.h>

#include "cvq_internal.cuh"

namespace cvq {

cudaError_t ensure_dyn_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kernel, dev}];
  if (bytes <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

std::atomic<unsigned long long> g_launches{0};
cudaError_t run_naive_attention(const AttnJob& job, const float* q, float* out, void* scratch,
                                size_t scratch_bytes, cudaStream_t st, bool exact);
size_t naive_scratch_bytes(const AttnJob& job, bool exact);
}  // namespace cvq

using namespace cvq;

namespace {

thread_local std::string g_err;

cvq_status fail(cvq_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CU(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess)                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? CVQ_ENOMEM : CVQ_ECUDA,        \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                \
  } while (0)

#define TRY(x)                      \
  do {                              \
    cvq_status s_ = (x);            \
    if (s_ != CVQ_OK) return s_;    \
  } while (0)

// Device buffer that only grows.
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    // grow geometrically: decode steps add one token at a time
    if (n) bytes = bytes + bytes / 2 > bytes ? bytes + bytes / 2 : bytes;
    n = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// KeyQuantConfig::validate (keyquant.cpp:46-60).
cvq_status validate_kc(const cvq_key_config* kc) {
  if (!kc) return fail(CVQ_EINVAL, "KeyQuantConfig: null");
  if (kc->d == 0 || kc->d % 2 != 0)
    return fail(CVQ_EINVAL, "KeyQuantConfig: d must be positive and even");
  if (kc->group_size == 0) return fail(CVQ_EINVAL, "KeyQuantConfig: group_size must be positive");
  if ((kc->d / 2) % kc->group_size != 0)
    return fail(CVQ_EINVAL, "KeyQuantConfig: group_size must divide d/2 evenly");
  if (kc->n_levels == 0 || (kc->n_levels & (kc->n_levels - 1)) != 0)
    return fail(CVQ_EINVAL, "KeyQuantConfig: n_levels must be a power of two");
  if (kc->n_levels > 65536) return fail(CVQ_EINVAL, "KeyQuantConfig: n_levels too large");
  if (kc->rounds == 0) return fail(CVQ_EINVAL, "KeyQuantConfig: rounds must be positive");
  return CVQ_OK;
}

int ilog2c(uint32_t v) {
  int b = 0;
  while ((1u << b) < v) ++b;
  return b;
}

Geom make_geom(const cvq_key_config* kc, uint32_t n_codes, uint32_t hidden, uint32_t G) {
  Geom g{};
  g.d = (int)kc->d;
  g.subs = g.d / 2;
  g.g = (int)kc->group_size;
  g.groups = g.subs / g.g;
  g.L = (int)kc->n_levels;
  g.lb = ilog2c(kc->n_levels);
  g.R = (int)kc->rounds;
  g.fpt = g.R * g.groups * 2;
  g.bpt = g.fpt * g.lb;
  g.n_codes = (int)n_codes;
  g.hidden = (int)hidden;
  g.G = (int)G;
  return g;
}

uint64_t words_for_bits(uint64_t bits) { return (bits + 63) / 64; }

// Per-stream pool strides (64-bit words) for `capacity` tokens: whole
// 128-token tiles, rounded to 32 B so tiles stay 32-B aligned, plus slack for
// the score kernels' window over-reads.
void pool_strides(const Geom& g, uint64_t capacity, uint64_t* ks, uint64_t* vs) {
  const uint64_t cap128 = (capacity + 127) / 128 * 128;
  *ks = (words_for_bits(cap128 * (uint64_t)g.bpt) + 8 + 3) / 4 * 4;
  *vs = (words_for_bits(cap128 * (uint64_t)g.n_codes) + 4 + 3) / 4 * 4;
}

std::vector<double> make_thetas(int d, double base) {  // rope.cpp:8-25
  std::vector<double> th(d / 2);
  for (int j = 0; j < d / 2; ++j) th[j] = std::pow(base, -2.0 * (double)j / (double)d);
  return th;
}

// fp64 atoms [R][subs][L][2] -> fp32 complex [R][L][subs] (decode layout:
// one row per (round, level) contiguous over subspaces).
std::vector<float> atoms_to_decode_layout(const Geom& g, const double* xy) {
  std::vector<float> out((size_t)g.R * g.L * g.subs * 2);
  for (int r = 0; r < g.R; ++r)
    for (int j = 0; j < g.subs; ++j)
      for (int l = 0; l < g.L; ++l) {
        const size_t src = (((size_t)r * g.subs + j) * g.L + l) * 2;
        const size_t dst = (((size_t)r * g.L + l) * g.subs + j) * 2;
        out[dst] = (float)xy[src];
        out[dst + 1] = (float)xy[src + 1];
      }
  return out;
}

}  // namespace

// ------------------------------------------------------------- structs
struct cvq_mirror;
void destroy_mirror(cvq_mirror* m);  // after its definition (mirrors section)
struct cvq_context {
  cvq_mirror* mirror = nullptr;  // single-stream mirrors' device cache (capi.cu)
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  unsigned long long* d_err = nullptr;  // single-stream encoder failure flag
  DevBuf scratch;
  // live timing of the dominant attention kernel (cvq_context_profile)
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;  // pairs
  size_t prof_used = 0;
  // side stream for the value encoder of an append (the key and value
  // encoders are independent: they overlap, joined before packing)
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaError_t ensure_side() {
    if (side) return cudaSuccess;
    cudaError_t e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    return e;
  }
  cudaEvent_t* next_prof_pair() {
    if (!prof) return nullptr;
    if (2 * (prof_used + 1) > prof_ev.size()) {
      cudaEvent_t a, b;
      if (cudaEventCreate(&a) != cudaSuccess) return nullptr;
      if (cudaEventCreate(&b) != cudaSuccess) return nullptr;
      prof_ev.push_back(a);
      prof_ev.push_back(b);
    }
    return &prof_ev[2 * prof_used++];
  }
};

struct cvq_cache {
  cvq_context* ctx = nullptr;
  cvq_cache_desc desc{};
  Geom geo{};
  int S = 0, n_slots = 0;
  uint64_t kstride = 0, vstride = 0, length = 0;
  uint64_t* kpool = nullptr;
  uint64_t* vpool = nullptr;
  double* atoms64 = nullptr;   // [slot][R][subs][L][2]
  double* base = nullptr;      // [slot][R][groups][L][L] (when it fits)
  float* keyf = nullptr;       // [slot]: fp32 atoms + base (head-preset key encoder)
  double* maxnorm = nullptr;   // [slot][R][groups]
  float2* cbk = nullptr;       // [slot][R][L][subs]
  uint32_t* cbk16 = nullptr;   // same, packed half2 (CVQ_CACHE_KEYS_FP16)
  uint16_t* cbtc = nullptr;    // tcgen05 A operand [slot][R][2][8192] (CVQ_CACHE_KEYS_TC)
  float* cbv = nullptr;        // [slot][n_codes][d]
  double *w1 = nullptr, *b1 = nullptr, *w2 = nullptr, *b2 = nullptr;
  float* w2f = nullptr;   // value-encoder screen tables: fp32 w2 and its fp64
  double* n2 = nullptr;   // column norms (k_encode_values_screen)
  double* thetas = nullptr;
  std::vector<char> key_set, val_set, enc_set;
  DevBuf attn_scratch, enc_scratch, stage_in, stage_out, stage_kv;
  uint32_t variant = 0;                   // CVQ_VARIANT_* kernel selection
  bool tc_demoted = false;                // a key codebook failed the fp16 guard
  unsigned long long* d_errpos = nullptr; // first failed append position (~0 = none)
  unsigned long long* h_errpos = nullptr; // pinned mirror, read at sync points
  void* h_stage = nullptr;                 // pinned [k | v | q] / out staging (small steps)
  size_t h_stage_n = 0;
  bool pending = false;                   // appends not yet checked for errors
};

namespace {

cvq_status ctx_check(cvq_context* ctx) {
  if (!ctx) return fail(CVQ_EINVAL, "null context");
  CU(cudaSetDevice(ctx->device));
  return CVQ_OK;
}

// fp16 guard of the tcgen05 path (fp16 codebook operand, fp32 accumulate):
// the key decode K_j = sum_r U[r,j,a] + i U[r,j,b] is exact in fp32 but each
// atom is rounded once to fp16 (relative 2^-11).  The absolute error of K_j
// grows with kappa = sum_r max_{j,l} |U|, and sharp softmaxes turn it into
// output error.  Measured (tests/test_tc_precision.py): kappa ~ 82 (R = 21,
// atoms N(0, 1)) gives 7.7e-4 relative output error against the 1e-3 bar, so
// codebooks beyond kappa = 96, or with an atom outside the fp16 range, demote
// the cache to the fp32-codebook CUDA-core kernels (exact to ~1e-6).
constexpr double kTcKappaMax = 96.0;
bool tc_codebook_ok(const Geom& g, const double* xy) {
  double kappa = 0.0;
  for (int r = 0; r < g.R; ++r) {
    double mx = 0.0;
    const size_t n = (size_t)g.subs * g.L * 2;
    for (size_t i = 0; i < n; ++i) mx = std::max(mx, std::fabs(xy[(size_t)r * n + i]));
    if (mx > 60000.0) return false;
    kappa += mx;
  }
  return kappa <= kTcKappaMax;
}

// Grows the packed pools so `need` tokens fit (amortised: x1.5, whole
// 128-token tiles).  The reference cache grows without bound on append
// (cache.cpp:256-285); pool pointers from cvq_cache_pools are invalidated.
cvq_status ensure_capacity(cvq_cache* c, uint64_t need) {
  if (need <= c->desc.capacity) return CVQ_OK;
  uint64_t cap = std::max<uint64_t>(need, c->desc.capacity + c->desc.capacity / 2);
  cap = (cap + 127) / 128 * 128;
  uint64_t ks = 0, vs = 0;
  pool_strides(c->geo, cap, &ks, &vs);
  cudaStream_t st = c->ctx->stream;
  uint64_t *kp = nullptr, *vp = nullptr;
  cudaError_t e = cudaMalloc(&kp, (size_t)c->S * ks * 8);
  if (e == cudaSuccess) e = cudaMalloc(&vp, (size_t)c->S * vs * 8);
  if (e == cudaSuccess) e = cudaMemsetAsync(kp, 0, (size_t)c->S * ks * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(vp, 0, (size_t)c->S * vs * 8, st);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(kp, ks * 8, c->kpool, c->kstride * 8, c->kstride * 8, c->S,
                          cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(vp, vs * 8, c->vpool, c->vstride * 8, c->vstride * 8, c->S,
                          cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    if (kp) cudaFree(kp);
    if (vp) cudaFree(vp);
    return fail(e == cudaErrorMemoryAllocation ? CVQ_ENOMEM : CVQ_ECUDA,
                std::string("cache grow: ") + cudaGetErrorString(e));
  }
  cudaFree(c->kpool);
  cudaFree(c->vpool);
  c->kpool = kp;
  c->vpool = vp;
  c->kstride = ks;
  c->vstride = vs;
  c->desc.capacity = cap;
  return CVQ_OK;
}

// Appends run without a host round trip: the value encoder records the first
// failed append position on the device (d_errpos) and the pack kernels skip
// that batch and every later one.  At the next synchronising call the error
// surfaces as CVQ_ETRAINING and the length rolls back to the failed append,
// as if it had thrown (valquant.cpp:86-87, cache.cpp:256-285).
cvq_status take_errors(cvq_cache* c) {
  if (!c->pending) return CVQ_OK;
  c->pending = false;
  const unsigned long long pos = *c->h_errpos;
  if (pos == ~0ull) return CVQ_OK;
  if (pos < c->length) c->length = pos;
  CU(cudaMemsetAsync(c->d_errpos, 0xFF, sizeof(unsigned long long), c->ctx->stream));
  return fail(CVQ_ETRAINING, "encoder_forward: non-finite activations");
}
cvq_status enqueue_error_read(cvq_cache* c) {
  if (c->pending)
    CU(cudaMemcpyAsync(c->h_errpos, c->d_errpos, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, c->ctx->stream));
  return CVQ_OK;
}
cvq_status sync_check(cvq_cache* c) {
  TRY(enqueue_error_read(c));
  CU(cudaStreamSynchronize(c->ctx->stream));
  return take_errors(c);
}

void free_cache(cvq_cache* c) {
  for (void* p : {(void*)c->kpool, (void*)c->vpool, (void*)c->atoms64, (void*)c->base, (void*)c->keyf,
                  (void*)c->maxnorm, (void*)c->cbk, (void*)c->cbk16, (void*)c->cbtc, (void*)c->cbv, (void*)c->w1, (void*)c->b1,
                  (void*)c->w2, (void*)c->b2, (void*)c->thetas, (void*)c->w2f, (void*)c->n2})
    if (p) cudaFree(p);
  c->attn_scratch.release();
  c->enc_scratch.release();
  c->stage_in.release();
  c->stage_out.release();
  c->stage_kv.release();
  if (c->d_errpos) cudaFree(c->d_errpos);
  if (c->h_errpos) cudaFreeHost(c->h_errpos);
  if (c->h_stage) cudaFreeHost(c->h_stage);
}

AttnJob make_job(const cvq_cache* c) {
  AttnJob j{};
  j.geo = c->geo;
  j.S = c->S;
  j.kpool = c->kpool;
  j.kstride = c->kstride;
  j.vpool = c->vpool;
  j.vstride = c->vstride;
  j.n_slots = c->n_slots;
  j.cb_key = c->cbk;
  j.cb_key16 = c->cbk16;
  j.cb_key_tc = c->tc_demoted ? nullptr : c->cbtc;  // demoted: fp32 CUDA-core path
  j.variant = c->variant;
  j.cb_val = c->cbv;
  j.thetas = c->thetas;
  j.n = (long long)c->length;
  j.pos0 = (long long)c->desc.position_offset;
  j.t = 0;
  return j;
}

cvq_status require_codebooks(const cvq_cache* c, bool keys, bool vrows, bool enc) {
  for (int s = 0; s < c->n_slots; ++s) {
    if (keys && !c->key_set[s]) return fail(CVQ_EINVAL, "cache: key codebook not set for a slot");
    if (vrows && !c->val_set[s]) return fail(CVQ_EINVAL, "cache: value codebook not set for a slot");
    if (enc && !c->enc_set[s]) return fail(CVQ_EINVAL, "cache: value encoder not set for a slot");
  }
  return CVQ_OK;
}

// Bring a caller buffer onto the device (staging copy when on host).
cvq_status to_device(cvq_cache* c, DevBuf& buf, const void* p, size_t bytes, int where,
                     const void** dev) {
  if (where == CVQ_DEVICE) {
    *dev = p;
    return CVQ_OK;
  }
  CU(buf.ensure(bytes));
  CU(cudaMemcpyAsync(buf.p, p, bytes, cudaMemcpyHostToDevice, c->ctx->stream));
  *dev = buf.p;
  return CVQ_OK;
}

}  // namespace

namespace cvq {
cvq_status set_error(cvq_status s, const std::string& msg) { return fail(s, msg); }
}  // namespace cvq

// ================================================================ general
CVQ_API const char* cvq_last_error(void) { return g_err.c_str(); }
CVQ_API int cvq_abi_version(void) { return 1; }
CVQ_API uint64_t cvq_launch_count(void) { return g_launches.load(); }

CVQ_API cvq_status cvq_context_create(int device, void* stream, cvq_context** out) {
  if (!out) return fail(CVQ_EINVAL, "null out");
  int n = 0;
  CU(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(CVQ_EINVAL, "context: bad device index");
  CU(cudaSetDevice(device));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(CVQ_ECUDA, std::string("context: sm_100a kernels need a Blackwell B200, got ") +
                               prop.name);
  cvq_context* c = new cvq_context;
  c->device = device;
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      return fail(CVQ_ECUDA, cudaGetErrorString(e));
    }
    c->own_stream = true;
  }
  cudaError_t e = cudaMalloc(&c->d_err, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    delete c;
    return fail(CVQ_ECUDA, cudaGetErrorString(e));
  }
  *out = c;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_context_profile(cvq_context* ctx, int enable) {
  TRY(ctx_check(ctx));
  ctx->prof = enable != 0;
  ctx->prof_used = 0;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_context_profile_read(cvq_context* ctx, double* ms, uint64_t* launches) {
  TRY(ctx_check(ctx));
  if (!ms || !launches) return fail(CVQ_EINVAL, "null argument");
  CU(cudaStreamSynchronize(ctx->stream));
  double tot = 0.0;
  for (size_t i = 0; i < ctx->prof_used; ++i) {
    float v = 0.f;
    CU(cudaEventElapsedTime(&v, ctx->prof_ev[2 * i], ctx->prof_ev[2 * i + 1]));
    tot += v;
  }
  *ms = tot;
  *launches = ctx->prof_used;
  ctx->prof_used = 0;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_context_destroy(cvq_context* ctx) {
  if (!ctx) return CVQ_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (cudaEvent_t e : ctx->prof_ev) cudaEventDestroy(e);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
    cudaEventDestroy(ctx->fork);
    cudaEventDestroy(ctx->join);
  }
  destroy_mirror(ctx->mirror);
  ctx->scratch.release();
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_context_stream(cvq_context* ctx, void** stream) {
  if (!ctx || !stream) return fail(CVQ_EINVAL, "null argument");
  *stream = ctx->stream;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_context_synchronize(cvq_context* ctx) {
  TRY(ctx_check(ctx));
  CU(cudaStreamSynchronize(ctx->stream));
  return CVQ_OK;
}

CVQ_API uint64_t cvq_predicted_flops_fused(uint64_t n, uint64_t d, uint64_t nc, uint64_t R,
                                           uint64_t L) {
  if (n == 0 || d == 0 || nc == 0 || R == 0 || L == 0) {
    g_err = "predicted_flops_fused: inputs must be > 0";
    return 0;
  }
  return (R * d + nc + 1) * n + d * (nc + R * L);  // attn.cpp:272-280
}

CVQ_API uint64_t cvq_predicted_flops_naive(uint64_t n, uint64_t d, uint64_t nc) {
  if (n == 0 || d == 0 || nc == 0) {
    g_err = "predicted_flops_naive: inputs must be > 0";
    return 0;
  }
  return (2 * d + 1) * n + 2 * d * nc * n;  // attn.cpp:265-270
}

CVQ_API uint32_t cvq_bits_per_token(const cvq_key_config* kc) {
  if (validate_kc(kc) != CVQ_OK) return 0;
  return kc->rounds * ((kc->d / 2) / kc->group_size) * 2 * (uint32_t)ilog2c(kc->n_levels);
}

// ================================================================== cache
CVQ_API cvq_status cvq_cache_create(cvq_context* ctx, const cvq_cache_desc* d, cvq_cache** out) {
  TRY(ctx_check(ctx));
  if (!d || !out) return fail(CVQ_EINVAL, "null argument");
  TRY(validate_kc(&d->key));
  if (d->n_codes == 0) return fail(CVQ_EINVAL, "ValueCodebook: zero dimension");
  if (d->n_seqs == 0 || d->n_layers == 0 || d->n_kv_heads == 0 || d->q_per_kv == 0)
    return fail(CVQ_EINVAL, "cache: empty shape");
  if (d->q_per_kv > 8) return fail(CVQ_EINVAL, "cache: q_per_kv > 8 unsupported");
  if (d->n_codes > 1024) return fail(CVQ_EINVAL, "cache: n_codes > 1024 unsupported");
  if (!(d->rope_base > 0.0)) return fail(CVQ_EINVAL, "theta: base must be positive");
  cvq_cache* c = new cvq_cache;
  c->ctx = ctx;
  c->desc = *d;
  c->geo = make_geom(&d->key, d->n_codes, d->hidden, d->q_per_kv);
  c->S = (int)(d->n_seqs * d->n_layers * d->n_kv_heads);
  c->n_slots = (int)(d->n_layers * d->n_kv_heads);
  const Geom& g = c->geo;
  pool_strides(g, d->capacity, &c->kstride, &c->vstride);
  c->key_set.assign(c->n_slots, 0);
  c->val_set.assign(c->n_slots, 0);
  c->enc_set.assign(c->n_slots, 0);
  const size_t na = (size_t)c->n_slots * g.R * g.subs * g.L;
  auto alloc = [&](void** p, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(*p, 0, bytes ? bytes : 8, ctx->stream);
    return e;
  };
  cudaError_t e = cudaMalloc(&c->d_errpos, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemsetAsync(c->d_errpos, 0xFF, sizeof(unsigned long long), ctx->stream);
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_errpos, sizeof(unsigned long long));
  if (e == cudaSuccess) e = alloc((void**)&c->kpool, (size_t)c->S * c->kstride * 8);
  if (e == cudaSuccess) e = alloc((void**)&c->vpool, (size_t)c->S * c->vstride * 8);
  if (e == cudaSuccess) e = alloc((void**)&c->atoms64, na * 2 * sizeof(double));
  if (e == cudaSuccess) e = alloc((void**)&c->cbk, na * sizeof(float2));
  if (e == cudaSuccess && (d->flags & CVQ_CACHE_KEYS_FP16))
    e = alloc((void**)&c->cbk16, na * sizeof(uint32_t));
  // tcgen05 path: head presets only (d=128, one 64-subspace group, L=64,
  // G in {1, 4} query heads per KV head)
  const bool tc_ok = g.d == 128 && g.groups == 1 && g.L == 64 && (g.G == 4 || g.G == 1);
  if (e == cudaSuccess && (d->flags & CVQ_CACHE_KEYS_TC) && tc_ok)
    e = alloc((void**)&c->cbtc, (size_t)c->n_slots * tc_codebook_elems(g.R) * sizeof(uint16_t));
  if (e == cudaSuccess) e = alloc((void**)&c->cbv, (size_t)c->n_slots * g.n_codes * g.d * 4);
  if (e == cudaSuccess)
    e = alloc((void**)&c->maxnorm, (size_t)c->n_slots * g.R * g.groups * sizeof(double));
  if (e == cudaSuccess && key_tables_fit(g))
    e = alloc((void**)&c->base, (size_t)c->n_slots * g.R * g.groups * g.L * g.L * sizeof(double));
  if (e == cudaSuccess && key_tables_fit(g) && key_t64_applies(g))
    e = alloc((void**)&c->keyf, (size_t)c->n_slots * key_t64_table_floats(g) * sizeof(float));
  if (e == cudaSuccess && d->hidden > 0) {
    e = alloc((void**)&c->w1, (size_t)c->n_slots * g.d * g.hidden * 8);
    if (e == cudaSuccess) e = alloc((void**)&c->b1, (size_t)c->n_slots * g.hidden * 8);
    if (e == cudaSuccess) e = alloc((void**)&c->w2, (size_t)c->n_slots * g.hidden * g.n_codes * 8);
    if (e == cudaSuccess) e = alloc((void**)&c->b2, (size_t)c->n_slots * g.n_codes * 8);
    if (e == cudaSuccess) e = alloc((void**)&c->w2f, (size_t)c->n_slots * g.hidden * g.n_codes * 4);
    if (e == cudaSuccess) e = alloc((void**)&c->n2, (size_t)c->n_slots * g.n_codes * 8);
  }
  if (e == cudaSuccess) {
    std::vector<double> th = make_thetas(g.d, d->rope_base);
    e = alloc((void**)&c->thetas, th.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(c->thetas, th.data(), th.size() * sizeof(double),
                          cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  }
  if (e != cudaSuccess) {
    free_cache(c);
    delete c;
    return fail(e == cudaErrorMemoryAllocation ? CVQ_ENOMEM : CVQ_ECUDA,
                std::string("cache_create: ") + cudaGetErrorString(e));
  }
  *out = c;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_destroy(cvq_cache* c) {
  if (!c) return CVQ_OK;
  cudaSetDevice(c->ctx->device);
  cudaStreamSynchronize(c->ctx->stream);
  free_cache(c);
  delete c;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_length(const cvq_cache* c, uint64_t* n) {
  if (!c || !n) return fail(CVQ_EINVAL, "null argument");
  if (c->pending) {  // surface deferred append errors (and their rollback)
    TRY(ctx_check(c->ctx));
    TRY(sync_check(const_cast<cvq_cache*>(c)));
  }
  *n = c->length;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_set_key_codebook(cvq_cache* c, uint32_t layer, uint32_t head,
                                              const double* xy) {
  if (!c || !xy) return fail(CVQ_EINVAL, "null argument");
  TRY(ctx_check(c->ctx));
  if (layer >= c->desc.n_layers || head >= c->desc.n_kv_heads)
    return fail(CVQ_EINVAL, "cache: slot out of range");
  const Geom& g = c->geo;
  const size_t na = (size_t)g.R * g.subs * g.L;
  for (size_t i = 0; i < 2 * na; ++i)
    if (!std::isfinite(xy[i])) return fail(CVQ_EINVAL, "comm_mat: entries must be finite");
  const int slot = (int)(layer * c->desc.n_kv_heads + head);
  cudaStream_t st = c->ctx->stream;
  CU(cudaMemcpyAsync(c->atoms64 + (size_t)slot * na * 2, xy, na * 2 * sizeof(double),
                     cudaMemcpyHostToDevice, st));
  std::vector<float> dl = atoms_to_decode_layout(g, xy);
  CU(cudaMemcpyAsync(c->cbk + (size_t)slot * na, dl.data(), dl.size() * sizeof(float),
                     cudaMemcpyHostToDevice, st));
  std::vector<uint32_t> dh;
  if (c->cbk16) {  // fp16 copy, rounded once from fp64
    dh.resize(na);
    for (int r = 0; r < g.R; ++r)
      for (int jj = 0; jj < g.subs; ++jj)
        for (int l = 0; l < g.L; ++l) {
          const size_t src = (((size_t)r * g.subs + jj) * g.L + l) * 2;
          const size_t dst = ((size_t)r * g.L + l) * g.subs + jj;
          const uint32_t hx = __half_as_ushort(__double2half(xy[src]));
          const uint32_t hy = __half_as_ushort(__double2half(xy[src + 1]));
          dh[dst] = hx | (hy << 16);
        }
    CU(cudaMemcpyAsync(c->cbk16 + (size_t)slot * na, dh.data(), na * 4, cudaMemcpyHostToDevice,
                       st));
  }
  std::vector<uint16_t> dt;
  if (c->cbtc && !tc_codebook_ok(g, xy)) c->tc_demoted = true;
  if (c->cbtc) {  // canonical K-major A operand of the one-hot MMA
    dt.assign(tc_codebook_elems(g.R), 0);
    tc_build_codebook(g.R, xy, dt.data(),
                      [](double v) -> uint16_t { return __half_as_ushort(__double2half(v)); });
    CU(cudaMemcpyAsync(c->cbtc + (size_t)slot * dt.size(), dt.data(), dt.size() * 2,
                       cudaMemcpyHostToDevice, st));
  }
  if (c->base) {
    float* af = c->keyf ? c->keyf + (size_t)slot * g.R * g.subs * g.L * 2 : nullptr;
    float* bf = c->keyf ? c->keyf + (size_t)c->n_slots * g.R * g.subs * g.L * 2 +
                              (size_t)slot * g.R * g.groups * g.L * g.L
                        : nullptr;
    CU(build_key_enc_tables(g, 1, c->atoms64 + (size_t)slot * na * 2,
                            c->base + (size_t)slot * g.R * g.groups * g.L * g.L,
                            c->maxnorm + (size_t)slot * g.R * g.groups, st, af, bf));
  }
  CU(cudaStreamSynchronize(st));  // host vector dl must outlive the copy
  c->key_set[slot] = 1;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_set_value_quantizer(cvq_cache* c, uint32_t layer, uint32_t head,
                                                 const double* w1, const double* b1,
                                                 const double* w2, const double* b2,
                                                 const double* rows) {
  if (!c || !rows) return fail(CVQ_EINVAL, "null argument");
  TRY(ctx_check(c->ctx));
  if (layer >= c->desc.n_layers || head >= c->desc.n_kv_heads)
    return fail(CVQ_EINVAL, "cache: slot out of range");
  const Geom& g = c->geo;
  const int slot = (int)(layer * c->desc.n_kv_heads + head);
  cudaStream_t st = c->ctx->stream;
  std::vector<float> rf((size_t)g.n_codes * g.d);
  for (size_t i = 0; i < rf.size(); ++i) rf[i] = (float)rows[i];
  CU(cudaMemcpyAsync(c->cbv + (size_t)slot * rf.size(), rf.data(), rf.size() * 4,
                     cudaMemcpyHostToDevice, st));
  const bool have_enc = w1 && b1 && w2 && b2;
  if (have_enc) {
    if (g.hidden == 0) return fail(CVQ_EINVAL, "cache: created with hidden = 0");
    CU(cudaMemcpyAsync(c->w1 + (size_t)slot * g.d * g.hidden, w1, (size_t)g.d * g.hidden * 8,
                       cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(c->b1 + (size_t)slot * g.hidden, b1, (size_t)g.hidden * 8,
                       cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(c->w2 + (size_t)slot * g.hidden * g.n_codes, w2,
                       (size_t)g.hidden * g.n_codes * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(c->b2 + (size_t)slot * g.n_codes, b2, (size_t)g.n_codes * 8,
                       cudaMemcpyHostToDevice, st));
    // screen tables: fp32 w2 and its fp64 column norms
    std::vector<float> f2((size_t)g.hidden * g.n_codes);
    std::vector<double> m2(g.n_codes, 0.0);
    for (size_t i = 0; i < f2.size(); ++i) {
      f2[i] = (float)w2[i];
      m2[i % g.n_codes] += w2[i] * w2[i];
    }
    for (double& v : m2) v = std::sqrt(v);
    CU(cudaMemcpyAsync(c->w2f + (size_t)slot * f2.size(), f2.data(), f2.size() * 4,
                       cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(c->n2 + (size_t)slot * g.n_codes, m2.data(), g.n_codes * 8,
                       cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));  // the host vectors go out of scope
  }
  CU(cudaStreamSynchronize(st));
  c->val_set[slot] = 1;
  if (have_enc) c->enc_set[slot] = 1;
  return CVQ_OK;
}

namespace {

// Encode + pack n tokens per stream (device K/V, element (s,i,k) at
// s*s_stride + i*d + k), appended at the current length.  err_at: the
// position a failure rolls back to (the start of the enclosing prefill).
cvq_status encode_append(cvq_cache* c, const void* K, const void* V, int dtype,
                         long long s_stride, long long n, uint64_t err_at) {
  const Geom& g = c->geo;
  cudaStream_t st = c->ctx->stream;
  const size_t per_tok = (size_t)c->S * (2 * sizeof(uint16_t) * g.R * g.groups + g.n_codes);
  CU(c->enc_scratch.ensure(per_tok * (size_t)n + 256));
  uint16_t* a = static_cast<uint16_t*>(c->enc_scratch.p);
  uint16_t* b = a + (size_t)c->S * n * g.R * g.groups;
  uint8_t* bits = reinterpret_cast<uint8_t*>(b + (size_t)c->S * n * g.R * g.groups);
  KeyEncTables tab{c->atoms64, c->base, c->maxnorm};
  if (c->keyf) {  // fp32 tables: slot-major atoms, then slot-major base
    tab.atomsf = c->keyf;
    tab.basef = c->keyf + (size_t)c->n_slots * g.R * g.subs * g.L * 2;
  }
  // decode-step appends (a few tokens per stream): the value encoder and
  // its pack run on the context's side stream, overlapping the key encoder
  // (both are latency-bound there); prefill chunks stay on one stream (two
  // large concurrent encoders measured slower)
  cudaStream_t vst = st;
  if (n <= 8) {
    CU(c->ctx->ensure_side());
    vst = c->ctx->side;
    CU(cudaEventRecord(c->ctx->fork, st));
    CU(cudaStreamWaitEvent(vst, c->ctx->fork, 0));
  }
  CU(run_encode_keys(g, c->S, c->n_slots, tab, K, dtype, s_stride, n, a, b, st));
  ValEncWeights w{c->w1, c->b1, c->w2, c->b2, c->w2f, c->n2};
  CU(run_encode_values(g, c->S, c->n_slots, w, V, dtype, s_stride, n, bits, nullptr, c->d_errpos,
                       err_at, vst));
  CU(run_pack_values(g, c->S, bits, n, (long long)c->length, c->vpool, c->vstride, vst,
                     c->d_errpos));
  if (vst != st) {
    CU(cudaEventRecord(c->ctx->join, vst));
    CU(cudaStreamWaitEvent(st, c->ctx->join, 0));  // the key pack reads the error position
  }
  CU(run_pack_keys(g, c->S, a, b, n, (long long)c->length, c->kpool, c->kstride, st, c->d_errpos));
  c->length += (uint64_t)n;
  c->pending = true;
  return CVQ_OK;
}

// QuantizedKVCache::prefill / append: n tokens for every stream; `check`
// synchronises and surfaces encoder errors before returning (prefill); the
// decode-step append leaves that to the step's own sync.
cvq_status append_tokens(cvq_cache* c, const void* K, const void* V, uint64_t n_tokens,
                         int dtype, int where, bool check) {
  if (!c) return fail(CVQ_EINVAL, "null cache");
  TRY(ctx_check(c->ctx));
  if (n_tokens == 0) return CVQ_OK;  // cache.cpp:225
  if (!K || !V) return fail(CVQ_EINVAL, "prefill: null input");
  if (dtype != CVQ_F32 && dtype != CVQ_F64) return fail(CVQ_EINVAL, "prefill: bad dtype");
  TRY(require_codebooks(c, true, true, true));
  TRY(ensure_capacity(c, c->length + n_tokens));
  const Geom& g = c->geo;
  const size_t es = dtype == CVQ_F32 ? 4 : 8;
  const long long s_stride = (long long)n_tokens * g.d;
  const uint64_t err_at = c->length;
  // chunk tokens so scratch stays bounded (~256 MB of inputs per chunk)
  const long long per_tok_bytes = (long long)c->S * g.d * (long long)es * 2;
  long long chunk = (256ll << 20) / (per_tok_bytes > 0 ? per_tok_bytes : 1);
  if (chunk < 1) chunk = 1;
  if (chunk > (long long)n_tokens) chunk = (long long)n_tokens;
  for (long long c0 = 0; c0 < (long long)n_tokens; c0 += chunk) {
    const long long nn = std::min<long long>(chunk, (long long)n_tokens - c0);
    const void* Kd;
    const void* Vd;
    long long stride = s_stride;
    if (where == CVQ_HOST) {
      const size_t row = (size_t)nn * g.d * es;
      if (c0 > 0) CU(cudaStreamSynchronize(c->ctx->stream));  // staging buffer reuse
      CU(c->stage_kv.ensure(2 * row * c->S));
      char* kd = static_cast<char*>(c->stage_kv.p);
      char* vd = kd + row * c->S;
      if (nn == (long long)n_tokens) {  // one contiguous block per tensor
        CU(cudaMemcpyAsync(kd, K, row * c->S, cudaMemcpyHostToDevice, c->ctx->stream));
        CU(cudaMemcpyAsync(vd, V, row * c->S, cudaMemcpyHostToDevice, c->ctx->stream));
      } else {
        CU(cudaMemcpy2DAsync(kd, row, static_cast<const char*>(K) + (size_t)c0 * g.d * es,
                             (size_t)s_stride * es, row, c->S, cudaMemcpyHostToDevice,
                             c->ctx->stream));
        CU(cudaMemcpy2DAsync(vd, row, static_cast<const char*>(V) + (size_t)c0 * g.d * es,
                             (size_t)s_stride * es, row, c->S, cudaMemcpyHostToDevice,
                             c->ctx->stream));
      }
      Kd = kd;
      Vd = vd;
      stride = nn * g.d;
    } else {
      Kd = static_cast<const char*>(K) + (size_t)c0 * g.d * es;
      Vd = static_cast<const char*>(V) + (size_t)c0 * g.d * es;
    }
    TRY(encode_append(c, Kd, Vd, dtype, stride, nn, err_at));
  }
  return check ? sync_check(c) : CVQ_OK;
}

}  // namespace

CVQ_API cvq_status cvq_cache_prefill(cvq_cache* c, const void* K, const void* V,
                                     uint64_t n_tokens, int dtype, int where) {
  return append_tokens(c, K, V, n_tokens, dtype, where, true);
}

CVQ_API cvq_status cvq_cache_append(cvq_cache* c, const void* k, const void* v, int dtype,
                                    int where) {
  // no host round trip: encoder errors surface at the next synchronising
  // call (cvq_cache_synchronize, cvq_cache_length, host-buffer attention)
  return append_tokens(c, k, v, 1, dtype, where, false);
}

namespace {

cvq_status attention_common(cvq_cache* c, const float* q, uint64_t t, float* out, float* m,
                            float* l, float* o, int where, bool naive = false) {
  TRY(ctx_check(c->ctx));
  if (c->length == 0) return fail(CVQ_EINVAL, "attention: empty cache");
  if (t + 1 < c->desc.position_offset + c->length)
    return fail(CVQ_EINVAL, "attention: query position precedes cache");
  TRY(require_codebooks(c, true, true, false));
  const Geom& g = c->geo;
  AttnJob job = make_job(c);
  job.t = (long long)t;
  AttnJob cap = job;  // size scratch for the full capacity once, not per step
  cap.n = (long long)c->desc.capacity;
  if (naive)
    CU(c->attn_scratch.ensure(naive_scratch_bytes(job, false)));
  else
    CU(c->attn_scratch.ensure(std::max(attn_scratch_bytes(job, nullptr),
                                       attn_scratch_bytes(cap, nullptr))));
  const size_t qbytes = (size_t)c->S * g.G * g.d * sizeof(float);
  const void* qd = nullptr;
  TRY(to_device(c, c->stage_in, q, qbytes, where, &qd));
  float* od = out;
  if (out && where == CVQ_HOST) {
    CU(c->stage_out.ensure(qbytes));
    od = static_cast<float*>(c->stage_out.p);
  }
  if (naive)
    CU(run_naive_attention(job, static_cast<const float*>(qd), od, c->attn_scratch.p,
                           c->attn_scratch.n, c->ctx->stream, false));
  else
    CU(run_attention(job, static_cast<const float*>(qd), od, m, l, o, nullptr, c->attn_scratch.p,
                     c->attn_scratch.n, c->ctx->stream, c->ctx->next_prof_pair()));
  if (out && where == CVQ_HOST) {  // the step's one sync also checks the appends
    CU(cudaMemcpyAsync(out, od, qbytes, cudaMemcpyDeviceToHost, c->ctx->stream));
    TRY(enqueue_error_read(c));
    CU(cudaStreamSynchronize(c->ctx->stream));
    return take_errors(c);
  }
  return CVQ_OK;
}

}  // namespace

CVQ_API cvq_status cvq_cache_attention(cvq_cache* c, const float* q, uint64_t t, float* out,
                                       int where) {
  if (!c || !q || !out) return fail(CVQ_EINVAL, "null argument");
  return attention_common(c, q, t, out, nullptr, nullptr, nullptr, where);
}

CVQ_API cvq_status cvq_cache_attention_naive(cvq_cache* c, const float* q, uint64_t t, float* out,
                                             int where) {
  if (!c || !q || !out) return fail(CVQ_EINVAL, "null argument");
  return attention_common(c, q, t, out, nullptr, nullptr, nullptr, where, true);
}

CVQ_API cvq_status cvq_cache_attention_partial(cvq_cache* c, const float* q, uint64_t t, float* m,
                                               float* l, float* o) {
  if (!c || !q || !m || !l || !o) return fail(CVQ_EINVAL, "null argument");
  return attention_common(c, q, t, nullptr, m, l, o, CVQ_DEVICE);
}

CVQ_API cvq_status cvq_lse_combine(cvq_context* ctx, const float* m, const float* l,
                                   const float* o, uint32_t n_parts, uint64_t rows, uint32_t d,
                                   float* out) {
  TRY(ctx_check(ctx));
  if (!m || !l || !o || !out || n_parts == 0) return fail(CVQ_EINVAL, "lse_combine: bad argument");
  CU(run_lse_combine(m, l, o, (int)n_parts, (long long)rows, (int)d, out, nullptr, nullptr,
                     ctx->stream));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_lse_combine_packed(cvq_context* ctx, const float* parts, uint32_t n_parts,
                                          uint64_t rows, uint32_t d, float* out) {
  TRY(ctx_check(ctx));
  if (!parts || !out || n_parts == 0) return fail(CVQ_EINVAL, "lse_combine: bad argument");
  const long long stride = (long long)rows * (d + 2);
  CU(run_lse_combine(parts, parts + rows, parts + 2 * rows, (int)n_parts, (long long)rows, (int)d,
                     out, nullptr, nullptr, ctx->stream, stride));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_lse_combine_ptrs(cvq_context* ctx, const float* const* parts,
                                        uint64_t offset, uint32_t n_parts, uint64_t rows,
                                        uint32_t d, float* out) {
  TRY(ctx_check(ctx));
  if (!parts || !out || n_parts == 0) return fail(CVQ_EINVAL, "lse_combine: bad argument");
  CU(run_lse_combine_ptrs(parts, (long long)offset, (int)n_parts, (long long)rows, (int)d, out,
                          ctx->stream));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_decode_step(cvq_cache* c, const void* k, const void* v, int kv_dtype,
                                         const float* q, float* out, int where) {
  if (!c) return fail(CVQ_EINVAL, "null cache");
  if (where == CVQ_HOST && k && v && q && out && (kv_dtype == CVQ_F32 || kv_dtype == CVQ_F64)) {
    // small steps: one H2D copy of [k | v | q] through pinned staging and one
    // D2H of out instead of three + one (copy latency dominates there)
    const Geom& g = c->geo;
    const size_t es = kv_dtype == CVQ_F32 ? 4 : 8;
    const size_t kvb = (size_t)c->S * g.d * es, qb = (size_t)c->S * g.G * g.d * sizeof(float);
    const size_t qo = (2 * kvb + 15) / 16 * 16, tot = qo + qb;
    if (tot <= (256u << 10)) {
      TRY(ctx_check(c->ctx));
      if (c->h_stage_n < tot) {
        if (c->h_stage) cudaFreeHost(c->h_stage);
        c->h_stage = nullptr;
        c->h_stage_n = 0;
        CU(cudaMallocHost(&c->h_stage, tot));
        c->h_stage_n = tot;
      }
      char* h = static_cast<char*>(c->h_stage);
      CU(cudaStreamSynchronize(c->ctx->stream));  // the previous step's D2H has landed
      std::memcpy(h, k, kvb);
      std::memcpy(h + kvb, v, kvb);
      std::memcpy(h + qo, q, qb);
      CU(c->stage_kv.ensure(tot));
      char* d = static_cast<char*>(c->stage_kv.p);
      CU(cudaMemcpyAsync(d, h, tot, cudaMemcpyHostToDevice, c->ctx->stream));
      TRY(append_tokens(c, d, d + kvb, 1, kv_dtype, CVQ_DEVICE, false));
      const uint64_t t = c->desc.position_offset + c->length - 1;  // cache.cpp:290
      CU(c->stage_out.ensure(qb));
      float* od = static_cast<float*>(c->stage_out.p);
      TRY(attention_common(c, reinterpret_cast<const float*>(d + qo), t, od, nullptr, nullptr,
                           nullptr, CVQ_DEVICE));
      CU(cudaMemcpyAsync(h, od, qb, cudaMemcpyDeviceToHost, c->ctx->stream));
      TRY(enqueue_error_read(c));
      CU(cudaStreamSynchronize(c->ctx->stream));
      TRY(take_errors(c));
      std::memcpy(out, h, qb);
      return CVQ_OK;
    }
  }
  TRY(cvq_cache_append(c, k, v, kv_dtype, where));
  const uint64_t t = c->desc.position_offset + c->length - 1;  // cache.cpp:290
  return cvq_cache_attention(c, q, t, out, where);
}

CVQ_API cvq_status cvq_cache_import_stream(cvq_cache* c, uint32_t seq, uint32_t layer,
                                           uint32_t head, const uint64_t* kw, const uint64_t* vw,
                                           uint64_t n, int where) {
  if (!c || !kw || !vw) return fail(CVQ_EINVAL, "null argument");
  TRY(ctx_check(c->ctx));
  if (seq >= c->desc.n_seqs || layer >= c->desc.n_layers || head >= c->desc.n_kv_heads)
    return fail(CVQ_EINVAL, "cache: stream out of range");
  TRY(ensure_capacity(c, n));
  const Geom& g = c->geo;
  const size_t s = ((size_t)seq * c->desc.n_layers + layer) * c->desc.n_kv_heads + head;
  const uint64_t nk = words_for_bits(n * (uint64_t)g.bpt), nv = words_for_bits(n * (uint64_t)g.n_codes);
  const cudaMemcpyKind kind = where == CVQ_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  cudaStream_t st = c->ctx->stream;
  CU(cudaMemsetAsync(c->kpool + s * c->kstride, 0, c->kstride * 8, st));
  CU(cudaMemsetAsync(c->vpool + s * c->vstride, 0, c->vstride * 8, st));
  CU(cudaMemcpyAsync(c->kpool + s * c->kstride, kw, nk * 8, kind, st));
  CU(cudaMemcpyAsync(c->vpool + s * c->vstride, vw, nv * 8, kind, st));
  CU(cudaStreamSynchronize(st));
  c->length = n;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_export_stream(const cvq_cache* c, uint32_t seq, uint32_t layer,
                                           uint32_t head, uint64_t* kw, uint64_t* vw, int where) {
  if (!c || !kw || !vw) return fail(CVQ_EINVAL, "null argument");
  CU(cudaSetDevice(c->ctx->device));
  if (seq >= c->desc.n_seqs || layer >= c->desc.n_layers || head >= c->desc.n_kv_heads)
    return fail(CVQ_EINVAL, "cache: stream out of range");
  TRY(sync_check(const_cast<cvq_cache*>(c)));
  const Geom& g = c->geo;
  const size_t s = ((size_t)seq * c->desc.n_layers + layer) * c->desc.n_kv_heads + head;
  const uint64_t nk = words_for_bits(c->length * (uint64_t)g.bpt);
  const uint64_t nv = words_for_bits(c->length * (uint64_t)g.n_codes);
  const cudaMemcpyKind kind = where == CVQ_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  CU(cudaMemcpyAsync(kw, c->kpool + s * c->kstride, nk * 8, kind, c->ctx->stream));
  CU(cudaMemcpyAsync(vw, c->vpool + s * c->vstride, nv * 8, kind, c->ctx->stream));
  CU(cudaStreamSynchronize(c->ctx->stream));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_pools(cvq_cache* c, uint64_t** kw, uint64_t* ks, uint64_t** vw,
                                   uint64_t* vs) {
  if (!c || !kw || !ks || !vw || !vs) return fail(CVQ_EINVAL, "null argument");
  *kw = c->kpool;
  *ks = c->kstride;
  *vw = c->vpool;
  *vs = c->vstride;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_set_length(cvq_cache* c, uint64_t n) {
  if (!c) return fail(CVQ_EINVAL, "null cache");
  TRY(ctx_check(c->ctx));
  TRY(ensure_capacity(c, n));
  c->length = n;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_shape_of(const cvq_cache* c, cvq_cache_shape* out) {
  if (!c || !out) return fail(CVQ_EINVAL, "null argument");
  out->n_seqs = c->desc.n_seqs;
  out->n_layers = c->desc.n_layers;
  out->n_kv_heads = c->desc.n_kv_heads;
  out->q_per_kv = c->desc.q_per_kv;
  out->d = c->desc.key.d;
  out->n_codes = c->desc.n_codes;
  out->position_offset = c->desc.position_offset;
  return CVQ_OK;
}

CVQ_API cvq_context* cvq_cache_context(const cvq_cache* c) { return c ? c->ctx : nullptr; }

CVQ_API cvq_status cvq_cache_reserve(cvq_cache* c, uint64_t n_tokens) {
  if (!c) return fail(CVQ_EINVAL, "null cache");
  TRY(ctx_check(c->ctx));
  return ensure_capacity(c, n_tokens);
}

CVQ_API cvq_status cvq_cache_capacity(const cvq_cache* c, uint64_t* n_tokens) {
  if (!c || !n_tokens) return fail(CVQ_EINVAL, "null argument");
  *n_tokens = c->desc.capacity;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_synchronize(cvq_cache* c) {
  if (!c) return fail(CVQ_EINVAL, "null cache");
  TRY(ctx_check(c->ctx));
  return sync_check(c);
}

CVQ_API cvq_status cvq_cache_set_variant(cvq_cache* c, uint32_t variant) {
  if (!c) return fail(CVQ_EINVAL, "null cache");
  if (variant & ~(uint32_t)(CVQ_VARIANT_GENERIC | CVQ_VARIANT_TC_DENSE | CVQ_VARIANT_TC_PAIR |
                            CVQ_VARIANT_FUSED | CVQ_VARIANT_F32_WEIGHTS))
    return fail(CVQ_EINVAL, "cache: unknown kernel variant");
  c->variant = variant;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_cache_key_mode(const cvq_cache* c, uint32_t* flags) {
  if (!c || !flags) return fail(CVQ_EINVAL, "null argument");
  uint32_t f = c->desc.flags & (CVQ_CACHE_KEYS_FP16 | CVQ_CACHE_KEYS_TC);
  if (!c->cbtc || c->tc_demoted) f &= ~CVQ_CACHE_KEYS_TC;
  *flags = f;
  return CVQ_OK;
}

// ===================================================== single-stream mirrors
namespace {

// The single-stream mirrors keep one device cache per context, reused across
// calls by identity (SURVEY 8b "Ownership": upload once, cache by identity):
// the key / value codebooks are re-uploaded only when their pointer or
// content hash changes, and the codes are treated as the reference's
// append-only vectors -- same buffers and n >= the cached n with the sampled
// earlier codes unchanged -> only the new tail tokens are uploaded and packed
// (a decode loop calling fused_attention per step re-sends one token, not N).
uint64_t fnv(const void* p, size_t bytes, uint64_t h = 1469598103934665603ull) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < bytes; ++i) h = (h ^ c[i]) * 1099511628211ull;
  return h;
}
// hash of up to 64 sampled tokens of [0, n) plus the last one
uint64_t sample_hash(const uint16_t* a, const uint16_t* b, const uint8_t* bits, uint64_t n,
                     size_t per_tok, uint32_t n_codes) {
  uint64_t h = fnv(&n, sizeof(n));
  if (n == 0) return h;
  const uint64_t step = n > 64 ? n / 64 : 1;
  for (uint64_t t = 0; t < n; t += step) {
    h = fnv(a + t * per_tok, per_tok * 2, h);
    h = fnv(b + t * per_tok, per_tok * 2, h);
    h = fnv(bits + t * n_codes, n_codes, h);
  }
  h = fnv(a + (n - 1) * per_tok, per_tok * 2, h);
  h = fnv(b + (n - 1) * per_tok, per_tok * 2, h);
  return fnv(bits + (n - 1) * n_codes, n_codes, h);
}

}  // namespace

struct cvq_mirror {
  cvq_cache* c = nullptr;
  cvq_key_config kc{};
  uint32_t n_codes = 0;
  double base = 0.0;
  const double* atoms = nullptr;
  uint64_t atoms_hash = 0;
  const double* vrows = nullptr;
  uint64_t vrows_hash = 0;
  const uint16_t* a = nullptr;
  const uint16_t* b = nullptr;
  const uint8_t* bits = nullptr;
  uint64_t n = 0, codes_hash = 0;
  ~cvq_mirror() {
    if (c) cvq_cache_destroy(c);
  }
};

void destroy_mirror(cvq_mirror* m) { delete m; }

namespace {

cvq_status mirror_cache(cvq_context* ctx, const cvq_key_config* kc, uint32_t n_codes,
                        const double* atoms, const uint16_t* a, const uint16_t* b, uint64_t n,
                        const uint8_t* bits, const double* vrows, double base, cvq_cache** out) {
  if (!ctx->mirror) ctx->mirror = new cvq_mirror;
  cvq_mirror& m = *ctx->mirror;
  const Geom g = make_geom(kc, n_codes, 0, 1);
  const size_t na = (size_t)g.R * g.subs * g.L;
  const bool same_geom = m.c && m.kc.d == kc->d && m.kc.group_size == kc->group_size &&
                         m.kc.n_levels == kc->n_levels && m.kc.rounds == kc->rounds &&
                         m.n_codes == n_codes && m.base == base;
  if (!same_geom) {
    if (m.c) cvq_cache_destroy(m.c);
    m = cvq_mirror{};
    cvq_cache_desc d{};
    d.key = *kc;
    d.n_codes = n_codes;
    d.hidden = 0;
    d.n_seqs = d.n_layers = d.n_kv_heads = d.q_per_kv = 1;
    d.capacity = n;
    d.position_offset = 0;
    d.rope_base = base;
    TRY(cvq_cache_create(ctx, &d, &m.c));
    m.kc = *kc;
    m.n_codes = n_codes;
    m.base = base;
  }
  cvq_cache* c = m.c;
  const uint64_t ah = fnv(atoms, na * 2 * sizeof(double));
  if (m.atoms != atoms || m.atoms_hash != ah) {
    TRY(cvq_cache_set_key_codebook(c, 0, 0, atoms));
    m.atoms = atoms;
    m.atoms_hash = ah;
  }
  const uint64_t vh = fnv(vrows, (size_t)n_codes * g.d * sizeof(double));
  if (m.vrows != vrows || m.vrows_hash != vh) {
    TRY(cvq_cache_set_value_quantizer(c, 0, 0, nullptr, nullptr, nullptr, nullptr, vrows));
    m.vrows = vrows;
    m.vrows_hash = vh;
  }
  const size_t per_tok = (size_t)g.R * g.groups;
  uint64_t from = 0;  // first token to (re)upload
  if (m.a == a && m.b == b && m.bits == bits && n >= m.n &&
      sample_hash(a, b, bits, m.n, per_tok, n_codes) == m.codes_hash)
    from = m.n;
  TRY(ensure_capacity(c, n));
  const uint64_t nn = n - from;
  if (nn > 0) {
    const size_t np = (size_t)nn * per_tok;
    CU(c->enc_scratch.ensure(np * 4 + (size_t)nn * n_codes + 64));
    uint16_t* da = static_cast<uint16_t*>(c->enc_scratch.p);
    uint16_t* db = da + np;
    uint8_t* dbits = reinterpret_cast<uint8_t*>(db + np);
    cudaStream_t st = ctx->stream;
    CU(cudaMemcpyAsync(da, a + from * per_tok, np * 2, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(db, b + from * per_tok, np * 2, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dbits, bits + from * n_codes, (size_t)nn * n_codes, cudaMemcpyHostToDevice,
                       st));
    CU(run_pack_keys(g, 1, da, db, (long long)nn, (long long)from, c->kpool, c->kstride, st));
    CU(run_pack_values(g, 1, dbits, (long long)nn, (long long)from, c->vpool, c->vstride, st));
  }
  c->length = n;
  m.a = a;
  m.b = b;
  m.bits = bits;
  m.n = n;
  m.codes_hash = sample_hash(a, b, bits, n, per_tok, n_codes);
  *out = c;
  return CVQ_OK;
}

// validate_input (attn.cpp:91-110) + the per-token code range check
// (attn.cpp:223-224).
cvq_status validate_attn(const cvq_key_config* kc, uint32_t n_codes, const uint16_t* a,
                         const uint16_t* b, uint64_t n, uint64_t t) {
  TRY(validate_kc(kc));
  if (n == 0) return fail(CVQ_EINVAL, "attention: empty cache");
  if (t + 1 < n) return fail(CVQ_EINVAL, "attention: query position precedes cache");
  if (n_codes == 0) return fail(CVQ_EINVAL, "attention: value codes/codebook mismatch");
  if (n_codes > 1024) return fail(CVQ_EINVAL, "attention: n_codes > 1024 unsupported");
  const uint64_t np = n * kc->rounds * ((kc->d / 2) / kc->group_size);
  for (uint64_t i = 0; i < np; ++i)
    if (a[i] >= kc->n_levels || b[i] >= kc->n_levels)
      return fail(CVQ_EINVAL, "fused_attention: code out of range");
  return CVQ_OK;
}

void fill_flops(cvq_flop_report* f, const cvq_key_config* kc, uint32_t n_codes, uint64_t n,
                bool naive) {
  if (!f) return;
  const uint64_t d = kc->d, R = kc->rounds, L = kc->n_levels;
  if (naive) {  // attn.cpp:155, 53, 77, 87
    f->predicted_mults = cvq_predicted_flops_naive(n, d, n_codes);
    f->measured_mults = n * n_codes * d + 2 * d + (2 * d + d + 1) * n + n * d;
  } else {  // attn.cpp:190, 207, 235, 256
    f->predicted_mults = cvq_predicted_flops_fused(n, d, n_codes, R, L);
    f->measured_mults = 2 * d + 2 * d * R * L + n * (R * d + 1) + (uint64_t)n_codes * d;
  }
}

}  // namespace

CVQ_API cvq_status cvq_fused_attention(cvq_context* ctx, const cvq_key_config* kc,
                                       uint32_t n_codes, const double* atoms, const uint16_t* a,
                                       const uint16_t* b, uint64_t n, const uint8_t* bits,
                                       const double* vrows, const double* q, uint64_t t,
                                       double base, double* out, double* scores_out,
                                       cvq_flop_report* flops) {
  TRY(ctx_check(ctx));
  if (!kc || !atoms || !q || !out || !vrows || (n && (!a || !b || !bits)))
    return fail(CVQ_EINVAL, "null argument");
  TRY(validate_attn(kc, n_codes, a, b, n, t));
  cvq_cache* c = nullptr;
  TRY(mirror_cache(ctx, kc, n_codes, atoms, a, b, n, bits, vrows, base, &c));
  const Geom& g = c->geo;
  AttnJob job = make_job(c);
  job.t = (long long)t;
  const size_t need = attn_scratch_bytes(job, nullptr);
  CU(c->attn_scratch.ensure(need));
  CU(c->stage_in.ensure((size_t)g.d * 4 * 2 + (size_t)n * 4 + 64));
  float* qd = static_cast<float*>(c->stage_in.p);
  float* od = qd + g.d;
  float* sd = od + g.d;
  std::vector<float> qf(g.d);
  for (int i = 0; i < g.d; ++i) qf[i] = (float)q[i];
  CU(cudaMemcpyAsync(qd, qf.data(), g.d * 4, cudaMemcpyHostToDevice, ctx->stream));
  CU(run_attention(job, qd, od, nullptr, nullptr, nullptr, scores_out ? sd : nullptr,
                   c->attn_scratch.p, c->attn_scratch.n, ctx->stream));
  std::vector<float> of(g.d), sf(scores_out ? n : 0);
  CU(cudaMemcpyAsync(of.data(), od, g.d * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (scores_out)
    CU(cudaMemcpyAsync(sf.data(), sd, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < g.d; ++i) out[i] = of[i];
  if (scores_out)
    for (uint64_t i = 0; i < n; ++i) scores_out[i] = sf[i];
  fill_flops(flops, kc, n_codes, n, false);
  return CVQ_OK;
}

CVQ_API cvq_status cvq_naive_attention(cvq_context* ctx, const cvq_key_config* kc,
                                       uint32_t n_codes, const double* atoms, const uint16_t* a,
                                       const uint16_t* b, uint64_t n, const uint8_t* bits,
                                       const double* vrows, const double* q, uint64_t t,
                                       double base, double* out, cvq_flop_report* flops) {
  TRY(ctx_check(ctx));
  if (!kc || !atoms || !q || !out || !vrows || (n && (!a || !b || !bits)))
    return fail(CVQ_EINVAL, "null argument");
  TRY(validate_attn(kc, n_codes, a, b, n, t));
  cvq_cache* c = nullptr;
  TRY(mirror_cache(ctx, kc, n_codes, atoms, a, b, n, bits, vrows, base, &c));
  const Geom& g = c->geo;
  AttnJob job = make_job(c);
  job.t = (long long)t;
  CU(c->attn_scratch.ensure(naive_scratch_bytes(job, true)));
  CU(c->stage_in.ensure((size_t)g.d * 8 + 64));
  float* qd = static_cast<float*>(c->stage_in.p);
  float* od = qd + g.d;
  std::vector<float> qf(g.d);
  for (int i = 0; i < g.d; ++i) qf[i] = (float)q[i];
  CU(cudaMemcpyAsync(qd, qf.data(), g.d * 4, cudaMemcpyHostToDevice, ctx->stream));
  CU(run_naive_attention(job, qd, od, c->attn_scratch.p, c->attn_scratch.n, ctx->stream, true));
  std::vector<float> of(g.d);
  CU(cudaMemcpyAsync(of.data(), od, g.d * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < g.d; ++i) out[i] = of[i];
  fill_flops(flops, kc, n_codes, n, true);
  return CVQ_OK;
}

CVQ_API cvq_status cvq_encode_keys(cvq_context* ctx, const cvq_key_config* kc, const double* atoms,
                                   const double* keys, uint64_t n, uint16_t* a, uint16_t* b) {
  TRY(ctx_check(ctx));
  TRY(validate_kc(kc));
  if (!atoms || (n && (!keys || !a || !b))) return fail(CVQ_EINVAL, "null argument");
  if (n == 0) return CVQ_OK;
  Geom g = make_geom(kc, 1, 0, 1);
  const size_t na = (size_t)g.R * g.subs * g.L;
  const bool tables = key_tables_fit(g);
  const size_t nb = tables ? (size_t)g.R * g.groups * g.L * g.L : 0;
  const size_t np = (size_t)n * g.R * g.groups;
  const size_t nf = tables && key_t64_applies(g) ? key_t64_table_floats(g) : 0;  // fp32 tables
  const size_t bytes =
      (na * 2 + nb + g.R * g.groups + (size_t)n * g.d) * 8 + 16 + nf * 4 + np * 4 + 256;
  CU(ctx->scratch.ensure(bytes));
  double* d_atoms = static_cast<double*>(ctx->scratch.p);
  double* d_base = d_atoms + na * 2;
  double* d_max = d_base + nb;
  double* d_keys = d_max + g.R * g.groups;
  float* d_f = reinterpret_cast<float*>(  // 16-B aligned (cp.async sources)
      (reinterpret_cast<uintptr_t>(d_keys + (size_t)n * g.d) + 15) & ~(uintptr_t)15);
  uint16_t* da = reinterpret_cast<uint16_t*>(d_f + nf);
  uint16_t* db = da + np;
  cudaStream_t st = ctx->stream;
  CU(cudaMemcpyAsync(d_atoms, atoms, na * 16, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_keys, keys, (size_t)n * g.d * 8, cudaMemcpyHostToDevice, st));
  if (tables)
    CU(build_key_enc_tables(g, 1, d_atoms, d_base, d_max, st, nf ? d_f : nullptr,
                            nf ? d_f + na * 2 : nullptr));
  KeyEncTables tab{d_atoms, tables ? d_base : nullptr, d_max};
  if (nf) {
    tab.atomsf = d_f;
    tab.basef = d_f + na * 2;
  }
  CU(run_encode_keys(g, 1, 1, tab, d_keys, CVQ_F64, 0, (long long)n, da, db, st));
  CU(cudaMemcpyAsync(a, da, np * 2, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(b, db, np * 2, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_decode_keys(cvq_context* ctx, const cvq_key_config* kc, const double* atoms,
                                   const uint16_t* a, const uint16_t* b, uint64_t n,
                                   double* out) {
  TRY(ctx_check(ctx));
  TRY(validate_kc(kc));
  if (!atoms || (n && (!a || !b || !out))) return fail(CVQ_EINVAL, "null argument");
  if (n == 0) return CVQ_OK;
  Geom g = make_geom(kc, 1, 0, 1);
  const size_t na = (size_t)g.R * g.subs * g.L, np = (size_t)n * g.R * g.groups;
  for (size_t i = 0; i < np; ++i)  // keyquant.cpp:756-757
    if (a[i] >= g.L || b[i] >= g.L) return fail(CVQ_EINVAL, "decode_keys: code out of range");
  CU(ctx->scratch.ensure((na * 2 + (size_t)n * g.d) * 8 + np * 4 + 256));
  double* d_atoms = static_cast<double*>(ctx->scratch.p);
  double* d_out = d_atoms + na * 2;
  uint16_t* da = reinterpret_cast<uint16_t*>(d_out + (size_t)n * g.d);
  uint16_t* db = da + np;
  cudaStream_t st = ctx->stream;
  CU(cudaMemcpyAsync(d_atoms, atoms, na * 16, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(da, a, np * 2, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(db, b, np * 2, cudaMemcpyHostToDevice, st));
  CU(run_decode_keys(g, d_atoms, da, db, (long long)n, d_out, st));
  CU(cudaMemcpyAsync(out, d_out, (size_t)n * g.d * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_decode_values(cvq_context* ctx, uint32_t n_codes, uint32_t d,
                                     const double* rows, const uint8_t* bits, uint64_t n,
                                     double* out) {
  TRY(ctx_check(ctx));
  if (n_codes == 0 || d == 0) return fail(CVQ_EINVAL, "decode_values: empty codebook");
  if (!rows || (n && (!bits || !out))) return fail(CVQ_EINVAL, "null argument");
  if (n == 0) return CVQ_OK;
  const size_t nr = (size_t)n_codes * d, nb = (size_t)n * n_codes;
  CU(ctx->scratch.ensure((nr + (size_t)n * d) * 8 + nb + 256));
  double* d_rows = static_cast<double*>(ctx->scratch.p);
  double* d_out = d_rows + nr;
  uint8_t* d_bits = reinterpret_cast<uint8_t*>(d_out + (size_t)n * d);
  cudaStream_t st = ctx->stream;
  CU(cudaMemcpyAsync(d_rows, rows, nr * 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_bits, bits, nb, cudaMemcpyHostToDevice, st));
  CU(run_decode_values((int)n_codes, (int)d, d_rows, d_bits, (long long)n, d_out, st));
  CU(cudaMemcpyAsync(out, d_out, (size_t)n * d * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_encode_keys_search(cvq_context* ctx, const cvq_key_config* kc,
                                          const double* atoms, const double* keys, uint64_t n,
                                          int32_t search, uint16_t* a, uint16_t* b) {
  if (search == 0) return cvq_encode_keys(ctx, kc, atoms, keys, n, a, b);
  TRY(ctx_check(ctx));
  TRY(validate_kc(kc));
  if (search != 1) return fail(CVQ_EINVAL, "encode_keys: unknown AssignSearch");
  if (!atoms || (n && (!keys || !a || !b))) return fail(CVQ_EINVAL, "null argument");
  if (n == 0) return CVQ_OK;
  Geom g = make_geom(kc, 1, 0, 1);
  const size_t na = (size_t)g.R * g.subs * g.L;
  const size_t np = (size_t)n * g.R * g.groups;
  CU(ctx->scratch.ensure((na * 2 + (size_t)n * g.d) * 8 + np * 4 + 256));
  double* d_atoms = static_cast<double*>(ctx->scratch.p);
  double* d_keys = d_atoms + na * 2;
  uint16_t* da = reinterpret_cast<uint16_t*>(d_keys + (size_t)n * g.d);
  uint16_t* db = da + np;
  cudaStream_t st = ctx->stream;
  CU(cudaMemcpyAsync(d_atoms, atoms, na * 16, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_keys, keys, (size_t)n * g.d * 8, cudaMemcpyHostToDevice, st));
  CU(encode_keys_factorized_gpu(g, d_atoms, d_keys, (long long)n, da, db, st));
  CU(cudaMemcpyAsync(a, da, np * 2, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(b, db, np * 2, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_train_key_codebook(cvq_context* ctx, const cvq_key_config* kc,
                                          const double* calib, uint64_t n, const cvq_em_config* em,
                                          double* atoms_out, double* objective_out,
                                          uint64_t objective_cap, uint64_t* objective_len,
                                          double* mse_out) {
  TRY(ctx_check(ctx));
  TRY(validate_kc(kc));
  if (!em || !atoms_out || !objective_len || !mse_out || (n && !calib))
    return fail(CVQ_EINVAL, "null argument");
  if (em->search != 0 && em->search != 1) return fail(CVQ_EINVAL, "EmConfig: unknown search");
  Geom g = make_geom(kc, 1, 0, 1);
  TrainConfig tc{em->soft_iters, em->hard_iters_max, em->t0, em->decay, em->tol,
                 em->ridge, em->seed, em->search == 1};
  std::vector<std::vector<double>> traces;
  std::vector<double> mse;
  std::string err;
  const int rc = train_key_codebook_gpu(g, calib, (long long)n, tc, atoms_out, &traces, &mse, &err,
                                        ctx->stream);
  if (rc == 1) return fail(CVQ_EINVAL, err);
  if (rc == 2) return fail(CVQ_ETRAINING, err);
  if (rc != 0) return fail(CVQ_ECUDA, err);
  uint64_t k = 0;
  for (size_t i = 0; i < traces.size(); ++i) {
    objective_len[i] = traces[i].size();
    for (double v : traces[i])
      if (objective_out && k < objective_cap) objective_out[k++] = v;
  }
  for (size_t r = 0; r < mse.size(); ++r) mse_out[r] = mse[r];
  return CVQ_OK;
}

CVQ_API cvq_status cvq_train_value_quantizer(cvq_context* ctx, const double* calib, uint64_t n,
                                             uint32_t d, uint32_t n_codes,
                                             const cvq_val_train_config* cfg,
                                             const double* init_codebook, double* w1, double* b1,
                                             double* w2, double* b2, double* codebook,
                                             double* loss_curve, uint64_t* curve_len,
                                             int32_t* diverged, uint64_t* steps_run) {
  TRY(ctx_check(ctx));
  if (!cfg || !w1 || !b1 || !w2 || !b2 || !codebook || !loss_curve || !curve_len || !diverged ||
      !steps_run || (n && !calib))
    return fail(CVQ_EINVAL, "null argument");
  ValTrainCfg vc{cfg->steps, cfg->batch, cfg->step_size, cfg->gumbel_t_start, cfg->gumbel_t_end,
                 cfg->hidden, cfg->seed, cfg->checkpoint_every, cfg->freeze_codebook != 0};
  std::string err;
  int dv = 0;
  long long sr = 0, cl = 0;
  const int rc = train_value_quantizer_gpu(calib, (long long)n, (int)d, (int)n_codes, vc,
                                           init_codebook, w1, b1, w2, b2, codebook, loss_curve,
                                           &dv, &sr, &cl, &err, ctx->stream);
  if (rc == 1) return fail(CVQ_EINVAL, err);
  if (rc != 0) return fail(CVQ_ECUDA, err);
  *diverged = dv;
  *steps_run = (uint64_t)sr;
  *curve_len = (uint64_t)cl;
  return CVQ_OK;
}

CVQ_API cvq_status cvq_encoder_forward_infer(cvq_context* ctx, uint32_t d, uint32_t hidden,
                                             uint32_t n_codes, const double* w1, const double* b1,
                                             const double* w2, const double* b2,
                                             const double* values, uint64_t n, uint8_t* bits,
                                             double* logits) {
  TRY(ctx_check(ctx));
  if (d == 0 || hidden == 0 || n_codes == 0) return fail(CVQ_EINVAL, "ValueEncoder: zero dimension");
  if (!w1 || !b1 || !w2 || !b2 || (n && (!values || !bits))) return fail(CVQ_EINVAL, "null argument");
  if (n == 0) return CVQ_OK;
  cvq_key_config kc{2, 1, 2, 1};
  Geom g = make_geom(&kc, n_codes, hidden, 1);
  g.d = (int)d;
  const size_t nw = (size_t)d * hidden + hidden + (size_t)hidden * n_codes + n_codes;
  const size_t bytes = (nw + (size_t)n * d + (size_t)n * n_codes) * 8 + (size_t)n * n_codes + 256;
  CU(ctx->scratch.ensure(bytes));
  double* dw1 = static_cast<double*>(ctx->scratch.p);
  double* db1 = dw1 + (size_t)d * hidden;
  double* dw2 = db1 + hidden;
  double* db2 = dw2 + (size_t)hidden * n_codes;
  double* dv = db2 + n_codes;
  double* dl = dv + (size_t)n * d;
  uint8_t* dbits = reinterpret_cast<uint8_t*>(dl + (size_t)n * n_codes);
  cudaStream_t st = ctx->stream;
  CU(cudaMemcpyAsync(dw1, w1, (size_t)d * hidden * 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(db1, b1, (size_t)hidden * 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dw2, w2, (size_t)hidden * n_codes * 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(db2, b2, (size_t)n_codes * 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dv, values, (size_t)n * d * 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(ctx->d_err, 0xFF, sizeof(unsigned long long), st));
  ValEncWeights w{dw1, db1, dw2, db2};
  CU(run_encode_values(g, 1, 1, w, dv, CVQ_F64, 0, (long long)n, dbits, dl, ctx->d_err, 0, st));
  unsigned long long herr = ~0ull;
  CU(cudaMemcpyAsync(&herr, ctx->d_err, sizeof(herr), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(bits, dbits, (size_t)n * n_codes, cudaMemcpyDeviceToHost, st));
  if (logits) CU(cudaMemcpyAsync(logits, dl, (size_t)n * n_codes * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (herr != ~0ull) return fail(CVQ_ETRAINING, "encoder_forward: non-finite activations");
  return CVQ_OK;
}

CVQ_API cvq_status cvq_pack_key_codes(cvq_context* ctx, const cvq_key_config* kc,
                                      const uint16_t* a, const uint16_t* b, uint64_t n,
                                      uint64_t* words) {
  TRY(ctx_check(ctx));
  TRY(validate_kc(kc));
  if (n == 0) return CVQ_OK;
  if (!a || !b || !words) return fail(CVQ_EINVAL, "null argument");
  Geom g = make_geom(kc, 1, 0, 1);
  const size_t np = (size_t)n * g.R * g.groups;
  const uint64_t nw = words_for_bits(n * (uint64_t)g.bpt);
  CU(ctx->scratch.ensure(np * 4 + nw * 8 + 64));
  uint64_t* dw = static_cast<uint64_t*>(ctx->scratch.p);
  uint16_t* da = reinterpret_cast<uint16_t*>(dw + nw);
  uint16_t* db = da + np;
  cudaStream_t st = ctx->stream;
  CU(cudaMemcpyAsync(da, a, np * 2, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(db, b, np * 2, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(dw, 0, nw * 8, st));
  CU(run_pack_keys(g, 1, da, db, (long long)n, 0, dw, nw, st));
  CU(cudaMemcpyAsync(words, dw, nw * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_pack_value_codes(cvq_context* ctx, uint32_t n_codes, const uint8_t* bits,
                                        uint64_t n, uint64_t* words) {
  TRY(ctx_check(ctx));
  if (n == 0 || n_codes == 0) return CVQ_OK;
  if (!bits || !words) return fail(CVQ_EINVAL, "null argument");
  cvq_key_config kc{2, 1, 2, 1};
  Geom g = make_geom(&kc, n_codes, 0, 1);
  const uint64_t nw = words_for_bits(n * (uint64_t)n_codes);
  CU(ctx->scratch.ensure((size_t)n * n_codes + nw * 8 + 64));
  uint64_t* dw = static_cast<uint64_t*>(ctx->scratch.p);
  uint8_t* dbits = reinterpret_cast<uint8_t*>(dw + nw);
  cudaStream_t st = ctx->stream;
  CU(cudaMemcpyAsync(dbits, bits, (size_t)n * n_codes, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(dw, 0, nw * 8, st));
  CU(run_pack_values(g, 1, dbits, (long long)n, 0, dw, nw, st));
  CU(cudaMemcpyAsync(words, dw, nw * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return CVQ_OK;
}

namespace {
// BitBuffer::from_words validation (cache.cpp:78-88).
cvq_status check_words(const uint64_t* words, uint64_t n_words, uint64_t bits) {
  if (n_words != words_for_bits(bits)) return fail(CVQ_EINVAL, "BitBuffer: word count mismatch");
  const unsigned tail = (unsigned)(bits % 64);
  if (tail != 0 && (words[n_words - 1] >> tail) != 0)
    return fail(CVQ_EINVAL, "BitBuffer: nonzero padding bits");
  return CVQ_OK;
}
}  // namespace

CVQ_API cvq_status cvq_unpack_key_codes(cvq_context* ctx, const cvq_key_config* kc,
                                        const uint64_t* words, uint64_t n_words, uint64_t n,
                                        uint16_t* a, uint16_t* b) {
  TRY(ctx_check(ctx));
  TRY(validate_kc(kc));
  Geom g = make_geom(kc, 1, 0, 1);
  TRY(check_words(words, n_words, n * (uint64_t)g.bpt));
  if (n == 0) return CVQ_OK;
  const size_t np = (size_t)n * g.R * g.groups;
  CU(ctx->scratch.ensure(np * 4 + n_words * 8 + 64));
  uint64_t* dw = static_cast<uint64_t*>(ctx->scratch.p);
  uint16_t* da = reinterpret_cast<uint16_t*>(dw + n_words);
  uint16_t* db = da + np;
  cudaStream_t st = ctx->stream;
  CU(cudaMemcpyAsync(dw, words, n_words * 8, cudaMemcpyHostToDevice, st));
  CU(run_unpack_keys(g, dw, (long long)n, da, db, st));
  CU(cudaMemcpyAsync(a, da, np * 2, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(b, db, np * 2, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_unpack_value_codes(cvq_context* ctx, uint32_t n_codes,
                                          const uint64_t* words, uint64_t n_words, uint64_t n,
                                          uint8_t* bits) {
  TRY(ctx_check(ctx));
  TRY(check_words(words, n_words, n * (uint64_t)n_codes));
  if (n == 0 || n_codes == 0) return CVQ_OK;
  cvq_key_config kc{2, 1, 2, 1};
  Geom g = make_geom(&kc, n_codes, 0, 1);
  CU(ctx->scratch.ensure((size_t)n * n_codes + n_words * 8 + 64));
  uint64_t* dw = static_cast<uint64_t*>(ctx->scratch.p);
  uint8_t* dbits = reinterpret_cast<uint8_t*>(dw + n_words);
  cudaStream_t st = ctx->stream;
  CU(cudaMemcpyAsync(dw, words, n_words * 8, cudaMemcpyHostToDevice, st));
  CU(run_unpack_values(g, dw, (long long)n, dbits, st));
  CU(cudaMemcpyAsync(bits, dbits, (size_t)n * n_codes, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return CVQ_OK;
}
