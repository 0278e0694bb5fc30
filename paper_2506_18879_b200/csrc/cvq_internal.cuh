// cvq_internal.cuh -- shared geometry, device helpers and launcher
// declarations for the sm_100a CommVQ kernels (attn.cu, encode.cu, pack.cu,
// capi.cu).  Not part of the public C-ABI (include/cvq.h).
#pragma once

#include <cfloat>

#include <cuda_runtime.h>
#include <string>

#include "../../include/cvq.h"
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

namespace cvq {

// Geometry of one quantizer configuration (KeyQuantConfig keyquant.hpp:16-28
// + value side).  fpt = code fields per token (rounds * groups * 2); the
// packed key stream is a plain sequence of lb-bit fields (cache.cpp:90-106),
// so field F of a stream sits at bit F * lb.
struct Geom {
  int d, subs, g, groups, L, lb, R, fpt, bpt;
  int n_codes, hidden;
  int G;  // query heads served per KV stream
};

// Work description shared by the attention launchers.
struct AttnJob {
  Geom geo;
  int S;                      // number of KV streams
  const uint64_t* kpool;      // [S][kstride] packed key words
  uint64_t kstride;
  const uint64_t* vpool;      // [S][vstride] packed value words
  uint64_t vstride;
  int n_slots;                // codebook slot of stream s = s % n_slots
  const float2* cb_key;       // [slot][R][L][subs] complex atoms (x, y), fp32
  const uint32_t* cb_key16;   // same as packed half2, or null (fp16-codebook mode)
  const uint16_t* cb_key_tc;  // [slot][R][2 sides][128 x 64 K-major fp16] tcgen05 A operand, or null
  const float* cb_val;        // [slot][n_codes][d] fp32
  const double* thetas;       // [subs] fp64, rope.cpp:8-25
  long long n;                // tokens per stream
  long long pos0;             // global position of token 0
  long long t;                // query position
  uint32_t variant;           // kVar* kernel-variant bits (cvq_cache_set_variant)
};

// Records the message returned by cvq_last_error() on this thread (capi.cu).
cvq_status set_error(cvq_status s, const std::string& msg);

// Kernel variants selectable per cache (cvq.h CVQ_VARIANT_*): cross-check /
// experimental kernels next to the defaults, chosen by the caller, never by
// the environment.
constexpr uint32_t kVarGeneric = 1u;  // generic kernels for every shape
constexpr uint32_t kVarTcDense = 2u;  // dense one-hot tcgen05 kernel (attn_tc.cu)
constexpr uint32_t kVarTcPair = 4u;   // CTA-pair (cta_group::2) sparse kernel
constexpr uint32_t kVarFused = 8u;    // single fused CUDA-core kernel (fp16 codebook)
constexpr uint32_t kVarF32W = 16u;    // fp32 score hand-off instead of fp16 weights

// Scratch handed to run_attention (sized by attn_scratch_bytes).
size_t attn_scratch_bytes(const AttnJob& job, int* n_chunks_out);

// q: [S][G][d] fp32 (device).  If out != nullptr writes normalised outputs
// [S][G][d]; if m/l/o != nullptr writes the merged partial (m, l, o[d]) of
// this job's tokens per row.  scores (optional) receives [S][G][n] fp32.
// prof (optional, 2 events) brackets the dominant (score) kernel so callers
// can time it live on the launching stream.
cudaError_t run_attention(const AttnJob& job, const float* q, float* out,
                          float* m, float* l, float* o, float* scores_out,
                          void* scratch, size_t scratch_bytes,
                          cudaStream_t st, cudaEvent_t* prof = nullptr);

// tcgen05 one-hot-MMA score kernel (attn_tc.cu).
size_t tc_smem_bytes(int G, int R);
int tc_blocks(const AttnJob& job);
// A operand of the one-hot MMA for one slot: [R][side][16 KiB core-matrix
// layout]; side b holds the rotated codebook (x <- -y, y <- x).
void tc_build_codebook(int R, const double* xy, uint16_t* out, uint16_t (*to_half)(double));
size_t tc_codebook_elems(int R);
// Half-weight output (HalfOut non-null, sparse kernel, one round part): the
// score epilogue writes fp16 exp(s - m32) per (token, head) and the max m32
// of each 32-token group instead of fp32 scores (k_fast_value<PH>).
struct HalfOut {
  void* ph;        // [S][nps][G] __half
  float* m32;      // [S][nps / 32][G]
  long long nps;   // tokens per stream, n rounded up to 128
};
bool tc_half_scores(const AttnJob& job);
cudaError_t run_tc_score(const AttnJob& job, const float* q, float* ps, int chunk,
                         cudaStream_t st, const HalfOut* ho = nullptr);
// 2:4-sparse tcgen05 score kernel (attn_sp.cu), R = 11: B blocks per slot
// [R][X rows | Y rows][64 levels] fp16, built by sp_build_codebook.
bool sp_supported(int R);
int sp_parts(int R);  // round parts (<= 11 resident rounds each) -> partial-score slices
size_t sp_codebook_elems(int R);
void sp_build_codebook(int R, const double* xy, uint16_t* out, uint16_t (*to_half)(double));
cudaError_t run_sp_score(const AttnJob& job, const uint16_t* cb, size_t slot_elems,
                         const float* q, float* ps, int chunk, cudaStream_t st,
                         const HalfOut* ho = nullptr);

// LSE merge over packed blocks reached through a device array of pointers
// (parts[p] + off), e.g. peers' symmetric-memory buffers over NVLink.
cudaError_t run_lse_combine_ptrs(const float* const* parts, long long off, int n_parts,
                                 long long rows, int d, float* out, cudaStream_t st);

// Block-wide max / sum; every thread gets the result (contains barriers).
__device__ __forceinline__ float block_reduce(float v, bool is_max, float* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  v = (threadIdx.x < nw) ? red[threadIdx.x] : (is_max ? -FLT_MAX : 0.f);
  if (wid == 0)
    for (int o = 16; o; o >>= 1) {
      float u = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmaxf(v, u) : v + u;
    }
  if (threadIdx.x == 0) red[32] = v;
  __syncthreads();
  return red[32];
}

// Log-sum-exp merge (device), parts-major.
// part_stride 0: m, l [parts][rows], o [parts][rows][d]; otherwise part p's
// m, l and o rows start at p * part_stride (packed exchange buffers).
cudaError_t run_lse_combine(const float* m, const float* l, const float* o,
                            int n_parts, long long rows, int d, float* out,
                            float* m_out, float* l_out, cudaStream_t st,
                            long long part_stride = 0);

// ---- encoders (encode.cu) -------------------------------------------------
// Per slot: atoms fp64 [R][subs][L][2] -> screen tables.
struct KeyEncTables {
  const double* atoms;   // [slot][R][subs][L][2] (reference order)
  const double* base;    // [slot][R][groups][L][L]
  const double* maxnorm; // [slot][R][groups]
  // fp32 copies of atoms / base for the head-preset encoder (k_encode_keys_t64)
  const float* atomsf = nullptr;
  const float* basef = nullptr;
};
// atomsf / basef (optional): fp32 copies for k_encode_keys_t64
cudaError_t build_key_enc_tables(const Geom& g, int n_slots,
                                 const double* atoms, double* base,
                                 double* maxnorm, cudaStream_t st, float* atomsf = nullptr,
                                 float* basef = nullptr);
// whether the head-preset key encoder applies (and wants the fp32 tables)
bool key_t64_applies(const Geom& g);
size_t key_t64_table_floats(const Geom& g);  // per slot: atoms + base
// keys: element (s, i, k) at keys + s*s_stride + i*d + k, dtype 0=f32 1=f64.
// Codes: a/b [s][n][R*groups] uint16.  err_flag (device int) set on failure.
cudaError_t run_encode_keys(const Geom& g, int S, int n_slots,
                            const KeyEncTables& tab, const void* keys,
                            int dtype, long long s_stride, long long n,
                            uint16_t* a, uint16_t* b, cudaStream_t st);
// Value encoder (infer): bits [s][n][n_codes] uint8, logits optional fp64.
struct ValEncWeights {
  const double* w1;  // [slot][d][hidden]
  const double* b1;  // [slot][hidden]
  const double* w2;  // [slot][hidden][n_codes]
  const double* b2;  // [slot][n_codes]
  // optional screen tables (prefill encoder, k_encode_values_screen): fp32
  // copy of w2 and its column 2-norms |w2[:, c]| (fp64)
  const float* w2f = nullptr;   // [slot][hidden][n_codes]
  const double* n2 = nullptr;   // [slot][n_codes]
};
cudaError_t run_encode_values(const Geom& g, int S, int n_slots,
                              const ValEncWeights& w, const void* vals,
                              int dtype, long long s_stride, long long n,
                              uint8_t* bits, double* logits,
                              unsigned long long* errpos, unsigned long long tok0,
                              cudaStream_t st);

// ---- key-codebook training (train.cu) -------------------------------------
bool key_tables_fit(const Geom& g);  // encode.cu
struct TrainConfig {  // EmConfig, keyquant.hpp:71-80
  size_t soft_iters, hard_iters_max;
  double t0, decay, tol, ridge;
  uint64_t seed;
  bool factorized;
};
// train_key_codebook (keyquant.cpp:641-703): calib [n][d] fp64 host;
// atoms_out [R][d/2][L][2]; traces: hard objective per (round, group);
// mse: reconstruction MSE per round.  Returns 0, or 1 (invalid argument),
// 2 (training error), 3 (CUDA error) with *err set.
cudaError_t encode_keys_factorized_gpu(const Geom& g, const double* atoms, const double* keys,
                                       long long n, uint16_t* a, uint16_t* b, cudaStream_t st);
int train_key_codebook_gpu(const Geom& g, const double* calib, long long n, const TrainConfig& em,
                           double* atoms_out, std::vector<std::vector<double>>* traces,
                           std::vector<double>* mse, std::string* err, cudaStream_t st);

// ---- value-quantizer training (train_value.cu) -----------------------------
struct ValTrainCfg {  // ValTrainConfig, valquant.hpp:76-86
  size_t steps, batch;
  double step_size, t_start, t_end;
  size_t hidden;
  uint64_t seed;
  size_t checkpoint_every;
  bool freeze_codebook;
};
// train_value_quantizer (valquant.cpp:172-383).  calib [n][d] host; outputs
// host arrays (w1 [d][H], b1 [H], w2 [H][C], b2 [C], cb [C][d], loss_curve
// [steps]).  Returns 0, 1 (invalid argument) or 3 (CUDA) with *err set.
int train_value_quantizer_gpu(const double* calib, long long n, int d, int n_codes,
                              const ValTrainCfg& cfg, const double* init_cb, double* w1,
                              double* b1, double* w2, double* b2, double* cb, double* loss_curve,
                              int* diverged, long long* steps_run, long long* curve_len,
                              std::string* err, cudaStream_t st);

// ---- packing (pack.cu) -----------------------------------------------------
// Writes n tokens' key codes (a/b [s][n][R*groups]) into stream words at
// token offset tok0 (read-modify-write of boundary words).
// errpos (optional): the cache's first-failed-append position; a batch at
// tok0 >= *errpos is not written (a failed append leaves the words as they
// were, cache.cpp:256-285 throws before mutating).
cudaError_t run_pack_keys(const Geom& g, int S, const uint16_t* a,
                          const uint16_t* b, long long n, long long tok0,
                          uint64_t* kpool, uint64_t kstride, cudaStream_t st,
                          const unsigned long long* errpos = nullptr);
cudaError_t run_pack_values(const Geom& g, int S, const uint8_t* bits,
                            long long n, long long tok0, uint64_t* vpool,
                            uint64_t vstride, cudaStream_t st,
                            const unsigned long long* errpos = nullptr);
cudaError_t run_unpack_keys(const Geom& g, const uint64_t* words, long long n,
                            uint16_t* a, uint16_t* b, cudaStream_t st);
// dense reconstruction, bit-identical to decode_keys / decode_values (decode.cu)
cudaError_t run_decode_keys(const Geom& g, const double* atoms, const uint16_t* a,
                            const uint16_t* b, long long n, double* out, cudaStream_t st);
cudaError_t run_decode_values(int n_codes, int d, const double* rows, const uint8_t* bits,
                              long long n, double* out, cudaStream_t st);
cudaError_t run_unpack_values(const Geom& g, const uint64_t* words,
                              long long n, uint8_t* bits, cudaStream_t st);

// cudaFuncAttributeMaxDynamicSharedMemorySize is per (kernel, device): the
// largest value set so far is remembered per pair (capi.cu), so a process
// driving several GPUs raises it on each device.
cudaError_t ensure_dyn_smem(const void* kernel, size_t bytes);

// Global launch counter (bench.py gpu_launches).
extern std::atomic<unsigned long long> g_launches;
inline void count_launch(unsigned long long k = 1) { g_launches += k; }

// ---- device helpers --------------------------------------------------------
__device__ __forceinline__ unsigned read_field(const uint64_t* __restrict__ w,
                                               unsigned long long bit,
                                               int nbits) {
  unsigned long long wi = bit >> 6;
  int off = (int)(bit & 63);
  unsigned long long v = __ldg(w + wi) >> off;
  if (off + nbits > 64) v |= __ldg(w + wi + 1) << (64 - off);
  return (unsigned)(v & ((1ull << nbits) - 1ull));
}

// e^{-i * delta * theta} with the angle formed and reduced mod 2*pi in fp64
// (fp32 angles break 1e-3 at long context).
__device__ __forceinline__ float2 phase_neg(long long delta, double theta) {
  const double kInv2Pi = 0.15915494309189535;
  const double k2PiHi = 6.283185307179586;
  const double k2PiLo = 2.4492935982947064e-16;
  double ang = (double)delta * theta;
  double k = rint(ang * kInv2Pi);
  double r = fma(-k, k2PiHi, ang);
  r = fma(-k, k2PiLo, r);
  float s, c;
  sincosf((float)r, &s, &c);
  return make_float2(c, -s);
}

}  // namespace cvq
