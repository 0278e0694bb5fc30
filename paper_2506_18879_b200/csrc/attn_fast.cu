// attn_fast.cu -- specialised CommVQ decode attention for the LLaMA-shaped
// head presets (d = 128, one 64-subspace group per round, L = 64 levels,
// R rounds, N_c value codes, G query heads per KV stream), sm_100a.
//
// Split of the work:
//  F1 k_fast_score  grid (context chunks, stream x subspace-split).  Each CTA
//     keeps its slice of the fp32 key codebook -- R x 64 levels x JC
//     subspaces, 176 KiB at R=11/JC=32 and 168 KiB at R=21/JC=16 -- resident
//     in shared memory, streams the packed key words of 128-token tiles with
//     cp.async (double-buffered), unpacks the 6-bit fields once per tile and
//     decodes K_j = sum_r U[r,a_r,j] + i U[r,b_r,j] with one lane per
//     subspace (conflict-free 256-B row reads), applies the per-position
//     RoPE phase (fp64-reduced base per 8-token run, fp32 recurrence inside),
//     and reduces the G query-head dot products across lanes with a
//     butterfly reduce-scatter.  Writes partial scores [S][JS][n][G].
//  F2 k_fast_value  grid (context chunks, stream).  Sums the JS partial
//     scores, softmax statistics of the chunk, z[k][h] += p_h(i) bit_k(i)
//     from cp.async-staged value words (attn.cpp:239-247).  Writes the chunk
//     partial (m, l, z), unnormalised.
//  k_combine_merge / k_combine_project  (row, 32-code slice) CTAs merge the
//                     chunk partials; then one CTA per row: LSE merge of the
//     chunk partials, then o = z . C_V / L (attn.cpp:249-255) once per row.
#include <cuda_fp16.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "cvq_internal.cuh"

namespace cvq {

namespace {

constexpr int kThreads = 256;
constexpr int kTile = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct FastArgs {
  const uint64_t* kpool;
  uint64_t kstride;
  const uint64_t* vpool;
  uint64_t vstride;
  const float2* cb;   // [slot][R][64][64]
  const uint32_t* cbh;  // same, packed (x, y) half2 (fp16-codebook mode) or null
  const float* cbv;   // [slot][NC][128]
  int n_slots;
  const float* q;     // [S][G][128]
  const double* thetas;
  long long t, pos0, n;
  int chunk;          // F1 tokens per CTA (multiple of 128)
  int chunk2;         // F2 tokens per CTA (multiple of 128)
  int S;
  float* ps;          // [S][JS][n][G] partial scores
  // half-weight mode (sparse tcgen05 scores, one round part): instead of ps,
  // ph[S][nps][G] = fp16 exp(s - m32) and m32[S][nps / 32][G] = the max of
  // each 32-token group (nps = n rounded up to 128)
  const __half* ph;
  const float* m32;
  long long nps;
  float* scores_out;  // optional [S][G][n]
  float *pm, *pl, *po;
};

// Butterfly reduce-scatter of NV values across the JC lanes of a group:
// afterwards lane keeps max(NV/JC, 1) sums starting at value index `base`.
// When NV < JC the last levels are plain butterfly sums; only lanes whose
// bits at those levels are zero report (`writer`).
template <int NV, int JC>
__device__ __forceinline__ int reduce_scatter(float (&v)[NV], int lane, bool& writer) {
  int base = 0;
  int cnt = NV;
  writer = true;
#pragma unroll
  for (int o = JC / 2; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
    if (cnt > 1) {
      const int half = cnt / 2;
#pragma unroll
      for (int i = 0; i < NV / 2; ++i) {
        if (i < half) {
          const float send = up ? v[i] : v[i + half];
          const float keep = up ? v[i + half] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (up) base += half;
      cnt = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      if (up) writer = false;
    }
  }
  return base;
}

// packed fp32x2 add (FADD2 on sm_100a)
__device__ __forceinline__ void add2(float2& acc, const float2 v) {
  asm("{.reg .b64 a, b;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 b, {%2, %3};\n\t"
      "add.rn.f32x2 a, a, b;\n\tmov.b64 {%0, %1}, a;}"
      : "+f"(acc.x), "+f"(acc.y)
      : "f"(v.x), "f"(v.y));
}

constexpr int kF1Threads = 512;  // 16 warps: one 8-token run each per 128-token tile

template <int R, int JC, int G>
__global__ void __launch_bounds__(kF1Threads, 1) k_fast_score(FastArgs a) {
  constexpr int JS = 64 / JC;
  constexpr int TP = 32 / JC;                  // tokens per warp step
  constexpr int NSTEP = 8 / TP;                // steps per run (8 tokens per warp)
  constexpr int CW = ((2 * R + 15) / 16) * 16; // code bytes per token
  constexpr int WPT = 24 * R;                  // words per 128-token tile (12R bits/token)
  constexpr int NV = NSTEP * G;                // values per lane before reduction
  static_assert(kF1Threads / 32 * 8 == kTile, "one pass per tile");
  extern __shared__ __align__(16) unsigned char smem[];
  float2* cbs = reinterpret_cast<float2*>(smem);                          // [R][64][JC]
  uint64_t* wbuf = reinterpret_cast<uint64_t*>(smem + (size_t)R * 64 * JC * 8);  // [2][WPT]
  uint8_t* codes = reinterpret_cast<uint8_t*>(wbuf + 2 * WPT);           // [kTile][CW]

  const int s = blockIdx.y / JS, js = blockIdx.y % JS;
  const long long i0 = (long long)blockIdx.x * a.chunk;
  const long long i1 = min(a.n, i0 + a.chunk);
  if (i0 >= i1) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = s % a.n_slots;

  const float2* cbg = a.cb + (size_t)slot * R * 64 * 64 + js * JC;
  for (int e = tid; e < R * 64 * (JC / 2); e += kF1Threads) {
    const int row = e / (JC / 2), c2 = e % (JC / 2);
    cp_async16(cbs + row * JC + 2 * c2, cbg + (size_t)row * 64 + 2 * c2);
  }
  cp_async_commit();
  const uint64_t* kw = a.kpool + (size_t)s * a.kstride + (size_t)(i0 / kTile) * WPT;
  const int ntiles = (int)((i1 - i0 + kTile - 1) / kTile);
  auto load_tile = [&](int k, int buf) {
    const uint64_t* src = kw + (size_t)k * WPT;
    for (int e = tid; e < WPT / 2; e += kF1Threads) cp_async16(wbuf + buf * WPT + 2 * e, src + 2 * e);
    cp_async_commit();
  };
  load_tile(0, 0);

  // per-lane constants: subspace j, query heads' conj(q_j)/sqrt(d), phase step
  const int tg = lane / JC, jc = lane % JC;
  const int j = js * JC + jc;
  const double theta = a.thetas[j];
  float2 w[G];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const float* qr = a.q + ((size_t)s * G + h) * 128;
    w[h] = make_float2(qr[2 * j] * 0.08838834764831845f, -qr[2 * j + 1] * 0.08838834764831845f);
  }
  float2 stepm;  // e^{+i TP theta}
  {
    double sn, cs;
    sincos((double)TP * theta, &sn, &cs);
    stepm = make_float2((float)cs, (float)sn);
  }
  float* ps = a.ps + ((size_t)(s * JS + js) * a.n) * G;

  for (int k = 0; k < ntiles; ++k) {
    if (k + 1 < ntiles) {
      load_tile(k + 1, (k + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    // unpack the tile's 6-bit fields (2R per token) into bytes
    const uint64_t* wt = wbuf + (k & 1) * WPT;
    for (int e = tid; e < kTile * 2 * R; e += kF1Threads) {
      const int tok = e / (2 * R), f = e % (2 * R);
      const unsigned bit = (unsigned)e * 6u;
      const unsigned wi = bit >> 6, off = bit & 63u;
      unsigned long long v = wt[wi] >> off;
      if (off > 58u) v |= wt[wi + 1] << (64u - off);
      codes[tok * CW + f] = (uint8_t)(v & 63u);
    }
    __syncthreads();
    const long long ti = i0 + (long long)k * kTile;
    const int valid = (int)min((long long)kTile, i1 - ti);
    {
      const int tok0 = warp * 8;
      if (tok0 < valid) {
      float2 ph = phase_neg(a.t - (a.pos0 + ti + tok0 + tg), theta);
      float acc[NV];
#pragma unroll
      for (int st = 0; st < NSTEP; ++st) {
        const int dlt = tok0 + st * TP + tg;
        const uint4* cd = reinterpret_cast<const uint4*>(codes + dlt * CW);
        uint4 cv[CW / 16];
#pragma unroll
        for (int c = 0; c < CW / 16; ++c) cv[c] = cd[c];
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(cv);
        float2 ka = make_float2(0.f, 0.f), kb = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t word = cw[(2 * r) >> 2];
          const unsigned ca = __byte_perm(word, 0, 0x4440 | ((2 * r) & 3));
          const unsigned cbb = __byte_perm(word, 0, 0x4440 | ((2 * r + 1) & 3));
          add2(ka, cbs[(r * 64 + ca) * JC + jc]);
          add2(kb, cbs[(r * 64 + cbb) * JC + jc]);
        }
        const float kx = ka.x - kb.y, ky = ka.y + kb.x;  // K = sum u_a + i sum u_b
        const float rx = ph.x * kx - ph.y * ky;
        const float ry = ph.x * ky + ph.y * kx;
#pragma unroll
        for (int h = 0; h < G; ++h) acc[st * G + h] = w[h].x * rx - w[h].y * ry;
        const float nx = ph.x * stepm.x - ph.y * stepm.y;
        ph.y = ph.x * stepm.y + ph.y * stepm.x;
        ph.x = nx;
      }
      bool writer;
      const int base = reduce_scatter<NV, JC>(acc, lane, writer);
      constexpr int VPL = NV / JC > 0 ? NV / JC : 1;
#pragma unroll
      for (int m = 0; m < VPL; ++m) {
        const int vi = base + m;
        const int st = vi / G, h = vi % G;
        const int dlt = tok0 + st * TP + tg;
        if (writer && dlt < valid) ps[(ti + dlt) * G + h] = acc[m];
      }
      }
    }
    __syncthreads();
  }
}


// f32 += f16 (FHADD on sm_100a) for both halves of a packed (x, y) half2.
__device__ __forceinline__ void hadd2_acc(float2& acc, uint32_t h2) {
  asm("{.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
      "add.rn.f32.f16 %0, lo, %0;\n\tadd.rn.f32.f16 %1, hi, %1;}"
      : "+f"(acc.x), "+f"(acc.y)
      : "r"(h2));
}

// fp16-codebook variant of k_fast_score: the slice is stored as packed
// (x, y) half2, accumulation stays fp32 (FHADD), so each gather moves half
// the shared-memory bytes.  LPT lanes decode one token, each owning SPL
// consecutive subspaces (SPL = 4: one 16-B LDS per row, so the per-gather
// address and load instructions are shared by 4 subspaces); a warp decodes
// TP = 32/LPT tokens per step.  JC = LPT*SPL subspaces per CTA: the whole
// 64-subspace codebook for R <= 13 (no split).
template <int R, int SPL, int LPT, int G>
__global__ void __launch_bounds__(kF1Threads, 1) k_fast_score_h(FastArgs a) {
  constexpr int JC = LPT * SPL;
  constexpr int JS = 64 / JC;
  constexpr int TP = 32 / LPT;
  constexpr int NSTEP = 8 / TP;  // 8 tokens per warp per tile
  constexpr int CW = ((2 * R + 15) / 16) * 16;
  constexpr int WPT = 24 * R;
  constexpr int NV = NSTEP * G;
  static_assert(kF1Threads / 32 * 8 == kTile, "one pass per tile");
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* cbs = reinterpret_cast<uint32_t*>(smem);                           // [R][64][JC] half2
  uint64_t* wbuf = reinterpret_cast<uint64_t*>(smem + (size_t)R * 64 * JC * 4);  // [2][WPT]
  uint8_t* codes = reinterpret_cast<uint8_t*>(wbuf + 2 * WPT);                 // [kTile][CW]

  const int s = blockIdx.y / JS, js = blockIdx.y % JS;
  const long long i0 = (long long)blockIdx.x * a.chunk;
  const long long i1 = min(a.n, i0 + a.chunk);
  if (i0 >= i1) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tg = lane / LPT, ln = lane % LPT;
  const int slot = s % a.n_slots;

  const uint32_t* cbg = a.cbh + (size_t)slot * R * 64 * 64 + js * JC;
  for (int e = tid; e < R * 64 * (JC / 4); e += kF1Threads) {
    const int row = e / (JC / 4), c4 = e % (JC / 4);
    cp_async16(cbs + row * JC + 4 * c4, cbg + (size_t)row * 64 + 4 * c4);
  }
  cp_async_commit();
  const uint64_t* kw = a.kpool + (size_t)s * a.kstride + (size_t)(i0 / kTile) * WPT;
  const int ntiles = (int)((i1 - i0 + kTile - 1) / kTile);
  auto load_tile = [&](int k, int buf) {
    const uint64_t* src = kw + (size_t)k * WPT;
    for (int e = tid; e < WPT / 2; e += kF1Threads) cp_async16(wbuf + buf * WPT + 2 * e, src + 2 * e);
    cp_async_commit();
  };
  load_tile(0, 0);

  double theta[SPL];
  float2 stepm[SPL], w[G][SPL];
#pragma unroll
  for (int m = 0; m < SPL; ++m) {
    const int j = js * JC + ln * SPL + m;
    theta[m] = a.thetas[j];
    double sn, cs;
    sincos((double)TP * theta[m], &sn, &cs);  // e^{+i TP theta}: next step's token
    stepm[m] = make_float2((float)cs, (float)sn);
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float* qr = a.q + ((size_t)s * G + h) * 128;
      w[h][m] = make_float2(qr[2 * j] * 0.08838834764831845f, -qr[2 * j + 1] * 0.08838834764831845f);
    }
  }
  float* ps = a.ps + ((size_t)(s * JS + js) * a.n) * G;
  const uint32_t* cb_lane = cbs + ln * SPL;

  for (int k = 0; k < ntiles; ++k) {
    if (k + 1 < ntiles) {
      load_tile(k + 1, (k + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint64_t* wt = wbuf + (k & 1) * WPT;
    for (int e = tid; e < kTile * 2 * R; e += kF1Threads) {
      const int tok = e / (2 * R), f = e % (2 * R);
      const unsigned bit = (unsigned)e * 6u;
      const unsigned wi = bit >> 6, off = bit & 63u;
      unsigned long long v = wt[wi] >> off;
      if (off > 58u) v |= wt[wi + 1] << (64u - off);
      codes[tok * CW + f] = (uint8_t)(v & 63u);
    }
    __syncthreads();
    const long long ti = i0 + (long long)k * kTile;
    const int valid = (int)min((long long)kTile, i1 - ti);
    const int tok0 = warp * 8;
    if (tok0 < valid) {
      float2 ph[SPL];
#pragma unroll
      for (int m = 0; m < SPL; ++m) ph[m] = phase_neg(a.t - (a.pos0 + ti + tok0 + tg), theta[m]);
      float acc[NV];
#pragma unroll
      for (int st = 0; st < NSTEP; ++st) {
        const int dlt = tok0 + st * TP + tg;
        const uint4* cd = reinterpret_cast<const uint4*>(codes + dlt * CW);
        uint4 cv[CW / 16];
#pragma unroll
        for (int c = 0; c < CW / 16; ++c) cv[c] = cd[c];
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(cv);
        float2 ka[SPL], kb[SPL];
#pragma unroll
        for (int m = 0; m < SPL; ++m) ka[m] = kb[m] = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t word = cw[(2 * r) >> 2];
          const unsigned ca = __byte_perm(word, 0, 0x4440 | ((2 * r) & 3));
          const unsigned cbb = __byte_perm(word, 0, 0x4440 | ((2 * r + 1) & 3));
          const uint32_t* ra = cb_lane + (r * 64 + ca) * JC;
          const uint32_t* rb = cb_lane + (r * 64 + cbb) * JC;
          if constexpr (SPL == 4) {
            const uint4 va = *reinterpret_cast<const uint4*>(ra);
            const uint4 vb = *reinterpret_cast<const uint4*>(rb);
            hadd2_acc(ka[0], va.x);
            hadd2_acc(ka[1], va.y);
            hadd2_acc(ka[2], va.z);
            hadd2_acc(ka[3], va.w);
            hadd2_acc(kb[0], vb.x);
            hadd2_acc(kb[1], vb.y);
            hadd2_acc(kb[2], vb.z);
            hadd2_acc(kb[3], vb.w);
          } else if constexpr (SPL == 2) {
            const uint2 va = *reinterpret_cast<const uint2*>(ra);
            const uint2 vb = *reinterpret_cast<const uint2*>(rb);
            hadd2_acc(ka[0], va.x);
            hadd2_acc(ka[1], va.y);
            hadd2_acc(kb[0], vb.x);
            hadd2_acc(kb[1], vb.y);
          } else {
            hadd2_acc(ka[0], *ra);
            hadd2_acc(kb[0], *rb);
          }
        }
        float part[G];
#pragma unroll
        for (int h = 0; h < G; ++h) part[h] = 0.f;
#pragma unroll
        for (int m = 0; m < SPL; ++m) {
          const float kx = ka[m].x - kb[m].y, ky = ka[m].y + kb[m].x;
          const float rx = ph[m].x * kx - ph[m].y * ky;
          const float ry = ph[m].x * ky + ph[m].y * kx;
#pragma unroll
          for (int h = 0; h < G; ++h) part[h] += w[h][m].x * rx - w[h][m].y * ry;
          const float nx = ph[m].x * stepm[m].x - ph[m].y * stepm[m].y;
          ph[m].y = ph[m].x * stepm[m].y + ph[m].y * stepm[m].x;
          ph[m].x = nx;
        }
#pragma unroll
        for (int h = 0; h < G; ++h) acc[st * G + h] = part[h];
      }
      bool writer;
      const int base = reduce_scatter<NV, LPT>(acc, lane, writer);
      constexpr int VPL = NV / LPT > 0 ? NV / LPT : 1;
#pragma unroll
      for (int m = 0; m < VPL; ++m) {
        const int vi = base + m;
        const int st = vi / G, h = vi % G;
        const int dlt = tok0 + st * TP + tg;
        if (writer && dlt < valid) ps[(ti + dlt) * G + h] = acc[m];
      }
    }
    __syncthreads();
  }
}

// Fused single-kernel decode attention for the 1-bit head preset with the
// fp16 codebook (whole codebook per CTA, so every CTA has complete scores):
// k_fast_score_h's key decode (R rounds, 16 lanes x 4 subspaces per token,
// G = 4 query heads) followed, per warp and per 8-token run, by an online
// softmax and the value accumulation z[c][h] += p_h bit_c (attn.cpp:
// 237-247) on value words streamed with the key words.  The 16 warps'
// (m, l, z) are merged at the end of the chunk and o = z C_V / l written as
// the chunk partial (attn.cpp:249-255).  Removes the partial-score round
// trip and the separate value kernel.
template <int R>
__global__ void __launch_bounds__(kF1Threads, 1) k_fast_attn_h(FastArgs a) {
  constexpr int G = 4, NC = 128, SPL = 4, LPT = 16, JC = 64, TP = 2, NSTEP = 4;
  constexpr int CW = ((2 * R + 15) / 16) * 16;
  constexpr int WPT = 24 * R;
  constexpr int VPT = 2 * kTile;  // value words per tile (128 bits per token)
  constexpr int NV = NSTEP * G;   // 16 = LPT: one (token, head) score per lane
  constexpr int NW = kF1Threads / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* cbs = reinterpret_cast<uint32_t*>(smem);                           // [R][64][64] half2
  uint64_t* wbuf = reinterpret_cast<uint64_t*>(smem + (size_t)R * 64 * JC * 4);  // [2][WPT]
  uint64_t* vbuf = wbuf + 2 * WPT;                                             // [2][VPT]
  float4* pw = reinterpret_cast<float4*>(vbuf + 2 * VPT);                      // [NW][8]
  uint8_t* codes = reinterpret_cast<uint8_t*>(pw + NW * 8);                    // [kTile][CW]

  const int s = blockIdx.y;
  const long long i0 = (long long)blockIdx.x * a.chunk;
  const long long i1 = min(a.n, i0 + a.chunk);
  if (i0 >= i1) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tg = lane / LPT, ln = lane % LPT;
  const int slot = s % a.n_slots;

  const uint32_t* cbg = a.cbh + (size_t)slot * R * 64 * 64;
  for (int e = tid; e < R * 64 * (JC / 4); e += kF1Threads) cp_async16(cbs + 4 * e, cbg + 4 * e);
  cp_async_commit();
  const uint64_t* kw = a.kpool + (size_t)s * a.kstride + (size_t)(i0 / kTile) * WPT;
  const uint64_t* vwg = a.vpool + (size_t)s * a.vstride + (size_t)(i0 / kTile) * VPT;
  const int ntiles = (int)((i1 - i0 + kTile - 1) / kTile);
  auto load_tile = [&](int k, int buf) {
    const uint64_t* src = kw + (size_t)k * WPT;
    for (int e = tid; e < WPT / 2; e += kF1Threads) cp_async16(wbuf + buf * WPT + 2 * e, src + 2 * e);
    const uint64_t* vsrc = vwg + (size_t)k * VPT;
    for (int e = tid; e < VPT / 2; e += kF1Threads) cp_async16(vbuf + buf * VPT + 2 * e, vsrc + 2 * e);
    cp_async_commit();
  };
  load_tile(0, 0);

  double theta[SPL];
  float2 stepm[SPL], w[G][SPL];
#pragma unroll
  for (int m = 0; m < SPL; ++m) {
    const int j = ln * SPL + m;
    theta[m] = a.thetas[j];
    double sn, cs;
    sincos((double)TP * theta[m], &sn, &cs);
    stepm[m] = make_float2((float)cs, (float)sn);
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float* qr = a.q + ((size_t)s * G + h) * 128;
      w[h][m] = make_float2(qr[2 * j] * 0.08838834764831845f, -qr[2 * j + 1] * 0.08838834764831845f);
    }
  }
  const uint32_t* cb_lane = cbs + ln * SPL;
  // per-warp online-softmax state; this lane's head is lane & 3, its codes
  // are 4*lane .. 4*lane+3 for all 4 heads (z as head pairs for FADD2)
  float m_run = -INFINITY, l_run = 0.f;
  float2 z[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) z[c][0] = z[c][1] = make_float2(0.f, 0.f);

  for (int k = 0; k < ntiles; ++k) {
    if (k + 1 < ntiles) {
      load_tile(k + 1, (k + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint64_t* wt = wbuf + (k & 1) * WPT;
    for (int e = tid; e < kTile * 2 * R; e += kF1Threads) {
      const int tok = e / (2 * R), f = e % (2 * R);
      const unsigned bit = (unsigned)e * 6u;
      const unsigned wi = bit >> 6, off = bit & 63u;
      unsigned long long v = wt[wi] >> off;
      if (off > 58u) v |= wt[wi + 1] << (64u - off);
      codes[tok * CW + f] = (uint8_t)(v & 63u);
    }
    __syncthreads();
    const long long ti = i0 + (long long)k * kTile;
    const int valid = (int)min((long long)kTile, i1 - ti);
    const int tok0 = warp * 8;
    if (tok0 < valid) {
      float2 ph[SPL];
#pragma unroll
      for (int m = 0; m < SPL; ++m) ph[m] = phase_neg(a.t - (a.pos0 + ti + tok0 + tg), theta[m]);
      float acc[NV];
#pragma unroll
      for (int st = 0; st < NSTEP; ++st) {
        const int dlt = tok0 + st * TP + tg;
        const uint4* cd = reinterpret_cast<const uint4*>(codes + dlt * CW);
        uint4 cv[CW / 16];
#pragma unroll
        for (int c = 0; c < CW / 16; ++c) cv[c] = cd[c];
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(cv);
        float2 ka[SPL], kb[SPL];
#pragma unroll
        for (int m = 0; m < SPL; ++m) ka[m] = kb[m] = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t word = cw[(2 * r) >> 2];
          const unsigned ca = __byte_perm(word, 0, 0x4440 | ((2 * r) & 3));
          const unsigned cbb = __byte_perm(word, 0, 0x4440 | ((2 * r + 1) & 3));
          const uint4 va = *reinterpret_cast<const uint4*>(cb_lane + (r * 64 + ca) * JC);
          const uint4 vb = *reinterpret_cast<const uint4*>(cb_lane + (r * 64 + cbb) * JC);
          hadd2_acc(ka[0], va.x);
          hadd2_acc(ka[1], va.y);
          hadd2_acc(ka[2], va.z);
          hadd2_acc(ka[3], va.w);
          hadd2_acc(kb[0], vb.x);
          hadd2_acc(kb[1], vb.y);
          hadd2_acc(kb[2], vb.z);
          hadd2_acc(kb[3], vb.w);
        }
        float part[G];
#pragma unroll
        for (int h = 0; h < G; ++h) part[h] = 0.f;
#pragma unroll
        for (int m = 0; m < SPL; ++m) {
          const float kx = ka[m].x - kb[m].y, ky = ka[m].y + kb[m].x;
          const float rx = ph[m].x * kx - ph[m].y * ky;
          const float ry = ph[m].x * ky + ph[m].y * kx;
#pragma unroll
          for (int h = 0; h < G; ++h) part[h] += w[h][m].x * rx - w[h][m].y * ry;
          const float nx = ph[m].x * stepm[m].x - ph[m].y * stepm[m].y;
          ph[m].y = ph[m].x * stepm[m].y + ph[m].y * stepm[m].x;
          ph[m].x = nx;
        }
#pragma unroll
        for (int h = 0; h < G; ++h) acc[st * G + h] = part[h];
      }
      bool writer;
      reduce_scatter<NV, LPT>(acc, lane, writer);
      // lane holds the score of (token tok0 + slot, head lane & 3), slot =
      // ((lane & 15) >> 2) * 2 + (lane >> 4)
      const int tslot = ((lane & 15) >> 2) * 2 + (lane >> 4);
      const bool ok = tok0 + tslot < valid;
      const float sv = ok ? acc[0] : -INFINITY;
      float tm = sv;
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 4));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 8));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
      const float mn = fmaxf(m_run, tm);
      const float scale = (m_run == -INFINITY) ? 0.f : __expf(m_run - mn);
      const float p = ok ? __expf(sv - mn) : 0.f;
      float psum = p;
      psum += __shfl_xor_sync(0xffffffffu, psum, 4);
      psum += __shfl_xor_sync(0xffffffffu, psum, 8);
      psum += __shfl_xor_sync(0xffffffffu, psum, 16);
      l_run = l_run * scale + psum;
      m_run = mn;
      const float2 s01 = make_float2(__shfl_sync(0xffffffffu, scale, 0),
                                     __shfl_sync(0xffffffffu, scale, 1));
      const float2 s23 = make_float2(__shfl_sync(0xffffffffu, scale, 2),
                                     __shfl_sync(0xffffffffu, scale, 3));
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        z[c][0].x *= s01.x;
        z[c][0].y *= s01.y;
        z[c][1].x *= s23.x;
        z[c][1].y *= s23.y;
      }
      reinterpret_cast<float*>(pw + warp * 8 + tslot)[lane & 3] = p;
      __syncwarp();
      const uint64_t* vt = vbuf + (k & 1) * VPT;
#pragma unroll
      for (int sl = 0; sl < 8; ++sl) {
        if (tok0 + sl < valid) {
          const float4 pp = pw[warp * 8 + sl];
          const unsigned bits =
              (unsigned)(vt[(tok0 + sl) * 2 + (lane >> 4)] >> (4 * (lane & 15)));
          const float2 p01 = make_float2(pp.x, pp.y), p23 = make_float2(pp.z, pp.w);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (bits & (1u << c)) {
              add2(z[c][0], p01);
              add2(z[c][1], p23);
            }
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
  // ---- merge the 16 warps' (m, l, z) (codebook smem is free now) ----
  float* red = reinterpret_cast<float*>(smem);  // [NW][8 + NC*G]
  float* mine = red + warp * (8 + NC * G);
  {  // lanes 0..3 hold heads 0..3 (every lane with the same lane & 3 agrees)
    const float mh = __shfl_sync(0xffffffffu, m_run, lane & 3);
    const float lh = __shfl_sync(0xffffffffu, l_run, lane & 3);
    if (lane < 4) {
      mine[lane] = mh;
      mine[4 + lane] = lh;
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float* zc = mine + 8 + (4 * lane + c) * G;
    zc[0] = z[c][0].x;
    zc[1] = z[c][0].y;
    zc[2] = z[c][1].x;
    zc[3] = z[c][1].y;
  }
  __syncthreads();
  __shared__ float Mh[G], Lh[G], Wt[NW][G];
  if (tid < G) {
    float M = -INFINITY;
    for (int ww = 0; ww < NW; ++ww) M = fmaxf(M, red[ww * (8 + NC * G) + tid]);
    float L = 0.f;
    for (int ww = 0; ww < NW; ++ww) {
      const float mw = red[ww * (8 + NC * G) + tid];
      const float wt = (mw == -INFINITY) ? 0.f : __expf(mw - M);
      Wt[ww][tid] = wt;
      L += red[ww * (8 + NC * G) + 4 + tid] * wt;
    }
    Mh[tid] = M;
    Lh[tid] = L;
  }
  __syncthreads();
  float* Z = red + NW * (8 + NC * G);  // [NC][G]
  for (int e = tid; e < NC * G; e += kF1Threads) {
    const int h = e % G;
    float v = 0.f;
    for (int ww = 0; ww < NW; ++ww) v += red[ww * (8 + NC * G) + 8 + e] * Wt[ww][h];
    Z[e] = v;
  }
  __syncthreads();
  const long long rows = (long long)a.S * G;
  for (int e = tid; e < G * NC; e += kF1Threads) {  // unnormalised z (k_combine_project)
    const int h = e / NC, kk = e % NC;
    a.po[((long long)blockIdx.x * rows + (long long)s * G + h) * NC + kk] = Z[kk * G + h];
  }
  if (tid < G) {
    a.pm[(long long)blockIdx.x * rows + (long long)s * G + tid] = Mh[tid];
    a.pl[(long long)blockIdx.x * rows + (long long)s * G + tid] = Lh[tid];
  }
}

// Sum of the per-warp z partials of a k_fast_value CTA and the chunk's
// (z, m, l) partial for the LSE merge.
template <int NC, int G>
__device__ __forceinline__ void fast_value_finish(const FastArgs& a, float* zr, const float* mh,
                                                  const float* lh, int s) {
  const int tid = threadIdx.x;
  __syncthreads();
  for (int e = tid; e < NC * G; e += kThreads) {
    float v = 0.f;
    for (int w = 0; w < kThreads / 32; ++w) v += zr[(size_t)w * NC * G + e];
    zr[e] = v;  // warp-0 slot reused for the total
  }
  __syncthreads();
  // unnormalised z of this chunk; the value codebook product happens once per
  // row after the merge (k_combine_project)
  const long long rows = (long long)a.S * G;
  for (int e = tid; e < G * NC; e += kThreads) {
    const int h = e / NC, k = e % NC;
    a.po[((long long)blockIdx.x * rows + (long long)s * G + h) * NC + k] = zr[k * G + h];
  }
  if (tid < G) {
    const long long row = (long long)s * G + tid;
    a.pm[(long long)blockIdx.x * rows + row] = mh[tid];
    a.pl[(long long)blockIdx.x * rows + row] = lh[tid];
  }
}

// one-thread bulk copies (TMA engine) into shared memory, completing on an
// mbarrier: a CTA's staging costs 3 instructions instead of a cp.async loop
__device__ __forceinline__ void fv_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void fv_bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;}"
        : "=r"(ok)
        : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Value accumulation z[c][h] = sum_i p_h(i) bit_c(i) of k_fast_value, either
// (MMA) as an fp16 tensor-core product z^T[NC][8] += Bits^T[NC][16 tokens] x
// P[16 tokens][8 heads] per 16-token step (mma.sync m16n8k16, fp32
// accumulators; bits expanded to fp16 0 / 1 by byte permutes; p rounded to
// fp16, relative 2^-11) or (!MMA) by predicated fp32 adds on CUDA cores.
template <int NC, int G, int JS, bool PH = false, bool MMA = false>
__global__ void __launch_bounds__(kThreads, MMA ? (NC <= 128 ? 4 : 2) : 1) k_fast_value(FastArgs a) {
  constexpr int CPL = NC / 32;       // codes per lane
  constexpr int WPTOK = NC / 64;     // value words per token
  extern __shared__ __align__(16) unsigned char smem[];
  float* sc = reinterpret_cast<float*>(smem);                                 // [chunk2][G]
  uint64_t* vw = reinterpret_cast<uint64_t*>(sc + (size_t)a.chunk2 * G);     // [chunk2][WPTOK]
  // per-warp z partials [8][NC][G] alias the score / value-word staging,
  // which is dead once the accumulate loop is done (fewer smem bytes per CTA
  // -> more resident CTAs for this latency-bound kernel)
  // (layout as f2_smem: scores, value words, group maxima, then zr unless
  // the staging is large enough to hold it)
  const size_t stage_bytes = (size_t)a.chunk2 * (G * 4 + WPTOK * 8) + (size_t)(a.chunk2 / 32) * G * 4;
  float* zr = stage_bytes >= (size_t)8 * NC * G * 4 ? reinterpret_cast<float*>(smem)
                                                    : reinterpret_cast<float*>(smem + stage_bytes);
  __shared__ float red[8][G];
  __shared__ float mh[G], lh[G];
  const int s = blockIdx.y;
  const long long i0 = (long long)blockIdx.x * a.chunk2;
  const long long i1 = min(a.n, i0 + a.chunk2);
  const int cnt = (int)(i1 - i0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // stage the chunk's value words (token-aligned, 16-B aligned) and, with
  // half weights, the weights and group maxima: bulk copies by one thread
  const uint64_t* vsrc = a.vpool + (size_t)s * a.vstride + (size_t)i0 * WPTOK;
  const int nw = ((cnt * WPTOK + 1) / 2) * 2;
  __shared__ __align__(8) uint64_t tbar;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tbar))
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t bytes = (uint32_t)nw * 8u;
    if constexpr (PH) {
      const int ngr0 = (cnt + 31) >> 5;
      bytes += (uint32_t)((cnt * G * 2 + 15) / 16) * 16u + (uint32_t)((ngr0 * G * 4 + 15) / 16) * 16u;
    }
    asm volatile("{.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tbar)),
                 "r"(bytes)
                 : "memory");
    fv_bulk(vw, vsrc, (uint32_t)nw * 8u, &tbar);
  }
  // programmatic dependent launch: the value words above do not depend on the
  // score kernel; everything below does
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float ls[G];
#pragma unroll
  for (int h = 0; h < G; ++h) ls[h] = 0.f;
  constexpr int kMaxPer = 4;  // tokens per thread: chunk2 <= 4 * kThreads (f2_chunk)
  float pv[kMaxPer][G];       // MMA: this thread's weights until the fp16 write
  if constexpr (PH) {
    // half weights [chunk2][G] in the upper half of the score buffer, the
    // group maxima after the value words (f2_smem adds them); the padded
    // stream stride keeps every source 16-B aligned (reads past cnt stay
    // inside the stream's padding)
    __half* hw = reinterpret_cast<__half*>(sc + (size_t)a.chunk2 * G / 2);
    float* gm = reinterpret_cast<float*>(vw + (size_t)a.chunk2 * WPTOK);  // [chunk2 / 32][G]
    const int ngr = (cnt + 31) >> 5;
    const __half* hsrc = a.ph + ((size_t)s * a.nps + i0) * G;
    const int nh = (cnt * G * 2 + 15) / 16;
    const float* msrc = a.m32 + ((size_t)s * (a.nps >> 5) + (i0 >> 5)) * G;
    const int nm = (ngr * G * 4 + 15) / 16;
    if (tid == 0) {
      fv_bulk(hw, hsrc, (uint32_t)nh * 16u, &tbar);
      fv_bulk(gm, msrc, (uint32_t)nm * 16u, &tbar);
    }
    fv_bar_wait(&tbar, 0);
    if (warp < G) {  // chunk max per head: warp h, lane = group (ngr <= 32)
      float v = lane < ngr ? gm[lane * G + warp] : -INFINITY;
      for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) mh[warp] = v;
    }
    __syncthreads();
    if (tid < ngr * G) {  // group scale exp(m32 - M) in place
      const float mg = gm[tid];
      gm[tid] = mg == -INFINITY ? 0.f : __expf(mg - mh[tid % G]);
    }
    __syncthreads();
    // p = half * group scale, once per (token, head) over the CTA; read
    // into registers first (sc[e] overlaps hw of lower tokens). MMA: the
    // thread takes token pairs (e, e + 1), e = 2 tid + 2 kThreads kp (one
    // 16-B load of both tokens' halves, one half2 store per head below)
    if constexpr (MMA) {
#pragma unroll
      for (int kp = 0; kp < kMaxPer / 2; ++kp) {
        const int e = 2 * tid + kp * 2 * kThreads;
        if (e < cnt) {
          __half hv[2 * G];
          if constexpr (G == 4) {
            *reinterpret_cast<uint4*>(hv) = *reinterpret_cast<const uint4*>(hw + (size_t)e * G);
          } else {
            *reinterpret_cast<__half2*>(hv) = *reinterpret_cast<const __half2*>(hw + (size_t)e * G);
          }
#pragma unroll
          for (int h = 0; h < G; ++h) {
            const float gs = gm[(e >> 5) * G + h];  // e even: e, e + 1 share a group
            pv[2 * kp][h] = __half2float(hv[h]) * gs;
            pv[2 * kp + 1][h] = __half2float(hv[G + h]) * gs;
          }
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < kMaxPer; ++k) {
        const int e = tid + k * kThreads;
        if (e < cnt) {
#pragma unroll
          for (int h = 0; h < G; ++h)
            pv[k][h] = __half2float(hw[(size_t)e * G + h]) * gm[(e >> 5) * G + h];
        }
      }
    }
    __syncthreads();
    if constexpr (!MMA) {
#pragma unroll
      for (int k = 0; k < kMaxPer; ++k) {
        const int e = tid + k * kThreads;
        if (e < cnt) {
#pragma unroll
          for (int h = 0; h < G; ++h) {
            sc[(size_t)e * G + h] = pv[k][h];
            ls[h] += pv[k][h];
          }
        }
      }
    }
  } else {
  // full scores = sum of the JS partials; chunk max per head
  float mx[G];
#pragma unroll
  for (int h = 0; h < G; ++h) mx[h] = -FLT_MAX;
  for (int e = tid; e < cnt; e += kThreads) {
    float v[G];
#pragma unroll
    for (int h = 0; h < G; ++h) v[h] = 0.f;
#pragma unroll
    for (int js = 0; js < JS; ++js) {
      const float* p = a.ps + (((size_t)(s * JS + js) * a.n) + i0 + e) * G;
#pragma unroll
      for (int h = 0; h < G; ++h) v[h] += p[h];
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
      sc[e * G + h] = v[h];
      mx[h] = fmaxf(mx[h], v[h]);
      if (a.scores_out) a.scores_out[((size_t)s * G + h) * a.n + i0 + e] = v[h];
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float v = mx[h];
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[warp][h] = v;
  }
  __syncthreads();
  if (tid < G) {
    float v = red[0][tid];
    for (int w = 1; w < kThreads / 32; ++w) v = fmaxf(v, red[w][tid]);
    mh[tid] = v;
  }
  __syncthreads();
  if constexpr (MMA) {
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) {
      const int e = tid + k * kThreads;
      if (e < cnt) {
#pragma unroll
        for (int h = 0; h < G; ++h) pv[k][h] = __expf(sc[e * G + h] - mh[h]);
      }
    }
    __syncthreads();  // the fp16 weights below overwrite sc
  } else {
    for (int e = tid; e < cnt; e += kThreads) {
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float p = __expf(sc[e * G + h] - mh[h]);
        sc[e * G + h] = p;
        ls[h] += p;
      }
    }
  }
  }  // !PH
  // MMA: fp16 weights PT[h][token] (rows padded by 8 halves: conflict-free
  // B-fragment loads), zero up to the 16-token step; l sums the rounded
  // weights the product uses
  __half* PT = reinterpret_cast<__half*>(smem);
  const int pst = a.chunk2 + 8;
  const int cpad = (cnt + 15) & ~15;
  if constexpr (MMA && PH) {
    // token pairs (e, e + 1) as above; cpad is a multiple of 16 and e even,
    // so e < cpad covers e + 1; weights carried as p 2^15 (see the
    // accumulation below)
#pragma unroll
    for (int kp = 0; kp < kMaxPer / 2; ++kp) {
      const int e = 2 * tid + kp * 2 * kThreads;
      if (e < cpad) {
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const __half2 hv = __floats2half2_rn(e < cnt ? pv[2 * kp][h] * 32768.f : 0.f,
                                               e + 1 < cnt ? pv[2 * kp + 1][h] * 32768.f : 0.f);
          *reinterpret_cast<__half2*>(PT + h * pst + e) = hv;
          const float2 hf = __half22float2(hv);
          ls[h] += (hf.x + hf.y) * (1.f / 32768.f);
        }
      }
    }
  } else if constexpr (MMA) {
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) {
      const int e = tid + k * kThreads;
      if (e < cpad) {
#pragma unroll
        for (int h = 0; h < G; ++h) {
          // weights carried as p 2^15 (see the accumulation below)
          const __half hv = __float2half_rn(e < cnt ? pv[k][h] * 32768.f : 0.f);
          PT[h * pst + e] = hv;
          ls[h] += __half2float(hv) * (1.f / 32768.f);
        }
      }
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float v = ls[h];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][h] = v;
  }
  if constexpr (!PH) fv_bar_wait(&tbar, 0);  // value words (PH waited with the weights)
  __syncthreads();
  if (tid < G) {
    float v = 0.f;
    for (int w = 0; w < kThreads / 32; ++w) v += red[w][tid];
    lh[tid] = v;
  }
  if constexpr (MMA) {
    // warp w takes 16-token steps w, w + 8, ...; thread (g, t) = (lane / 4,
    // lane % 4) holds the fragments of tokens 2t, 2t+1, 2t+8, 2t+9 of the
    // step and codes 16 mt + g (+ 8): byte j of u32 word i of a token's code
    // bits, masked at bit g, is code 32 i + 8 j + g, i.e. m-tile 2 i + j / 2,
    // row g + 8 (j & 1). The mask stays in place (one LOP3 per word): a byte
    // m in {0, 2^g} doubled into both bytes of an fp16 (m << 8 | m, one prmt
    // pairs two tokens' bytes into an A register) is 0 or c_g = fp16(0x0101
    // << g), the same constant for every row this thread supplies (c_7 =
    // -2^-17 has the sign bit; subnormals are exact in the tensor core), so
    // z = D / (2^15 c_g) at the end.
    constexpr int MT = NC / 16, NW32 = NC / 32;
    const int g = lane >> 2, t = lane & 3;
    const uint32_t gmask = 0x01010101u << g;
    float d[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) d[mt][0] = d[mt][1] = d[mt][2] = d[mt][3] = 0.f;
    const uint32_t* vw32 = reinterpret_cast<const uint32_t*>(vw);
    const int nks = cpad >> 4;
#pragma unroll 2
    for (int ks = warp; ks < nks; ks += kThreads / 32) {
      const int k0 = ks << 4;
      uint32_t b0 = 0, b1 = 0;
      if (g < G) {
        b0 = *reinterpret_cast<const uint32_t*>(PT + g * pst + k0 + 2 * t);
        b1 = *reinterpret_cast<const uint32_t*>(PT + g * pst + k0 + 2 * t + 8);
      }
      const uint32_t* wa = vw32 + (size_t)(k0 + 2 * t) * NW32;
#pragma unroll
      for (int i4 = 0; i4 < NW32; i4 += 4) {
        const uint4 A4 = *reinterpret_cast<const uint4*>(wa + i4);
        const uint4 B4 = *reinterpret_cast<const uint4*>(wa + NW32 + i4);
        const uint4 C4 = *reinterpret_cast<const uint4*>(wa + 8 * NW32 + i4);
        const uint4 D4 = *reinterpret_cast<const uint4*>(wa + 9 * NW32 + i4);
        const uint32_t av[4] = {A4.x, A4.y, A4.z, A4.w}, bv[4] = {B4.x, B4.y, B4.z, B4.w};
        const uint32_t cv[4] = {C4.x, C4.y, C4.z, C4.w}, dv[4] = {D4.x, D4.y, D4.z, D4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int mt = 2 * (i4 + u);
          const uint32_t mA = av[u] & gmask, mB = bv[u] & gmask;
          const uint32_t mC = cv[u] & gmask, mD = dv[u] & gmask;
          uint32_t fa[4] = {prmt(mA, mB, 0x4400), prmt(mA, mB, 0x5511), prmt(mC, mD, 0x4400),
                            prmt(mC, mD, 0x5511)};
          mma16816(d[mt], fa, b0, b1);
          uint32_t fb[4] = {prmt(mA, mB, 0x6622), prmt(mA, mB, 0x7733), prmt(mC, mD, 0x6622),
                            prmt(mC, mD, 0x7733)};
          mma16816(d[mt + 1], fb, b0, b1);
        }
      }
    }
    __syncthreads();  // all warps are done with PT / vw (zr may alias them)
    // bits were c_g, weights p 2^15 (fast division: a couple of ulp on z,
    // far inside the fp16 weights' 2^-11)
    const float zsc =
        __fdividef(1.f, 32768.f * __half2float(__ushort_as_half((unsigned short)(0x0101u << g))));
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      float* z0 = zr + ((size_t)warp * NC + 16 * mt + g) * G;
      float* z1 = z0 + 8 * G;
      if (2 * t < G) {
        z0[2 * t] = zsc * d[mt][0];
        z1[2 * t] = zsc * d[mt][2];
      }
      if (2 * t + 1 < G) {
        z0[2 * t + 1] = zsc * d[mt][1];
        z1[2 * t + 1] = zsc * d[mt][3];
      }
    }
    fast_value_finish<NC, G>(a, zr, mh, lh, s);
    return;
  }
  // z[c][h] += p_h(i) * bit_c(i); lane owns codes [CPL*lane, CPL*lane+CPL)
  // heads in pairs so the conditional adds are packed fp32x2 (FADD2)
  constexpr int G2 = (G + 1) / 2;
  float2 z[CPL][G2];
#pragma unroll
  for (int c = 0; c < CPL; ++c)
#pragma unroll
    for (int h = 0; h < G2; ++h) z[c][h] = make_float2(0.f, 0.f);
  const int wsel = (CPL * lane) >> 6, sh = (CPL * lane) & 63;
#pragma unroll 4
  for (int e = warp; e < cnt; e += kThreads / 32) {
    const unsigned bits = (unsigned)(vw[(size_t)e * WPTOK + wsel] >> sh);
    float2 p[G2];
#pragma unroll
    for (int h = 0; h < G2; ++h)
      p[h] = make_float2(sc[e * G + 2 * h], 2 * h + 1 < G ? sc[e * G + 2 * h + 1] : 0.f);
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (bits & (1u << c)) {
#pragma unroll
        for (int h = 0; h < G2; ++h) add2(z[c][h], p[h]);
      }
  }
  __syncthreads();  // all warps are done with sc / vw (zr may alias them)
#pragma unroll
  for (int c = 0; c < CPL; ++c)
#pragma unroll
    for (int h = 0; h < G; ++h)
      zr[((size_t)warp * NC + CPL * lane + c) * G + h] = (h & 1) ? z[c][h / 2].y : z[c][h / 2].x;
  fast_value_finish<NC, G>(a, zr, mh, lh, s);
}

// subspace split (CTAs per stream) so the codebook slice fits in smem
int js_for(const AttnJob& job) {
  if (job.cb_key_tc) return tc_blocks(job);          // tcgen05: round blocks of 11
  if (job.cb_key16) return job.geo.R <= 13 ? 1 : 2;  // fp16: 16 KiB per round
  return job.geo.R <= 12 ? 2 : 4;                    // fp32: 32 KiB per round
}

size_t f1_smem(int R, int JC, int esize) {
  return (size_t)R * 64 * JC * esize + 2 * 24 * R * 8 + (size_t)kTile * (((2 * R + 15) / 16) * 16);
}

int f1_chunk(const AttnJob& job) {
  const int JS = js_for(job);
  long long want = (job.n * (long long)job.S * JS + 2 * 148 - 1) / (2 * 148);
  long long ch = (want + kTile - 1) / kTile * kTile;
  if (ch < 512) ch = 512;
  if (ch > 8192) ch = 8192;
  return (int)ch;
}

int f2_chunk(const AttnJob& job) {
  long long want = (job.n * (long long)job.S + 2 * 148 - 1) / (2 * 148);
  long long ch = (want + kTile - 1) / kTile * kTile;
  if (ch < 256) ch = 256;
  // 32 KiB smem -> 6 CTAs/SM (latency-bound kernel); measured on C3: 1024 and
  // 2048 tie, 512 and 4096 are slower
#ifndef CVQ_F2_MAXCHUNK
#define CVQ_F2_MAXCHUNK 1024
#endif
  if (ch > CVQ_F2_MAXCHUNK) ch = CVQ_F2_MAXCHUNK;
  return (int)ch;
}

size_t f2_smem(const AttnJob& job, int chunk2) {
  const Geom& g = job.geo;
  // scores / weights, value words, group maxima (half-weight mode)
  const size_t stage = (size_t)chunk2 * g.G * 4 + (size_t)chunk2 * (g.n_codes / 64) * 8 +
                       (size_t)(chunk2 / 32) * g.G * 4;
  const size_t zr = (size_t)8 * g.n_codes * g.G * 4;
  return (stage >= zr ? stage : stage + zr) + 16;  // zr aliases the staging when it fits
}

// launch with programmatic stream serialization: the kernel may start while
// its predecessor drains and waits in griddepcontrol.wait for its results
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

template <class K>
cudaError_t set_smem(K kernel, size_t sm) {
  return ensure_dyn_smem(reinterpret_cast<const void*>(kernel), sm);
}

template <int R, int G>
cudaError_t launch_f1(const FastArgs& a, int S, cudaStream_t st) {
  constexpr int JC = R <= 12 ? 32 : 16;
  constexpr int JS = 64 / JC;
  const size_t sm = f1_smem(R, JC, 8);
  cudaError_t e = set_smem(k_fast_score<R, JC, G>, sm);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.n + a.chunk - 1) / a.chunk), S * JS);
  k_fast_score<R, JC, G><<<grid, kF1Threads, sm, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <int R, int G>
cudaError_t launch_f1h(const FastArgs& a, int S, cudaStream_t st) {
  // 16 lanes x 4 subspaces per token; the whole codebook per CTA for R <= 13
  constexpr int SPL = R <= 13 ? 4 : 2;
  constexpr int LPT = 16;
  constexpr int JS = 64 / (SPL * LPT);
  const size_t sm = f1_smem(R, SPL * LPT, 4);
  cudaError_t e = set_smem(k_fast_score_h<R, SPL, LPT, G>, sm);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.n + a.chunk - 1) / a.chunk), S * JS);
  k_fast_score_h<R, SPL, LPT, G><<<grid, kF1Threads, sm, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <int NC, int G, int JS, bool PH = false, bool MMA = false>
cudaError_t launch_f2(const FastArgs& a, size_t sm, cudaStream_t st) {
  cudaError_t e = set_smem(k_fast_value<NC, G, JS, PH, MMA>, sm);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.n + a.chunk2 - 1) / a.chunk2), a.S);
  e = launch_pdl(k_fast_value<NC, G, JS, PH, MMA>, grid, dim3(kThreads), sm, st, a);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

template <int NC, int G>
cudaError_t launch_f2_js(const FastArgs& a, int JS, bool mma, size_t sm, cudaStream_t st) {
  if (a.ph) return launch_f2<NC, G, 1, true, true>(a, sm, st);
  if (mma) return JS == 1 ? launch_f2<NC, G, 1, false, true>(a, sm, st)
                          : launch_f2<NC, G, 2, false, true>(a, sm, st);
  switch (JS) {
    case 1: return launch_f2<NC, G, 1>(a, sm, st);
    case 2: return launch_f2<NC, G, 2>(a, sm, st);
    default: return launch_f2<NC, G, 4>(a, sm, st);
  }
}

// Merge of the chunk partials (m_p, l_p, z_p) of one row (flash-decoding
// LSE merge; the reference softmax is global, linalg.cpp:63-75), then the
// value codebook product o = z . C_V / L once per row (attn.cpp:249-256).
// LSE merge of the chunk partials of every row, parallel over (row, 32-code
// slice): grid (rows, NC / 32), 8 warps; warp w takes the parts p = w (mod
// 8), lane = code -> coalesced 128-B rows of z.  Writes the merged,
// unnormalised z[row][NC] and (M, L) per row.  (One CTA per row serialised
// over the parts took 0.5 ms at C5: 32 rows x 128 chunks.)
template <int NC>
__global__ void __launch_bounds__(256) k_combine_merge(const float* __restrict__ m,
                                                       const float* __restrict__ l,
                                                       const float* __restrict__ z, int P,
                                                       long long rows, float* __restrict__ zm) {
  __shared__ float part[8][32];
  __shared__ float red[8];
  __shared__ float Ms, Lsh;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the value kernel's partials
  const long long row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float M = -FLT_MAX;
  for (int p = tid; p < P; p += 256)
    if (l[p * rows + row] > 0.f) M = fmaxf(M, m[p * rows + row]);
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  if (lane == 0) red[warp] = M;
  __syncthreads();
  if (tid == 0) {
    float v = red[0];
    for (int w = 1; w < 8; ++w) v = fmaxf(v, red[w]);
    Ms = v;
  }
  __syncthreads();
  M = Ms;
  const int k = blockIdx.y * 32 + lane;
  float acc = 0.f, Lp = 0.f;
#pragma unroll 4
  for (int p = warp; p < P; p += 8) {
    const float lp = l[p * rows + row];
    const float wgt = lp > 0.f ? expf(m[p * rows + row] - M) : 0.f;
    Lp += lp * wgt;
    if (wgt != 0.f) acc += z[(p * rows + row) * NC + k] * wgt;
  }
  part[warp][lane] = acc;
  if (lane == 0) red[warp] = Lp;
  __syncthreads();
  if (warp == 0) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += part[w][lane];
    zm[row * (NC + 2) + k] = v;
    if (blockIdx.y == 0 && lane == 0) {
      float L = 0.f;
      for (int w = 0; w < 8; ++w) L += red[w];
      zm[row * (NC + 2) + NC] = M;
      zm[row * (NC + 2) + NC + 1] = L;
    }
  }
}

// o = z C_V / L per row (attn.cpp:249-256): one CTA of 128 threads per row,
// thread = output dim, value codebook rows coalesced.
template <int NC>
__global__ void __launch_bounds__(128) k_combine_project(const float* __restrict__ zm,
                                                         long long rows, int G,
                                                         const float* __restrict__ cbv, int n_slots,
                                                         float* __restrict__ out,
                                                         float* __restrict__ m_out,
                                                         float* __restrict__ l_out) {
  __shared__ float zs[NC];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the merged z rows
  const long long row = blockIdx.x;
  const float* zr = zm + row * (NC + 2);
  for (int k = threadIdx.x; k < NC; k += 128) zs[k] = zr[k];
  __syncthreads();
  const float Lsum = zr[NC + 1];
  const float* cb = cbv + (size_t)((row / G) % n_slots) * NC * 128;
  const int jd = threadIdx.x;
  float acc = 0.f;
#pragma unroll 8
  for (int k = 0; k < NC; ++k) acc += zs[k] * __ldg(cb + (size_t)k * 128 + jd);
  out[row * 128 + jd] = acc / Lsum;
  if (jd == 0) {
    if (m_out) m_out[row] = zr[NC];
    if (l_out) l_out[row] = Lsum;
  }
}

// Small jobs (few chunk partials): merge + project in ONE kernel, a CTA per
// row (grid streams x G): the LSE weights of the P parts (warp 0), z[k] =
// sum_p w_p z_p[k] with the parts split over 4 thread groups, then
// o[:] = z . C_V / L with the k range split over 4 thread groups.  One
// launch instead of two, no zm round trip, every sequential chain <= P/4 or
// NC/4 long.
constexpr int kCfThreads = 512, kCfMaxP = 64;
template <int NC>
__global__ void __launch_bounds__(kCfThreads) k_combine_fused(
    const float* __restrict__ m, const float* __restrict__ l, const float* __restrict__ z, int P,
    long long rows, int G, const float* __restrict__ cbv, int n_slots, float* __restrict__ out,
    float* __restrict__ m_out, float* __restrict__ l_out) {
  __shared__ float wts[kCfMaxP];
  __shared__ float Ms, Ls;
  __shared__ float zp[4][NC];
  __shared__ float zs[NC];
  __shared__ float part[4][128];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the value kernel's partials
  const int s = blockIdx.x, tid = threadIdx.x, q = tid >> 7, t = tid & 127;
  const long long row = (long long)s * G + blockIdx.y;
  if (tid < 32) {
    float M = -FLT_MAX;
    for (int p = tid; p < P; p += 32)
      if (l[p * rows + row] > 0.f) M = fmaxf(M, m[p * rows + row]);
    for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    for (int p = tid; p < P; p += 32) {
      const float lp = l[p * rows + row];
      const float w = lp > 0.f ? expf(m[p * rows + row] - M) : 0.f;
      wts[p] = w;
      L += lp * w;
    }
    for (int o = 16; o; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (tid == 0) {
      Ms = M;
      Ls = L;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = t; k < NC; k += 128) {
    float acc = 0.f;
#pragma unroll 4
    for (int p = q; p < P; p += 4) {
      const float w = wts[p];
      if (w != 0.f) acc += z[(p * rows + row) * NC + k] * w;
    }
    zp[q][k] = acc;
  }
  __syncthreads();
  for (int k = tid; k < NC; k += kCfThreads) zs[k] = zp[0][k] + zp[1][k] + zp[2][k] + zp[3][k];
  __syncthreads();
  const float* cb = cbv + (size_t)(s % n_slots) * NC * 128;
  float acc = 0.f;
#pragma unroll 8
  for (int k = q * (NC / 4); k < (q + 1) * (NC / 4); ++k) acc += zs[k] * __ldg(cb + (size_t)k * 128 + t);
  part[q][t] = acc;
  __syncthreads();
  if (tid < 128) out[row * 128 + tid] = (part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid]) / Ls;
  if (tid == 0) {
    if (m_out) m_out[row] = Ms;
    if (l_out) l_out[row] = Ls;
  }
}

}  // namespace

cudaError_t run_fast_combine(const AttnJob& job, const float* pm, const float* pl,
                             const float* pz, int n_parts, float* out, float* m_out,
                             float* l_out, float* zm, cudaStream_t st) {
  const long long rows = (long long)job.S * job.geo.G;
  if (rows == 0) return cudaSuccess;
  const int NC = job.geo.n_codes;
  dim3 gm((unsigned)rows, NC / 32);
  if (n_parts <= kCfMaxP && job.geo.d == 128) {
    const dim3 grid((unsigned)job.S, (unsigned)job.geo.G);
    if (NC == 128)
      launch_pdl(k_combine_fused<128>, grid, dim3(kCfThreads), 0, st, pm, pl, pz, n_parts, rows,
                 job.geo.G, job.cb_val, job.n_slots, out, m_out, l_out);
    else
      launch_pdl(k_combine_fused<256>, grid, dim3(kCfThreads), 0, st, pm, pl, pz, n_parts, rows,
                 job.geo.G, job.cb_val, job.n_slots, out, m_out, l_out);
    count_launch(1);
    return cudaGetLastError();
  }
  if (NC == 128) {
    launch_pdl(k_combine_merge<128>, gm, dim3(256), 0, st, pm, pl, pz, n_parts, rows, zm);
    launch_pdl(k_combine_project<128>, dim3((unsigned)rows), dim3(128), 0, st, zm, rows,
               job.geo.G, job.cb_val, job.n_slots, out, m_out, l_out);
  } else {
    launch_pdl(k_combine_merge<256>, gm, dim3(256), 0, st, pm, pl, pz, n_parts, rows, zm);
    launch_pdl(k_combine_project<256>, dim3((unsigned)rows), dim3(128), 0, st, zm, rows,
               job.geo.G, job.cb_val, job.n_slots, out, m_out, l_out);
  }
  count_launch(2);
  return cudaGetLastError();
}

bool fast_path_applies(const AttnJob& job) {
  const Geom& g = job.geo;
  if (job.variant & kVarGeneric) return false;
  return g.d == 128 && g.groups == 1 && g.L == 64 && (g.R == 11 || g.R == 21) &&
         (g.n_codes == 128 || g.n_codes == 256) && (g.G == 1 || g.G == 4) && job.n > 0;
}

// single fused kernel (k_fast_attn_h): 1-bit fp16-codebook preset, GQA 4
bool fused_applies(const AttnJob& job) {
  const Geom& g = job.geo;
  // Measured slower than score + value kernels on C3 (20.2 vs 19.5 ms: the
  // score loop is issue-bound, so in-loop value work costs more than the
  // separate kernel); opt-in only.
  return job.cb_key16 && !job.cb_key_tc && g.R == 11 && g.G == 4 && g.n_codes == 128 &&
         (job.variant & kVarFused);
}

size_t fast_scratch_bytes(const AttnJob& job, int* n_chunks) {
  const int JS = js_for(job);
  const int c2 = f2_chunk(job);
  *n_chunks = (int)((job.n + c2 - 1) / c2);
  if (fused_applies(job)) {
    const int c1 = f1_chunk(job);
    *n_chunks = std::max(*n_chunks, (int)((job.n + c1 - 1) / c1));
  }
  size_t ps = (size_t)job.S * JS * job.n * job.geo.G * sizeof(float);
  if (tc_half_scores(job)) {  // half weights + group maxima (run_attention_fast)
    const size_t nps = (size_t)(job.n + kTile - 1) / kTile * kTile;
    const size_t hb = ((size_t)job.S * nps * job.geo.G * 2 + 255) / 256 * 256 +
                      (size_t)job.S * (nps / 32) * job.geo.G * 4;
    ps = std::max(ps, hb);
  }
  return (ps + 255) / 256 * 256;
}

cudaError_t run_attention_fast(const AttnJob& job, const float* q, float* pm, float* pl,
                               float* po, int* n_chunks, void* scratch, cudaStream_t st,
                               cudaEvent_t* prof, float* scores_out) {
  const Geom& g = job.geo;
  FastArgs a{};
  a.kpool = job.kpool;
  a.kstride = job.kstride;
  a.vpool = job.vpool;
  a.vstride = job.vstride;
  a.cb = job.cb_key;
  a.cbh = job.cb_key16;
  a.cbv = job.cb_val;
  a.n_slots = job.n_slots;
  a.q = q;
  a.thetas = job.thetas;
  a.t = job.t;
  a.pos0 = job.pos0;
  a.n = job.n;
  a.chunk = f1_chunk(job);
  a.chunk2 = f2_chunk(job);
  a.S = job.S;
  a.ps = static_cast<float*>(scratch);
  a.scores_out = scores_out;
  a.pm = pm;
  a.pl = pl;
  a.po = po;
  cudaError_t e;
  if (fused_applies(job) && !scores_out) {
    const size_t sm = (size_t)11 * 64 * 64 * 4 + 2 * 24 * 11 * 8 + 2 * 2 * kTile * 8 +
                      (kF1Threads / 32) * 8 * 16 + (size_t)kTile * 32;
    if ((e = set_smem(k_fast_attn_h<11>, sm)) != cudaSuccess) return e;
    const int nc = (int)((job.n + a.chunk - 1) / a.chunk);
    if (prof) cudaEventRecord(prof[0], st);
    k_fast_attn_h<11><<<dim3((unsigned)nc, job.S), kF1Threads, sm, st>>>(a);
    count_launch();
    if (prof) cudaEventRecord(prof[1], st);
    *n_chunks = nc;
    return cudaGetLastError();
  }
  *n_chunks = (int)((job.n + a.chunk2 - 1) / a.chunk2);
  if (prof) cudaEventRecord(prof[0], st);
  if (job.cb_key_tc) {
    HalfOut ho{};
    const bool half = !scores_out && tc_half_scores(job);
    if (half) {
      ho.nps = (job.n + kTile - 1) / kTile * kTile;
      ho.ph = scratch;
      ho.m32 = reinterpret_cast<float*>(static_cast<char*>(scratch) +
                                        ((size_t)job.S * ho.nps * g.G * 2 + 255) / 256 * 256);
      a.ph = static_cast<const __half*>(ho.ph);
      a.m32 = ho.m32;
      a.nps = ho.nps;
    }
    e = run_tc_score(job, q, a.ps, a.chunk, st, half ? &ho : nullptr);
  } else if (job.cb_key16) {
    if (g.R == 11)
      e = g.G == 4 ? launch_f1h<11, 4>(a, job.S, st) : launch_f1h<11, 1>(a, job.S, st);
    else
      e = g.G == 4 ? launch_f1h<21, 4>(a, job.S, st) : launch_f1h<21, 1>(a, job.S, st);
  } else {
    if (g.R == 11)
      e = g.G == 4 ? launch_f1<11, 4>(a, job.S, st) : launch_f1<11, 1>(a, job.S, st);
    else
      e = g.G == 4 ? launch_f1<21, 4>(a, job.S, st) : launch_f1<21, 1>(a, job.S, st);
  }
  if (prof) cudaEventRecord(prof[1], st);
  if (e != cudaSuccess) return e;
  const size_t sm2 = f2_smem(job, a.chunk2);
  const int JS = js_for(job);
  // tensor-core value accumulation (fp16 weights) in the tcgen05 key modes
  // unless the cache asked for the fp32 hand-off
  const bool mma = job.cb_key_tc && !(job.variant & kVarF32W) && !scores_out && JS <= 2;
  if (g.n_codes == 128)
    e = g.G == 4 ? launch_f2_js<128, 4>(a, JS, mma, sm2, st)
                 : launch_f2_js<128, 1>(a, JS, mma, sm2, st);
  else
    e = g.G == 4 ? launch_f2_js<256, 4>(a, JS, mma, sm2, st)
                 : launch_f2_js<256, 1>(a, JS, mma, sm2, st);
  return e;
}

}  // namespace cvq
