// naive.cu -- the decode-then-attend pathway (naive_quantized_attention,
// attn.cpp:130-162) as a real GPU baseline for the fused kernels
// (Table 4 compares the two).
//
// What a KV-cache implementation without the commutative trick does at
// every decode step:
//   1. dequantise the whole cache: every key K_hat_j(i) = sum_r U[r,j,a_r] +
//      i U[r,j,b_r] rotated to its own position (apply_rope, rope.cpp:44-58),
//      every value V_hat(i) = sum_c bit_c(i) C_V[c] (valquant.cpp:115-128),
//      stored fp16 (a dense KV cache) -- 512 B per token and stream at d = 128
//      against 32.5 B of codes;
//   2. dense decode attention over it: q rotated to t, s_i = q.K_hat(i) /
//      sqrt(d), flash-decoding split over context chunks, each chunk's
//      (m, l, o) merged by the LSE combine kernel.
// Multi-stream (every (seq, layer, kv head) stream, G query heads each) and
// any key geometry (groups, L, R); fp32 arithmetic, fp16 storage.
#include <cuda_fp16.h>

#include "cvq_internal.cuh"

namespace cvq {

namespace {

constexpr int kDqTok = 32;      // tokens per dequantisation CTA
constexpr int kAtChunk = 1024;  // tokens per attention CTA (flash-decoding split)

// grid (ceil(n / kDqTok), S), blockDim = max(d, 64): thread e < d/2 owns
// subspace j = e for the keys of tokens of parity (e / (d/2)), every thread
// owns value dim e.
template <class T>
__device__ __forceinline__ T to_store(float v);
template <>
__device__ __forceinline__ __half to_store<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ float to_store<float>(float v) { return v; }
__device__ __forceinline__ float from_store(__half v) { return __half2float(v); }
__device__ __forceinline__ float from_store(float v) { return v; }

template <class T>
__global__ void k_naive_dequant(Geom g, const uint64_t* __restrict__ kpool, uint64_t kstride,
                                const uint64_t* __restrict__ vpool, uint64_t vstride,
                                const float2* __restrict__ cbk, const float* __restrict__ cbv,
                                int n_slots, const double* __restrict__ thetas, long long pos0,
                                long long n, T* __restrict__ Kh, T* __restrict__ Vh,
                                bool values_by_mma) {
  const int s = blockIdx.y, tid = threadIdx.x, slot = s % n_slots;
  const long long t0 = (long long)blockIdx.x * kDqTok;
  const int nt = (int)min((long long)kDqTok, n - t0);
  const uint64_t* kw = kpool + (size_t)s * kstride;
  const uint64_t* vw = vpool + (size_t)s * vstride;
  const float2* cb = cbk + (size_t)slot * g.R * g.L * g.subs;
  const float* cv = cbv + (size_t)slot * g.n_codes * g.d;
  // keys: two tokens per pass (threads [0, subs) and [subs, 2 subs))
  const int half = tid / g.subs, j = tid % g.subs;
  if (half < 2) {
    const int grp = j / g.g;
    const double th = thetas[j];
    for (int tt = half; tt < nt; tt += 2) {
      const long long i = t0 + tt;
      const unsigned long long f0 = (unsigned long long)i * g.fpt;
      float kx = 0.f, ky = 0.f;
      for (int r = 0; r < g.R; ++r) {
        const unsigned long long f = f0 + (unsigned long long)(r * g.groups + grp) * 2;
        const unsigned a = read_field(kw, f * g.lb, g.lb);
        const unsigned b = read_field(kw, (f + 1) * g.lb, g.lb);
        const float2 ua = __ldg(cb + ((size_t)r * g.L + a) * g.subs + j);
        const float2 ub = __ldg(cb + ((size_t)r * g.L + b) * g.subs + j);
        kx += ua.x - ub.y;  // u_a + v_b, v_b = (-y_b, x_b)
        ky += ua.y + ub.x;
      }
      const float2 p = phase_neg(-(pos0 + i), th);  // e^{+i pos theta}
      T* kr = Kh + ((size_t)s * n + i) * g.d;
      kr[2 * j] = to_store<T>(kx * p.x - ky * p.y);
      kr[2 * j + 1] = to_store<T>(kx * p.y + ky * p.x);
    }
  }
  if (values_by_mma) return;  // k_naive_values_mma reconstructs V
  // values: dim e of every token (coalesced codebook rows, broadcast bits)
  for (int e = tid; e < g.d; e += blockDim.x) {
    for (int tt = 0; tt < nt; ++tt) {
      const long long i = t0 + tt;
      float v = 0.f;
      const unsigned long long b0 = (unsigned long long)i * g.n_codes;
      for (int c = 0; c < g.n_codes; ++c) {
        const unsigned long long bit = b0 + c;
        if ((__ldg(vw + (bit >> 6)) >> (bit & 63)) & 1ull) v += __ldg(cv + (size_t)c * g.d + e);
      }
      Vh[((size_t)s * n + i) * g.d + e] = to_store<T>(v);
    }
  }
}

// Value dequantisation as the dense GEMM it is: V_hat[64 tok][d] =
// bits[64 tok][N_c] (exact fp16 0/1) x C_V[N_c][d] (fp16) on the tensor cores
// (mma.sync m16n8k16, fp32 accumulate), d = 128, N_c a multiple of 16
// (<= 256).  grid (ceil(n / 64), S), 4 warps x 16 tokens.
constexpr int kVmTok = 64;
__global__ void __launch_bounds__(128) k_naive_values_mma(Geom g, const uint64_t* __restrict__ vpool,
                                                          uint64_t vstride,
                                                          const float* __restrict__ cbv, int n_slots,
                                                          long long n, __half* __restrict__ Vh) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int NCP = g.n_codes + 8;                            // padded row (bank spread)
  __half* Bt = reinterpret_cast<__half*>(smem);             // [128 d][NCP] = C_V^T
  __half* As = Bt + (size_t)128 * NCP;                      // [64 tok][NCP] bits
  const int s = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long t0 = (long long)blockIdx.x * kVmTok;
  const int nt = (int)min((long long)kVmTok, n - t0);
  const float* cv = cbv + (size_t)(s % n_slots) * g.n_codes * 128;
  for (int e = tid; e < g.n_codes * 128; e += blockDim.x) {
    const int c = e / 128, dd = e % 128;
    Bt[(size_t)dd * NCP + c] = __float2half_rn(cv[e]);
  }
  const uint64_t* vw = vpool + (size_t)s * vstride;
  for (int e = tid; e < kVmTok * g.n_codes; e += blockDim.x) {
    const int tt = e / g.n_codes, c = e % g.n_codes;
    float bit = 0.f;
    if (tt < nt) {
      const unsigned long long b = (unsigned long long)(t0 + tt) * g.n_codes + c;
      bit = (float)((__ldg(vw + (b >> 6)) >> (b & 63)) & 1ull);
    }
    As[(size_t)tt * NCP + c] = __float2half_rn(bit);
  }
  __syncthreads();
  const int r0 = warp * 16 + (lane >> 2), kq = (lane & 3) * 2;
  for (int nb = 0; nb < 16; ++nb) {  // 8 output dims per n-tile
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    for (int ks = 0; ks < g.n_codes; ks += 16) {
      const uint32_t a0 = *reinterpret_cast<const uint32_t*>(As + (size_t)r0 * NCP + ks + kq);
      const uint32_t a1 = *reinterpret_cast<const uint32_t*>(As + (size_t)(r0 + 8) * NCP + ks + kq);
      const uint32_t a2 = *reinterpret_cast<const uint32_t*>(As + (size_t)r0 * NCP + ks + kq + 8);
      const uint32_t a3 = *reinterpret_cast<const uint32_t*>(As + (size_t)(r0 + 8) * NCP + ks + kq + 8);
      const int ncol = nb * 8 + (lane >> 2);
      const uint32_t b0 = *reinterpret_cast<const uint32_t*>(Bt + (size_t)ncol * NCP + ks + kq);
      const uint32_t b1 = *reinterpret_cast<const uint32_t*>(Bt + (size_t)ncol * NCP + ks + kq + 8);
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
          "{%8, %9}, {%0, %1, %2, %3};"
          : "+f"(c0), "+f"(c1), "+f"(c2), "+f"(c3)
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    const int col = nb * 8 + kq;
    if (r0 < nt)
      *reinterpret_cast<__half2*>(Vh + ((size_t)s * n + t0 + r0) * 128 + col) = __floats2half2_rn(c0, c1);
    if (r0 + 8 < nt)
      *reinterpret_cast<__half2*>(Vh + ((size_t)s * n + t0 + r0 + 8) * 128 + col) =
          __floats2half2_rn(c2, c3);
  }
}

// grid (chunks, S), 128 threads.  Scores: a warp per token, lanes over the
// dims (half2 each); then chunk softmax stats per head; then o_d = sum p V.
template <int G, class T>
__global__ void __launch_bounds__(128) k_naive_attend(Geom g, const T* __restrict__ Kh,
                                                      const T* __restrict__ Vh,
                                                      const float* __restrict__ q,
                                                      const double* __restrict__ thetas,
                                                      long long t, long long n,
                                                      float* __restrict__ pm, float* __restrict__ pl,
                                                      float* __restrict__ po, long long rows) {
  __shared__ float qs[G][256];
  __shared__ float sc[kAtChunk][G];
  __shared__ float red[4][G];
  __shared__ float mh[G], lh[G];
  const int s = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long i0 = (long long)blockIdx.x * kAtChunk;
  const int cnt = (int)min((long long)kAtChunk, n - i0);
  const float rs = rsqrtf((float)g.d);
  // q_h rotated to t (apply_rope) and scaled by 1/sqrt(d)
  for (int e = tid; e < G * g.subs; e += blockDim.x) {
    const int h = e / g.subs, j = e % g.subs;
    const float2 p = phase_neg(-t, thetas[j]);
    const float* qh = q + ((size_t)s * G + h) * g.d;
    const float qx = qh[2 * j], qy = qh[2 * j + 1];
    qs[h][2 * j] = (qx * p.x - qy * p.y) * rs;
    qs[h][2 * j + 1] = (qx * p.y + qy * p.x) * rs;
  }
  __syncthreads();
  for (int tt = warp; tt < cnt; tt += 4) {
    const T* kr = Kh + ((size_t)s * n + i0 + tt) * g.d;
    float acc[G];
#pragma unroll
    for (int h = 0; h < G; ++h) acc[h] = 0.f;
    for (int e = 2 * lane; e < g.d; e += 64) {
      const float k0 = from_store(kr[e]), k1 = from_store(kr[e + 1]);
#pragma unroll
      for (int h = 0; h < G; ++h) acc[h] += qs[h][e] * k0 + qs[h][e + 1] * k1;
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float v = acc[h];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) sc[tt][h] = v;
    }
  }
  __syncthreads();
  float mx[G];
#pragma unroll
  for (int h = 0; h < G; ++h) mx[h] = -FLT_MAX;
  for (int tt = tid; tt < cnt; tt += blockDim.x)
#pragma unroll
    for (int h = 0; h < G; ++h) mx[h] = fmaxf(mx[h], sc[tt][h]);
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float v = mx[h];
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[warp][h] = v;
  }
  __syncthreads();
  if (tid < G) mh[tid] = fmaxf(fmaxf(red[0][tid], red[1][tid]), fmaxf(red[2][tid], red[3][tid]));
  __syncthreads();
  float ls[G];
#pragma unroll
  for (int h = 0; h < G; ++h) ls[h] = 0.f;
  for (int tt = tid; tt < cnt; tt += blockDim.x)
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float p = __expf(sc[tt][h] - mh[h]);
      sc[tt][h] = p;
      ls[h] += p;
    }
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float v = ls[h];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][h] = v;
  }
  __syncthreads();
  if (tid < G) lh[tid] = red[0][tid] + red[1][tid] + red[2][tid] + red[3][tid];
  __syncthreads();
  for (int e = tid; e < g.d; e += blockDim.x) {
    float o[G];
#pragma unroll
    for (int h = 0; h < G; ++h) o[h] = 0.f;
    for (int tt = 0; tt < cnt; ++tt) {
      const float v = from_store(Vh[((size_t)s * n + i0 + tt) * g.d + e]);
#pragma unroll
      for (int h = 0; h < G; ++h) o[h] += sc[tt][h] * v;
    }
#pragma unroll
    for (int h = 0; h < G; ++h)
      po[((size_t)blockIdx.x * rows + (size_t)s * G + h) * g.d + e] = o[h] / lh[h];
  }
  if (tid < G) {
    pm[(size_t)blockIdx.x * rows + (size_t)s * G + tid] = mh[tid];
    pl[(size_t)blockIdx.x * rows + (size_t)s * G + tid] = lh[tid];
  }
}

template <int G, class T>
cudaError_t launch_attend(const AttnJob& job, const T* Kh, const T* Vh, const float* q,
                          float* pm, float* pl, float* po, int nc, cudaStream_t st) {
  dim3 grid((unsigned)nc, job.S);
  k_naive_attend<G, T><<<grid, 128, 0, st>>>(job.geo, Kh, Vh, q, job.thetas, job.t, job.n, pm, pl, po,
                                          (long long)job.S * G);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

size_t naive_scratch_bytes(const AttnJob& job, bool exact) {
  const Geom& g = job.geo;
  const size_t kv = (size_t)job.S * job.n * g.d * 2 * (exact ? sizeof(float) : sizeof(__half));
  const size_t nc = (size_t)((job.n + kAtChunk - 1) / kAtChunk);
  const size_t rows = (size_t)job.S * g.G;
  return kv + nc * rows * (2 + g.d) * sizeof(float) + 512;
}

template <class T>
static cudaError_t naive_impl(const AttnJob& job, const float* q, float* out, void* scratch,
                              cudaStream_t st, bool mma) {
  const Geom& g = job.geo;
  T* Kh = static_cast<T*>(scratch);
  T* Vh = Kh + (size_t)job.S * job.n * g.d;
  const int nc = (int)((job.n + kAtChunk - 1) / kAtChunk);
  const size_t rows = (size_t)job.S * g.G;
  float* pm = reinterpret_cast<float*>(Vh + (size_t)job.S * job.n * g.d);
  float* pl = pm + (size_t)nc * rows;
  float* po = pl + (size_t)nc * rows;
  dim3 gd((unsigned)((job.n + kDqTok - 1) / kDqTok), job.S);
  const int thr = g.d > 64 ? (g.d + 31) / 32 * 32 : 64;
  k_naive_dequant<T><<<gd, thr, 0, st>>>(g, job.kpool, job.kstride, job.vpool, job.vstride,
                                         job.cb_key, job.cb_val, job.n_slots, job.thetas, job.pos0,
                                         job.n, Kh, Vh, mma);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if constexpr (sizeof(T) == 2) {
    if (mma) {
      const size_t sm = (size_t)(128 + kVmTok) * (g.n_codes + 8) * sizeof(__half);
      if ((e = ensure_dyn_smem(reinterpret_cast<const void*>(k_naive_values_mma), sm)) != cudaSuccess)
        return e;
      dim3 gv((unsigned)((job.n + kVmTok - 1) / kVmTok), job.S);
      k_naive_values_mma<<<gv, 128, sm, st>>>(g, job.vpool, job.vstride, job.cb_val, job.n_slots,
                                               job.n, Vh);
      count_launch();
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  switch (g.G) {
    case 1: e = launch_attend<1, T>(job, Kh, Vh, q, pm, pl, po, nc, st); break;
    case 2: e = launch_attend<2, T>(job, Kh, Vh, q, pm, pl, po, nc, st); break;
    case 4: e = launch_attend<4, T>(job, Kh, Vh, q, pm, pl, po, nc, st); break;
    case 8: e = launch_attend<8, T>(job, Kh, Vh, q, pm, pl, po, nc, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return run_lse_combine(pm, pl, po, nc, (long long)rows, g.d, out, nullptr, nullptr, st);
}

// Decode-then-attend for every (stream, q head): out [S][G][d] (device).
// exact: fp32 storage and CUDA-core value sums (the reference-API mirror,
// cvq_naive_attention); otherwise the fp16 dense-cache baseline with the
// value dequantisation on the tensor cores (d = 128).
cudaError_t run_naive_attention(const AttnJob& job, const float* q, float* out, void* scratch,
                                size_t scratch_bytes, cudaStream_t st, bool exact) {
  const Geom& g = job.geo;
  if (scratch_bytes < naive_scratch_bytes(job, exact) || g.d > 256 || g.G > 8 || job.n <= 0)
    return cudaErrorInvalidValue;
  if (exact) return naive_impl<float>(job, q, out, scratch, st, false);
  const bool mma = g.d == 128 && g.n_codes % 16 == 0 && g.n_codes <= 256;
  return naive_impl<__half>(job, q, out, scratch, st, mma);
}

}  // namespace cvq
