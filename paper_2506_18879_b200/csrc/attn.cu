// attn.cu -- CommVQ decode attention over a packed code cache (sm_100a).
//
// Replaces fused_attention (attn.cpp:164-263).  Algebra (verified against
// attn.cpp:192-234): with q_j = q[2j] + i q[2j+1], atoms U = x + iy and the
// per-round key k_j = U[r,j,a_r] + i U[r,j,b_r] (cluster_center,
// keyquant.cpp:98-114),
//
//   score(i) = Re sum_j conj(q_j) e^{-i (t - pos_i) theta_j} K_j / sqrt(d),
//   K_j      = sum_r U[r,j,a_r(i)] + i U[r,j,b_r(i)].
//
// The reference folds q through the atoms (px, py) and rotates per token; we
// decode K once per KV stream and share it across the q_per_kv query heads
// (GQA), which is 4x less gather work than a per-query LUT.
//
// This file holds the generic path (any d, g, L, R, N_c -- the reference's
// pinned test shapes) and the dispatcher; the specialised fast path for the
// LLaMA-shaped presets lives in attn_fast.cu.
#include <cfloat>
#include <cmath>

#include <algorithm>

#include "cvq_internal.cuh"

namespace cvq {

constexpr int kMaxG = 8;  // query heads per KV stream supported

// ---------------------------------------------------------------- scores
// One thread per token; K_j decoded on the fly from the packed stream
// (L1/L2-resident codebook), phase per (token, subspace) from an fp64
// reduced angle.  Writes scores[s][h][i].
template <int MAXG>
__global__ void __launch_bounds__(128)
k_score_generic(Geom g, const uint64_t* __restrict__ kpool, uint64_t kstride,
                const float2* __restrict__ cb, int n_slots,
                const float* __restrict__ q, const double* __restrict__ thetas,
                long long t, long long pos0, long long n,
                float* __restrict__ scores) {
  extern __shared__ float2 sw[];  // [G][subs] conj(q)/sqrt(d)
  const int s = blockIdx.y;
  const float inv = rsqrtf((float)g.d);
  for (int k = threadIdx.x; k < g.G * g.subs; k += blockDim.x) {
    int h = k / g.subs, j = k % g.subs;
    const float* qr = q + ((size_t)s * g.G + h) * g.d;
    sw[k] = make_float2(qr[2 * j] * inv, -qr[2 * j + 1] * inv);
  }
  __syncthreads();
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t* words = kpool + (size_t)s * kstride;
  const float2* cbs = cb + (size_t)(s % n_slots) * g.R * g.L * g.subs;
  float acc[MAXG];
#pragma unroll
  for (int h = 0; h < MAXG; ++h) acc[h] = 0.f;
  const long long delta = t - (pos0 + i);
  const unsigned long long f0 = (unsigned long long)i * g.fpt;
  for (int j = 0; j < g.subs; ++j) {
    const int grp = j / g.g;
    float kx = 0.f, ky = 0.f;
    for (int r = 0; r < g.R; ++r) {
      unsigned long long f = f0 + (unsigned long long)(r * g.groups + grp) * 2;
      unsigned a = read_field(words, f * g.lb, g.lb);
      unsigned b = read_field(words, (f + 1) * g.lb, g.lb);
      float2 ua = __ldg(cbs + ((size_t)r * g.L + a) * g.subs + j);
      float2 ub = __ldg(cbs + ((size_t)r * g.L + b) * g.subs + j);
      kx += ua.x - ub.y;
      ky += ua.y + ub.x;
    }
    float2 ph = phase_neg(delta, thetas[j]);
    float rx = ph.x * kx - ph.y * ky, ry = ph.x * ky + ph.y * kx;
#pragma unroll
    for (int h = 0; h < MAXG; ++h)
      if (h < g.G) acc[h] += sw[h * g.subs + j].x * rx - sw[h * g.subs + j].y * ry;
  }
#pragma unroll
  for (int h = 0; h < MAXG; ++h)
    if (h < g.G) scores[((size_t)s * g.G + h) * n + i] = acc[h];
}

// ---------------------------------------------------------------- values
// One CTA per (chunk, stream): softmax statistics of the chunk, z[h][k] =
// sum_i p_h(i) bit_k(i) (attn.cpp:239-247), then o = z . C_V / l
// (attn.cpp:249-255).  Writes the chunk partial (m, l, o).
constexpr int kValThreads = 256;
constexpr int kValKpt = 4;  // codes per thread -> n_codes <= 1024


template <int MAXG>
__global__ void __launch_bounds__(kValThreads)
k_value_generic(Geom g, const uint64_t* __restrict__ vpool, uint64_t vstride,
                const float* __restrict__ cbv, int n_slots,
                const float* __restrict__ scores, long long n, int CH, int S,
                float* __restrict__ pm, float* __restrict__ pl,
                float* __restrict__ po) {
  extern __shared__ float sh[];
  float* ptile = sh;                         // [G][kValThreads]
  float* zs = sh + MAXG * kValThreads;       // [G][n_codes]
  __shared__ float red[33];
  __shared__ float mh[MAXG], lh[MAXG];
  const int s = blockIdx.y, c = blockIdx.x, tid = threadIdx.x;
  const long long i0 = (long long)c * CH;
  const long long i1 = min(n, i0 + CH);
  const float* sc = scores + (size_t)s * g.G * n;
  const uint64_t* words = vpool + (size_t)s * vstride;

  for (int h = 0; h < g.G; ++h) {
    float mx = -FLT_MAX;
    for (long long i = i0 + tid; i < i1; i += blockDim.x) mx = fmaxf(mx, sc[h * n + i]);
    mx = block_reduce(mx, true, red);
    if (tid == 0) mh[h] = mx;
  }
  __syncthreads();

  float z[MAXG][kValKpt];
  float lsum[MAXG];
#pragma unroll
  for (int h = 0; h < MAXG; ++h) {
    lsum[h] = 0.f;
#pragma unroll
    for (int j = 0; j < kValKpt; ++j) z[h][j] = 0.f;
  }
  for (long long ts = i0; ts < i1; ts += kValThreads) {
    const long long i = ts + tid;
#pragma unroll
    for (int h = 0; h < MAXG; ++h)
      if (h < g.G) {
        float p = (i < i1) ? expf(sc[h * n + i] - mh[h]) : 0.f;
        ptile[h * kValThreads + tid] = p;
        lsum[h] += p;
      }
    __syncthreads();
    const int cnt = (int)min((long long)kValThreads, i1 - ts);
    for (int tk = 0; tk < cnt; ++tk) {
      const unsigned long long base = (unsigned long long)(ts + tk) * g.n_codes;
#pragma unroll
      for (int j = 0; j < kValKpt; ++j) {
        const int k = tid + j * kValThreads;
        if (k < g.n_codes) {
          unsigned long long bit = base + k;
          const float on = (float)((__ldg(words + (bit >> 6)) >> (bit & 63)) & 1ull);
#pragma unroll
          for (int h = 0; h < MAXG; ++h)
            if (h < g.G) z[h][j] += on * ptile[h * kValThreads + tk];
        }
      }
    }
    __syncthreads();
  }
  for (int h = 0; h < g.G; ++h) {
    float v = block_reduce(lsum[h], false, red);
    if (tid == 0) lh[h] = v;
  }
#pragma unroll
  for (int h = 0; h < MAXG; ++h)
#pragma unroll
    for (int j = 0; j < kValKpt; ++j) {
      const int k = tid + j * kValThreads;
      if (h < g.G && k < g.n_codes) zs[h * g.n_codes + k] = z[h][j];
    }
  __syncthreads();
  const float* cb = cbv + (size_t)(s % n_slots) * g.n_codes * g.d;
  const long long rows = (long long)S * g.G;
  for (int e = tid; e < g.G * g.d; e += blockDim.x) {
    const int h = e / g.d, jd = e % g.d;
    float acc = 0.f;
    for (int k = 0; k < g.n_codes; ++k) acc += zs[h * g.n_codes + k] * __ldg(cb + (size_t)k * g.d + jd);
    const long long row = (long long)s * g.G + h;
    po[((long long)c * rows + row) * g.d + jd] = acc / lh[h];
  }
  if (tid < g.G) {
    const long long row = (long long)s * g.G + tid;
    pm[(long long)c * rows + row] = mh[tid];
    pl[(long long)c * rows + row] = lh[tid];
  }
}

// --------------------------------------------------------------- combine
// out = sum_p o_p l_p e^{m_p - M} / sum_p l_p e^{m_p - M}  (flash-decoding
// merge; the reference softmax is global, linalg.cpp:63-75).
// Part p's m / l rows at p * sm, its o rows at p * so (elements).
__global__ void k_combine(const float* __restrict__ m, const float* __restrict__ l,
                          const float* __restrict__ o, int P, long long rows, int d,
                          long long sm, long long so, float* __restrict__ out,
                          float* __restrict__ m_out, float* __restrict__ l_out) {
  // part weights l_p e^{m_p - M} computed once per part (smem), then each
  // thread sums its output column over the parts
  extern __shared__ float wsh[];  // [P]
  __shared__ float red[33];
  const long long row = blockIdx.x;
  float M = -FLT_MAX;
  for (int p = threadIdx.x; p < P; p += blockDim.x)
    if (l[p * sm + row] > 0.f) M = fmaxf(M, m[p * sm + row]);
  M = block_reduce(M, true, red);
  float Ls = 0.f;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const float lp = l[p * sm + row];
    const float wgt = lp > 0.f ? lp * expf(m[p * sm + row] - M) : 0.f;
    wsh[p] = wgt;
    Ls += wgt;
  }
  const float Lsum = block_reduce(Ls, false, red);  // (its barriers publish wsh)
  for (int jd = threadIdx.x; jd < d; jd += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < P; ++p) {
      const float wgt = wsh[p];
      if (wgt != 0.f) acc += o[p * so + row * d + jd] * wgt;
    }
    out[row * d + jd] = acc / Lsum;
  }
  if (threadIdx.x == 0) {
    if (m_out) m_out[row] = M;
    if (l_out) l_out[row] = Lsum;
  }
}

// Same merge, part p's packed block [m | l | o] read through parts[p] + off:
// the parts may live in peer GPUs' memory (symmetric / IPC buffers mapped
// over NVLink), so the gather is the combine's own loads -- no collective.
__global__ void k_combine_ptrs(const float* const* __restrict__ parts, long long off, int P,
                               long long rows, int d, float* __restrict__ out) {
  extern __shared__ float wsh[];  // [P]
  __shared__ float red[33];
  const long long row = blockIdx.x;
  float M = -FLT_MAX;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const float* b = parts[p] + off;
    if (b[rows + row] > 0.f) M = fmaxf(M, b[row]);
  }
  M = block_reduce(M, true, red);
  float Ls = 0.f;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const float* b = parts[p] + off;
    const float lp = b[rows + row];
    const float wgt = lp > 0.f ? lp * expf(b[row] - M) : 0.f;
    wsh[p] = wgt;
    Ls += wgt;
  }
  const float Lsum = block_reduce(Ls, false, red);
  for (int jd = threadIdx.x; jd < d; jd += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < P; ++p) {
      const float wgt = wsh[p];
      if (wgt != 0.f) acc += parts[p][off + 2 * rows + row * d + jd] * wgt;
    }
    out[row * d + jd] = acc / Lsum;
  }
}

cudaError_t run_lse_combine_ptrs(const float* const* parts, long long off, int n_parts,
                                 long long rows, int d, float* out, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  k_combine_ptrs<<<(unsigned)rows, 128, (size_t)n_parts * sizeof(float), st>>>(parts, off, n_parts,
                                                                               rows, d, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t run_lse_combine(const float* m, const float* l, const float* o,
                            int n_parts, long long rows, int d, float* out,
                            float* m_out, float* l_out, cudaStream_t st,
                            long long part_stride) {
  if (rows == 0) return cudaSuccess;
  const long long sm = part_stride ? part_stride : rows;
  const long long so = part_stride ? part_stride : rows * d;
  k_combine<<<(unsigned)rows, 128, (size_t)n_parts * sizeof(float), st>>>(
      m, l, o, n_parts, rows, d, sm, so, out, m_out, l_out);
  count_launch();
  return cudaGetLastError();
}


// ------------------------------------------------------------- dispatcher
bool fast_path_applies(const AttnJob& job);
size_t fast_scratch_bytes(const AttnJob& job, int* n_chunks);
cudaError_t run_attention_fast(const AttnJob& job, const float* q, float* pm,
                               float* pl, float* po, int* n_chunks, void* scratch,
                               cudaStream_t st, cudaEvent_t* prof, float* scores_out);
cudaError_t run_fast_combine(const AttnJob& job, const float* pm, const float* pl,
                             const float* pz, int n_parts, float* out, float* m_out,
                             float* l_out, float* zm, cudaStream_t st);

static int generic_chunk(const AttnJob& job) {
  long long want = (job.n * (long long)job.S + 591) / 592;  // >= ~4 CTAs/SM
  long long ch = ((want + 255) / 256) * 256;
  if (ch < 256) ch = 256;
  if (ch > 16384) ch = 16384;
  return (int)ch;
}

size_t attn_scratch_bytes(const AttnJob& job, int* n_chunks_out) {
  const Geom& g = job.geo;
  const long long rows = (long long)job.S * g.G;
  if (fast_path_applies(job)) {
    int nc = 0;
    size_t extra = fast_scratch_bytes(job, &nc);
    if (n_chunks_out) *n_chunks_out = nc;
    // partials (m, l, z[n_codes]) per chunk and row
    // + the merged z of every row and its (M, L) for k_combine_project
    return extra + (size_t)nc * rows * (2 + std::max(g.d, g.n_codes)) * sizeof(float) +
           (size_t)rows * (g.n_codes + 2) * sizeof(float) + 512;
  }
  const int CH = generic_chunk(job);
  const int nc = (int)((job.n + CH - 1) / CH);
  if (n_chunks_out) *n_chunks_out = nc;
  return (size_t)rows * job.n * sizeof(float) + (size_t)nc * rows * (2 + g.d) * sizeof(float) + 256;
}

cudaError_t run_attention(const AttnJob& job, const float* q, float* out,
                          float* m, float* l, float* o, float* scores_out,
                          void* scratch, size_t scratch_bytes, cudaStream_t st,
                          cudaEvent_t* prof) {
  const Geom& g = job.geo;
  const long long rows = (long long)job.S * g.G;
  int nc = 0;
  const size_t need = attn_scratch_bytes(job, &nc);
  if (scratch_bytes < need || g.G > kMaxG) return cudaErrorInvalidValue;
  char* p = static_cast<char*>(scratch);
  const bool fast = fast_path_applies(job);
  float* pm;
  float* pl;
  float* po;
  float* zm = nullptr;  // merged z rows (fast path)
  cudaError_t e;
  if (fast) {
    size_t extra = fast_scratch_bytes(job, &nc);
    pm = reinterpret_cast<float*>(p + extra);
    pl = pm + (size_t)nc * rows;
    po = pl + (size_t)nc * rows;
    zm = po + (size_t)nc * rows * std::max(g.d, g.n_codes);
    e = run_attention_fast(job, q, pm, pl, po, &nc, p, st, prof, scores_out);
    if (e != cudaSuccess) return e;
  } else {
    const int CH = generic_chunk(job);
    nc = (int)((job.n + CH - 1) / CH);
    float* scores = reinterpret_cast<float*>(p);
    pm = scores + (size_t)rows * job.n;
    pl = pm + (size_t)nc * rows;
    po = pl + (size_t)nc * rows;
    dim3 gs((unsigned)((job.n + 127) / 128), job.S);
    size_t shs = (size_t)g.G * g.subs * sizeof(float2);
    if (prof) cudaEventRecord(prof[0], st);
    k_score_generic<kMaxG><<<gs, 128, shs, st>>>(g, job.kpool, job.kstride, job.cb_key,
                                                 job.n_slots, q, job.thetas, job.t, job.pos0,
                                                 job.n, scores);
    if (prof) cudaEventRecord(prof[1], st);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (scores_out)
      if ((e = cudaMemcpyAsync(scores_out, scores, (size_t)rows * job.n * sizeof(float),
                               cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return e;
    dim3 gv((unsigned)nc, job.S);
    size_t shv = (size_t)kMaxG * kValThreads * sizeof(float) + (size_t)g.G * g.n_codes * sizeof(float);
    k_value_generic<kMaxG><<<gv, kValThreads, shv, st>>>(g, job.vpool, job.vstride, job.cb_val,
                                                         job.n_slots, scores, job.n, CH, job.S,
                                                         pm, pl, po);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  float* mo = m;
  float* lo = l;
  if (fast) {  // partials hold unnormalised z: merge, then the codebook product
    if (out) {
      e = run_fast_combine(job, pm, pl, po, nc, out, mo, lo, zm, st);
      if (e != cudaSuccess) return e;
      if (o) e = cudaMemcpyAsync(o, out, (size_t)rows * g.d * sizeof(float), cudaMemcpyDeviceToDevice, st);
      return e;
    }
    if (o) return run_fast_combine(job, pm, pl, po, nc, o, mo, lo, zm, st);
    return cudaSuccess;
  }
  if (out) {
    e = run_lse_combine(pm, pl, po, nc, rows, g.d, out, mo, lo, st);
    if (e != cudaSuccess) return e;
    if (o) e = cudaMemcpyAsync(o, out, (size_t)rows * g.d * sizeof(float), cudaMemcpyDeviceToDevice, st);
    return e;
  }
  if (o) return run_lse_combine(pm, pl, po, nc, rows, g.d, o, mo, lo, st);
  return cudaSuccess;
}

}  // namespace cvq
