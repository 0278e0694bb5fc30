// train.cu -- key-codebook training on the GPU:
// train_key_codebook (keyquant.cpp:641-703) with GroupEm's soft-to-hard
// schedule (keyquant.cpp:319-544), the heavy passes on sm_100a.
//
// Per (round, group) clustering problem the host runs the reference's
// control flow unchanged (init_atoms with the reference Rng stream,
// auto_temperature, the annealed soft schedule, the hard phase with
// repair_empty / rollback / tolerance stop, refit_atoms with the reference
// Cholesky).  The device does the O(n L^2 2g) work:
//
//   * projections p.u_l, p.v_l and center tables, in the reference's exact
//     fp64 operation order (no FMA), so distances are bit-identical;
//   * soft E-step (keyquant.cpp:411-437): per point the L^2 unsquared
//     distances, the annealed weights exp(-(d - lo)/T) / sum and their
//     moments (joint weights in registers per CTA, marginals per point, then
//     the marginal-weighted point sums).  Summation order differs from the
//     sequential reference (fp64, ~1e-16 relative per step);
//   * hard E-step (keyquant.cpp:441-461): brute-force assignments by the
//     bit-exact key encoder (encode.cu) or the factorised scan, the exact
//     distances, and the hard moments summed in the reference's point order,
//     so from identical atoms the hard phase is bit-identical.
//
// Parity: tests/test_train_gpu.py against the compiled reference
// (oracle/_ref) -- identical hard assignments / codes, atoms within 1e-9.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "cvq_internal.cuh"

namespace cvq {

namespace {

// ------------------------------------------------------------ host helpers
uint64_t mix_seed(uint64_t seed, size_t round, size_t group) {  // keyquant.cpp:27-35
  uint64_t h = seed;
  h ^= (round + 1) * 0x9E3779B97F4A7C15ull;
  h ^= (h >> 29);
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= (group + 1) * 0x94D049BB133111EBull;
  h ^= (h >> 32);
  return h;
}

// commvq::Rng::normal (rng.hpp:27-39): mt19937_64 + Box-Muller, spare cached.
struct RefRng {
  std::mt19937_64 gen;
  bool has_spare = false;
  double spare = 0.0;
  explicit RefRng(uint64_t seed) : gen(seed) {}
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = (static_cast<double>(gen() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    has_spare = true;
    return r * std::cos(a);
  }
};

struct TrainFail {
  int code;  // 1 = invalid argument, 2 = training error, 3 = cuda
  std::string msg;
};

#define TCU(x)                                                      \
  do {                                                              \
    cudaError_t e_ = (x);                                           \
    if (e_ != cudaSuccess) throw TrainFail{3, cudaGetErrorString(e_)}; \
  } while (0)

struct Moments {  // keyquant.cpp:228-279
  size_t g, L;
  std::vector<double> joint, num_a, num_b;
  Moments(size_t g_, size_t L_)
      : g(g_), L(L_), joint(L_ * L_, 0.0), num_a(L_ * 2 * g_, 0.0), num_b(L_ * 2 * g_, 0.0) {}
};

// refit_atoms (keyquant.cpp:284-336) with cholesky_factor / solve
// (linalg.cpp:95-132), same operation order.
std::vector<double> refit_atoms(const Moments& mom, double ridge) {
  const size_t L = mom.L, g = mom.g, w = 2 * g, n = 2 * L;
  std::vector<double> a(n * n, 0.0);
  auto A = [&](size_t i, size_t j) -> double& { return a[i * n + j]; };
  for (size_t ia = 0; ia < L; ++ia)
    for (size_t ib = 0; ib < L; ++ib) {
      const double wt = mom.joint[ia * L + ib];
      if (wt == 0.0) continue;
      const size_t xa = 2 * ia, ya = 2 * ia + 1, xb = 2 * ib, yb = 2 * ib + 1;
      A(xa, xa) += wt;
      A(yb, yb) += wt;
      A(xa, yb) -= wt;
      A(yb, xa) -= wt;
      A(xb, xb) += wt;
      A(ya, ya) += wt;
      A(xb, ya) += wt;
      A(ya, xb) += wt;
    }
  double lam = ridge;
  if (lam < 0.0) {
    double trace = 0.0;
    for (size_t i = 0; i < n; ++i) trace += A(i, i);
    lam = 1e-8 * trace / static_cast<double>(n);
    if (!(lam > 0.0)) lam = 1e-12;
  }
  for (size_t i = 0; i < n; ++i) A(i, i) += lam;
  std::vector<double> l(n * n, 0.0);
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j <= i; ++j) {
      double s = A(i, j);
      for (size_t k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
      if (i == j) {
        if (s <= 0.0 || !std::isfinite(s))
          throw TrainFail{2,
                          "refit_atoms: normal equations singular after ridge; the group's "
                          "weights are too degenerate to fit atoms"};
        l[i * n + i] = std::sqrt(s);
      } else {
        l[i * n + j] = s / l[j * n + j];
      }
    }
  std::vector<double> out(g * L * 2), rhs(n), y(n), x(n);
  for (size_t s = 0; s < g; ++s) {
    for (size_t lv = 0; lv < L; ++lv) {
      rhs[2 * lv] = mom.num_a[lv * w + 2 * s] + mom.num_b[lv * w + 2 * s + 1];
      rhs[2 * lv + 1] = mom.num_a[lv * w + 2 * s + 1] - mom.num_b[lv * w + 2 * s];
    }
    for (size_t i = 0; i < n; ++i) {
      double t = rhs[i];
      for (size_t k = 0; k < i; ++k) t -= l[i * n + k] * y[k];
      y[i] = t / l[i * n + i];
    }
    for (size_t ii = n; ii-- > 0;) {
      double t = y[ii];
      for (size_t k = ii + 1; k < n; ++k) t -= l[k * n + ii] * x[k];
      x[ii] = t / l[ii * n + ii];
    }
    for (size_t lv = 0; lv < L; ++lv) {
      out[(s * L + lv) * 2] = x[2 * lv];
      out[(s * L + lv) * 2 + 1] = x[2 * lv + 1];
    }
  }
  return out;
}

// ------------------------------------------------------------ kernels
// Points of one group: element (p, i) at P[p * ld + i], i < w = 2g.

// |p|^2 as the reference dot (sequential, no FMA).
__global__ void k_em_pnorm(const double* __restrict__ P, int ld, int w, long long n,
                           double* __restrict__ pnorm) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double* r = P + p * ld;
  double s = 0.0;
  for (int i = 0; i < w; ++i) s = __dadd_rn(s, __dmul_rn(r[i], r[i]));
  pnorm[p] = s;
}

// init_atoms' per-subspace spread (keyquant.cpp:362-372): sequential over
// points, one thread per subspace.
__global__ void k_em_var(const double* __restrict__ P, int ld, int g, long long n,
                         double* __restrict__ var) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= g) return;
  double v = 0.0;
  for (long long p = 0; p < n; ++p) {
    const double x = P[p * ld + 2 * s], y = P[p * ld + 2 * s + 1];
    v = __dadd_rn(v, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
  }
  var[s] = v;
}

// CenterCache tables (keyquant.cpp:127-155): u_l = (x_s, y_s)_s,
// v_l = (-y_s, x_s)_s; base[a][b] = |u_a|^2 + |v_b|^2 + 2 u_a.v_b, all as
// the reference's sequential dots.  uT / vT are [w][L] for coalesced reads.
__global__ void k_em_tables(const double* __restrict__ atoms, int g, int L,
                            double* __restrict__ uT, double* __restrict__ vT,
                            double* __restrict__ unorm, double* __restrict__ vnorm,
                            double* __restrict__ base, int phase) {
  const int w = 2 * g;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  auto U = [&](int l, int i) {  // u_l[i]
    const double* m = atoms + ((size_t)(i >> 1) * L + l) * 2;
    return (i & 1) ? m[1] : m[0];
  };
  auto V = [&](int l, int i) {  // v_l[i]
    const double* m = atoms + ((size_t)(i >> 1) * L + l) * 2;
    return (i & 1) ? m[0] : -m[1];
  };
  if (phase == 0) {
    if (e < (long long)w * L) {
      const int i = (int)(e / L), l = (int)(e % L);
      uT[e] = U(l, i);
      vT[e] = V(l, i);
    }
    if (e < L) {
      double su = 0.0, sv = 0.0;
      for (int i = 0; i < w; ++i) {
        const double u = U((int)e, i), v = V((int)e, i);
        su = __dadd_rn(su, __dmul_rn(u, u));
        sv = __dadd_rn(sv, __dmul_rn(v, v));
      }
      unorm[e] = su;
      vnorm[e] = sv;
    }
  } else if (e < (long long)L * L) {
    const int a = (int)(e / L), b = (int)(e % L);
    double uv = 0.0;
    for (int i = 0; i < w; ++i) uv = __dadd_rn(uv, __dmul_rn(U(a, i), V(b, i)));
    base[e] = __dadd_rn(__dadd_rn(unorm[a], vnorm[b]), __dmul_rn(2.0, uv));
  }
}

// CenterCache::project (keyquant.cpp:163-176): pu[p][l] = p.u_l,
// pv[p][l] = p.v_l, sequential over i.  Block: 8 points x L levels.
constexpr int kProjPts = 8;
__global__ void k_em_project(const double* __restrict__ P, int ld, int w, long long n,
                             const double* __restrict__ uT, const double* __restrict__ vT,
                             int L, double* __restrict__ pu, double* __restrict__ pv) {
  extern __shared__ double prow[];  // [kProjPts][w]
  const long long p0 = (long long)blockIdx.x * kProjPts;
  for (int e = threadIdx.x; e < kProjPts * w; e += blockDim.x) {
    const long long p = p0 + e / w;
    prow[e] = p < n ? P[p * ld + e % w] : 0.0;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    double su[kProjPts], sv[kProjPts];
#pragma unroll
    for (int k = 0; k < kProjPts; ++k) su[k] = sv[k] = 0.0;
    for (int i = 0; i < w; ++i) {
      const double u = uT[(size_t)i * L + l], v = vT[(size_t)i * L + l];
#pragma unroll
      for (int k = 0; k < kProjPts; ++k) {
        su[k] = __dadd_rn(su[k], __dmul_rn(prow[k * w + i], u));
        sv[k] = __dadd_rn(sv[k], __dmul_rn(prow[k * w + i], v));
      }
    }
#pragma unroll
    for (int k = 0; k < kProjPts; ++k)
      if (p0 + k < n) {
        pu[(p0 + k) * L + l] = su[k];
        pv[(p0 + k) * L + l] = sv[k];
      }
  }
}

// Unsquared distance of the soft pass / auto_temperature
// (keyquant.cpp:399-401, 420-423): sqrt(max(base - 2 (pu + pv) + |p|^2, 0)).
__device__ __forceinline__ double soft_dist(double base, double pu, double pv, double pn) {
  const double d2 = __dadd_rn(__dsub_rn(base, __dmul_rn(2.0, __dadd_rn(pu, pv))), pn);
  return sqrt(fmax(d2, 0.0));
}

// auto_temperature samples (keyquant.cpp:389-410): points 0, stride, ...
__global__ void k_em_temp_samples(const double* __restrict__ pu, const double* __restrict__ pv,
                                  const double* __restrict__ pnorm, const double* __restrict__ base,
                                  int L, long long stride, long long n_samp,
                                  double* __restrict__ out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long C = (long long)L * L;
  if (e >= n_samp * C) return;
  const long long si = e / C, p = si * stride;
  const int c = (int)(e % C), a = c / L, b = c % L;
  out[e] = soft_dist(base[c], pu[p * L + a], pv[p * L + b], pnorm[p]);
}

__device__ __forceinline__ double block_min_d(double v, double* red) {
  for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) r = fmin(r, red[i]);
  return r;
}
__device__ __forceinline__ double block_sum_d(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) r += red[i];
  return r;
}

// Soft E-step (keyquant.cpp:411-437): one CTA per group of points, one point
// at a time; thread t owns centers c = t + kSoftThreads k.  Joint weights
// accumulate in registers across the CTA's points; the marginals of each
// point go to global for the marginal-weighted point sums.
constexpr int kSoftThreads = 256;
constexpr int kSoftMaxK = 16;  // L^2 <= 4096
__global__ void __launch_bounds__(kSoftThreads)
k_em_soft(const double* __restrict__ pu, const double* __restrict__ pv,
          const double* __restrict__ pnorm, const double* __restrict__ base, int L, long long n,
          double temp, double* __restrict__ joint, double* __restrict__ marg_a,
          double* __restrict__ marg_b) {
  extern __shared__ double sm[];  // ma[L], mb[L]
  __shared__ double red[kSoftThreads / 32];
  double* ma = sm;
  double* mb = sm + L;
  const int C = L * L, t = threadIdx.x;
  double jacc[kSoftMaxK], dv[kSoftMaxK];
#pragma unroll
  for (int k = 0; k < kSoftMaxK; ++k) jacc[k] = 0.0;
  for (long long p = blockIdx.x; p < n; p += gridDim.x) {
    const double pn = pnorm[p];
    double lo = INFINITY;
#pragma unroll
    for (int k = 0; k < kSoftMaxK; ++k) {
      const int c = t + kSoftThreads * k;
      dv[k] = INFINITY;
      if (c < C) {
        dv[k] = soft_dist(base[c], pu[p * L + c / L], pv[p * L + c % L], pn);
        lo = fmin(lo, dv[k]);
      }
    }
    lo = block_min_d(lo, red);
    for (int e = t; e < 2 * L; e += kSoftThreads) sm[e] = 0.0;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kSoftMaxK; ++k) {
      const int c = t + kSoftThreads * k;
      if (c < C) {
        dv[k] = exp(-(dv[k] - lo) / temp);
        s += dv[k];
      }
    }
    const double sum = block_sum_d(s, red);  // (its barriers also order the ma/mb zeroing)
#pragma unroll
    for (int k = 0; k < kSoftMaxK; ++k) {
      const int c = t + kSoftThreads * k;
      if (c < C) {
        const double wv = dv[k] / sum;
        jacc[k] += wv;
        atomicAdd(ma + c / L, wv);
        atomicAdd(mb + c % L, wv);
      }
    }
    __syncthreads();
    for (int e = t; e < L; e += kSoftThreads) {
      marg_a[p * L + e] = ma[e];
      marg_b[p * L + e] = mb[e];
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < kSoftMaxK; ++k) {
    const int c = t + kSoftThreads * k;
    if (c < C && jacc[k] != 0.0) atomicAdd(joint + c, jacc[k]);
  }
}

// out[l][i] += sum_p A[p][l] P[p][i] over a chunk of points (soft moments).
constexpr int kGemmChunk = 512;
__global__ void k_em_wsum(const double* __restrict__ A, int L, const double* __restrict__ P, int ld,
                          int w, long long n, double* __restrict__ out) {
  const int l = blockIdx.y;
  const long long p0 = (long long)blockIdx.x * kGemmChunk;
  const long long p1 = min(n, p0 + kGemmChunk);
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
    double s = 0.0;
    for (long long p = p0; p < p1; ++p) {
      const double wa = A[p * L + l];
      if (wa != 0.0) s += wa * P[p * ld + i];
    }
    atomicAdd(out + (size_t)l * w + i, s);
  }
}

// Hard moments (Moments::add_hard, keyquant.cpp:241-248) in the reference's
// point order: thread (level, i) sums the points assigned to that level,
// listed in increasing index (CSR from the host).
__global__ void k_em_hard_sum(const long long* __restrict__ off, const int* __restrict__ idx,
                              const double* __restrict__ P, int ld, int w, int L,
                              double* __restrict__ out) {
  const int l = blockIdx.x;
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
    double s = 0.0;
    for (long long k = off[l]; k < off[l + 1]; ++k) s = __dadd_rn(s, P[(long long)idx[k] * ld + i]);
    out[(size_t)l * w + i] = s;
  }
}

// Exact distance of the assigned center (the `best` of assign_brute,
// keyquant.cpp:180-200: centers c_i = u_a[i] + v_b[i], sum of squares).
__global__ void k_em_assigned_dist(const double* __restrict__ P, int ld, int g, int L, long long n,
                                   const double* __restrict__ atoms, const uint16_t* __restrict__ a,
                                   const uint16_t* __restrict__ b, double* __restrict__ d2) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double* r = P + p * ld;
  const int aa = a[p], bb = b[p];
  double s = 0.0;
  for (int si = 0; si < g; ++si) {
    const double* ua = atoms + ((size_t)si * L + aa) * 2;
    const double* ub = atoms + ((size_t)si * L + bb) * 2;
    const double c0 = __dadd_rn(ua[0], -ub[1]);
    const double c1 = __dadd_rn(ua[1], ub[0]);
    const double d0 = __dsub_rn(r[2 * si], c0);
    s = __dadd_rn(s, __dmul_rn(d0, d0));
    const double d1 = __dsub_rn(r[2 * si + 1], c1);
    s = __dadd_rn(s, __dmul_rn(d1, d1));
  }
  d2[p] = s;
}

// assign_factorized (keyquant.cpp:204-224): argmin over (a, b) of
// base[a][b] - 2 pu[a] - 2 pv[b], strict '<' in c order; d2 = best + |p|^2.
__global__ void k_em_assign_factorized(const double* __restrict__ pu, const double* __restrict__ pv,
                                       const double* __restrict__ pnorm,
                                       const double* __restrict__ base, int L, long long n,
                                       uint16_t* __restrict__ a_out, uint16_t* __restrict__ b_out,
                                       double* __restrict__ d2, int ostride = 1) {
  const long long p = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= n) return;
  double best = INFINITY;
  int bc = 0x7fffffff;
  for (int c = lane; c < L * L; c += 32) {
    const int a = c / L, b = c % L;
    const double pa2 = __dmul_rn(2.0, pu[p * L + a]);
    const double s = __dsub_rn(__dsub_rn(base[c], pa2), __dmul_rn(2.0, pv[p * L + b]));
    if (s < best) {
      best = s;
      bc = c;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
    if (v2 < best || (v2 == best && c2 < bc)) {
      best = v2;
      bc = c2;
    }
  }
  if (lane == 0) {
    if (bc == 0x7fffffff) bc = 0;
    a_out[p * ostride] = (uint16_t)(bc / L);
    b_out[p * ostride] = (uint16_t)(bc % L);
    if (d2) d2[p] = best + pnorm[p];
  }
}

// Residual update after a group (keyquant.cpp:686-694).
__global__ void k_em_residual(double* __restrict__ R, int d, int col0, int g, int L, long long n,
                              const double* __restrict__ atoms, const uint16_t* __restrict__ a,
                              const uint16_t* __restrict__ b, int cstride = 1) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * g) return;
  const long long p = e / g;
  const int s = (int)(e % g);
  const double* ua = atoms + ((size_t)s * L + a[p * cstride]) * 2;
  const double* ub = atoms + ((size_t)s * L + b[p * cstride]) * 2;
  double* row = R + p * d + col0;
  row[2 * s] = __dsub_rn(row[2 * s], __dsub_rn(ua[0], ub[1]));
  row[2 * s + 1] = __dsub_rn(row[2 * s + 1], __dadd_rn(ua[1], ub[0]));
}

__global__ void k_em_copy_cols(const double* __restrict__ R, int d, int col0, int w, long long n,
                               double* __restrict__ out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * w) return;
  out[e] = R[(e / w) * d + col0 + e % w];
}

unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

struct DevBufs {
  std::vector<void*> ptrs;
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
    TCU(cudaMalloc(&p, std::max<size_t>(count * sizeof(T), 8)));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~DevBufs() {
    for (void* p : ptrs) cudaFree(p);
  }
};

// One (round, group) problem: GroupEm::run (keyquant.cpp:342-352).
class GroupEmGpu {
 public:
  GroupEmGpu(const double* P, int ld, long long n, int g, int L, const TrainConfig& em,
             uint64_t seed, cudaStream_t st)
      : P_(P), ld_(ld), n_(n), g_(g), L_(L), w_(2 * g), em_(em), rng_(seed), st_(st) {
    pnorm_ = buf_.get<double>(n);
    pu_ = buf_.get<double>((size_t)n * L);
    pv_ = buf_.get<double>((size_t)n * L);
    ma_ = buf_.get<double>((size_t)n * L);
    mb_ = buf_.get<double>((size_t)n * L);
    atoms_d_ = buf_.get<double>((size_t)g * L * 2);
    uT_ = buf_.get<double>((size_t)w_ * L);
    vT_ = buf_.get<double>((size_t)w_ * L);
    un_ = buf_.get<double>(L);
    vn_ = buf_.get<double>(L);
    base_ = buf_.get<double>((size_t)L * L);
    joint_ = buf_.get<double>((size_t)L * L);
    numa_ = buf_.get<double>((size_t)L * w_);
    numb_ = buf_.get<double>((size_t)L * w_);
    a_ = buf_.get<uint16_t>(n);
    b_ = buf_.get<uint16_t>(n);
    d2_ = buf_.get<double>(n);
    k_em_pnorm<<<nblk(n, 256), 256, 0, st_>>>(P_, ld_, w_, n_, pnorm_);
    count_launch();
    TCU(cudaGetLastError());
  }

  void run() {
    init_atoms();
    const double t0 = em_.t0 > 0.0 ? em_.t0 : auto_temperature();
    for (size_t it = 0; it < em_.soft_iters; ++it) {
      const double temp = std::max(t0 * std::pow(em_.decay, static_cast<double>(it)), 1e-12);
      soft_update(temp);
    }
    hard_phase();
  }

  const std::vector<double>& atoms() const { return atoms_; }
  const std::vector<double>& objective_trace() const { return obj_trace_; }
  const double* atoms_dev() const { return atoms_d_; }
  const uint16_t* a_dev() const { return a_; }
  const uint16_t* b_dev() const { return b_; }

 private:
  void upload_atoms() {
    TCU(cudaMemcpyAsync(atoms_d_, atoms_.data(), atoms_.size() * 8, cudaMemcpyHostToDevice, st_));
  }
  void tables() {
    upload_atoms();
    const long long e0 = std::max<long long>((long long)w_ * L_, L_);
    k_em_tables<<<nblk(e0, 256), 256, 0, st_>>>(atoms_d_, g_, L_, uT_, vT_, un_, vn_, base_, 0);
    k_em_tables<<<nblk((long long)L_ * L_, 256), 256, 0, st_>>>(atoms_d_, g_, L_, uT_, vT_, un_, vn_,
                                                                base_, 1);
    count_launch(2);
    TCU(cudaGetLastError());
  }
  void project() {
    k_em_project<<<nblk(n_, kProjPts), 128, (size_t)kProjPts * w_ * 8, st_>>>(P_, ld_, w_, n_, uT_,
                                                                             vT_, L_, pu_, pv_);
    count_launch();
    TCU(cudaGetLastError());
  }

  void init_atoms() {  // keyquant.cpp:356-373
    std::vector<double> var(g_);
    double* dv = buf_.get<double>(g_);
    k_em_var<<<nblk(g_, 64), 64, 0, st_>>>(P_, ld_, g_, n_, dv);
    count_launch();
    TCU(cudaGetLastError());
    TCU(cudaMemcpyAsync(var.data(), dv, g_ * 8, cudaMemcpyDeviceToHost, st_));
    TCU(cudaStreamSynchronize(st_));
    atoms_.assign((size_t)g_ * L_ * 2, 0.0);
    for (int s = 0; s < g_; ++s) {
      double v = var[s] / static_cast<double>(2 * n_);
      double sigma = std::sqrt(v / 2.0);
      if (!(sigma > 0.0)) sigma = 1e-3;
      for (int l = 0; l < L_; ++l) {
        const double x = sigma * rng_.normal();
        const double y = sigma * rng_.normal();
        atoms_[((size_t)s * L_ + l) * 2] = x;
        atoms_[((size_t)s * L_ + l) * 2 + 1] = y;
      }
    }
  }

  double auto_temperature() {  // keyquant.cpp:389-410
    tables();
    project();
    const long long stride = std::max<long long>(1, n_ / 512);
    const long long ns = (n_ + stride - 1) / stride;
    const long long total = ns * (long long)L_ * L_;
    double* dsm = buf_.get<double>(total);
    k_em_temp_samples<<<nblk(total, 256), 256, 0, st_>>>(pu_, pv_, pnorm_, base_, L_, stride, ns, dsm);
    count_launch();
    TCU(cudaGetLastError());
    std::vector<double> samples(total);
    TCU(cudaMemcpyAsync(samples.data(), dsm, total * 8, cudaMemcpyDeviceToHost, st_));
    TCU(cudaStreamSynchronize(st_));
    const size_t mid = samples.size() / 2;
    std::nth_element(samples.begin(), samples.begin() + mid, samples.end());
    const double med = samples[mid];
    return med > 0.0 ? med : 1.0;
  }

  Moments download_moments() {
    Moments mom(g_, L_);
    TCU(cudaMemcpyAsync(mom.joint.data(), joint_, mom.joint.size() * 8, cudaMemcpyDeviceToHost, st_));
    TCU(cudaMemcpyAsync(mom.num_a.data(), numa_, mom.num_a.size() * 8, cudaMemcpyDeviceToHost, st_));
    TCU(cudaMemcpyAsync(mom.num_b.data(), numb_, mom.num_b.size() * 8, cudaMemcpyDeviceToHost, st_));
    TCU(cudaStreamSynchronize(st_));
    return mom;
  }

  void soft_update(double temp) {  // keyquant.cpp:411-437
    tables();
    project();
    TCU(cudaMemsetAsync(joint_, 0, (size_t)L_ * L_ * 8, st_));
    TCU(cudaMemsetAsync(numa_, 0, (size_t)L_ * w_ * 8, st_));
    TCU(cudaMemsetAsync(numb_, 0, (size_t)L_ * w_ * 8, st_));
    const unsigned grid = (unsigned)std::min<long long>(n_, 148 * 8);
    k_em_soft<<<grid, kSoftThreads, (size_t)2 * L_ * 8, st_>>>(pu_, pv_, pnorm_, base_, L_, n_, temp,
                                                                joint_, ma_, mb_);
    dim3 gg(nblk(n_, kGemmChunk), L_);
    k_em_wsum<<<gg, 128, 0, st_>>>(ma_, L_, P_, ld_, w_, n_, numa_);
    k_em_wsum<<<gg, 128, 0, st_>>>(mb_, L_, P_, ld_, w_, n_, numb_);
    count_launch(3);
    TCU(cudaGetLastError());
    atoms_ = refit_atoms(download_moments(), em_.ridge);
  }

  // Hard E-step (keyquant.cpp:441-461): assignments, exact distances and the
  // hard moments; returns the objective (sequential sum as the reference).
  double e_step(Moments& mom) {
    if (em_.factorized) {
      tables();
      project();
      k_em_assign_factorized<<<nblk(n_, 8), 256, 0, st_>>>(pu_, pv_, pnorm_, base_, L_, n_, a_, b_,
                                                           d2_);
      count_launch();
      TCU(cudaGetLastError());
    } else {
      upload_atoms();
      Geom eg{};
      eg.d = w_;
      eg.subs = g_;
      eg.g = g_;
      eg.groups = 1;
      eg.L = L_;
      eg.R = 1;
      eg.fpt = 2;
      eg.n_codes = 1;
      eg.G = 1;
      const bool fit = key_tables_fit(eg);
      double* ebase = fit ? base_ : nullptr;  // encoder screen table (its own layout)
      double* emax = un_;
      if (fit) TCU(build_key_enc_tables(eg, 1, atoms_d_, ebase, emax, st_));
      const double* keys = P_;
      if (ld_ != w_) {  // the encoder reads contiguous rows
        if (!slice_) slice_ = buf_.get<double>((size_t)n_ * w_);
        k_em_copy_cols<<<nblk(n_ * w_, 256), 256, 0, st_>>>(P_, ld_, 0, w_, n_, slice_);
        count_launch();
        keys = slice_;
      }
      KeyEncTables tab{atoms_d_, ebase, emax};
      TCU(run_encode_keys(eg, 1, 1, tab, keys, 1, 0, n_, a_, b_, st_));
      k_em_assigned_dist<<<nblk(n_, 256), 256, 0, st_>>>(P_, ld_, g_, L_, n_, atoms_d_, a_, b_, d2_);
      count_launch();
      TCU(cudaGetLastError());
    }
    ha_.resize(n_);
    hb_.resize(n_);
    dist_.resize(n_);
    TCU(cudaMemcpyAsync(ha_.data(), a_, n_ * 2, cudaMemcpyDeviceToHost, st_));
    TCU(cudaMemcpyAsync(hb_.data(), b_, n_ * 2, cudaMemcpyDeviceToHost, st_));
    TCU(cudaMemcpyAsync(dist_.data(), d2_, n_ * 8, cudaMemcpyDeviceToHost, st_));
    TCU(cudaStreamSynchronize(st_));
    double obj = 0.0;
    for (long long p = 0; p < n_; ++p) obj += dist_[p];
    hard_moments(mom);
    return obj;
  }

  // Moments of the current host assignments, in the reference point order.
  void hard_moments(Moments& mom) {
    mom = Moments(g_, L_);
    for (long long p = 0; p < n_; ++p) mom.joint[(size_t)ha_[p] * L_ + hb_[p]] += 1.0;
    for (int side = 0; side < 2; ++side) {
      const std::vector<uint16_t>& asg = side ? hb_ : ha_;
      std::vector<long long> off(L_ + 1, 0);
      for (long long p = 0; p < n_; ++p) off[asg[p] + 1]++;
      for (int l = 0; l < L_; ++l) off[l + 1] += off[l];
      std::vector<int> idx(n_);
      std::vector<long long> pos(off.begin(), off.end() - 1);
      for (long long p = 0; p < n_; ++p) idx[pos[asg[p]]++] = (int)p;
      if (!csr_off_) {
        csr_off_ = buf_.get<long long>(L_ + 1);
        csr_idx_ = buf_.get<int>(n_);
      }
      TCU(cudaMemcpyAsync(csr_off_, off.data(), off.size() * 8, cudaMemcpyHostToDevice, st_));
      TCU(cudaMemcpyAsync(csr_idx_, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, st_));
      double* out = side ? numb_ : numa_;
      k_em_hard_sum<<<L_, 128, 0, st_>>>(csr_off_, csr_idx_, P_, ld_, w_, L_, out);
      count_launch();
      TCU(cudaGetLastError());
      std::vector<double>& dst = side ? mom.num_b : mom.num_a;
      TCU(cudaMemcpyAsync(dst.data(), out, dst.size() * 8, cudaMemcpyDeviceToHost, st_));
      TCU(cudaStreamSynchronize(st_));  // host idx/off must outlive the copies
    }
  }

  bool repair_empty(Moments& mom) {  // keyquant.cpp:465-490
    const double threshold =
        1e-6 * static_cast<double>(n_) / static_cast<double>((size_t)L_ * L_);
    std::vector<size_t> empty;
    for (size_t c = 0; c < (size_t)L_ * L_; ++c)
      if (mom.joint[c] <= threshold) empty.push_back(c);
    if (empty.empty()) return false;
    std::vector<size_t> order(n_);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](size_t x, size_t y) {
      if (dist_[x] != dist_[y]) return dist_[x] > dist_[y];
      return x < y;
    });
    const size_t take = std::min(empty.size(), (size_t)n_);
    for (size_t k = 0; k < take; ++k) {
      const size_t c = empty[k];
      ha_[order[k]] = static_cast<uint16_t>(c / L_);
      hb_[order[k]] = static_cast<uint16_t>(c % L_);
    }
    hard_moments(mom);
    return true;
  }

  void hard_phase() {  // keyquant.cpp:492-531
    bool repair_enabled = true;
    Moments mom(g_, L_);
    double obj = e_step(mom);
    obj_trace_.push_back(obj);
    for (size_t it = 0; it < em_.hard_iters_max; ++it) {
      Moments mom_snap(g_, L_);
      bool repaired = false;
      if (repair_enabled) {
        mom_snap = mom;
        repaired = repair_empty(mom);
      }
      atoms_ = refit_atoms(mom, em_.ridge);
      Moments next(g_, L_);
      double new_obj = e_step(next);
      if (repaired && new_obj > obj * (1.0 + 1e-12) + 1e-300) {
        atoms_ = refit_atoms(mom_snap, em_.ridge);
        next = Moments(g_, L_);
        new_obj = e_step(next);
        repair_enabled = false;
      }
      obj_trace_.push_back(new_obj);
      mom = std::move(next);
      const double drop = obj - new_obj;
      obj = new_obj;
      if (drop <= em_.tol * std::max(obj, 1e-300)) break;
    }
    upload_atoms();  // final atoms (and the last assignments in a_, b_)
    TCU(cudaMemcpyAsync(a_, ha_.data(), n_ * 2, cudaMemcpyHostToDevice, st_));
    TCU(cudaMemcpyAsync(b_, hb_.data(), n_ * 2, cudaMemcpyHostToDevice, st_));
    TCU(cudaStreamSynchronize(st_));
  }

  const double* P_;
  int ld_;
  long long n_;
  int g_, L_, w_;
  TrainConfig em_;
  RefRng rng_;
  cudaStream_t st_;
  DevBufs buf_;
  double *pnorm_, *pu_, *pv_, *ma_, *mb_, *atoms_d_, *uT_, *vT_, *un_, *vn_, *base_;
  double *joint_, *numa_, *numb_, *d2_;
  double* slice_ = nullptr;
  long long* csr_off_ = nullptr;
  int* csr_idx_ = nullptr;
  uint16_t *a_, *b_;
  std::vector<double> atoms_, dist_, obj_trace_;
  std::vector<uint16_t> ha_, hb_;
};

}  // namespace

int train_key_codebook_gpu(const Geom& g, const double* calib, long long n, const TrainConfig& em,
                           double* atoms_out, std::vector<std::vector<double>>* traces,
                           std::vector<double>* mse, std::string* err, cudaStream_t st) {
  try {
    if (n < (long long)g.L * g.L)
      throw TrainFail{1, "train_key_codebook: need at least n_levels^2 calibration rows"};
    if (g.L * g.L > kSoftThreads * kSoftMaxK)
      throw TrainFail{1, "train_key_codebook: n_levels^2 > 4096 not supported on the GPU"};
    bool all_zero = true;
    for (long long i = 0; i < n * g.d; ++i) {
      if (!std::isfinite(calib[i])) throw TrainFail{1, "train_key_codebook: calib not finite"};
      if (calib[i] != 0.0) all_zero = false;
    }
    if (all_zero) throw TrainFail{2, "train_key_codebook: degenerate all-zero calibration"};
    DevBufs buf;
    double* res = buf.get<double>((size_t)n * g.d);
    TCU(cudaMemcpyAsync(res, calib, (size_t)n * g.d * 8, cudaMemcpyHostToDevice, st));
    const double denom = static_cast<double>(n * g.d);
    std::vector<double> host_res((size_t)n * g.d);
    for (int r = 0; r < g.R; ++r) {
      for (int grp = 0; grp < g.groups; ++grp) {
        GroupEmGpu fit(res + (size_t)grp * 2 * g.g, g.d, n, g.g, g.L, em,
                       mix_seed(em.seed, (size_t)r, (size_t)grp), st);
        fit.run();
        traces->push_back(fit.objective_trace());
        const std::vector<double>& at = fit.atoms();
        for (int s = 0; s < g.g; ++s)
          for (int l = 0; l < g.L; ++l) {
            const size_t dst = (((size_t)r * g.subs + (size_t)grp * g.g + s) * g.L + l) * 2;
            atoms_out[dst] = at[((size_t)s * g.L + l) * 2];
            atoms_out[dst + 1] = at[((size_t)s * g.L + l) * 2 + 1];
          }
        k_em_residual<<<nblk(n * g.g, 256), 256, 0, st>>>(res, g.d, grp * 2 * g.g, g.g, g.L, n,
                                                          fit.atoms_dev(), fit.a_dev(), fit.b_dev());
        count_launch();
        TCU(cudaGetLastError());
        TCU(cudaStreamSynchronize(st));
      }
      TCU(cudaMemcpyAsync(host_res.data(), res, host_res.size() * 8, cudaMemcpyDeviceToHost, st));
      TCU(cudaStreamSynchronize(st));
      double sq = 0.0;
      for (double x : host_res) sq += x * x;
      mse->push_back(sq / denom);
    }
    return 0;
  } catch (const TrainFail& f) {
    *err = f.msg;
    return f.code;
  }
}

// encode_keys with AssignSearch::factorized (keyquant.cpp:705-739 with
// assign_factorized 204-224): per (round, group) the CenterCache tables, the
// sequential projections and |p|^2, the base - 2 pu - 2 pv argmin (strict
// '<' in a*L+b order), then the exact residual update -- the same kernels
// (and therefore the same fp64 operation order) as the factorized EM E-step.
// keys: device fp64 [n][d]; a, b: device, KeyCodes::idx order.
cudaError_t encode_keys_factorized_gpu(const Geom& g, const double* atoms, const double* keys,
                                       long long n, uint16_t* a, uint16_t* b, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  try {
  const int w = 2 * g.g, L = g.L;
  DevBufs buf;
  double* res = buf.get<double>((size_t)n * g.d);
  double* uT = buf.get<double>((size_t)w * L);
  double* vT = buf.get<double>((size_t)w * L);
  double* un = buf.get<double>((size_t)L);
  double* vn = buf.get<double>((size_t)L);
  double* base = buf.get<double>((size_t)L * L);
  double* pu = buf.get<double>((size_t)n * L);
  double* pv = buf.get<double>((size_t)n * L);
  double* pn = buf.get<double>((size_t)n);
  cudaError_t e = cudaMemcpyAsync(res, keys, (size_t)n * g.d * 8, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  const int cs = g.R * g.groups;  // codes per token
  for (int r = 0; r < g.R; ++r)
    for (int grp = 0; grp < g.groups; ++grp) {
      const double* slice = atoms + ((size_t)r * g.subs + (size_t)grp * g.g) * L * 2;
      k_em_tables<<<nblk((long long)w * L, 256), 256, 0, st>>>(slice, g.g, L, uT, vT, un, vn, base, 0);
      k_em_tables<<<nblk((long long)L * L, 256), 256, 0, st>>>(slice, g.g, L, uT, vT, un, vn, base, 1);
      double* P = res + (size_t)grp * w;
      k_em_pnorm<<<nblk(n, 256), 256, 0, st>>>(P, g.d, w, n, pn);
      k_em_project<<<nblk(n, kProjPts), 128, (size_t)kProjPts * w * 8, st>>>(P, g.d, w, n, uT, vT,
                                                                          L, pu, pv);
      const int off = r * g.groups + grp;
      k_em_assign_factorized<<<nblk(n, 8), 256, 0, st>>>(pu, pv, pn, base, L, n, a + off, b + off,
                                                         nullptr, cs);
      k_em_residual<<<nblk(n * g.g, 256), 256, 0, st>>>(res, g.d, grp * w, g.g, L, n, slice, a + off,
                                                        b + off, cs);
      count_launch(6);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  return cudaStreamSynchronize(st);  // DevBufs frees on return
  } catch (const TrainFail&) {
    return cudaErrorMemoryAllocation;
  }
}

}  // namespace cvq
