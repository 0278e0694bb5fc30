// encode.cu -- bit-exact KV encoders on sm_100a.
//
// Keys: replaces encode_keys with brute-force search (keyquant.cpp:705-739,
// CenterCache::assign_brute 180-200).  The reference scans all L^2 centers
// c_ab = u_a + v_b of each (round, group) slice with an fp64 sequential
// squared distance (no FMA) and strict '<', so ties go to the smallest
// a*L+b.  Codes must be bit-identical, including near-ties.
//
// Device algorithm per (token, round, group):
//   1. screen: s(a,b) = base[a,b] - 2 p.u_a - 2 p.v_b  (fp64, FMA allowed),
//      the factorised form of keyquant.cpp:204-224; |p|^2 is shared.
//   2. if the runner-up screen value is > best + margin, the best pair is
//      the reference argmin (margin bounds screen + reference rounding,
//      see kMarginRel below); otherwise every pair within the margin is
//      re-evaluated with the reference's exact fp64 sequence
//      (__dsub_rn/__dmul_rn/__dadd_rn, increasing c, strict '<').
//   3. residual -= (u_a + v_b) in fp64 exactly as keyquant.cpp:733-734.
// Non-finite or overflowing residuals take the exact brute-force path for
// every pair (the reference then returns pair 0).
//
// Values: replaces encoder_forward in infer mode (valquant.cpp:50-101):
// h = relu(t.w1 + b1), logit = h.w2 + b2 in the reference's summation order
// with zero-skips (valquant.cpp:53-68), bit = logit > 0.  Exact fp64, no
// FMA, so logits and bits are bit-identical.
#include <cfloat>
#include <cmath>

#include "cvq_internal.cuh"

namespace cvq {

// Screen error bound, relative to (|p| + 2 max|u|)^2: worst-case fp64
// rounding of the screen and of the reference sum is ~4*(2g+4)*2^-53 of that
// scale (< 6e-14 at g = 64); 1e-11 leaves a ~90x safety factor.
constexpr double kMarginRel = 1e-11;
// fp32 screen: worst-case error 3 * 2^-24 of scale^2 per value (see the
// table kernel), 3.6e-7 pair to pair; 4e-6 leaves an 11x safety factor.
constexpr double kMarginRel32 = 4e-6;

// ---------------------------------------------------------------- tables
// base[a][b] = |u_a|^2 + |v_b|^2 + 2 u_a.v_b per (slot, round, group) and
// max_l |u_l| (= max |v_l|, v is u rotated per subspace).
__global__ void k_key_base(Geom g, const double* __restrict__ atoms,
                           double* __restrict__ base, double* __restrict__ maxnorm,
                           float* __restrict__ atomsf, float* __restrict__ basef) {
  const int rg = blockIdx.x;  // r * groups + grp
  const int slot = blockIdx.y;
  const int r = rg / g.groups, grp = rg % g.groups;
  const double2* U = reinterpret_cast<const double2*>(atoms) +
                     ((size_t)(slot * g.R + r) * g.subs + (size_t)grp * g.g) * g.L;
  double* B = base + ((size_t)slot * g.R * g.groups + rg) * g.L * g.L;
  __shared__ double nrm[1024];
  for (int l = threadIdx.x; l < g.L; l += blockDim.x) {
    double s = 0.0;
    for (int si = 0; si < g.g; ++si) {
      double2 u = U[(size_t)si * g.L + l];
      s += u.x * u.x + u.y * u.y;
    }
    if (l < 1024) nrm[l] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < g.L * g.L; e += blockDim.x) {
    const int a = e / g.L, b = e % g.L;
    double uv = 0.0;
    for (int si = 0; si < g.g; ++si) {
      double2 ua = U[(size_t)si * g.L + a], ub = U[(size_t)si * g.L + b];
      uv += ua.x * (-ub.y) + ua.y * ub.x;  // u_a . v_b, v_b = (-y_b, x_b)
    }
    B[e] = nrm[a] + nrm[b] + 2.0 * uv;
    if (basef) basef[((size_t)slot * g.R * g.groups + rg) * g.L * g.L + e] = (float)B[e];
  }
  if (atomsf) {
    const size_t o = ((size_t)(slot * g.R + r) * g.subs + (size_t)grp * g.g) * g.L * 2;
    for (int e = threadIdx.x; e < g.g * g.L * 2; e += blockDim.x) atomsf[o + e] = (float)atoms[o + e];
  }
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int l = 0; l < g.L; ++l) m = fmax(m, nrm[l]);
    maxnorm[(size_t)slot * g.R * g.groups + rg] = sqrt(m);
  }
}

cudaError_t build_key_enc_tables(const Geom& g, int n_slots, const double* atoms,
                                 double* base, double* maxnorm, cudaStream_t st, float* atomsf,
                                 float* basef) {
  if (g.L > 1024) return cudaErrorInvalidValue;
  dim3 grid(g.R * g.groups, n_slots);
  k_key_base<<<grid, 256, 0, st>>>(g, atoms, base, maxnorm, atomsf, basef);
  count_launch();
  return cudaGetLastError();
}

__device__ __forceinline__ double load_elem(const void* p, int dtype, long long idx) {
  return dtype == 0 ? (double)static_cast<const float*>(p)[idx]
                    : static_cast<const double*>(p)[idx];
}

// Exact reference distance of residual p (2g values) to center (a, b).
// U rows are us double2 apart (us = L in global memory, L + 1 in the padded
// shared-memory copy of k_encode_keys_table).
__device__ __forceinline__ double exact_dist(const double* p, const double2* U, int us, int gsz,
                                             int a, int b) {
  double s = 0.0;
  for (int si = 0; si < gsz; ++si) {
    const double2 ua = U[(size_t)si * us + a], ub = U[(size_t)si * us + b];
    const double c0 = __dadd_rn(ua.x, -ub.y);  // u_a + v_b, keyquant.cpp:152-156
    const double c1 = __dadd_rn(ua.y, ub.x);
    const double d0 = __dsub_rn(p[2 * si], c0);
    s = __dadd_rn(s, __dmul_rn(d0, d0));
    const double d1 = __dsub_rn(p[2 * si + 1], c1);
    s = __dadd_rn(s, __dmul_rn(d1, d1));
  }
  return s;
}

__device__ __forceinline__ void argmin_merge(double& v, int& c, double v2, int c2) {
  if (v2 < v || (v2 == v && c2 < c)) {
    v = v2;
    c = c2;
  }
}

__device__ __forceinline__ void warp_argmin(double& v, int& c) {
  for (int o = 16; o; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int c2 = __shfl_xor_sync(0xffffffffu, c, o);
    argmin_merge(v, c, v2, c2);
  }
}

// Exact search over all pairs (or those whose screen value is <= thr when
// use_thr) for one token; U may be shared or global.
__device__ __forceinline__ double screen_val(const double* B, const double* PU, const double* PV,
                                             int L, int a, int b) {
  return B[(size_t)a * L + b] - 2.0 * PU[a] - 2.0 * PV[b];
}
// fp32 screen: (B - 2 pu) by one FMA, then - 2 pv (2 pv exact): two roundings
__device__ __forceinline__ float screen_val(const float* B, const float* PU, const float* PV, int L,
                                            int a, int b) {
  return fmaf(-2.f, PU[a], B[(size_t)a * L + b]) - 2.f * PV[b];
}

template <class T>
__device__ int exact_search(const double* p, const double2* U, int us, int L, int gsz, const T* B,
                            const T* PU, const T* PV, bool use_thr, T thr) {
  const int lane = threadIdx.x & 31;
  double best = INFINITY;
  int bc = 0x7fffffff;
  for (int c = lane; c < L * L; c += 32) {
    const int a = c / L, b = c % L;
    if (use_thr) {
      const T sc = screen_val(B, PU, PV, L, a, b);
      if (!(sc <= thr)) continue;
    }
    const double d = exact_dist(p, U, us, gsz, a, b);
    if (d < best) {  // increasing c per lane: strict '<' keeps the smallest
      best = d;
      bc = c;
    }
  }
  // Lanes whose candidates were all NaN/inf keep bc = INT_MAX unless the
  // reference would pick them: assign_brute picks c = 0 when nothing is
  // strictly below +inf.
  warp_argmin(best, bc);
  if (bc == 0x7fffffff) bc = 0;
  return bc;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

constexpr int kEncTok = 32;
constexpr int kEncWarps = 16;  // measured: 8 -> 4.5e6, 16 -> 6.9e6, 32 -> 3.2e6 token-heads/s (C4 sample)

// Table-screen encoder: one CTA per (32-token tile, stream); one warp per
// token at a time.  Requires g*L*16 + L*L*8 bytes of the slice in smem.
__global__ void __launch_bounds__(kEncWarps * 32)
k_encode_keys_table(Geom g, int n_slots, const double* __restrict__ atoms,
                    const double* __restrict__ base, const double* __restrict__ maxnorm,
                    const void* __restrict__ keys, int dtype, long long s_stride, long long n,
                    uint16_t* __restrict__ a_out, uint16_t* __restrict__ b_out) {
  extern __shared__ double sm[];
  // U rows padded to L + 1 double2: the residual update reads one column
  // down all rows (stride L double2 = 1 KiB would be a 32-way bank conflict)
  const int us = g.L + 1;
  double2* U = reinterpret_cast<double2*>(sm);          // [g][L + 1]
  double* B = sm + 2 * (size_t)g.g * us;                // [L][L]
  double* P = B + (size_t)g.L * g.L;                    // [kEncTok][d]
  double* PU = P + (size_t)kEncTok * g.d;               // [warps][L]
  double* PV = PU + (size_t)kEncWarps * g.L;            // [warps][L]
  float* Bf = reinterpret_cast<float*>(PV + (size_t)kEncWarps * g.L);  // [L][L] fp32 screen table
  // (reassigned below for the tiled layout)
  float* PUf = Bf + (size_t)g.L * g.L;                  // [warps][L]
  float* PVf = PUf + (size_t)kEncWarps * g.L;           // [warps][L]
  // head presets (L = 64, 64 subspaces per group): projections of the whole
  // tile per round into [tok][L] tables, which then take the place of the
  // per-warp PU / PV / PUf / PVf rows (same smem offset)
  const bool tiled = g.L == 64 && g.g == 64 && kEncTok == 32 && kEncWarps == 16;
  double* TPU = PU;                                    // [tok][L]
  double* TPV = TPU + (size_t)kEncTok * g.L;
  float* TPUf = reinterpret_cast<float*>(TPV + (size_t)kEncTok * g.L);
  float* TPVf = TPUf + (size_t)kEncTok * g.L;
  if (tiled) Bf = TPVf + (size_t)kEncTok * g.L;       // the fp32 screen table after them
  const int s = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long i0 = (long long)blockIdx.x * kEncTok;
  const int nt = (int)min((long long)kEncTok, n - i0);
  const int slot = s % n_slots;
  for (int e = tid; e < nt * g.d; e += blockDim.x)
    P[e] = load_elem(keys, dtype, (long long)s * s_stride + (i0 + e / g.d) * g.d + e % g.d);
  const int L = g.L, gs = g.g, w2 = 2 * g.g;
  for (int r = 0; r < g.R; ++r) {
    for (int grp = 0; grp < g.groups; ++grp) {
      __syncthreads();
      const double2* Ug = reinterpret_cast<const double2*>(atoms) +
                          ((size_t)(slot * g.R + r) * g.subs + (size_t)grp * gs) * L;
      const double* Bg = base + ((size_t)(slot * g.R + r) * g.groups + grp) * L * L;
      // the round's slice and base table by cp.async (16 B per request, no
      // register round trip: the plain load/store loop was latency-bound)
      for (int e = tid; e < gs * L; e += blockDim.x) cp_async16(U + (e / L) * us + e % L, Ug + e);
      for (int e = 2 * tid; e < L * L; e += 2 * blockDim.x) cp_async16(B + e, Bg + e);
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;\n" ::: "memory");
      const double mn = maxnorm[(size_t)(slot * g.R + r) * g.groups + grp];
      __syncthreads();
      for (int e = tid; e < L * L; e += blockDim.x) Bf[e] = (float)B[e];
      if (!tiled) __syncthreads();  // tiled: the barrier after the projections
      if (tiled) {
        // projections of every token of the tile at once, register-tiled:
        // thread = 4 tokens x 2 levels x (u, v) over one half of the
        // subspaces (threads 256..511 the upper half, added through smem).
        // Per subspace 2 LDS.128 of U (levels lg and lg + 32: 4 wavefronts
        // each) + 4 broadcast P loads feed 32 DFMA.
        // (Summation order is free here: pu / pv only feed the screen.)
        const int hs = tid >> 8, lg = tid & 31, tq = (tid >> 5) & 7;  // tokens 4 tq .. 4 tq + 3
        double su[4][2], sv[4][2];
#pragma unroll
        for (int t = 0; t < 4; ++t) su[t][0] = su[t][1] = sv[t][0] = sv[t][1] = 0.0;
        const double* p0 = P + (size_t)(4 * tq) * g.d + grp * w2;
        const int sh = gs >> 1;
#pragma unroll 2
        for (int si = hs * sh; si < (hs + 1) * sh; ++si) {
          const double2 u0 = U[(size_t)si * us + lg], u1 = U[(size_t)si * us + lg + 32];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const double2 pa = *reinterpret_cast<const double2*>(p0 + (size_t)t * g.d + 2 * si);
            su[t][0] = fma(pa.x, u0.x, fma(pa.y, u0.y, su[t][0]));
            sv[t][0] = fma(pa.y, u0.x, fma(-pa.x, u0.y, sv[t][0]));
            su[t][1] = fma(pa.x, u1.x, fma(pa.y, u1.y, su[t][1]));
            sv[t][1] = fma(pa.y, u1.x, fma(-pa.x, u1.y, sv[t][1]));
          }
        }
        if (hs) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const size_t o = (size_t)(4 * tq + t) * L + lg;
            TPU[o] = su[t][0];
            TPU[o + 32] = su[t][1];
            TPV[o] = sv[t][0];
            TPV[o + 32] = sv[t][1];
          }
        }
        __syncthreads();
        if (!hs) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const size_t o = (size_t)(4 * tq + t) * L + lg;
            const double u0 = su[t][0] + TPU[o], u1 = su[t][1] + TPU[o + 32];
            const double v0 = sv[t][0] + TPV[o], v1 = sv[t][1] + TPV[o + 32];
            TPU[o] = u0;
            TPU[o + 32] = u1;
            TPV[o] = v0;
            TPV[o + 32] = v1;
            TPUf[o] = (float)u0;
            TPUf[o + 32] = (float)u1;
            TPVf[o] = (float)v0;
            TPVf[o + 32] = (float)v1;
          }
        }
        __syncthreads();
      }
      for (int tk = warp; tk < nt; tk += kEncWarps) {
        double* p = P + (size_t)tk * g.d + grp * w2;
        double* pu = tiled ? TPU + (size_t)tk * L : PU + warp * L;
        double* pv = tiled ? TPV + (size_t)tk * L : PV + warp * L;
        float* puf = tiled ? TPUf + (size_t)tk * L : PUf + warp * L;
        float* pvf = tiled ? TPVf + (size_t)tk * L : PVf + warp * L;
        if (!tiled) {
          for (int l = lane; l < L; l += 32) {
            double su = 0.0, sv = 0.0;
            for (int si = 0; si < gs; ++si) {
              const double2 u = U[(size_t)si * us + l];
              const double px = p[2 * si], py = p[2 * si + 1];
              su = fma(px, u.x, fma(py, u.y, su));
              sv = fma(py, u.x, fma(-px, u.y, sv));
            }
            pu[l] = su;
            pv[l] = sv;
            puf[l] = (float)su;
            pvf[l] = (float)sv;
          }
        }
        double pn = 0.0;
        for (int e = lane; e < w2; e += 32) pn = fma(p[e], p[e], pn);
        for (int o = 16; o; o >>= 1) pn += __shfl_xor_sync(0xffffffffu, pn, o);
        __syncwarp();
        int chosen;
        const double scale = sqrt(pn) + 2.0 * mn;
        const double scale2 = scale * scale * fmax(1.0, w2 / 128.0);
        if (!(pn < 1e300) || !(mn < 1e150)) {
          chosen = exact_search(p, U, us, L, gs, B, pu, pv, false, 0.0);
        } else if (scale2 > 1e-30 && scale2 < 1e30) {
          // fp32 screen (twice the pair rate of fp64).  Each screen value is
          // within 3 * 2^-24 * scale^2 of the exact shifted distance (inputs
          // rounded once to fp32, two fp32 roundings; |B| + 2|pu| + 2|pv| <=
          // scale^2), so a pair-to-pair error below 3.6e-7 scale^2: with the
          // 4e-6 margin every pair that can be the reference argmin is
          // re-checked exactly whenever the screen is not decisive.
          float b1 = INFINITY, b2 = INFINITY;
          int c1 = 0x7fffffff;
          float m1a = INFINITY, m1b = INFINITY;
          if (L == 64) {
            // lane = columns b = 2 lane, 2 lane + 1 (one LDS.64 per row);
            // per column only the running min and runner-up of
            // x = fl(B - 2 pu) over a (4 instructions per pair), the
            // "- 2 pv[b]" applied at the end: fl(x - t) is monotone in x, so
            // the column's best and runner-up screen values are those of x.
            // No index is tracked: when the screen is decisive the best is
            // unique and its row is recovered from the winning column below;
            // ties leave the runner-up equal to the best, i.e. not decisive.
            const int b0 = 2 * lane;
            float m2a = INFINITY, m2b = INFINITY;
#pragma unroll 4
            for (int a0 = 0; a0 < 64; a0 += 4) {
              const float4 pu4 = *reinterpret_cast<const float4*>(puf + a0);
              const float pus[4] = {pu4.x, pu4.y, pu4.z, pu4.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float2 bb = *reinterpret_cast<const float2*>(Bf + (a0 + u) * 64 + b0);
                const float xa = fmaf(-2.f, pus[u], bb.x), xb = fmaf(-2.f, pus[u], bb.y);
                m2a = fminf(m2a, fmaxf(m1a, xa));
                m1a = fminf(m1a, xa);
                m2b = fminf(m2b, fmaxf(m1b, xb));
                m1b = fminf(m1b, xb);
              }
            }
            const float2 pv2 = *reinterpret_cast<const float2*>(pvf + b0);
            const float va = m1a - 2.f * pv2.x, vb = m1b - 2.f * pv2.y;
            const float ra = m2a - 2.f * pv2.x, rb = m2b - 2.f * pv2.y;
            if (vb < va) {  // c1 = the column (the row comes later)
              b1 = vb; c1 = b0 + 1; b2 = fminf(rb, va);
            } else {
              b1 = va; c1 = b0; b2 = fminf(ra, vb);
            }
          } else {
            for (int b = lane; b < L; b += 32) {
              const float t2 = 2.f * pvf[b];
              for (int a = 0; a < L; ++a) {
                const float sc = fmaf(-2.f, puf[a], Bf[a * L + b]) - t2;
                const int c = a * L + b;
                if (sc < b1 || (sc == b1 && c < c1)) {
                  b2 = b1;
                  b1 = sc;
                  c1 = c;
                } else if (sc < b2) {
                  b2 = sc;
                }
              }
            }
          }
          float gb = b1;
          int gc = c1;
          for (int o = 16; o; o >>= 1) {
            const float v2 = __shfl_xor_sync(0xffffffffu, gb, o);
            const int c2 = __shfl_xor_sync(0xffffffffu, gc, o);
            if (v2 < gb || (v2 == gb && c2 < gc)) {
              gb = v2;
              gc = c2;
            }
          }
          float ru = (c1 == gc) ? b2 : b1;
          for (int o = 16; o; o >>= 1) ru = fminf(ru, __shfl_xor_sync(0xffffffffu, ru, o));
          const float margin = (float)(kMarginRel32 * scale2);
          if (ru > gb + margin) {
            if (L == 64) {
              // row of the unique best in column gc: the a whose x (same
              // fmaf, same inputs) equals the column minimum
              const float mc = __shfl_sync(0xffffffffu, (gc & 1) ? m1b : m1a, gc >> 1);
              const float x0 = fmaf(-2.f, puf[lane], Bf[lane * 64 + gc]);
              const float x1 = fmaf(-2.f, puf[lane + 32], Bf[(lane + 32) * 64 + gc]);
              const unsigned k0 = __ballot_sync(0xffffffffu, x0 == mc);
              const unsigned k1 = __ballot_sync(0xffffffffu, x1 == mc);
              chosen = (k0 ? __ffs(k0) - 1 : 31 + __ffs(k1)) * 64 + gc;
            } else {
              chosen = gc;
            }
          } else {
            chosen = exact_search(p, U, us, L, gs, Bf, puf, pvf, true, gb + margin);
          }
        } else {
          // single pass: lane-local best and runner-up, then warp merge
          double b1 = INFINITY, b2 = INFINITY;
          int c1 = 0x7fffffff;
          for (int b = lane; b < L; b += 32) {
            const double t2 = 2.0 * pv[b];
            for (int a = 0; a < L; ++a) {
              const double sc = B[a * L + b] - 2.0 * pu[a] - t2;
              const int c = a * L + b;
              if (sc < b1 || (sc == b1 && c < c1)) {
                b2 = b1;
                b1 = sc;
                c1 = c;
              } else if (sc < b2) {
                b2 = sc;
              }
            }
          }
          double gb = b1;
          int gc = c1;
          warp_argmin(gb, gc);
          // runner-up over the warp: every lane's b2, plus other lanes' b1
          double ru = (c1 == gc) ? b2 : b1;
          for (int o = 16; o; o >>= 1) ru = fmin(ru, __shfl_xor_sync(0xffffffffu, ru, o));
          const double margin = kMarginRel * scale2;
          if (ru > gb + margin) {
            chosen = gc;
          } else {
            chosen = exact_search(p, U, us, L, gs, B, pu, pv, true, gb + margin);
          }
        }
        const int ca = chosen / L, cb = chosen % L;
        if (lane == 0) {
          const size_t idx = ((size_t)s * n + i0 + tk) * (g.R * g.groups) + (size_t)r * g.groups + grp;
          a_out[idx] = (uint16_t)ca;
          b_out[idx] = (uint16_t)cb;
        }
        for (int si = lane; si < gs; si += 32) {
          const double2 ua = U[(size_t)si * us + ca], ub = U[(size_t)si * us + cb];
          p[2 * si] = __dsub_rn(p[2 * si], __dadd_rn(ua.x, -ub.y));
          p[2 * si + 1] = __dsub_rn(p[2 * si + 1], __dadd_rn(ua.y, ub.x));
        }
        __syncwarp();
      }
    }
  }
}

// Head-preset key encoder (L = 64 levels, g = 64 subspaces per group):
// one CTA per (32-token tile, stream), 512 threads.  Per (round, group):
//  * the fp64 slice U (exact distances, residual update; rows padded to 65)
//    and the fp32 copies of the slice and of the base table arrive by
//    cp.async from global fp32 tables built with the codebook;
//  * projections p.u / p.v of all 32 tokens in fp32 (thread = 4 tokens x
//    levels lg, lg + 32 over half the subspaces): twice the fp64 rate;
//  * the index-free column screen of k_encode_keys_table, margin kMarginT64.
// Screen error with fp32 projections (u = 2^-24, |p.u_a| sums 2g = 128
// products, computed as two 64-FMA halves + one add, inputs rounded once):
// |err(pu)| <= 68 u |p| |u_a| <= 68 u |p| mn, the same for pv; with the base
// rounding and the two screen roundings a screen value is within
// 3 u scale^2 + 4 * 68 u |p| mn <= 37 u scale^2 (|p| mn <= scale^2 / 8)
// of the exact shifted distance: 4.4e-6 scale^2 pair to pair, so the margin
// 8e-6 keeps a 1.8x factor.  Out-of-range scales and non-finite residuals
// take the exact search over all pairs.
constexpr double kMarginT64 = 8e-6;
__global__ void __launch_bounds__(kEncWarps * 32, 1)
k_encode_keys_t64(Geom g, int n_slots, const double* __restrict__ atoms,
                  const float* __restrict__ atomsf, const float* __restrict__ basef,
                  const double* __restrict__ maxnorm, const void* __restrict__ keys, int dtype,
                  long long s_stride, long long n, uint16_t* __restrict__ a_out,
                  uint16_t* __restrict__ b_out) {
  constexpr int L = 64, gs = 64, w2 = 128, us = L + 1;
  extern __shared__ double sm[];
  double2* U = reinterpret_cast<double2*>(sm);                     // [64][65]
  float2* Uf = reinterpret_cast<float2*>(U + gs * us);             // [64][64]
  float* Bf = reinterpret_cast<float*>(Uf + gs * L);               // [64][64]
  double* P = reinterpret_cast<double*>(Bf + L * L);               // [32][d]
  float* Pf = reinterpret_cast<float*>(P + (size_t)kEncTok * g.d); // [32][128] (this group)
  float* TPUf = Pf + kEncTok * w2;                                 // [32][64]
  float* TPVf = TPUf + kEncTok * L;                                // [32][64]
  const int s = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long i0 = (long long)blockIdx.x * kEncTok;
  const int nt = (int)min((long long)kEncTok, n - i0);
  const int slot = s % n_slots;
  for (int e = tid; e < nt * g.d; e += blockDim.x)
    P[e] = load_elem(keys, dtype, (long long)s * s_stride + (i0 + e / g.d) * g.d + e % g.d);
  for (int r = 0; r < g.R; ++r) {
    for (int grp = 0; grp < g.groups; ++grp) {
      __syncthreads();
      const size_t rg = (size_t)(slot * g.R + r) * g.groups + grp;
      const size_t uo = ((size_t)(slot * g.R + r) * g.subs + (size_t)grp * gs) * L;
      const double2* Ug = reinterpret_cast<const double2*>(atoms) + uo;
      for (int e = tid; e < gs * L; e += blockDim.x) cp_async16(U + (e / L) * us + e % L, Ug + e);
      const float2* Ufg = reinterpret_cast<const float2*>(atomsf) + uo;
      for (int e = 2 * tid; e < gs * L; e += 2 * blockDim.x) cp_async16(Uf + e, Ufg + e);
      const float* Bg = basef + rg * L * L;
      for (int e = 4 * tid; e < L * L; e += 4 * blockDim.x) cp_async16(Bf + e, Bg + e);
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;\n" ::: "memory");
      for (int e = tid; e < kEncTok * w2; e += blockDim.x)
        Pf[e] = (float)P[(size_t)(e / w2) * g.d + grp * w2 + e % w2];
      const double mn = maxnorm[rg];
      __syncthreads();
      {  // fp32 projections, halves of the subspaces added through smem
        const int hs = tid >> 8, lg = tid & 31, tq = (tid >> 5) & 7;
        float su[4][2], sv[4][2];
#pragma unroll
        for (int t = 0; t < 4; ++t) su[t][0] = su[t][1] = sv[t][0] = sv[t][1] = 0.f;
        const float* p0 = Pf + (size_t)(4 * tq) * w2;
#pragma unroll 4
        for (int si = hs * 32; si < hs * 32 + 32; si += 2) {  // two subspaces per P load
          const float2 u0 = Uf[si * L + lg], u1 = Uf[si * L + lg + 32];
          const float2 v0 = Uf[(si + 1) * L + lg], v1 = Uf[(si + 1) * L + lg + 32];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float4 pq = *reinterpret_cast<const float4*>(p0 + t * w2 + 2 * si);
            su[t][0] = fmaf(pq.x, u0.x, fmaf(pq.y, u0.y, su[t][0]));
            sv[t][0] = fmaf(pq.y, u0.x, fmaf(-pq.x, u0.y, sv[t][0]));
            su[t][1] = fmaf(pq.x, u1.x, fmaf(pq.y, u1.y, su[t][1]));
            sv[t][1] = fmaf(pq.y, u1.x, fmaf(-pq.x, u1.y, sv[t][1]));
            su[t][0] = fmaf(pq.z, v0.x, fmaf(pq.w, v0.y, su[t][0]));
            sv[t][0] = fmaf(pq.w, v0.x, fmaf(-pq.z, v0.y, sv[t][0]));
            su[t][1] = fmaf(pq.z, v1.x, fmaf(pq.w, v1.y, su[t][1]));
            sv[t][1] = fmaf(pq.w, v1.x, fmaf(-pq.z, v1.y, sv[t][1]));
          }
        }
        if (hs) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int o = (4 * tq + t) * L + lg;
            TPUf[o] = su[t][0];
            TPUf[o + 32] = su[t][1];
            TPVf[o] = sv[t][0];
            TPVf[o + 32] = sv[t][1];
          }
        }
        __syncthreads();
        if (!hs) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int o = (4 * tq + t) * L + lg;
            TPUf[o] += su[t][0];
            TPUf[o + 32] += su[t][1];
            TPVf[o] += sv[t][0];
            TPVf[o + 32] += sv[t][1];
          }
        }
        __syncthreads();
      }
      for (int tk = warp; tk < nt; tk += kEncWarps) {
        double* p = P + (size_t)tk * g.d + grp * w2;
        const float* puf = TPUf + tk * L;
        const float* pvf = TPVf + tk * L;
        double pn = 0.0;
        for (int e = lane; e < w2; e += 32) pn = fma(p[e], p[e], pn);
        for (int o = 16; o; o >>= 1) pn += __shfl_xor_sync(0xffffffffu, pn, o);
        const double scale = sqrt(pn) + 2.0 * mn;
        const double scale2 = scale * scale;
        int chosen;
        if (!(pn < 1e300) || !(mn < 1e150) || !(scale2 > 1e-30 && scale2 < 1e30)) {
          chosen = exact_search<float>(p, U, us, L, gs, nullptr, nullptr, nullptr, false, 0.f);
        } else {
          // column screen (k_encode_keys_table): lane = columns 2 lane, 2 lane + 1
          const int b0 = 2 * lane;
          float m1a = INFINITY, m2a = INFINITY, m1b = INFINITY, m2b = INFINITY;
#pragma unroll 4
          for (int a0 = 0; a0 < L; a0 += 4) {
            const float4 pu4 = *reinterpret_cast<const float4*>(puf + a0);
            const float pus[4] = {pu4.x, pu4.y, pu4.z, pu4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float2 bb = *reinterpret_cast<const float2*>(Bf + (a0 + u) * L + b0);
              const float xa = fmaf(-2.f, pus[u], bb.x), xb = fmaf(-2.f, pus[u], bb.y);
              m2a = fminf(m2a, fmaxf(m1a, xa));
              m1a = fminf(m1a, xa);
              m2b = fminf(m2b, fmaxf(m1b, xb));
              m1b = fminf(m1b, xb);
            }
          }
          const float2 pv2 = *reinterpret_cast<const float2*>(pvf + b0);
          const float va = m1a - 2.f * pv2.x, vb = m1b - 2.f * pv2.y;
          const float ra = m2a - 2.f * pv2.x, rb = m2b - 2.f * pv2.y;
          float b1, b2;
          int c1;
          if (vb < va) {
            b1 = vb; c1 = b0 + 1; b2 = fminf(rb, va);
          } else {
            b1 = va; c1 = b0; b2 = fminf(ra, vb);
          }
          float gb = b1;
          int gc = c1;
          for (int o = 16; o; o >>= 1) {
            const float v2 = __shfl_xor_sync(0xffffffffu, gb, o);
            const int c2 = __shfl_xor_sync(0xffffffffu, gc, o);
            if (v2 < gb || (v2 == gb && c2 < gc)) {
              gb = v2;
              gc = c2;
            }
          }
          float ru = (c1 == gc) ? b2 : b1;
          for (int o = 16; o; o >>= 1) ru = fminf(ru, __shfl_xor_sync(0xffffffffu, ru, o));
          const float margin = (float)(kMarginT64 * scale2);
          if (ru > gb + margin) {
            const float mc = __shfl_sync(0xffffffffu, (gc & 1) ? m1b : m1a, gc >> 1);
            const float x0 = fmaf(-2.f, puf[lane], Bf[lane * L + gc]);
            const float x1 = fmaf(-2.f, puf[lane + 32], Bf[(lane + 32) * L + gc]);
            const unsigned k0 = __ballot_sync(0xffffffffu, x0 == mc);
            const unsigned k1 = __ballot_sync(0xffffffffu, x1 == mc);
            chosen = (k0 ? __ffs(k0) - 1 : 31 + __ffs(k1)) * L + gc;
          } else {
            chosen = exact_search(p, U, us, L, gs, Bf, puf, pvf, true, gb + margin);
          }
        }
        const int ca = chosen / L, cb = chosen % L;
        if (lane == 0) {
          const size_t idx = ((size_t)s * n + i0 + tk) * (g.R * g.groups) + (size_t)r * g.groups + grp;
          a_out[idx] = (uint16_t)ca;
          b_out[idx] = (uint16_t)cb;
        }
        for (int si = lane; si < gs; si += 32) {
          const double2 ua = U[(size_t)si * us + ca], ub = U[(size_t)si * us + cb];
          p[2 * si] = __dsub_rn(p[2 * si], __dadd_rn(ua.x, -ub.y));
          p[2 * si + 1] = __dsub_rn(p[2 * si + 1], __dadd_rn(ua.y, ub.x));
        }
        __syncwarp();
      }
    }
  }
}

static size_t t64_smem(const Geom& g) {
  return (size_t)64 * 65 * 16 + 64 * 64 * 8 + 64 * 64 * 4 + (size_t)kEncTok * g.d * 8 +
         kEncTok * 128 * 4 + 2 * kEncTok * 64 * 4;
}

// Exact brute-force encoder for shapes whose slice does not fit on chip:
// one warp per token, centers read from global/L1.
__global__ void __launch_bounds__(128)
k_encode_keys_brute(Geom g, int n_slots, const double* __restrict__ atoms,
                    const void* __restrict__ keys, int dtype, long long s_stride, long long n,
                    uint16_t* __restrict__ a_out, uint16_t* __restrict__ b_out) {
  extern __shared__ double sm[];  // [4 warps][d]
  const int s = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * 4 + warp;
  if (i >= n) return;
  double* p = sm + (size_t)warp * g.d;
  for (int e = lane; e < g.d; e += 32)
    p[e] = load_elem(keys, dtype, (long long)s * s_stride + i * g.d + e);
  __syncwarp();
  const int slot = s % n_slots;
  for (int r = 0; r < g.R; ++r)
    for (int grp = 0; grp < g.groups; ++grp) {
      const double2* U = reinterpret_cast<const double2*>(atoms) +
                         ((size_t)(slot * g.R + r) * g.subs + (size_t)grp * g.g) * g.L;
      double* pg = p + grp * 2 * g.g;
      const int c = exact_search<double>(pg, U, g.L, g.L, g.g, nullptr, nullptr, nullptr, false, 0.0);
      const int ca = c / g.L, cb = c % g.L;
      if (lane == 0) {
        const size_t idx = ((size_t)s * n + i) * (g.R * g.groups) + (size_t)r * g.groups + grp;
        a_out[idx] = (uint16_t)ca;
        b_out[idx] = (uint16_t)cb;
      }
      __syncwarp();
      for (int si = lane; si < g.g; si += 32) {
        const double2 ua = U[(size_t)si * g.L + ca], ub = U[(size_t)si * g.L + cb];
        pg[2 * si] = __dsub_rn(pg[2 * si], __dadd_rn(ua.x, -ub.y));
        pg[2 * si + 1] = __dsub_rn(pg[2 * si + 1], __dadd_rn(ua.y, ub.x));
      }
      __syncwarp();
    }
}


// Decode-step key encoder: one 128-thread CTA per (token, stream), the
// round's slice and screen table read straight from L2 (no smem staging --
// appends encode one token per stream).  Same screen + exact re-check as
// k_encode_keys_table; requires 2L <= 128 (L <= 64).
constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;

__device__ __forceinline__ void block_argmin2(double& b1, int& c1, double& b2, double* rv, int* rc) {
  // per-warp: argmin with smallest index, runner-up = min over the rest
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = b1;
  int c = c1;
  warp_argmin(v, c);
  double ru = (c1 == c) ? b2 : b1;
  for (int o = 16; o; o >>= 1) ru = fmin(ru, __shfl_xor_sync(0xffffffffu, ru, o));
  constexpr int W = kSmallWarps;
  if (lane == 0) {
    rv[warp] = v;
    rc[warp] = c;
    rv[W + warp] = ru;
  }
  __syncthreads();
  if (warp == 0) {  // the same merge over the warps' (best, index, runner-up)
    const double wv = lane < W ? rv[lane] : INFINITY;
    const int wc = lane < W ? rc[lane] : 0x7fffffff;
    const double wr = lane < W ? rv[W + lane] : INFINITY;
    double gv = wv;
    int gc = wc;
    warp_argmin(gv, gc);
    double gr = (wc == gc) ? wr : wv;
    for (int o = 16; o; o >>= 1) gr = fmin(gr, __shfl_xor_sync(0xffffffffu, gr, o));
    if (lane == 0) {
      rv[2 * W] = gv;
      rv[2 * W + 1] = gr;
      rc[W] = gc;
    }
  }
  __syncthreads();
  b1 = rv[2 * W];
  b2 = rv[2 * W + 1];
  c1 = rc[W];
  __syncthreads();
}

// Decode-step key encoder for the head presets (L = g = 64) with the fp32
// tables of k_encode_keys_t64: a CTA of 512 threads per (token, stream).
// Per (round, group) only the fp32 slice and base table (48 KiB) stream in,
// double-buffered by cp.async; projections and the screen run in fp32 with
// the t64 margin (kMarginT64, same error analysis: each projection is four
// 32-product FMA partials plus three adds).  The fp64 slice is read from
// global memory only for the residual update and the (rare) exact search.
__global__ void __launch_bounds__(kSmallThreads)
k_encode_keys_small32(Geom g, int n_slots, const double* __restrict__ atoms,
                      const float* __restrict__ atomsf, const float* __restrict__ basef,
                      const double* __restrict__ maxnorm, const void* __restrict__ keys,
                      int dtype, long long s_stride, long long n, uint16_t* __restrict__ a_out,
                      uint16_t* __restrict__ b_out) {
  constexpr int L = 64, gs = 64, w2 = 128;
  extern __shared__ double sm[];
  float2* UB = reinterpret_cast<float2*>(sm);            // [2][64][64]
  float* BB = reinterpret_cast<float*>(UB + 2 * gs * L); // [2][64][64]
  double* P = reinterpret_cast<double*>(BB + 2 * L * L); // [d]
  float* Pf = reinterpret_cast<float*>(P + g.d);         // [128]
  float* PR = Pf + w2;                                   // [4][128] projection partials
  float* PUf = PR + 4 * w2;                              // [64]
  float* PVf = PUf + L;                                  // [64]
  __shared__ float rv[2 * kSmallWarps + 2];
  __shared__ int rc[kSmallWarps + 2];
  __shared__ double pns;
  const int s = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long i = blockIdx.x;
  const int slot = s % n_slots;
  for (int e = tid; e < g.d; e += blockDim.x)
    P[e] = load_elem(keys, dtype, (long long)s * s_stride + i * g.d + e);
  const int total = g.R * g.groups;
  auto stage = [&](int idx, int buf) {
    const int rr = idx / g.groups, gg = idx % g.groups;
    const size_t uo = ((size_t)(slot * g.R + rr) * g.subs + (size_t)gg * gs) * L;
    const float* Ug = atomsf + 2 * uo;
    const float* Bg = basef + ((size_t)(slot * g.R + rr) * g.groups + gg) * L * L;
    float* Ud = reinterpret_cast<float*>(UB + buf * gs * L);
    for (int e = 4 * tid; e < 2 * gs * L; e += 4 * kSmallThreads) cp_async16(Ud + e, Ug + e);
    for (int e = 4 * tid; e < L * L; e += 4 * kSmallThreads) cp_async16(BB + buf * L * L + e, Bg + e);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage(0, 0);
  for (int r = 0; r < g.R; ++r) {
    for (int grp = 0; grp < g.groups; ++grp) {
      const int idx = r * g.groups + grp, buf = idx & 1;
      if (idx + 1 < total) {
        stage(idx + 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      double* p = P + grp * w2;
      if (tid < w2) Pf[tid] = (float)p[tid];
      if (tid < 32) {
        double pn = 0.0;
        for (int e = tid; e < w2; e += 32) pn = fma(p[e], p[e], pn);
        for (int o = 16; o; o >>= 1) pn += __shfl_xor_sync(0xffffffffu, pn, o);
        if (tid == 0) pns = pn;
      }
      __syncthreads();
      const float2* Uf = UB + buf * gs * L;
      const float* Bf = BB + buf * L * L;
      {  // projections: thread (q, o) sums subspaces [16 q, 16 q + 16) of output o
        const int o = tid & 127, q = tid >> 7, l = o & 63;
        const bool isv = o >= L;
        float acc = 0.f;
#pragma unroll 8
        for (int si = 16 * q; si < 16 * q + 16; ++si) {
          const float2 u = Uf[si * L + l];
          const float px = Pf[2 * si], py = Pf[2 * si + 1];
          acc = isv ? fmaf(py, u.x, fmaf(-px, u.y, acc)) : fmaf(px, u.x, fmaf(py, u.y, acc));
        }
        PR[q * w2 + o] = acc;
      }
      __syncthreads();
      if (tid < w2) {
        const float v = ((PR[tid] + PR[w2 + tid]) + PR[2 * w2 + tid]) + PR[3 * w2 + tid];
        (tid >= L ? PVf : PUf)[tid & 63] = v;
      }
      __syncthreads();
      const double pn = pns;
      const double mn = maxnorm[(size_t)(slot * g.R + r) * g.groups + grp];
      const double scale = sqrt(pn) + 2.0 * mn, scale2 = scale * scale;
      const bool screen = pn < 1e300 && mn < 1e150 && scale2 > 1e-30 && scale2 < 1e30;
      const double2* U = reinterpret_cast<const double2*>(atoms) +
                         ((size_t)(slot * g.R + r) * g.subs + (size_t)grp * gs) * L;
      int chosen = 0;
      bool exact = !screen;
      float gb = 0.f, margin = 0.f;
      if (screen) {
        // thread: column b = tid & 63, rows a = (tid >> 6) + 8 k (increasing c)
        const int b = tid & 63;
        float m1 = INFINITY, m2 = INFINITY;
        int ia = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int a = (tid >> 6) + 8 * k;
          const float x = fmaf(-2.f, PUf[a], Bf[a * L + b]);
          if (x < m1) ia = a;
          m2 = fminf(m2, fmaxf(m1, x));
          m1 = fminf(m1, x);
        }
        const float t2 = 2.f * PVf[b];
        float v = m1 - t2, ru = m2 - t2;
        int c = ia * L + b;
        // block argmin (value, then smallest index) and runner-up
        float gv = v;
        int gc = c;
        for (int o = 16; o; o >>= 1) {
          const float v2 = __shfl_xor_sync(0xffffffffu, gv, o);
          const int c2 = __shfl_xor_sync(0xffffffffu, gc, o);
          if (v2 < gv || (v2 == gv && c2 < gc)) {
            gv = v2;
            gc = c2;
          }
        }
        float wr = (c == gc) ? ru : v;
        for (int o = 16; o; o >>= 1) wr = fminf(wr, __shfl_xor_sync(0xffffffffu, wr, o));
        if (lane == 0) {
          rv[warp] = gv;
          rc[warp] = gc;
          rv[kSmallWarps + warp] = wr;
        }
        __syncthreads();
        if (warp == 0) {
          const float wv = lane < kSmallWarps ? rv[lane] : INFINITY;
          const int wc = lane < kSmallWarps ? rc[lane] : 0x7fffffff;
          const float wrr = lane < kSmallWarps ? rv[kSmallWarps + lane] : INFINITY;
          float bv = wv;
          int bc = wc;
          for (int o = 16; o; o >>= 1) {
            const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
            const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
            if (v2 < bv || (v2 == bv && c2 < bc)) {
              bv = v2;
              bc = c2;
            }
          }
          float br = (wc == bc) ? wrr : wv;
          for (int o = 16; o; o >>= 1) br = fminf(br, __shfl_xor_sync(0xffffffffu, br, o));
          if (lane == 0) {
            rv[2 * kSmallWarps] = bv;
            rv[2 * kSmallWarps + 1] = br;
            rc[kSmallWarps] = bc;
          }
        }
        __syncthreads();
        gb = rv[2 * kSmallWarps];
        margin = (float)(kMarginT64 * scale2);
        chosen = rc[kSmallWarps];
        exact = !(rv[2 * kSmallWarps + 1] > gb + margin);
      }
      if (exact) {  // warp 0: exact search (screen-filtered when in range); rare
        if (warp == 0) {
          const int c = screen ? exact_search(p, U, L, L, gs, Bf, PUf, PVf, true, gb + margin)
                               : exact_search<float>(p, U, L, L, gs, nullptr, nullptr, nullptr,
                                                     false, 0.f);
          if (lane == 0) rc[kSmallWarps + 1] = c;
        }
        __syncthreads();
        chosen = rc[kSmallWarps + 1];
      }
      const int ca = chosen / L, cb = chosen % L;
      if (tid == 0) {
        const size_t o = ((size_t)s * n + i) * (g.R * g.groups) + (size_t)r * g.groups + grp;
        a_out[o] = (uint16_t)ca;
        b_out[o] = (uint16_t)cb;
      }
      if (tid < gs) {
        const double2 ua = U[(size_t)tid * L + ca], vb = U[(size_t)tid * L + cb];
        p[2 * tid] = __dsub_rn(p[2 * tid], __dadd_rn(ua.x, -vb.y));
        p[2 * tid + 1] = __dsub_rn(p[2 * tid + 1], __dadd_rn(ua.y, vb.x));
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kSmallThreads)
k_encode_keys_small(Geom g, int n_slots, const double* __restrict__ atoms,
                    const double* __restrict__ base, const double* __restrict__ maxnorm,
                    const void* __restrict__ keys, int dtype, long long s_stride, long long n,
                    uint16_t* __restrict__ a_out, uint16_t* __restrict__ b_out) {
  extern __shared__ double sm[];
  // the (round, group) slices and base tables double-buffered in smem by
  // cp.async: the next one streams in while this one is searched
  const size_t ub = (size_t)g.g * g.L * 2, bb_ = ((size_t)g.L * g.L + 1) & ~(size_t)1;  // doubles per buffer (16-B multiples)
  double* UB = sm;                    // [2][g][L] double2
  double* BB = UB + 2 * ub;           // [2][L][L]
  double* P = BB + 2 * bb_;           // [d]
  double* PU = P + g.d;               // [L]
  double* PV = PU + g.L;              // [L]
  double* PR = PV + g.L;              // [nsplit][2L] projection partials
  __shared__ double rv[2 * kSmallWarps + 2];
  __shared__ int rc[kSmallWarps + 1];
  __shared__ double pns;
  const int s = blockIdx.y, tid = threadIdx.x;
  const long long i = blockIdx.x;
  const int slot = s % n_slots;
  for (int e = tid; e < g.d; e += blockDim.x)
    P[e] = load_elem(keys, dtype, (long long)s * s_stride + i * g.d + e);
  __syncthreads();
  const int L = g.L, gs = g.g, w2 = 2 * g.g;
  const int total = g.R * g.groups;
  auto stage = [&](int idx, int buf) {
    const int rr = idx / g.groups, gg = idx % g.groups;
    const double* Ug = atoms + 2 * (((size_t)(slot * g.R + rr) * g.subs + (size_t)gg * gs) * L);
    const double* Bg = base + ((size_t)(slot * g.R + rr) * g.groups + gg) * L * L;
    for (size_t e = 2 * (size_t)tid; e < ub; e += 2 * kSmallThreads) cp_async16(UB + buf * ub + e, Ug + e);
    if ((L * L) & 1) {  // odd table: 8-B copies (the source is only 8-B aligned)
      for (size_t e = tid; e < (size_t)L * L; e += kSmallThreads) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(BB + buf * bb_ + e);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(Bg + e) : "memory");
      }
    } else {
      for (size_t e = 2 * (size_t)tid; e < bb_; e += 2 * kSmallThreads) cp_async16(BB + buf * bb_ + e, Bg + e);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage(0, 0);
  for (int r = 0; r < g.R; ++r) {
    for (int grp = 0; grp < g.groups; ++grp) {
      const int idx = r * g.groups + grp, buf = idx & 1;
      if (idx + 1 < total) {
        stage(idx + 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const double2* U = reinterpret_cast<const double2*>(UB + buf * ub);
      const double* B = BB + buf * bb_;
      const double mn = maxnorm[(size_t)(slot * g.R + r) * g.groups + grp];
      double* p = P + grp * w2;
      // projections: thread (q, o) sums subspaces [q sper, (q + 1) sper) of
      // output o (o < L: p.u_l, else p.v_l); partials summed below
      const int nsplit = kSmallThreads / (2 * L), sper = (gs + nsplit - 1) / nsplit;
      if (tid < nsplit * 2 * L) {
        const int o = tid % (2 * L), q = tid / (2 * L), l = o % L;
        const bool isv = o >= L;
        const int s0 = q * sper, s1 = min(gs, s0 + sper);
        double acc = 0.0;
#pragma unroll 8
        for (int si = s0; si < s1; ++si) {
          const double2 u = U[(size_t)si * L + l];
          const double px = p[2 * si], py = p[2 * si + 1];
          acc = isv ? fma(py, u.x, fma(-px, u.y, acc)) : fma(px, u.x, fma(py, u.y, acc));
        }
        PR[q * 2 * L + o] = acc;
      }
      if (tid < 32) {
        double pn = 0.0;
        for (int e = tid; e < w2; e += 32) pn = fma(p[e], p[e], pn);
        for (int o = 16; o; o >>= 1) pn += __shfl_xor_sync(0xffffffffu, pn, o);
        if (tid == 0) pns = pn;
      }
      __syncthreads();
      if (tid < 2 * L) {
        double acc = 0.0;
        for (int q = 0; q < nsplit; ++q) acc += PR[q * 2 * L + tid];
        (tid >= L ? PV : PU)[tid % L] = acc;
      }
      __syncthreads();
      const double pn = pns;
      int chosen;
      bool exact = !(pn < 1e300) || !(mn < 1e150);
      double gb = 0.0, margin = 0.0;
      if (!exact) {
        double b1 = INFINITY, b2 = INFINITY;
        int c1 = 0x7fffffff;
        // candidates c = tid + k * threads in increasing order; (a, b)
        // stepped without a division per candidate
        const int da = kSmallThreads / L, db = kSmallThreads % L;
        int aa = tid / L, bb = tid % L;
#pragma unroll 4
        for (int c = tid; c < L * L; c += kSmallThreads) {
          const double sc = B[c] - 2.0 * PU[aa] - 2.0 * PV[bb];
          aa += da;
          bb += db;
          if (bb >= L) {
            bb -= L;
            ++aa;
          }
          if (sc < b1 || (sc == b1 && c < c1)) {
            b2 = b1;
            b1 = sc;
            c1 = c;
          } else if (sc < b2) {
            b2 = sc;
          }
        }
        block_argmin2(b1, c1, b2, rv, rc);
        const double scale = sqrt(pn) + 2.0 * mn;
        margin = kMarginRel * scale * scale * fmax(1.0, w2 / 128.0);
        gb = b1;
        chosen = c1;
        exact = !(b2 > b1 + margin);
      }
      if (exact) {  // re-evaluate every candidate within the margin exactly
        const bool all = !(pn < 1e300) || !(mn < 1e150);
        double best = INFINITY;
        int bc = 0x7fffffff;
        for (int c = tid; c < L * L; c += blockDim.x) {
          const int aa = c / L, bb = c % L;
          if (!all) {
            const double sc = B[c] - 2.0 * PU[aa] - 2.0 * PV[bb];
            if (!(sc <= gb + margin)) continue;
          }
          const double dd = exact_dist(p, U, L, gs, aa, bb);
          if (dd < best || (dd == best && c < bc)) {
            best = dd;
            bc = c;
          }
        }
        double dummy = INFINITY;
        block_argmin2(best, bc, dummy, rv, rc);
        chosen = (bc == 0x7fffffff) ? 0 : bc;
      }
      const int ca = chosen / L, cb = chosen % L;
      if (tid == 0) {
        const size_t o = ((size_t)s * n + i) * (g.R * g.groups) + (size_t)r * g.groups + grp;
        a_out[o] = (uint16_t)ca;
        b_out[o] = (uint16_t)cb;
      }
      for (int si = tid; si < gs; si += blockDim.x) {
        const double2 ua = U[(size_t)si * L + ca], vb = U[(size_t)si * L + cb];
        p[2 * si] = __dsub_rn(p[2 * si], __dadd_rn(ua.x, -vb.y));
        p[2 * si + 1] = __dsub_rn(p[2 * si + 1], __dadd_rn(ua.y, vb.x));
      }
      __syncthreads();
    }
  }
}

static size_t table_smem(const Geom& g) {
  // per-warp projection rows, or (head presets) per-token projection tables
  const size_t rows = (g.L == 64 && g.g == 64) ? kEncTok : kEncWarps;
  return sizeof(double) * (2 * (size_t)g.g * (g.L + 1) + (size_t)g.L * g.L + (size_t)kEncTok * g.d +
                           2 * rows * g.L) +
         sizeof(float) * ((size_t)g.L * g.L + 2 * rows * g.L);
}

bool key_t64_applies(const Geom& g) { return g.L == 64 && g.g == 64 && g.d % 128 == 0; }
size_t key_t64_table_floats(const Geom& g) {
  return (size_t)g.R * g.subs * g.L * 2 + (size_t)g.R * g.groups * g.L * g.L;
}

cudaError_t run_encode_keys(const Geom& g, int S, int n_slots, const KeyEncTables& tab,
                            const void* keys, int dtype, long long s_stride, long long n,
                            uint16_t* a, uint16_t* b, cudaStream_t st) {
  if (n <= 0 || S <= 0) return cudaSuccess;
  if (tab.atomsf && tab.basef && tab.maxnorm && key_t64_applies(g) && n >= 8 &&
      t64_smem(g) <= 200 * 1024) {
    const size_t sm = t64_smem(g);
    cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(k_encode_keys_t64), sm);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((n + kEncTok - 1) / kEncTok), S);
    k_encode_keys_t64<<<grid, kEncWarps * 32, sm, st>>>(g, n_slots, tab.atoms, tab.atomsf,
                                                        tab.basef, tab.maxnorm, keys, dtype,
                                                        s_stride, n, a, b);
    count_launch();
    return cudaGetLastError();
  }
  const size_t sm = table_smem(g);
  cudaError_t e;
  const size_t sm_small =
      sizeof(double) * (4 * (size_t)g.g * g.L + 2 * (((size_t)g.L * g.L + 1) & ~(size_t)1) + g.d + 2 * g.L +
                        (size_t)(kSmallThreads / (2 * g.L)) * 2 * g.L);
  if (tab.atomsf && tab.basef && key_t64_applies(g) && n < 8) {
    // decode-step appends, head presets: fp32 screen from the fp32 tables
    const size_t sm32 = (size_t)2 * 64 * 64 * 8 + 2 * 64 * 64 * 4 + g.d * 8 + (128 + 4 * 128 + 128) * 4;
    e = ensure_dyn_smem(reinterpret_cast<const void*>(k_encode_keys_small32), sm32);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)n, S);
    k_encode_keys_small32<<<grid, kSmallThreads, sm32, st>>>(
        g, n_slots, tab.atoms, tab.atomsf, tab.basef, tab.maxnorm, keys, dtype, s_stride, n, a, b);
    count_launch();
    return cudaGetLastError();
  }
  if (tab.base != nullptr && n < 8 && 2 * g.L <= kSmallThreads && sm_small <= 220 * 1024) {
    // decode-step appends: a CTA per token, the round slices double-buffered
    e = ensure_dyn_smem(reinterpret_cast<const void*>(k_encode_keys_small), sm_small);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)n, S);
    k_encode_keys_small<<<grid, kSmallThreads, sm_small, st>>>(
        g, n_slots, tab.atoms, tab.base, tab.maxnorm, keys, dtype, s_stride, n, a, b);
  } else if (tab.base != nullptr && sm <= 200 * 1024) {
    e = ensure_dyn_smem(reinterpret_cast<const void*>(k_encode_keys_table), sm);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((n + kEncTok - 1) / kEncTok), S);
    k_encode_keys_table<<<grid, kEncWarps * 32, sm, st>>>(g, n_slots, tab.atoms, tab.base,
                                                         tab.maxnorm, keys, dtype, s_stride, n,
                                                         a, b);
  } else {
    dim3 grid((unsigned)((n + 3) / 4), S);
    k_encode_keys_brute<<<grid, 128, 4 * g.d * sizeof(double), st>>>(g, n_slots, tab.atoms, keys,
                                                                     dtype, s_stride, n, a, b);
  }
  count_launch();
  return cudaGetLastError();
}

bool key_tables_fit(const Geom& g) { return table_smem(g) <= 200 * 1024 && g.L <= 1024; }

// ------------------------------------------------------------ values
// One CTA per (TV-token tile, stream), blockDim = max(hidden, n_codes)
// rounded to a warp multiple (<= 1024).  TV = 16 for prefill (weights read
// once per 16 tokens), TV = 1 for decode-step appends.
template <int TV>
__global__ void k_encode_values(Geom g, int n_slots, ValEncWeights w,
                                const void* __restrict__ vals, int dtype, long long s_stride,
                                long long n, uint8_t* __restrict__ bits,
                                double* __restrict__ logits,
                                unsigned long long* __restrict__ errpos, unsigned long long tok0) {
  extern __shared__ double sm[];
  double* T = sm;                          // [TV][d]
  double* H = T + (size_t)TV * g.d;        // [TV][hidden]
  const int s = blockIdx.y, tid = threadIdx.x;
  const long long i0 = (long long)blockIdx.x * TV;
  const int nt = (int)min((long long)TV, n - i0);
  const int slot = s % n_slots;
  for (int e = tid; e < TV * g.d; e += blockDim.x)
    T[e] = (e / g.d < nt)
               ? load_elem(vals, dtype, (long long)s * s_stride + (i0 + e / g.d) * g.d + e % g.d)
               : 0.0;
  __syncthreads();
  const double* w1 = w.w1 + (size_t)slot * g.d * g.hidden;
  const double* b1 = w.b1 + (size_t)slot * g.hidden;
  const double* w2 = w.w2 + (size_t)slot * g.hidden * g.n_codes;
  const double* b2 = w.b2 + (size_t)slot * g.n_codes;
  for (int j = tid; j < g.hidden; j += blockDim.x) {  // valquant.cpp:52-62
    double h[TV];
#pragma unroll
    for (int k = 0; k < TV; ++k) h[k] = 0.0;
    // weights 16 rows at a time into registers (the loads do not depend on
    // the sequential, zero-skipping sums: keep 16 in flight)
    for (int i0 = 0; i0 < g.d; i0 += 16) {
      double wv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        wv[u] = i0 + u < g.d ? __ldg(w1 + (size_t)(i0 + u) * g.hidden + j) : 0.0;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
#pragma unroll
        for (int k = 0; k < TV; ++k) {
          // a skipped term (t_i == 0) adds -0.0, which leaves every value
          // (signed zeros, inf, NaN included) bit-identical: no branch on the
          // sequential chain
          const double ti = i0 + u < g.d ? T[k * g.d + i0 + u] : 0.0;
          h[k] = __dadd_rn(h[k], ti != 0.0 ? __dmul_rn(ti, wv[u]) : -0.0);
        }
      }
    }
    const double bj = b1[j];
#pragma unroll
    for (int k = 0; k < TV; ++k) {
      double v = __dadd_rn(h[k], bj);
      if (v < 0.0) v = 0.0;
      H[k * g.hidden + j] = v;
    }
  }
  __syncthreads();
  for (int c = tid; c < g.n_codes; c += blockDim.x) {  // valquant.cpp:63-69, 98
    double lg[TV];
#pragma unroll
    for (int k = 0; k < TV; ++k) lg[k] = 0.0;
    for (int j0 = 0; j0 < g.hidden; j0 += 16) {
      double wv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        wv[u] = j0 + u < g.hidden ? __ldg(w2 + (size_t)(j0 + u) * g.n_codes + c) : 0.0;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
#pragma unroll
        for (int k = 0; k < TV; ++k) {
          const double hj = j0 + u < g.hidden ? H[k * g.hidden + j0 + u] : 0.0;
          lg[k] = __dadd_rn(lg[k], hj != 0.0 ? __dmul_rn(hj, wv[u]) : -0.0);
        }
      }
    }
    const double bc = b2[c];
    for (int k = 0; k < nt; ++k) {
      const double v = __dadd_rn(lg[k], bc);
      if (!isfinite(v)) atomicMin(errpos, tok0);  // valquant.cpp:86-87 (TrainingError)
      const size_t o = ((size_t)s * n + i0 + k) * g.n_codes + c;
      bits[o] = v > 0.0 ? 1 : 0;
      if (logits) logits[o] = v;
    }
  }
}

// Prefill value encoder as two exact-order fp64 GEMMs per 32-token tile:
// H = relu(T W1 + b1), logits = H W2 + b2 (valquant.cpp:50-70), every output
// accumulated sequentially over the reduction index in the reference order
// with its zero-skips (t_i == 0, h_j == 0) and no FMA -- bit-identical to the
// reference, but register-tiled (thread = 4 tokens x 4 columns, W rows staged
// in smem 16 at a time) instead of a thread per column re-reading T per
// product (k_encode_values<16>: fp64 pipe 20%).  grid (ceil(n / 32), S),
// 256 threads; smem T[32][d], H[32][hidden], W chunk [16][128].
constexpr int kVgTok = 32, kVgCols = 128, kVgK = 16;
__global__ void __launch_bounds__(256) k_encode_values_gemm(
    Geom g, int n_slots, ValEncWeights w, const void* __restrict__ vals, int dtype,
    long long s_stride, long long n, uint8_t* __restrict__ bits, double* __restrict__ logits,
    unsigned long long* __restrict__ errpos, unsigned long long tok0) {
  extern __shared__ double smv[];
  double* T = smv;                              // [32][d]
  double* H = T + (size_t)kVgTok * g.d;         // [32][hidden]
  double* W = H + (size_t)kVgTok * g.hidden;    // [16][128]
  const int s = blockIdx.y, tid = threadIdx.x;
  const long long i0 = (long long)blockIdx.x * kVgTok;
  const int nt = (int)min((long long)kVgTok, n - i0);
  const int slot = s % n_slots;
  const int tg = tid >> 5, cg = tid & 31;  // tokens 4 tg .. +3, columns 4 cg .. +3 of a block
  for (int e = tid; e < kVgTok * g.d; e += 256)
    T[e] = (e / g.d < nt)
               ? load_elem(vals, dtype, (long long)s * s_stride + (i0 + e / g.d) * g.d + e % g.d)
               : 0.0;
  // one exact-order GEMM: out[32][N] = A[32][K] x B[K][N] (+ bias), per
  // output sequential over k, skipping A == 0; `post` finishes a column
  auto gemm = [&](const double* A, int K, const double* B, int N, auto post) {
    for (int c0 = 0; c0 < N; c0 += kVgCols) {
      double acc[4][4];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[m][c] = 0.0;
      for (int k0 = 0; k0 < K; k0 += kVgK) {
        __syncthreads();  // previous chunk consumed (and A complete)
        for (int e = tid; e < kVgK * kVgCols; e += 256) {
          const int kk = e / kVgCols, cc = e % kVgCols;
          W[e] = (k0 + kk < K && c0 + cc < N) ? __ldg(B + (size_t)(k0 + kk) * N + c0 + cc) : 0.0;
        }
        __syncthreads();
        const int kn = min(kVgK, K - k0);
        for (int kk = 0; kk < kn; ++kk) {
          double a[4], b[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) a[m] = A[(size_t)(4 * tg + m) * K + k0 + kk];
#pragma unroll
          for (int c = 0; c < 4; ++c) b[c] = W[kk * kVgCols + 4 * cg + c];
#pragma unroll
          for (int m = 0; m < 4; ++m)
            if (a[m] != 0.0)
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[m][c] = __dadd_rn(acc[m][c], __dmul_rn(a[m], b[c]));
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int col = c0 + 4 * cg + c;
          if (col < N) post(4 * tg + m, col, acc[m][c]);
        }
    }
  };
  const double* b1 = w.b1 + (size_t)slot * g.hidden;
  const double* b2 = w.b2 + (size_t)slot * g.n_codes;
  gemm(T, g.d, w.w1 + (size_t)slot * g.d * g.hidden, g.hidden, [&](int m, int col, double v) {
    v = __dadd_rn(v, b1[col]);  // valquant.cpp:58-61
    H[(size_t)m * g.hidden + col] = v < 0.0 ? 0.0 : v;
  });
  __syncthreads();  // H complete before it is read as A
  gemm(H, g.hidden, w.w2 + (size_t)slot * g.hidden * g.n_codes, g.n_codes,
       [&](int m, int col, double v) {
         if (m >= nt) return;
         v = __dadd_rn(v, b2[col]);  // valquant.cpp:69
         if (!isfinite(v)) atomicMin(errpos, tok0);
         const size_t o = ((size_t)s * n + i0 + m) * g.n_codes + col;
         bits[o] = v > 0.0 ? 1 : 0;
         if (logits) logits[o] = v;
       });
}

// Screened prefill value encoder.  The logits are only needed for their
// sign (bits = logit > 0).  The hidden layer h = relu(t w1 + b1) runs as the
// exact-order fp64 GEMM of k_encode_values_gemm (bit-identical to the
// reference's h); the output layer runs as an fp32 GEMM of fl32(h) with
// fp32 weights, whose distance to the reference's fp64 logit is bounded by
//   |l~_c - l_c| <= k2 (|h| |w2[:, c]| + |b2_c|),  k2 = 1.01 (hidden + 4) 2^-24
// (rounding of h, w2, b2 to fp32 and the FMA dot product of hidden terms,
// Cauchy-Schwarz; the 1.01 covers the fp64 rounding of the reference sum and
// of the bound).  A logit farther from 0 than its bound has the reference's
// sign; a token with any undecided or non-finite logit gets its output layer
// recomputed exactly (reference order, zero-skips, no FMA) from the exact h,
// so bits and the TrainingError position are bit-identical.
constexpr double kU32 = 5.9604644775390625e-08;  // 2^-24
__global__ void __launch_bounds__(256) k_encode_values_screen(
    Geom g, int n_slots, ValEncWeights w, const void* __restrict__ vals, int dtype,
    long long s_stride, long long n, uint8_t* __restrict__ bits,
    unsigned long long* __restrict__ errpos, unsigned long long tok0) {
  extern __shared__ double smv[];
  double* T = smv;                              // [32][d]
  double* H = T + (size_t)kVgTok * g.d;         // [32][hidden] (exact)
  double* W = H + (size_t)kVgTok * g.hidden;    // [16][128] fp64 chunk (layer 1)
  float* Wf = reinterpret_cast<float*>(W);      // [16][128] fp32 chunk (layer 2)
  __shared__ double hn[kVgTok];
  __shared__ int flag[kVgTok];
  const int s = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long i0 = (long long)blockIdx.x * kVgTok;
  const int nt = (int)min((long long)kVgTok, n - i0);
  const int slot = s % n_slots;
  const int tg = warp, cg = lane;  // tokens 4 tg .. +3, columns 4 cg .. +3 of a block
  for (int e = tid; e < kVgTok * g.d; e += 256)
    T[e] = (e / g.d < nt)
               ? load_elem(vals, dtype, (long long)s * s_stride + (i0 + e / g.d) * g.d + e % g.d)
               : 0.0;
  if (tid < kVgTok) flag[tid] = 0;
  const double* b1 = w.b1 + (size_t)slot * g.hidden;
  const double* b2 = w.b2 + (size_t)slot * g.n_codes;
  const double* n2 = w.n2 + (size_t)slot * g.n_codes;
  // layer 1: exact-order fp64 (as k_encode_values_gemm)
  {
    const double* B = w.w1 + (size_t)slot * g.d * g.hidden;
    const int K = g.d, N = g.hidden;
    for (int c0 = 0; c0 < N; c0 += kVgCols) {
      double acc[4][4];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[m][c] = 0.0;
      for (int k0 = 0; k0 < K; k0 += kVgK) {
        __syncthreads();
        for (int e = tid; e < kVgK * kVgCols; e += 256) {
          const int kk = e / kVgCols, cc = e % kVgCols;
          W[e] = (k0 + kk < K && c0 + cc < N) ? __ldg(B + (size_t)(k0 + kk) * N + c0 + cc) : 0.0;
        }
        __syncthreads();
        const int kn = min(kVgK, K - k0);
        for (int kk = 0; kk < kn; ++kk) {
          double a[4], b[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) a[m] = T[(size_t)(4 * tg + m) * K + k0 + kk];
#pragma unroll
          for (int c = 0; c < 4; ++c) b[c] = W[kk * kVgCols + 4 * cg + c];
#pragma unroll
          for (int m = 0; m < 4; ++m)
            if (a[m] != 0.0)
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[m][c] = __dadd_rn(acc[m][c], __dmul_rn(a[m], b[c]));
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int col = c0 + 4 * cg + c;
          if (col < N) {
            double v = __dadd_rn(acc[m][c], b1[col]);  // valquant.cpp:58-61
            H[(size_t)(4 * tg + m) * N + col] = v < 0.0 ? 0.0 : v;
          }
        }
    }
  }
  __syncthreads();
  if (tid < kVgTok * 8) {  // |h| per token: 8 threads per token
    const int m = tid >> 3, q = tid & 7;
    double a = 0.0;
    for (int j = q; j < g.hidden; j += 8) a = fma(H[(size_t)m * g.hidden + j], H[(size_t)m * g.hidden + j], a);
    a += __shfl_xor_sync(0xffffffffu, a, 1);
    a += __shfl_xor_sync(0xffffffffu, a, 2);
    a += __shfl_xor_sync(0xffffffffu, a, 4);
    if (q == 0) hn[m] = sqrt(a);
  }
  // layer 2: fp32 screen
  const double k2 = 1.01 * (g.hidden + 4) * kU32;
  {
    const float* B = w.w2f + (size_t)slot * g.hidden * g.n_codes;
    const int K = g.hidden, N = g.n_codes;
    for (int c0 = 0; c0 < N; c0 += kVgCols) {
      float acc[4][4];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[m][c] = 0.f;
      for (int k0 = 0; k0 < K; k0 += kVgK) {
        __syncthreads();
        for (int e = tid; e < kVgK * kVgCols / 4; e += 256) {
          const int kk = e / (kVgCols / 4), cc = 4 * (e % (kVgCols / 4));
          *reinterpret_cast<float4*>(Wf + kk * kVgCols + cc) =
              __ldg(reinterpret_cast<const float4*>(B + (size_t)(k0 + kk) * N + c0 + cc));
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < kVgK; ++kk) {
          float a[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) a[m] = (float)H[(size_t)(4 * tg + m) * K + k0 + kk];
          const float4 b = *reinterpret_cast<const float4*>(Wf + kk * kVgCols + 4 * cg);
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            acc[m][0] = fmaf(a[m], b.x, acc[m][0]);
            acc[m][1] = fmaf(a[m], b.y, acc[m][1]);
            acc[m][2] = fmaf(a[m], b.z, acc[m][2]);
            acc[m][3] = fmaf(a[m], b.w, acc[m][3]);
          }
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int tok = 4 * tg + m;
        if (tok >= nt) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int col = c0 + 4 * cg + c;
          const float v = acc[m][c] + (float)b2[col];
          const double bound = k2 * (hn[tok] * n2[col] + fabs(b2[col]));
          if (!(fabs((double)v) > bound)) flag[tok] = 1;  // undecided or non-finite
          else bits[((size_t)s * n + i0 + tok) * N + col] = v > 0.f ? 1 : 0;
        }
      }
    }
  }
  __syncthreads();
  // exact output layer for the flagged tokens (h is exact already)
  const double* w2 = w.w2 + (size_t)slot * g.hidden * g.n_codes;
#pragma unroll 1
  for (int m = 0; m < nt; ++m) {
    if (!flag[m]) continue;  // uniform (smem)
    const double* hm = H + (size_t)m * g.hidden;
    for (int c = tid; c < g.n_codes; c += 256) {
      double lg = 0.0;
      for (int j0 = 0; j0 < g.hidden; j0 += 16) {
        double wv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u)
          wv[u] = j0 + u < g.hidden ? __ldg(w2 + (size_t)(j0 + u) * g.n_codes + c) : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double hj = j0 + u < g.hidden ? hm[j0 + u] : 0.0;
          lg = __dadd_rn(lg, hj != 0.0 ? __dmul_rn(hj, wv[u]) : -0.0);  // valquant.cpp:63-69
        }
      }
      const double v = __dadd_rn(lg, b2[c]);
      if (!isfinite(v)) atomicMin(errpos, tok0);  // valquant.cpp:86-87 (TrainingError)
      bits[((size_t)s * n + i0 + m) * g.n_codes + c] = v > 0.0 ? 1 : 0;
    }
  }
}

template <int TV>
static cudaError_t launch_values(const Geom& g, int S, int n_slots, const ValEncWeights& w,
                                 const void* vals, int dtype, long long s_stride, long long n,
                                 uint8_t* bits, double* logits, unsigned long long* errpos,
                                 unsigned long long tok0, cudaStream_t st) {
  int threads = ((g.hidden > g.n_codes ? g.hidden : g.n_codes) + 31) / 32 * 32;
  if (threads > 1024) threads = 1024;
  if (threads < 64) threads = 64;
  const size_t sm = sizeof(double) * (size_t)TV * (g.d + g.hidden);
  cudaError_t e;
  if (sm > 48 * 1024) {
    e = ensure_dyn_smem(reinterpret_cast<const void*>(k_encode_values<TV>), sm);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((unsigned)((n + TV - 1) / TV), S);
  k_encode_values<TV><<<grid, threads, sm, st>>>(g, n_slots, w, vals, dtype, s_stride, n, bits,
                                                 logits, errpos, tok0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t run_encode_values(const Geom& g, int S, int n_slots, const ValEncWeights& w,
                              const void* vals, int dtype, long long s_stride, long long n,
                              uint8_t* bits, double* logits, unsigned long long* errpos,
                              unsigned long long tok0, cudaStream_t st) {
  if (n <= 0 || S <= 0) return cudaSuccess;
  if (n < 16)  // decode-step appends: one token per CTA, no wasted lanes
    return launch_values<1>(g, S, n_slots, w, vals, dtype, s_stride, n, bits, logits, errpos, tok0,
                            st);
  if (w.w2f && !logits && g.d % kVgK == 0 && g.hidden % kVgCols == 0 &&
      g.hidden % kVgK == 0 && g.n_codes % kVgCols == 0) {
    const size_t sm = sizeof(double) * ((size_t)kVgTok * (g.d + g.hidden) + kVgK * kVgCols);
    if (sm <= 200 * 1024) {
      cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(k_encode_values_screen), sm);
      if (e != cudaSuccess) return e;
      dim3 grid((unsigned)((n + kVgTok - 1) / kVgTok), S);
      k_encode_values_screen<<<grid, 256, sm, st>>>(g, n_slots, w, vals, dtype, s_stride, n, bits,
                                                     errpos, tok0);
      count_launch();
      return cudaGetLastError();
    }
  }
  if (g.d % 4 == 0 && g.hidden % 4 == 0 && g.n_codes % 4 == 0) {
    const size_t sm = sizeof(double) * ((size_t)kVgTok * (g.d + g.hidden) + kVgK * kVgCols);
    if (sm <= 200 * 1024) {
      cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(k_encode_values_gemm), sm);
      if (e != cudaSuccess) return e;
      dim3 grid((unsigned)((n + kVgTok - 1) / kVgTok), S);
      k_encode_values_gemm<<<grid, 256, sm, st>>>(g, n_slots, w, vals, dtype, s_stride, n, bits,
                                                   logits, errpos, tok0);
      count_launch();
      return cudaGetLastError();
    }
  }
  return launch_values<16>(g, S, n_slots, w, vals, dtype, s_stride, n, bits, logits, errpos, tok0,
                           st);
}

}  // namespace cvq
