// Round-2 question: why does the sparse score kernel's MMA warp lose ~200
// clk per elected issue region (profiles/r01_umma_issue_sync_costs.txt,
// kres3)?  The SASS of k_sp_score shows each region as
// ELECT / BSSY / 16 x UTCHMMA / UTCBAR / BSYNC, and BSYNC waits on the
// scoreboards the UTCHMMAs set.  This benchmark runs the kernel's producer ->
// issuer handoff (8 producer warps writing one-hot A + metadata into 6 TMEM
// round stages, one MMA warp issuing 88 sparse M128 N64 MMAs per 128-token
// tile) with different issue codings:
//   mode 0: one branchy elected region per round pair (round-1 kernel)
//   mode 1: per-MMA `if (elect_one())` (compiler if-converts to @UP UTCHMMA)
//   mode 2: per-MMA asm with its own elect.sync and a predicated mma
//   mode 3: one asm per round: elect.sync, 8 predicated mmas, predicated commit
// prod = 0 drops the producers (stage barriers are never waited on).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_pred_bench tools/umma_pred_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;}" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ bool mtry(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
               : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mma_plain(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc, uint32_t e) {
  asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc), "r"(e));
}
__device__ __forceinline__ void mma_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc, uint32_t e) {
  asm volatile("{.reg .pred p, q;\n\telect.sync _|q, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc), "r"(e));
}
__device__ __forceinline__ void commit_plain(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile("{.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\t"
               "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(su32(bar)) : "memory");
}
// one round (both sides, both K halves, Re/Im blocks) = 8 MMAs + commit, one elect
__device__ __forceinline__ void round_elect(uint32_t d, uint32_t a_st, uint32_t e_st, uint64_t br, uint32_t idesc,
                                            uint32_t first, uint64_t* bar) {
  // side a: (d, a_st, br + 0), (d+64, a_st, br+Y); side b: (d, a_st+16, br+Y, neg), (d+64, a_st+16, br)
  // K halves at +8 columns / + 4*2048 bytes
  const uint32_t neg = idesc | (1u << 13);
  asm volatile(
      "{.reg .pred q, p;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      ".reg .pred t;\n\tsetp.eq.u32 t, %6, %6;\n\t"
      ".reg .b32 a0, a1, a2, a3, d1, e1;\n\t"
      ".reg .b64 b0, b1, b2, b3;\n\t"
      "add.u32 a1, %1, 8;\n\t"
      "add.u32 a2, %1, 16;\n\t"
      "add.u32 a3, %1, 24;\n\t"
      "add.u32 d1, %0, 64;\n\t"
      "add.u32 e1, %2, 2;\n\t"
      "add.u64 b1, %3, 64;\n\t"      // Y rows: +64 rows * 16 B >> 4
      "add.u64 b2, %3, 512;\n\t"     // K half 1: + 4 * 2048 >> 4
      "add.u64 b3, %3, 576;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %3, [%2], %4, p;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [d1], [%1], b1, [%2], %4, p;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [a1], b2, [%2], %4, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [d1], [a1], b3, [%2], %4, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [a2], b1, [e1], %5, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [d1], [a2], %3, [e1], %4, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [a3], b3, [e1], %5, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [d1], [a3], b2, [e1], %4, t;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];}" ::"r"(d),
      "r"(a_st), "r"(e_st), "l"(br), "r"(idesc), "r"(neg), "r"(first), "r"(su32(bar))
      : "memory");
}

__device__ long long g_tr[10 * 44];
constexpr int kG0 = 30 * 11;
template <int MODE, int PROD, int SLEEP, int NST>
__global__ void __launch_bounds__(576, 1) khand(int tiles, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t afull[8], aempty[8], fin;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 176 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&afull[i])), "r"(4));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&aempty[i])), "r"(1));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&fin)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  constexpr int R = 11;
  if (warp >= 8 && warp < 16) {  // producers
    if (PROD) {
      const int p = warp - 8, quarter = p & 3, sub = p >> 2;
      const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
      uint32_t v[16];
      for (int i = 0; i < 16; ++i) v[i] = (i == (lane & 15)) ? 0x3C00u : 0u;
      uint32_t gbase = 0;
      long long pw = 0, pb = 0;
      for (int t = 0; t < tiles; ++t) {
        for (int r = sub; r < R; r += 2) {
          const uint32_t g = gbase + r, st = g % NST, use = g / NST;
          long long b0 = 0;
          if (use > 0) {
            long long w0 = clock64();
            while (!mtry(&aempty[st], (use - 1) & 1)) if (SLEEP) __nanosleep(SLEEP);
            pw += clock64() - w0;
            b0 = clock64();
            if (blockIdx.x == 0 && lane == 0 && g >= kG0 && g < kG0 + 44) g_tr[(2 + quarter) * 44 + g - kG0] = b0;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          } else {
            b0 = clock64();
          }
          for (int s2 = 0; s2 < 2; ++s2) {
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
                         ::"r"(tmem + lane_base + 256 + 32 * st + 16 * s2), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]),
                         "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
                         "r"(v[14]), "r"(v[15]) : "memory");
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lane_base + 256 + 32 * NST + 4 * st + 2 * s2),
                         "r"(0x44444444u) : "memory");
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) asm volatile("{.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];}" ::"r"(su32(&afull[st])) : "memory");
          pb += clock64() - b0;
          if (blockIdx.x == 0 && lane == 0 && g >= kG0 && g < kG0 + 44) g_tr[(6 + quarter) * 44 + g - kG0] = clock64();
        }
        gbase += R;
      }
      if (blockIdx.x == 0 && warp == 8 && lane == 0) { out[2] = pw; out[3] = pb; }
    }
  } else if (warp == 16) {  // MMA issuer
    const uint32_t idesc = (1u << 4) | (8u << 17) | (8u << 24) | (1u << 2);
    const uint64_t bdesc0 = sdesc(su32(sm), 2048, 128);
    uint32_t gst = 0, gph = 0;
    long long waited = 0;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dcol = tmem + (uint32_t)(t & 1) * 128u;
      uint64_t br = bdesc0;
#pragma unroll 1
      for (int r = 0; r < R; r += 2) {
        const bool two = r + 1 < R;
        const uint32_t st0 = gst, ph0 = gph;
        uint32_t st1 = gst + 1, ph1 = gph;
        if (st1 == NST) { st1 = 0; ph1 ^= 1u; }
        if (MODE == 4) {
          const int g0 = t * 11 + r - kG0;
          long long w0 = clock64();
          if (PROD) while (!mtry(&afull[st0], ph0)) {}
          waited += clock64() - w0;
          if (blockIdx.x == 0 && lane == 0 && g0 >= 0 && g0 < 44) { g_tr[g0] = w0; g_tr[44 + g0] = clock64(); }
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          round_elect(dcol, tmem + 256 + 32 * st0, tmem + 256 + 32 * NST + 4 * st0, br, idesc, r ? 1u : 0u, &aempty[st0]);
          if (two) {
            w0 = clock64();
            if (PROD) while (!mtry(&afull[st1], ph1)) {}
            waited += clock64() - w0;
            if (blockIdx.x == 0 && lane == 0 && g0 + 1 >= 0 && g0 + 1 < 44) { g_tr[g0 + 1] = w0; g_tr[44 + g0 + 1] = clock64(); }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            round_elect(dcol, tmem + 256 + 32 * st1, tmem + 256 + 32 * NST + 4 * st1, br + (16384 >> 4), idesc, 1u, &aempty[st1]);
          }
          br += (uint64_t)((2 * 16384) >> 4);
          gst += two ? 2u : 1u;
          if (gst >= NST) { gst -= NST; gph ^= 1u; }
          continue;
        }
        {
          long long w0 = clock64();
          if (PROD) {
            while (!mtry(&afull[st0], ph0)) {}
            if (two) while (!mtry(&afull[st1], ph1)) {}
          }
          waited += clock64() - w0;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (MODE == 0) {
          if (elect_one()) {
            for (int u = 0; u < 2; ++u) {
              if (u == 1 && !two) break;
              const uint32_t st = u ? st1 : st0;
              for (int s = 0; s < 2; ++s) {
                const uint32_t a_tm = tmem + 256 + 32 * st + 16 * s;
                const uint32_t e_tm = tmem + 256 + 32 * NST + 4 * st + 2 * s;
                for (int h = 0; h < 2; ++h)
                  for (int blk = 0; blk < 2; ++blk) {
                    const int rows = s ? (blk ? 0 : 64) : (blk ? 64 : 0);
                    const uint64_t bd = br + (uint64_t)(((u * 16384) + h * 4 * 2048 + rows * 16) >> 4);
                    mma_plain(dcol + blk * 64, a_tm + h * 8, bd, idesc | ((s && !blk) ? (1u << 13) : 0u),
                              (u | s | h | r) ? 1 : 0, e_tm);
                  }
              }
              commit_plain(&aempty[u ? st1 : st0]);
            }
          }
          __syncwarp();
        } else if (MODE == 1 || MODE == 2) {
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !two) break;
            const uint32_t st = u ? st1 : st0;
            for (int s = 0; s < 2; ++s) {
              const uint32_t a_tm = tmem + 256 + 32 * st + 16 * s;
              const uint32_t e_tm = tmem + 256 + 32 * NST + 4 * st + 2 * s;
              for (int h = 0; h < 2; ++h)
                for (int blk = 0; blk < 2; ++blk) {
                  const int rows = s ? (blk ? 0 : 64) : (blk ? 64 : 0);
                  const uint64_t bd = br + (uint64_t)(((u * 16384) + h * 4 * 2048 + rows * 16) >> 4);
                  const uint32_t id = idesc | ((s && !blk) ? (1u << 13) : 0u);
                  const uint32_t acc = (u | s | h | r) ? 1 : 0;
                  if (MODE == 1) {
                    if (elect_one()) mma_plain(dcol + blk * 64, a_tm + h * 8, bd, id, acc, e_tm);
                    __syncwarp();
                  } else {
                    mma_elect(dcol + blk * 64, a_tm + h * 8, bd, id, acc, e_tm);
                  }
                }
            }
            if (MODE == 1) {
              if (elect_one()) commit_plain(&aempty[st]);
              __syncwarp();
            } else {
              commit_elect(&aempty[st]);
            }
          }
        } else {  // MODE 3
          round_elect(dcol, tmem + 256 + 32 * st0, tmem + 256 + 32 * NST + 4 * st0, br, idesc, r ? 1u : 0u, &aempty[st0]);
          if (two)
            round_elect(dcol, tmem + 256 + 32 * st1, tmem + 256 + 32 * NST + 4 * st1, br + (16384 >> 4), idesc, 1u, &aempty[st1]);
        }
        br += (uint64_t)((2 * 16384) >> 4);
        gst += two ? 2u : 1u;
        if (gst >= NST) { gst -= NST; gph ^= 1u; }
      }
    }
    if (elect_one()) commit_plain(&fin);
    __syncwarp();
    while (!mtry(&fin, 0)) {}
    if (blockIdx.x == 0 && lane == 0) { out[0] = clock64() - t0; out[1] = waited; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// Issuer-only: before each round, wait on an already-satisfied condition with
// variant W: 0 none, 1 mbarrier.try_wait, 2 mbarrier.test_wait loop,
// 3 ld.acquire.shared flag, 4 ld.volatile.shared flag, 5 try_wait without commit in rounds
template <int W>
__global__ void __launch_bounds__(128, 1) kwait(int tiles, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8], fin;
  __shared__ uint32_t flag[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 176 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[i])), "r"(1));
      flag[i] = 1;
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&fin)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid < 6) asm volatile("{.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];}" ::"r"(su32(&bar[tid])) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (8u << 17) | (8u << 24) | (1u << 2);
    const uint64_t bdesc0 = sdesc(su32(sm), 2048, 128);
    long long waited = 0;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dcol = tmem + (uint32_t)(t & 1) * 128u;
      uint64_t br = bdesc0;
#pragma unroll 1
      for (int r = 0; r < 11; ++r) {
        const uint32_t st = (uint32_t)(r % 6);
        const long long w0 = clock64();
        if (W == 1 || W == 5) {
          while (!mtry(&bar[st], 0)) {}
        } else if (W == 2) {
          uint32_t ok = 0;
          while (!ok)
            asm volatile("{.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                         : "=r"(ok) : "r"(su32(&bar[st])), "r"(0) : "memory");
        } else if (W == 3) {
          uint32_t v = 0;
          while (!v) asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(su32(&flag[st])) : "memory");
        } else if (W == 4) {
          uint32_t v = 0;
          while (!v) asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(su32(&flag[st])) : "memory");
        }
        waited += clock64() - w0;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        round_elect(dcol, tmem + 256 + 32 * st, tmem + 256 + 32 * 6 + 4 * st, br, idesc, r ? 1u : 0u,
                    W == 5 ? &bar[7] : &bar[6]);
        br += (uint64_t)(16384 >> 4);
      }
    }
    if (elect_one()) commit_plain(&fin);
    __syncwarp();
    while (!mtry(&fin, 0)) {}
    if (blockIdx.x == 0 && lane == 0) { out[0] = clock64() - t0; out[1] = waited; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
template <int W>
void runw(long long* d) {
  auto k = kwait<W>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 176 * 1024);
  k<<<148, 128, 176 * 1024>>>(2, d);
  k<<<148, 128, 176 * 1024>>>(64, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long cyc[2];
  cudaMemcpy(cyc, d, 16, cudaMemcpyDeviceToHost);
  const char* nm[] = {"none", "mbarrier.try_wait", "mbarrier.test_wait loop", "ld.acquire.shared flag", "ld.volatile.shared flag",
                      "try_wait, commits to another barrier"};
  printf("issuer-only wait=%s: %.1f clk/tile, %.1f clk/mma, wait %.1f clk/round\n", nm[W], cyc[0] / 64.0, cyc[0] / 64.0 / 88,
         cyc[1] / 64.0 / 11);
}

template <int MODE, int PROD, int SLEEP = 64, int NST = 6>
void run(long long* d) {
  auto k = khand<MODE, PROD, SLEEP, NST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 176 * 1024);
  k<<<148, 576, 176 * 1024>>>(2, d);
  k<<<148, 576, 176 * 1024>>>(64, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long cyc[4] = {0, 0, 0, 0};
  cudaMemcpy(cyc, d, 32, cudaMemcpyDeviceToHost);
  const char* names[] = {"branchy 16-MMA region", "per-MMA if(elect)", "per-MMA asm elect+@p", "per-round asm elect+@p x8",
                         "per-round wait + asm x8"};
  printf("mode %d (%s) producers=%d sleep=%d: %.1f clk per 128-token tile, %.1f clk/mma; issuer waits %.1f, producer waits %.1f, producer busy %.1f clk/tile, stages %d\n",
         MODE, names[MODE], PROD, SLEEP, cyc[0] / 64.0, cyc[0] / 64.0 / 88, cyc[1] / 64.0, cyc[2] / 64.0, cyc[3] / 64.0, NST);
  if (MODE == 4 && PROD) {
    long long tr[440];
    cudaMemcpyFromSymbol(tr, g_tr, sizeof(tr));
    const long long z = tr[0];
    printf("  g: iss_wait_begin iss_wait_end | prod_start q0..q3 | prod_arrive q0..q3 (clk rel. to first)\n");
    for (int i = 0; i < 44; ++i) {
      printf("  %2d: %6lld %6lld |", i, tr[i] - z, tr[44 + i] - z);
      for (int q = 0; q < 4; ++q) printf(" %6lld", tr[(2 + q) * 44 + i] - z);
      printf(" |");
      for (int q = 0; q < 4; ++q) printf(" %6lld", tr[(6 + q) * 44 + i] - z);
      printf("\n");
    }
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 32);
  runw<0>(d);
  runw<1>(d);
  runw<2>(d);
  runw<3>(d);
  runw<4>(d);
  runw<5>(d);
  return 0;
}
