// Microbenchmark of the MMA issue pattern a tokens-in-M sparse score kernel
// would use: I issuer warps (whole warp walks the loop, one elected lane
// issues, warp-uniform operands), each with its own accumulator, B walking
// 4 x 16 KiB stages, A from smem or TMEM.  Reports SM clocks per MMA per SM.
#include <cstdio>
#include <cstdint>
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
template <int SPARSE, int ATM, int N>
__global__ void kb(int issuers, int tiles, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 80 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < 8) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[tid])), "r"(1));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp < 4) {
    const uint32_t z = 0, m = 0x44444444u;
    for (int c = 256; c < 512; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c),
                   "r"(c >= 448 ? m : z) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = __shfl_sync(0xffffffffu, warp, 0);
  if (w < issuers) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24) | (SPARSE ? (1u << 2) : 0u);
    const uint32_t d = tmem + (uint32_t)(w * (N == 256 ? 0 : 128));
    const uint32_t a_tm = tmem + 384 + (uint32_t)(w * 16);
    const uint32_t te = tmem + 448 + (uint32_t)w;
    const uint32_t sA = su32(sm + 65536);  // 16 KiB A region
    const uint32_t sB = su32(sm);          // 4 x 16 KiB B stages
    const int per_tile = SPARSE ? 44 : 88;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      for (int i = 0; i < per_tile; ++i) {
        const uint32_t stage = (uint32_t)((i >> 1) & 3);
        const uint32_t half = (uint32_t)(i & 1);
        const uint64_t bd = sdesc(sB + stage * 16384 + half * (SPARSE ? 4 : 2) * 128, 128 * 16, 128);
        const uint64_t ad = sdesc(sA + half * 4096, 128 * 16, 128);
        if (elect_one()) {
          if (SPARSE && ATM)
            asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(d),
                         "r"(a_tm + half * 8), "l"(bd), "r"(idesc), "r"(i), "r"(te));
          else if (SPARSE)
            asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;}" ::"r"(d),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(i), "r"(te));
          else if (ATM)
            asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
                         "r"(a_tm + half * 8), "l"(bd), "r"(idesc), "r"(i));
          else
            asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(i));
        }
        __syncwarp();
      }
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[w])) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(su32(&bar[w])), "r"(0) : "memory");
    if (blockIdx.x == 0 && w == 0 && (tid & 31) == 0) out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// Resident-codebook pattern: N = 64, 4 MMAs per (round, K32 half) into two
// 64-column blocks (Re, Im), B walking an 11 x 16 KiB resident codebook,
// A and metadata from TMEM stage regions, negate-A on one MMA in four.
__global__ void kres(int tiles, int ms, long long* out, int rnd = 0) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 176 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < 8) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[tid])), "r"(1));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp < 4) {
    const int lane = tid & 31;
    for (int c = 256; c < 512; ++c) {
      uint32_t h = (uint32_t)(c * 2654435761u) ^ (uint32_t)((warp * 32 + lane) * 40503u);
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      uint32_t v;
      if (c >= 448) {  // metadata: each 16-bit half picks (0,1) or (2,3) for its row
        v = rnd ? (((h & 1) ? 0x0000EEEEu : 0x00004444u) | ((h & 2) ? 0xEEEE0000u : 0x44440000u)) : 0x44444444u;
      } else {  // A: a one-hot fp16 1.0 per row and stage (random column) or zeros
        v = (rnd == 2 && ((h >> 4) & 15) == (uint32_t)(c & 15)) ? ((h & 4) ? 0x3C000000u : 0x3C00u) : 0u;
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c),
                   "r"(v) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (8u << 17) | (8u << 24) | (1u << 2);  // N = 64
    const uint32_t sB = su32(sm);
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (uint32_t)((t & 1) * 128);
      for (int r = 0; r < 11; ++r) {
        for (int s = 0; s < 2; ++s) {
          const uint32_t st = (uint32_t)((r * 2 + s) & 7);
          const uint32_t a_tm = tmem + 256 + st * 16;
          const uint32_t te = tmem + 448 + st * (uint32_t)ms;
          for (int h = 0; h < 2; ++h) {
            for (int blk = 0; blk < 2; ++blk) {
              // side a: Re += X, Im += Y;  side b: Re -= Y, Im += X
              const uint32_t rows = (uint32_t)(s ? (blk ? 0 : 64) : (blk ? 64 : 0));
              const uint64_t bd = sdesc(sB + r * 16384 + h * 4 * 2048 + rows * 16, 2048, 128);
              const uint32_t id = idesc | ((s && !blk) ? (1u << 13) : 0u);
              if (elect_one())
                asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(d + blk * 64),
                             "r"(a_tm + h * 8), "l"(bd), "r"(id), "r"(r | s | h), "r"(te));
              __syncwarp();
            }
          }
        }
      }
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0])) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(su32(&bar[0])), "r"(0) : "memory");
    if (blockIdx.x == 0 && (tid & 31) == 0) out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// kres with `nprod` extra warps hammering tcgen05.st (x16 zeros into the A
// stage columns 256..447, wait::st each time) and `nld` warps doing
// tcgen05.ld x16 of the accumulator columns: does TMEM store / load traffic
// slow the sparse MMAs?
__global__ void kres2(int tiles, int nprod, int nld, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8];
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 176 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (tid == 0) done = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < 8) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[tid])), "r"(1));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp < 4) {
    for (int c = 256; c < 512; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c),
                   "r"(c >= 448 ? 0x44444444u : 0u) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = warp;
  if (w == 4) {
    const uint32_t idesc = (1u << 4) | (8u << 17) | (8u << 24) | (1u << 2);
    const uint32_t sB = su32(sm);
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (uint32_t)((t & 1) * 128);
      for (int r = 0; r < 11; ++r) {
        for (int s = 0; s < 2; ++s) {
          const uint32_t st = (uint32_t)((r * 2 + s) % 6);
          const uint32_t a_tm = tmem + 256 + st * 32 + s * 16;
          const uint32_t te = tmem + 448 + st * 4 + 2 * s;
          for (int h = 0; h < 2; ++h) {
            for (int blk = 0; blk < 2; ++blk) {
              const uint32_t rows = (uint32_t)(s ? (blk ? 0 : 64) : (blk ? 64 : 0));
              const uint64_t bd = sdesc(sB + r * 16384 + h * 4 * 2048 + rows * 16, 2048, 128);
              const uint32_t id = idesc | ((s && !blk) ? (1u << 13) : 0u);
              if (elect_one())
                asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(d + blk * 64),
                             "r"(a_tm + h * 8), "l"(bd), "r"(id), "r"(r | s | h), "r"(te));
              __syncwarp();
            }
          }
        }
      }
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0])) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(su32(&bar[0])), "r"(0) : "memory");
    if (blockIdx.x == 0 && (tid & 31) == 0) out[0] = clock64() - t0;
    if ((tid & 31) == 0) done = 1;
  } else if (w >= 8 && w < 8 + nprod) {
    const uint32_t lane_base = (uint32_t)((w & 3) * 32) << 16;
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = 0u;
    uint32_t st = 0;
    while (!done) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
                   ::"r"(tmem + lane_base + 256 + 16 * st), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                   "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      st = st == 11 ? 0 : st + 1;
    }
  } else if (w >= 24 && w < 24 + nld) {
    const uint32_t lane_base = (uint32_t)((w & 3) * 32) << 16;
    uint32_t acc = 0;
    while (!done) {
      uint32_t v[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tmem + lane_base));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += v[0] ^ v[15];
    }
    if (acc == 12345u) out[1] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// kres with the per-round synchronisation of the real kernel: mode bit 0 =
// tcgen05.commit to an mbarrier after every round (nobody waits on it), bit 1
// = mbarrier try_wait on an already-completed barrier + tcgen05 fence before
// every round, bit 2 = rounds issued in pairs (one elected region of 16).
__global__ void kres3(int tiles, int mode, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[16];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 176 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < 16) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[tid])), "r"(tid < 8 ? 1 : 1));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  // complete phase 0 of barriers 8..15 (the "already full" stages)
  if (tid >= 8 && tid < 16) asm volatile("{.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];}" ::"r"(su32(&bar[tid])) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp < 4) {
    for (int c = 256; c < 512; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c),
                   "r"(c >= 448 ? 0x44444444u : 0u) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (8u << 17) | (8u << 24) | (1u << 2);
    const uint32_t sB = su32(sm);
    const int per = (mode & 4) ? 2 : 1;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (uint32_t)((t & 1) * 128);
#pragma unroll 1
      for (int r0 = 0; r0 < 11; r0 += per) {
        if (mode & 2) {
          uint32_t ok = 0;
          while (!ok)
            asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                         : "=r"(ok) : "r"(su32(&bar[8 + (r0 % 6)])), "r"(0) : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (elect_one()) {
          for (int u = 0; u < per; ++u) {
            const int r = r0 + u;
            if (r >= 11) break;
            for (int s = 0; s < 2; ++s) {
              const uint32_t st = (uint32_t)(r % 6);
              const uint32_t a_tm = tmem + 256 + st * 32 + s * 16;
              const uint32_t te = tmem + 448 + st * 4 + 2 * s;
              for (int h = 0; h < 2; ++h) {
                for (int blk = 0; blk < 2; ++blk) {
                  const uint32_t rows = (uint32_t)(s ? (blk ? 0 : 64) : (blk ? 64 : 0));
                  const uint64_t bd = sdesc(sB + r * 16384 + h * 4 * 2048 + rows * 16, 2048, 128);
                  const uint32_t id = idesc | ((s && !blk) ? (1u << 13) : 0u);
                  asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                               "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(d + blk * 64),
                               "r"(a_tm + h * 8), "l"(bd), "r"(id), "r"(r | s | h), "r"(te));
                }
              }
            }
            if (mode & 1)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[1 + (r % 6)])) : "memory");
          }
        }
        __syncwarp();
      }
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0])) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(su32(&bar[0])), "r"(0) : "memory");
    if (blockIdx.x == 0 && (tid & 31) == 0) out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


__device__ __forceinline__ bool mtry(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
               : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok != 0;
}
// The kernel's producer -> issuer handoff in isolation: 6 round stages in
// TMEM, 8 producer warps (2 per lane quarter, even / odd rounds) writing 2 x
// (16 A + 1 metadata) columns per round with tcgen05.st, wait::st, fence,
// arrive; the MMA warp waits both stages of a round pair, issues 16 sparse
// N = 64 MMAs in one elected region and commits each round's stage.
// sleep_ns: producer backoff while waiting (0 = spin).
__global__ void kres4(int tiles, int sleep_ns, int mode, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t afull[6], aempty[6], fin;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 176 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 6; ++i) {
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
  const int R = 11;
  if (warp >= 8 && warp < 16) {  // producers
    const int p = warp - 8, quarter = p & 3, sub = p >> 2;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = (i == (lane & 15)) ? 0x3C00u : 0u;
    uint32_t gbase = 0;
    for (int t = 0; t < tiles; ++t) {
      for (int r = sub; r < R; r += 2) {
        const uint32_t g = gbase + r, st = g % 6, use = g / 6;
        if (use > 0) {
          while (!mtry(&aempty[st], (use - 1) & 1)) if (sleep_ns) __nanosleep(64);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        for (int s2 = 0; s2 < 2; ++s2) {
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
                       ::"r"(tmem + lane_base + 256 + 32 * st + 16 * s2), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]),
                       "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
                       "r"(v[14]), "r"(v[15]) : "memory");
          asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lane_base + 448 + 4 * st + 2 * s2),
                       "r"(0x44444444u) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) asm volatile("{.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];}" ::"r"(su32(&afull[st])) : "memory");
      }
      gbase += R;
    }
  } else if (warp == 16 || (mode == 2 && warp == 17)) {  // MMA issuer(s)
    const int iss = warp - 16;  // mode 2: warp iss takes round pairs p = iss (mod 2)
    const uint32_t idesc = (1u << 4) | (8u << 17) | (8u << 24) | (1u << 2);
    const uint64_t bdesc0 = sdesc(su32(sm), 2048, 128);
    uint32_t gst = 0, gph = 0;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dcol = tmem + (uint32_t)(t & 1) * 128u;
#pragma unroll 1
      for (int r = 0; r < R; r += 2) {
        const bool two = r + 1 < R;
        const uint32_t st0 = gst, ph0 = gph;
        uint32_t st1 = gst + 1, ph1 = gph;
        if (st1 == 6) { st1 = 0; ph1 ^= 1u; }
        if (mode == 2 && ((r >> 1) & 1) != iss) {  // the other issuer's pair
          gst += two ? 2u : 1u;
          if (gst >= 6) { gst -= 6; gph ^= 1u; }
          continue;
        }
        while (!mtry(&afull[st0], ph0)) {}
        if (two) while (!mtry(&afull[st1], ph1)) {}
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (mode != 1) {
        if (elect_one()) {
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !two) break;
            const uint32_t st = u ? st1 : st0;
            for (int s = 0; s < 2; ++s) {
              const uint32_t a_tm = tmem + 256 + 32 * st + 16 * s;
              const uint32_t e_tm = tmem + 448 + 4 * st + 2 * s;
              for (int h = 0; h < 2; ++h)
                for (int blk = 0; blk < 2; ++blk) {
                  const int rows = s ? (blk ? 0 : 64) : (blk ? 64 : 0);
                  const uint64_t bd = bdesc0 + (uint64_t)((((r + u) * 16384) + h * 4 * 2048 + rows * 16) >> 4);
                  asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                               "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(dcol + blk * 64),
                               "r"(a_tm + h * 8), "l"(bd), "r"(idesc | ((s && !blk) ? (1u << 13) : 0u)),
                               "r"(mode == 2 ? 1 : ((u | s | h | r) ? 1 : 0)), "r"(e_tm));
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&aempty[st])) : "memory");
          }
        }
        __syncwarp();
        } else {
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !two) break;
            const uint32_t st = u ? st1 : st0;
            for (int s = 0; s < 2; ++s) {
              const uint32_t a_tm = tmem + 256 + 32 * st + 16 * s;
              const uint32_t e_tm = tmem + 448 + 4 * st + 2 * s;
              for (int h = 0; h < 2; ++h)
                for (int blk = 0; blk < 2; ++blk) {
                  const int rows = s ? (blk ? 0 : 64) : (blk ? 64 : 0);
                  const uint64_t bd = bdesc0 + (uint64_t)((((r + u) * 16384) + h * 4 * 2048 + rows * 16) >> 4);
                  if (elect_one())
                    asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(dcol + blk * 64),
                                 "r"(a_tm + h * 8), "l"(bd), "r"(idesc | ((s && !blk) ? (1u << 13) : 0u)),
                                 "r"((u | s | h | r) ? 1 : 0), "r"(e_tm));
                  __syncwarp();
                }
            }
            if (elect_one())
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&aempty[st])) : "memory");
            __syncwarp();
          }
        }
        gst += two ? 2u : 1u;
        if (gst >= 6) { gst -= 6; gph ^= 1u; }
      }
    }
    if (iss == 0) {
      if (elect_one())
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&fin)) : "memory");
      __syncwarp();
      while (!mtry(&fin, 0)) {}
      if (blockIdx.x == 0 && lane == 0) out[0] = clock64() - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int SP, int ATM, int N>
void run(int iss, long long* d) {
  auto k = kb<SP, ATM, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int tiles = 64;
  k<<<148, 128, 96 * 1024>>>(iss, 2, d);
  k<<<148, 128, 96 * 1024>>>(iss, tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const int per_tile = SP ? 44 : 88;
  const double per = (double)cyc / ((double)tiles * per_tile * iss);
  const double macs = 128.0 * N * (SP ? 32 : 16);
  printf("%s A=%s N=%d issuers=%d: %.1f clk/mma per SM, %.0f logical MAC/clk (%.0f%% of dense), %.1f clk per 128 tok x 22 steps\n",
         SP ? "sparse" : "dense ", ATM ? "tmem" : "smem", N, iss, per, macs / per, 100 * macs / per / 4096,
         per * (SP ? 44 : 88) * (N == 256 && !SP ? 0.5 : 1.0) * (N == 128 && !SP ? 2.0 : 1.0));
}
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 8);
  run<0, 0, 256>(1, d);
  run<0, 1, 256>(1, d);
  run<1, 0, 128>(1, d);
  run<1, 1, 128>(1, d);
  run<1, 1, 64>(1, d);
  {
    cudaFuncSetAttribute(kres, cudaFuncAttributeMaxDynamicSharedMemorySize, 176 * 1024);
   for (int ms : {4, 2, 102, 202}) {
    const int rnd = ms / 100;
    kres<<<148, 128, 176 * 1024>>>(2, ms % 100, d, rnd);
    kres<<<148, 128, 176 * 1024>>>(64, ms % 100, d, rnd);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
    long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("resident-codebook N=64 pattern: %.1f clk per 128-token tile (88 MMAs), %.1f clk/mma, %.2f clk/token\n",
           cyc / 64.0, cyc / 64.0 / 88, cyc / 64.0 / 128);
    printf("  (metadata column stride %d, %s)\n", ms % 100, ms >= 200 ? "random metadata + random one-hot A" : ms >= 100 ? "random metadata per row" : "uniform metadata");
   }
  }
  {
    cudaFuncSetAttribute(kres2, cudaFuncAttributeMaxDynamicSharedMemorySize, 176 * 1024);
    long long* d2;
    cudaMalloc(&d2, 16);
    const int cfg[][2] = {{0, 0}, {8, 0}, {16, 0}, {0, 8}, {8, 8}};
    for (auto& c : cfg) {
      kres2<<<148, 1024, 176 * 1024>>>(2, c[0], c[1], d2);
      kres2<<<148, 1024, 176 * 1024>>>(64, c[0], c[1], d2);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
      long long cyc = 0;
      cudaMemcpy(&cyc, d2, 8, cudaMemcpyDeviceToHost);
      printf("kres2 store-warps=%d load-warps=%d: %.1f clk per 128-token tile (88 sparse N=64 MMAs), %.1f clk/mma\n",
             c[0], c[1], cyc / 64.0, cyc / 64.0 / 88);
    }
  }
  {
    cudaFuncSetAttribute(kres3, cudaFuncAttributeMaxDynamicSharedMemorySize, 176 * 1024);
    long long* d3;
    cudaMalloc(&d3, 16);
    for (int mode : {0, 1, 2, 3, 4, 5, 7}) {
      kres3<<<148, 128, 176 * 1024>>>(2, mode, d3);
      kres3<<<148, 128, 176 * 1024>>>(64, mode, d3);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
      long long cyc = 0;
      cudaMemcpy(&cyc, d3, 8, cudaMemcpyDeviceToHost);
      printf("kres3 commit=%d wait+fence=%d pairs=%d: %.1f clk per tile, %.1f clk/mma\n", mode & 1, (mode >> 1) & 1,
             (mode >> 2) & 1, cyc / 64.0, cyc / 64.0 / 88);
    }
  }
  {
    cudaFuncSetAttribute(kres4, cudaFuncAttributeMaxDynamicSharedMemorySize, 176 * 1024);
    long long* d4;
    cudaMalloc(&d4, 16);
    for (int md = 0; md < 3; ++md) {
      const int sl = 1;
      kres4<<<148, 576, 176 * 1024>>>(2, sl, md, d4);
      kres4<<<148, 576, 176 * 1024>>>(64, sl, md, d4);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
      long long cyc = 0;
      cudaMemcpy(&cyc, d4, 8, cudaMemcpyDeviceToHost);
      printf("kres4 handoff (%s): %.1f clk per 128-token tile, %.1f clk/mma\n", md == 2 ? "2 issuers, alternate pairs" : md ? "per-MMA elect" : "16-MMA region",
             cyc / 64.0, cyc / 64.0 / 88);
    }
  }
  return 0;
}
