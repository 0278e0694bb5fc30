// Microbenchmark: dense tcgen05.mma kind::f16 (K16) vs sparse
// tcgen05.mma.sp kind::f16 (K32 logical, 2:4 A, metadata in TMEM) issue
// cost per SM, M=128, several N and issuer counts.  Operand data are zeros
// (timing only); metadata words hold the (0,1) index pair in every group.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__global__ void kbench(int N, int issuers, int iters, int sparse, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
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
  // metadata: columns 448..511, every lane: 0x44444444 ((0,1) pairs)
  if (warp < 4) {
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) v[i] = 0x44444444u;
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 448;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (lane == 0 && warp < issuers) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24) | (sparse ? (1u << 2) : 0u);
    const uint64_t ad = sdesc(su32(sm), 128 * 16, 128);
    const uint64_t bd = sdesc(su32(sm + 16384), 256 * 16, 128);
    const int per = 448 / issuers / 8 * 8;
    const uint32_t d = tmem + warp * per;
    const uint32_t te = tmem + 448;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (sparse) {
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;}" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(1), "r"(te));
      } else {
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(su32(&bar[warp])), "r"(0) : "memory");
    if (blockIdx.x == 0 && warp == 0) out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// Variant: A operand from TMEM (cols 256..263) or smem, `chains` accumulators
// per issuer used round-robin (independent accumulate chains).
__global__ void kbench2(int N, int issuers, int chains, int iters, int sparse, int atm, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
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
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) v[i] = 0x44444444u;
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 448;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    for (int i = 0; i < 8; ++i) v[i] = 0u;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 ::"r"(ta - 192), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if ((tid & 31) == 0 && warp < issuers) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24) | (sparse ? (1u << 2) : 0u);
    const uint64_t ad = sdesc(su32(sm), 128 * 16, 128);
    const uint64_t bd = sdesc(su32(sm + 16384), 256 * 16, 128);
    const uint32_t ta = tmem + 256;
    const uint32_t te = tmem + 448;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (uint32_t)((warp * chains + it % chains) * N);
      if (sparse && atm) {
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(d),
                     "r"(ta), "l"(bd), "r"(idesc), "r"(1), "r"(te));
      } else if (sparse) {
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;}" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(1), "r"(te));
      } else if (atm) {
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
                     "r"(ta), "l"(bd), "r"(idesc), "r"(1));
      } else {
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(su32(&bar[warp])), "r"(0) : "memory");
    if (blockIdx.x == 0 && warp == 0) out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(kbench, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048;
  for (int sparse = 0; sparse < 2; ++sparse)
    for (int N : {64, 128, 256})
      for (int iss : {1, 2, 4}) {
        if (N == 256 && iss > 1) continue;  // D columns
        kbench<<<148, 128, 49152>>>(N, iss, 16, sparse, d);
        cudaEventRecord(e0);
        kbench<<<148, 128, 49152>>>(N, iss, iters, sparse, d);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double clk = ms * 1e-3 * 1.9e9;
        const double per = clk / ((double)iters * iss);
        const double kl = sparse ? 32 : 16;
        printf("%s N=%3d issuers=%d : %.1f clk/mma per SM, %.0f logical MAC/clk/SM (%.0f%% of dense 4096)\n",
               sparse ? "sparse K32" : "dense  K16", N, iss, per, 128.0 * N * kl / per, 100 * 128.0 * N * kl / per / 4096);
      }

  cudaFuncSetAttribute(kbench2, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152);
  struct Cfg { int N, iss, ch, sp, atm; };
  const Cfg cfgs[] = {
      {256, 1, 1, 0, 0}, {256, 1, 1, 0, 1}, {256, 1, 1, 1, 0}, {256, 1, 1, 1, 1},
      {128, 1, 1, 1, 0}, {128, 1, 1, 1, 1}, {128, 1, 2, 1, 0}, {128, 1, 2, 1, 1},
      {128, 2, 1, 1, 1}, {128, 1, 2, 0, 0}, {128, 1, 2, 0, 1}, {64, 1, 4, 1, 1}, {64, 2, 2, 1, 1}};
  for (const Cfg& c : cfgs) {
    long long* dd = d;
    kbench2<<<148, 128, 49152>>>(c.N, c.iss, c.ch, 16, c.sp, c.atm, dd);
    cudaEventRecord(e0);
    kbench2<<<148, 128, 49152>>>(c.N, c.iss, c.ch, iters, c.sp, c.atm, dd);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)cyc / ((double)iters * c.iss);
    const double kl = c.sp ? 32 : 16;
    printf("v2 %s A=%s N=%3d issuers=%d chains=%d : %.1f clk/mma (SM clock), %.0f logical MAC/clk (%.0f%% of dense 4096), %.3f ms\n",
           c.sp ? "sparse K32" : "dense  K16", c.atm ? "tmem" : "smem", c.N, c.iss, c.ch, per,
           128.0 * c.N * kl / per, 100 * 128.0 * c.N * kl / per / 4096, ms);
  }
  return 0;
}
