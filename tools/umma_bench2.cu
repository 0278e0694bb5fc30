// Microbenchmark 2: is the ~125 clk/tcgen05.mma cost per issuing thread or
// per SM?  `issuers` warps of one CTA each issue `chains` independent
// accumulator chains (M=128, kind::f16, A/B in smem) into their own TMEM
// columns; grid = ctas_per_sm * 148, timed with events over the whole grid.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__global__ void kbench(int N, int chains, int issuers, int iters, int cols, int m256, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < 8) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[tid])), "r"(1));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if ((tid & 31) == 0 && warp < issuers) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((m256 ? 4u : 8u) << 24);
    const uint64_t ad = sdesc(su32(sm), 128 * 16, 128);
    const uint64_t bd = sdesc(su32(sm + 16384), 256 * 16, 128);
    const int per = cols / issuers;  // columns owned by this issuer
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int c = 0; c < chains; ++c) {
        const uint32_t d = tmem + warp * per + (uint32_t)((c * N) % per);
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(1));
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(kbench, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1024;
  struct Cfg { int N, chains, issuers, cps, m256; };
  Cfg cfgs[] = {
      {256, 2, 1, 1, 0}, {256, 1, 2, 1, 0}, {128, 4, 1, 1, 0}, {128, 2, 2, 1, 0}, {128, 1, 4, 1, 0},
      {128, 2, 1, 2, 0}, {64, 4, 1, 1, 0},  {64, 2, 2, 1, 0},  {64, 1, 4, 1, 0},  {64, 4, 1, 2, 0},
      {256, 2, 1, 1, 1}, {128, 4, 1, 1, 1}, {64, 4, 1, 1, 1},
  };
  for (const Cfg& c : cfgs) {
    const int cols = 512 / c.cps;
    const int grid = 148 * c.cps;
    kbench<<<grid, 128, 49152>>>(c.N, c.chains, c.issuers, 16, cols, c.m256, d);  // warm
    cudaEventRecord(e0);
    kbench<<<grid, 128, 49152>>>(c.N, c.chains, c.issuers, iters, cols, c.m256, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double mmas_per_sm = (double)iters * c.chains * c.issuers * c.cps;
    const double clk = ms * 1e-3 * 1.965e9;
    const int M = c.m256 ? 64 : 128;
    const double macs = mmas_per_sm * M * c.N * 16;
    printf("M=%d N=%3d chains=%d issuers=%d ctas/sm=%d : %.1f clk/mma per SM (event), %.0f MAC/clk/SM (%.0f%% of 4096); cta0 clock %.1f clk/mma\n",
           M, c.N, c.chains, c.issuers, c.cps, clk / mmas_per_sm, macs / clk, 100 * macs / clk / 4096,
           (double)h / (iters * c.chains));
  }
  return 0;
}
