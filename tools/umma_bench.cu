// Microbenchmark: tcgen05.mma (kind::f16, M=128) issue cost vs N, number of
// independent accumulator chains, and A operand source (smem / TMEM).
// Single CTA; clock64 around `iters` rounds of `chains` MMAs + final commit.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__global__ void kbench(int N, int chains, int iters, int a_tmem, int commit_every, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, bar2;
  const int tid = threadIdx.x;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint64_t ad = sdesc(su32(sm), 128 * 16, 128);
    const uint64_t bd = sdesc(su32(sm + 32768), 128 * 16, 128);
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int c = 0; c < chains; ++c) {
        const uint32_t d = a_tmem ? tmem + 256 + (uint32_t)((c * N) % 256) : tmem + (uint32_t)((c * N) % 512);
        if (a_tmem) {
          asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
                       "r"(tmem + (uint32_t)(it % 8) * 8), "l"(bd), "r"(idesc), "r"(1));
        } else {
          asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(idesc), "r"(1));
        }
      }
      if (commit_every && (it + 1) % commit_every == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        if (commit_every < 0) {}
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)) : "memory");
    {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                     : "=r"(ok) : "r"(su32(&bar2)), "r"(phase) : "memory");
    }
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(kbench, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 512;
  for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
    for (int commit = 0; commit <= 1; ++commit)
      for (int N : {32, 64, 128, 256})
        for (int chains : {1, 2, 4, 8}) {
          if (commit && chains != 4) continue;
          kbench<<<1, 128, 65536>>>(N, chains, iters, a_tmem, commit, d);
          long long h = 0;
          cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
          const double per = (double)h / (iters * chains);
          printf("A=%s commit_every=%d N=%3d chains=%d : %.1f clk/mma (floor %.0f) -> %.0f%% of peak\n",
                 a_tmem ? "tmem" : "smem", commit, N, chains, per, 128.0 * N / 256, 100.0 * (128.0 * N / 256) / per);
        }
  return 0;
}
