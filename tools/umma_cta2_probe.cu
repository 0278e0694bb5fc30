// Probe of tcgen05.mma.sp.cta_group::2 (CTA pair, M = 256) with the sparse
// A operand in TMEM: correctness of the operand split (each CTA holds its
// 128 rows of A + metadata in its own TMEM and N/2 rows of B in its smem)
// and the issue rate of the resident-codebook pattern at M = 256, N = 128.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;}" : "=r"(p));
  return p != 0;
}

// A: [256 rows][16 compressed fp16] (rows 128r.. in CTA r); B: [N rows][32 K]
// (rows N/2 r .. in CTA r); uniform metadata 0x4444 (pairs (0,1)).
// D: [256][N] fp32.  iters > 1: timing mode (same MMA repeated).
template <int N>
__global__ void __cluster_dims__(2, 1, 1) kprobe2(const __half* A, const __half* B, float* D, int iters,
                                                  long long* cyc) {
  __shared__ __align__(1024) unsigned char sB[N / 2 * 64];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = ctarank();
  // B half: rows [N/2 rank, +N/2), K-major canonical: core (kc, g) at (kc * N/16 + g) * 128
  for (int e = tid; e < N / 2 * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    *reinterpret_cast<__half*>(sB + ((k / 8) * (N / 16) + n / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) =
        B[(N / 2 * rank + n) * 32 + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  // A rows of this CTA -> TMEM columns 256..263, metadata column 448
  if (warp < 4) {
    const int r = 128 * rank + warp * 32 + lane;
    for (int c = 0; c < 8; ++c) {
      __half2 h2 = __halves2half2(A[r * 16 + 2 * c], A[r * 16 + 2 * c + 1]);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c),
                   "r"(*reinterpret_cast<uint32_t*>(&h2)) : "memory");
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + 448),
                 "r"(0x44444444u) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (rank == 0 && warp == 0) {
    // M = 256 (idesc M >> 4 = 16), N, f32 accumulate, f16 A/B, sparse
    const uint32_t idesc = (1u << 2) | (1u << 4) | ((uint32_t)(N >> 3) << 17) | (16u << 24);
    const uint64_t bd = sdesc(su32(sB), (N / 16) * 128, 128);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one())
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(tmem),
                     "r"(tmem + 256), "l"(bd), "r"(idesc), "r"(it > 0 ? 1 : 0), "r"(tmem + 448));
      __syncwarp();
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(su32(&bar)), "h"((uint16_t)3) : "memory");
    __syncwarp();
    if (lane == 0 && blockIdx.x == 0) cyc[0] = clock64() - t0;
  }
  if (warp == 0) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(su32(&bar)), "r"(0) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4 && blockIdx.x < 2) {
    for (int n0 = 0; n0 < N; n0 += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + n0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int r = 128 * rank + warp * 32 + lane;
      for (int i = 0; i < 8; ++i) D[r * N + n0 + i] = __uint_as_float(v[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

static float hf(__half h) { return __half2float(h); }

template <int N>
void run() {
  static __half hA[256 * 16], hB[N * 32];
  srand(3);
  for (int i = 0; i < 256 * 16; ++i) hA[i] = __float2half((float)(rand() % 17 - 8) / 8.f);
  for (int i = 0; i < N * 32; ++i) hB[i] = __float2half((float)(rand() % 17 - 8) / 8.f);
  __half *dA, *dB;
  float* dD;
  long long* dc;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, 256 * N * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  kprobe2<N><<<2, 128>>>(dA, dB, dD, 1, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d launch failed: %s\n", N, cudaGetErrorString(e)); exit(1); }
  static float D[256 * N];
  cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
  double worst = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int g = 0; g < 8; ++g)
        ref += hf(hA[m * 16 + 2 * g]) * hf(hB[n * 32 + 4 * g]) + hf(hA[m * 16 + 2 * g + 1]) * hf(hB[n * 32 + 4 * g + 1]);
      worst = fmax(worst, fabs(ref - D[m * N + n]));
    }
  printf("cta_group::2 sparse M=256 N=%d, A in TMEM: max |err| = %g\n", N, worst);
  // timing: 148 CTAs = 74 pairs, 4096 MMAs per pair
  kprobe2<N><<<148, 128>>>(dA, dB, dD, 64, dc);
  kprobe2<N><<<148, 128>>>(dA, dB, dD, 4096, dc);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("timing launch failed: %s\n", cudaGetErrorString(e)); exit(1); }
  long long cyc = 0;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)cyc / 4096;
  printf("  issue rate: %.1f clk per MMA (M256 N%d K32 sparse = %.0f logical MAC/clk per SM, %.0f%% of dense 4096)\n",
         per, N, 128.0 * N * 32 / per, 100 * 128.0 * N * 32 / per / 4096);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  run<64>();
  run<128>();
  run<256>();
  return 0;
}
