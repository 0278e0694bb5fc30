// Probe of the tcgen05.mma.sp kind::f16 operand formats (M=128, N=8,
// K=32 logical): A compressed [128][16] fp16 in the canonical K-major
// no-swizzle smem layout, B [8][32] K-major, metadata in TMEM.  Test 1/2:
// uniform metadata words (every lane / column) with index pairs (0,1) and
// (2,3); test 3: metadata that differs by TMEM lane and column, to map
// (lane, column, nibble) -> (row, group).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// A_c [128][16] fp16 row-major in global -> canonical K-major core matrices:
// (kc, g) at (kc*16 + g)*128 B, row r%8 at 16 B, element k%8 at 2 B.
// B [8][32] row-major -> (kc, 0) at kc*128.
// meta [128 lanes][ncol] u32 written to TMEM columns 448.. by warps 0-3.
__global__ void kprobe(const __half* Ac, const __half* B, const uint32_t* meta, int ncol,
                       float* D, int atm, int neg, int acol) {
  __shared__ __align__(1024) unsigned char sA[4096];
  __shared__ __align__(1024) unsigned char sB[512];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 16; e += blockDim.x) {
    const int r = e / 16, k = e % 16;
    *reinterpret_cast<__half*>(sA + ((k / 8) * 16 + r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) = Ac[e];
  }
  for (int e = tid; e < 8 * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    *reinterpret_cast<__half*>(sB + (k / 8) * 128 + n * 16 + (k % 8) * 2) = B[e];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const int lane = tid & 31;
  for (int c = 0; c < ncol; ++c) {  // 32x32b.x1 per column
    const uint32_t v = meta[(warp * 32 + lane) * ncol + c];
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + 448 + c), "r"(v) : "memory");
  }
  if (atm && warp < 4) {
    const int r = warp * 32 + lane;
    for (int c = 0; c < 8; ++c) {
      __half2 h2 = __halves2half2(Ac[r * 16 + 2 * c], Ac[r * 16 + 2 * c + 1]);
      const uint32_t v = *reinterpret_cast<uint32_t*>(&h2);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + 256 + acol + c), "r"(v) : "memory");
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 17) | (8u << 24) | (1u << 2) | (neg ? (1u << 13) : 0u);  // f32 acc, N=8, M=128, sparse
    const uint64_t ad = sdesc(su32(sA), 2048, 128);
    const uint64_t bd = sdesc(su32(sB), 128, 512);
    if (atm)
      asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(tmem),
                   "r"(tmem + 256 + acol), "l"(bd), "r"(idesc), "r"(0), "r"(tmem + 448));
    else
      asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;}" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(0), "r"(tmem + 448));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(su32(&bar)), "r"(0) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int n = 0; n < 8; ++n) D[(warp * 32 + lane) * 8 + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

static float hf(__half h) { return __half2float(h); }

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int atm = argc > 1;
  const int neg = argc > 2 && argv[2][0] == '1';
  const int acol = argc > 3 ? atoi(argv[3]) : 0;
  printf("A column offset %d\n", acol);
  const double sg = neg ? -1.0 : 1.0;
  printf("A from %s\n", atm ? "TMEM" : "smem");
  const int NC = 8;  // metadata columns written
  __half hA[128 * 16], hB[8 * 32];
  srand(1);
  for (int i = 0; i < 128 * 16; ++i) hA[i] = __float2half((float)(rand() % 17 - 8) / 8.f);
  for (int i = 0; i < 8 * 32; ++i) hB[i] = __float2half((float)(rand() % 17 - 8) / 8.f);
  __half *dA, *dB;
  uint32_t* dM;
  float* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dM, 128 * NC * 4);
  cudaMalloc(&dD, 128 * 8 * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  static uint32_t meta[128 * NC];
  float D[128 * 8];
  // tests 1/2: uniform pairs
  struct Pair { int i0, i1; } pairs[] = {{0, 1}, {2, 3}, {0, 2}, {1, 3}};
  for (auto pr : pairs) {
    const uint32_t nib = (uint32_t)pr.i0 | ((uint32_t)pr.i1 << 2);
    uint32_t w = 0;
    for (int i = 0; i < 8; ++i) w |= nib << (4 * i);
    for (int i = 0; i < 128 * NC; ++i) meta[i] = w;
    cudaMemcpy(dM, meta, sizeof(meta), cudaMemcpyHostToDevice);
    kprobe<<<1, 128>>>(dA, dB, dM, NC, dD, atm, neg, acol);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed\n"); return 1; }
    cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 8; ++n) {
        double ref = 0;
        for (int gI = 0; gI < 8; ++gI) {  // 8 groups of 4 logical K
          ref += hf(hA[m * 16 + 2 * gI]) * hf(hB[n * 32 + 4 * gI + pr.i0]);
          ref += hf(hA[m * 16 + 2 * gI + 1]) * hf(hB[n * 32 + 4 * gI + pr.i1]);
        }
        worst = fmax(worst, fabs(sg * ref - D[m * 8 + n]));
      }
    printf("uniform pair (%d,%d) nibble 0x%x: max |err| = %g\n", pr.i0, pr.i1, nib, worst);
  }
  if (argc > 4) {  // lane map: metadata lane L word -> (2,3) everywhere; which rows change?
    for (int L = 0; L < 128; ++L) {
      for (int i = 0; i < 128 * NC; ++i) meta[i] = 0x44444444u;
      meta[L * NC + 0] = 0xEEEEEEEEu;
      cudaMemcpy(dM, meta, sizeof(meta), cudaMemcpyHostToDevice);
      kprobe<<<1, 128>>>(dA, dB, dM, NC, dD, atm, neg, acol);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed\n"); return 1; }
      cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
      printf("L%d:", L);
      for (int m = 0; m < 128; ++m) {
        double e = 0;
        for (int n = 0; n < 8; ++n) {
          double ref = 0;
          for (int gI = 0; gI < 8; ++gI)
            ref += hf(hA[m * 16 + 2 * gI]) * hf(hB[n * 32 + 4 * gI]) + hf(hA[m * 16 + 2 * gI + 1]) * hf(hB[n * 32 + 4 * gI + 1]);
          e = fmax(e, fabs(ref - D[m * 8 + n]));
        }
        if (e > 1e-3) printf(" %d", m);
      }
      printf("\n");
    }
    return 0;
  }
  // test 3: per (lane, column) distinct: lane L column c nibble pattern
  // (0,1) everywhere except one nibble set to (2,3); find which D rows change
  for (int probe = 0; probe < 6; ++probe) {
    const int lane = (probe % 3) * 40 + 3, col = probe / 3 == 0 ? 0 : 1, nibi = (probe % 2) ? 5 : 0;
    for (int i = 0; i < 128 * NC; ++i) meta[i] = 0x44444444u;
    meta[lane * NC + col] = (0x44444444u & ~(0xFu << (4 * nibi))) | (0xEu << (4 * nibi));
    cudaMemcpy(dM, meta, sizeof(meta), cudaMemcpyHostToDevice);
    kprobe<<<1, 128>>>(dA, dB, dM, NC, dD, atm, neg, acol);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed\n"); return 1; }
    cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
    printf("meta lane %d col %d nibble %d -> changed rows/groups:", lane, col, nibi);
    for (int m = 0; m < 128; ++m) {
      // which single group g, if switched to (2,3), explains row m?
      double base_err = 0;
      double ref01[8];
      for (int n = 0; n < 8; ++n) {
        double ref = 0;
        for (int gI = 0; gI < 8; ++gI)
          ref += hf(hA[m * 16 + 2 * gI]) * hf(hB[n * 32 + 4 * gI]) +
                 hf(hA[m * 16 + 2 * gI + 1]) * hf(hB[n * 32 + 4 * gI + 1]);
        ref01[n] = ref;
        base_err = fmax(base_err, fabs(ref - D[m * 8 + n]));
      }
      if (base_err < 1e-3) continue;
      int found = -1;
      for (int gI = 0; gI < 8 && found < 0; ++gI) {
        double e = 0;
        for (int n = 0; n < 8; ++n) {
          double ref = ref01[n] - hf(hA[m * 16 + 2 * gI]) * hf(hB[n * 32 + 4 * gI]) -
                       hf(hA[m * 16 + 2 * gI + 1]) * hf(hB[n * 32 + 4 * gI + 1]) +
                       hf(hA[m * 16 + 2 * gI]) * hf(hB[n * 32 + 4 * gI + 2]) +
                       hf(hA[m * 16 + 2 * gI + 1]) * hf(hB[n * 32 + 4 * gI + 3]);
          e = fmax(e, fabs(ref - D[m * 8 + n]));
        }
        if (e < 1e-3) found = gI;
      }
      printf(" row %d grp %d;", m, found);
    }
    printf("\n");
  }
  return 0;
}
