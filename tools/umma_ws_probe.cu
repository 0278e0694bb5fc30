// Round-2 probe: tcgen05.mma.ws.sp (weight-stationary) with B collector
// buffers for the sparse score kernel's resident-codebook round.
//
// Each round issues 8 sparse M128 x N64 x K32 MMAs that read only 4 distinct
// B slices (X_h, Y_h for K halves h = 0, 1): side a uses (X_h -> Re, Y_h ->
// Im), side b (-Y_h -> Re, X_h -> Im).  With .collector::bN::fill on the
// first use and ::lastuse on the second, each slice should be read from smem
// once per round instead of twice -- half the B bandwidth (the plain .sp
// pattern reads 128 B/clk of B, all the smem bandwidth there is).
//
// test 1: one round with random A (TMEM, uniform metadata) and random B
//         (exact fp16 products): D from .sp vs .ws.sp (+ collectors), bitwise.
// test 2: 64 tiles x 11 rounds, issuer only, with `nld` extra warps
//         streaming ld.shared (the epilogue's smem traffic): clk per tile.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_ws_probe tools/umma_ws_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ bool mtry(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;}"
               : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok != 0;
}

// one round, plain sparse MMAs (the round-1 schedule)
__device__ __forceinline__ void round_sp(uint32_t d, uint32_t a, uint32_t e, uint64_t br, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{.reg .pred q, p, t;\n\t"
      ".reg .b32 a1, a2, a3, d1, e1;\n\t"
      ".reg .b64 b1, b2, b3;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.u32 t, %5, %5;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.u32 d1, %0, 64;\n\tadd.u32 e1, %2, 2;\n\t"
      "add.u64 b1, %3, 64;\n\tadd.u64 b2, %3, 512;\n\tadd.u64 b3, %3, 576;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %3, [%2], %4, p;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [d1], [%1], b1, [%2], %4, p;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [a1], b2, [%2], %4, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [d1], [a1], b3, [%2], %4, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [a2], b1, [e1], %6, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [d1], [a2], %3, [e1], %4, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [a3], b3, [e1], %6, t;\n\t"
      "@q tcgen05.mma.sp.cta_group::1.kind::f16 [d1], [a3], b2, [e1], %4, t;}" ::"r"(d),
      "r"(a), "r"(e), "l"(br), "r"(idesc), "r"(accum), "r"(idesc | (1u << 13)) : "memory");
}
// same round as weight-stationary MMAs, each B slice read once: X_0 -> b0,
// Y_0 -> b1, X_1 -> b2, Y_1 -> b3 (fill on the side-a use, lastuse on side b)
__device__ __forceinline__ void round_ws(uint32_t d, uint32_t a, uint32_t e, uint64_t br, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{.reg .pred q, p, t;\n\t"
      ".reg .b32 a1, a2, a3, d1, e1;\n\t"
      ".reg .b64 b1, b2, b3;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.u32 t, %5, %5;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.u32 d1, %0, 64;\n\tadd.u32 e1, %2, 2;\n\t"
      "add.u64 b1, %3, 64;\n\tadd.u64 b2, %3, 512;\n\tadd.u64 b3, %3, 576;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16.collector::b0::fill [%0], [%1], %3, [%2], %4, p;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16.collector::b1::fill [d1], [%1], b1, [%2], %4, p;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16.collector::b2::fill [%0], [a1], b2, [%2], %4, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16.collector::b3::fill [d1], [a1], b3, [%2], %4, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16.collector::b1::lastuse [%0], [a2], b1, [e1], %6, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16.collector::b0::lastuse [d1], [a2], %3, [e1], %4, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16.collector::b3::lastuse [%0], [a3], b3, [e1], %6, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16.collector::b2::lastuse [d1], [a3], b2, [e1], %4, t;}" ::"r"(d),
      "r"(a), "r"(e), "l"(br), "r"(idesc), "r"(accum), "r"(idesc | (1u << 13)) : "memory");
}
// weight-stationary without collector reuse
__device__ __forceinline__ void round_ws_plain(uint32_t d, uint32_t a, uint32_t e, uint64_t br, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{.reg .pred q, p, t;\n\t"
      ".reg .b32 a1, a2, a3, d1, e1;\n\t"
      ".reg .b64 b1, b2, b3;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.u32 t, %5, %5;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.u32 d1, %0, 64;\n\tadd.u32 e1, %2, 2;\n\t"
      "add.u64 b1, %3, 64;\n\tadd.u64 b2, %3, 512;\n\tadd.u64 b3, %3, 576;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16 [%0], [%1], %3, [%2], %4, p;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16 [d1], [%1], b1, [%2], %4, p;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16 [%0], [a1], b2, [%2], %4, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16 [d1], [a1], b3, [%2], %4, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16 [%0], [a2], b1, [e1], %6, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16 [d1], [a2], %3, [e1], %4, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16 [%0], [a3], b3, [e1], %6, t;\n\t"
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16 [d1], [a3], b2, [e1], %4, t;}" ::"r"(d),
      "r"(a), "r"(e), "l"(br), "r"(idesc), "r"(accum), "r"(idesc | (1u << 13)) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("{.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\t"
               "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(su32(bar)) : "memory");
}

constexpr uint32_t kIdesc = (1u << 4) | (8u << 17) | (8u << 24) | (1u << 2);  // f32 acc, N=64, M=128, sparse

// test 1: D[0..127] from .sp, D[128..255] from .ws.sp + collectors, D[256..383]
// from .ws.sp plain; A = 32 columns at 384.., metadata 448.. (uniform 0x4444)
__global__ void kcheck(const uint32_t* Atm, const __half* Bs, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 16384 / 2; i += blockDim.x) reinterpret_cast<__half*>(sm)[i] = Bs[i];
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
  const uint32_t lb = (uint32_t)(warp * 32) << 16;
  for (int c = 0; c < 32; ++c)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lb + 384 + c), "r"(Atm[(warp * 32 + lane) * 32 + c]) : "memory");
  for (int c = 0; c < 4; ++c)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lb + 448 + c), "r"(0x44444444u) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    const uint64_t br = sdesc(su32(sm), 2048, 128);
    round_sp(tmem, tmem + 384, tmem + 448, br, kIdesc, 0);
    round_ws(tmem + 128, tmem + 384, tmem + 448, br, kIdesc, 0);
    round_ws_plain(tmem + 256, tmem + 384, tmem + 448, br, kIdesc, 0);
    commit(&bar);
    __syncwarp();
    while (!mtry(&bar, 0)) {}
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < 384; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + lb + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    D[(warp * 32 + lane) * 384 + c] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// test 2: issuer-only tile loop; warps 4.. stream ld.shared over a 16 KiB
// window (outside the codebook) until the issuer is done
template <int MODE>
__global__ void __launch_bounds__(1024, 1) krate(int tiles, int nld, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t fin;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (176 + 16) * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (tid == 0) done = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&fin)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
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
    const uint64_t bdesc0 = sdesc(su32(sm), 2048, 128);
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dcol = tmem + (uint32_t)(t & 1) * 128u;
      uint64_t br = bdesc0;
#pragma unroll 1
      for (int r = 0; r < 11; ++r) {
        const uint32_t st = (uint32_t)(r % 6);
        if (MODE == 0) round_sp(dcol, tmem + 256 + 32 * st, tmem + 448 + 4 * st, br, kIdesc, r ? 1u : 0u);
        else if (MODE == 1) round_ws(dcol, tmem + 256 + 32 * st, tmem + 448 + 4 * st, br, kIdesc, r ? 1u : 0u);
        else round_ws_plain(dcol, tmem + 256 + 32 * st, tmem + 448 + 4 * st, br, kIdesc, r ? 1u : 0u);
        br += (uint64_t)(16384 >> 4);
      }
    }
    commit(&fin);
    __syncwarp();
    while (!mtry(&fin, 0)) {}
    if (blockIdx.x == 0 && lane == 0) out[0] = clock64() - t0;
    if (lane == 0) done = 1;
  } else if (warp >= 4 && warp < 4 + nld) {
    const float4* win = reinterpret_cast<const float4*>(sm + 176 * 1024);
    float4 acc = make_float4(0, 0, 0, 0);
    int i = lane;
    while (!done) {
#pragma unroll 8
      for (int u = 0; u < 8; ++u) {
        const float4 v = win[(i + 32 * u) & 1023];
        acc.x += v.x;
        acc.y += v.y;
      }
      i += 7;
    }
    if (acc.x == 1234.5f) out[1] = (long long)acc.y;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// test 3: issue-queue depth.  One thread issues 24 sparse N=64 MMAs back to
// back (pipe idle at the start) and reads clock64 after each issue: the
// first ones return at once, later ones only when the tensor pipe has room.
__global__ void kqueue(long long* out, int ws) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t fin;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&fin)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint64_t b = sdesc(su32(sm), 2048, 128);
    long long ts[25];
    ts[0] = clock64();
#pragma unroll
    for (int i = 0; i < 24; ++i) {
      if (ws)
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                     "tcgen05.mma.ws.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%4], %3, p;}" ::"r"(tmem + (i & 1) * 64),
                     "r"(tmem + 256), "l"(b), "r"(kIdesc), "r"(tmem + 448) : "memory");
      else
        asm volatile("{.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%4], %3, p;}" ::"r"(tmem + (i & 1) * 64),
                     "r"(tmem + 256), "l"(b), "r"(kIdesc), "r"(tmem + 448) : "memory");
      ts[i + 1] = clock64();
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&fin)) : "memory");
    while (!mtry(&fin, 0)) {}
    const long long te = clock64();
    for (int i = 0; i < 25; ++i) out[i] = ts[i] - ts[0];
    out[25] = te - ts[0];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int MODE>
void rate(int nld, long long* d) {
  auto k = krate<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (176 + 16) * 1024);
  k<<<148, 1024, (176 + 16) * 1024>>>(2, nld, d);
  k<<<148, 1024, (176 + 16) * 1024>>>(64, nld, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {".sp", ".ws.sp + B collectors", ".ws.sp plain"};
  printf("rate %-24s ld.shared warps %2d: %.1f clk per 128-token tile (88 MMAs), %.1f clk/mma\n", nm[MODE], nld, cyc / 64.0,
         cyc / 64.0 / 88);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  // test 1
  srand(7);
  uint32_t* hA = (uint32_t*)malloc(128 * 32 * 4);
  __half* hB = (__half*)malloc(16384);
  for (int i = 0; i < 128 * 32; ++i) {
    const __half lo = __float2half((float)(rand() % 17 - 8) / 8.f), hi = __float2half((float)(rand() % 17 - 8) / 8.f);
    hA[i] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
  }
  for (int i = 0; i < 8192; ++i) hB[i] = __float2half((float)(rand() % 17 - 8) / 8.f);
  uint32_t* dA;
  __half* dB;
  float* dD;
  cudaMalloc(&dA, 128 * 32 * 4);
  cudaMalloc(&dB, 16384);
  cudaMalloc(&dD, 128 * 384 * 4);
  cudaMemcpy(dA, hA, 128 * 32 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, 16384, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kcheck, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  kcheck<<<1, 128, 16384>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("check err %s\n", cudaGetErrorString(e)); return 1; }
  float* hD = (float*)malloc(128 * 384 * 4);
  cudaMemcpy(hD, dD, 128 * 384 * 4, cudaMemcpyDeviceToHost);
  int diff_ws = 0, diff_wsp = 0, nz = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 128; ++c) {
      const float a = hD[r * 384 + c], b = hD[r * 384 + 128 + c], p = hD[r * 384 + 256 + c];
      nz += a != 0.f;
      diff_ws += memcmp(&a, &b, 4) != 0;
      diff_wsp += memcmp(&a, &p, 4) != 0;
    }
  printf("check: %d / 16384 nonzero; .ws.sp+collectors differs from .sp at %d, .ws.sp plain at %d\n", nz, diff_ws, diff_wsp);
  if (diff_ws)
    for (int r = 0; r < 4; ++r)
      printf("  row %d: sp %g %g %g  ws %g %g %g  wsp %g %g %g\n", r, hD[r * 384], hD[r * 384 + 1], hD[r * 384 + 64],
             hD[r * 384 + 128], hD[r * 384 + 129], hD[r * 384 + 192], hD[r * 384 + 256], hD[r * 384 + 257], hD[r * 384 + 320]);
  long long* d;
  cudaMalloc(&d, 32 * 8);
  for (int ws = 0; ws < 2; ++ws) {
    cudaFuncSetAttribute(kqueue, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    kqueue<<<1, 128, 16384>>>(d, ws);
    kqueue<<<1, 128, 16384>>>(d, ws);
    cudaDeviceSynchronize();
    long long q[26];
    cudaMemcpy(q, d, 26 * 8, cudaMemcpyDeviceToHost);
    printf("queue%s: clk after each issue:", ws ? " (.ws)" : "");
    for (int i = 1; i < 25; ++i) printf(" %lld", q[i]);
    printf("; all complete at %lld\n", q[25]);
  }
  for (int nld : {0, 8, 16, 24}) {
    rate<0>(nld, d);
    rate<1>(nld, d);
    rate<2>(nld, d);
  }
  return 0;
}
