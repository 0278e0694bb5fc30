// attn_tc.cu -- tcgen05 (5th-gen tensor core) score kernel for the head
// presets: the key decode K_j(i) = sum_r U[r,j,a_r] + i U[r,j,b_r] as a
// one-hot GEMM with the accumulators in TMEM.
//
// Per 128-token tile and per (round r, side s in {a, b}):
//     D_s[token, n] += A_{r,s}[token, l] * B_r[n, l]      (M=128, N=128, K=64)
// A_{r,s} is the one-hot of the token's code (fp16 1.0 at l = code), B_r the
// round-r codebook as fp16 with n = 2j + {x, y}.  D_a and D_b live in TMEM
// (128 columns each); K = D_a + i D_b.  The epilogue (one thread per token =
// one TMEM lane) rotates K by the RoPE phase -- the tile-independent
// e^{+i delta theta_j} table also lives in TMEM, the per-tile factor
// e^{-i (t - pos_tile) theta_j} is folded into the query -- and forms the G
// query-head partial scores.
//
// Warp roles (160 threads): warps 0-3 = one-hot producers (thread = token;
// only the 1.0 entries are set and later cleared, so a stage costs one 2-B
// store per token instead of 16 KB of smem traffic) and epilogue; warp 4 =
// TMEM allocator + single-thread tcgen05.mma issuer.  Synchronisation is by
// mbarriers: full[stage] (128 producer arrivals), empty[stage] and d_full
// (tcgen05.commit), d_empty (128 epilogue arrivals).
//
// Codebook precision is fp16 (as CVQ_CACHE_KEYS_FP16); accumulation fp32.
// Rounds are processed in blocks of <= 11 (176 KiB of B per block); a 2-bit
// stream (R = 21) uses two blocks whose partial scores the value kernel sums.
#include "cvq_internal.cuh"

namespace cvq {

namespace {

constexpr int kTcTile = 128;
constexpr int kTcThreads = 160;
constexpr int kTcRR = 11;        // rounds per block
constexpr int kNB = 64;          // MMA N per CTA: 32 subspaces x (x, y)
constexpr int kSub = kNB / 2;    // subspaces per CTA (a stream is split in 2 halves)
constexpr int kBBytes = kNB * 64 * 2;  // one round of B: 64 levels x 64 reals fp16
constexpr int kTcStages = 8;     // one-hot A stages (16 KiB each)
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColPh = 256;  // D buffers at [0,128) and [128,256): Da | Db

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];}" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;}"
      : "=r"(ok)
      : "r"(su32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}
// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of
// 8 rows x 16 B; lbo = byte stride between K-adjacent core matrices, sbo =
// between M/N-adjacent ones; version 1 (Blackwell) at bit 46.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;"); }

// Byte offset of element (row, l) in a K-major, no-swizzle 128-row x 64-K
// fp16 operand: core matrix (kc = l/8, g = row/8) at (kc*16 + g)*128.
__device__ __forceinline__ uint32_t kmaj_off(int row, int l) {
  return (uint32_t)((((l >> 3) * 16 + (row >> 3)) << 7) + ((row & 7) << 4) + ((l & 7) << 1));
}

struct TcArgs {
  const uint64_t* kpool;
  uint64_t kstride;
  const uint16_t* cbtc;  // [slot][R][2 halves][8 KiB canonical B] fp16
  int n_slots;
  const float* q;        // [S][G][128]
  const double* thetas;
  long long t, pos0, n;
  int chunk;             // tokens per CTA (multiple of 128)
  int R;                 // total rounds
  int nblk;              // round blocks
  float* ps;             // [S][nblk*2][n][G]
};

template <int G>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_score(TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* Bs = smem;                                    // [kTcRR][8 KiB]
  unsigned char* As = smem + kTcRR * kBBytes;                  // [kTcStages][16 KiB]
  float2* wq = reinterpret_cast<float2*>(As + kTcStages * 16384);  // [3][32][G]
  uint16_t* lastoff = reinterpret_cast<uint16_t*>(wq + 3 * kSub * G);  // [kTcStages][128]/16
  uint64_t* bars = reinterpret_cast<uint64_t*>(lastoff + kTcStages * 128);
  uint64_t* full = bars;                       // [kTcStages]
  uint64_t* empty = bars + kTcStages;          // [kTcStages]
  uint64_t* dfull = bars + 2 * kTcStages;      // [2]
  uint64_t* dempty = dfull + 2;                // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int per = 2 * a.nblk;
  const int s = blockIdx.y / per, part = blockIdx.y % per;
  const int blk = part >> 1, half = part & 1;
  const int r0 = blk * kTcRR;
  const int rr = min(kTcRR, a.R - r0);
  const long long i0 = (long long)blockIdx.x * a.chunk;
  const long long i1 = min(a.n, i0 + a.chunk);
  if (i0 >= i1) return;
  const int ntiles = (int)((i1 - i0 + kTcTile - 1) / kTcTile);
  const int slot = s % a.n_slots;
  const int j0 = half * kSub;  // first subspace of this CTA

  // ---- setup: TMEM, barriers, B (codebook block/half), zeroed A stages ----
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(full + i, 4);  // one arrival per producer warp
      mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(dfull + i, 1);
      mbar_init(dempty + i, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.cbtc);
    uint4* dst = reinterpret_cast<uint4*>(Bs);
    for (int e = tid; e < rr * (kBBytes / 16); e += kTcThreads) {
      const int r = e / (kBBytes / 16), o = e % (kBBytes / 16);
      dst[e] = __ldg(src + ((((size_t)slot * a.R + r0 + r) * 2 + half) * (kBBytes / 16)) + o);
    }
    uint4* az = reinterpret_cast<uint4*>(As);
    for (int e = tid; e < kTcStages * 1024; e += kTcThreads) az[e] = make_uint4(0, 0, 0, 0);
    for (int e = tid; e < kTcStages * 128; e += kTcThreads) lastoff[e] = 0xffffu;
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ================= producers + epilogue (thread = token row) =========
    const int d = tid;  // row in the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    // tile-independent phase table e^{+i d theta_j}, j in this half
#pragma unroll 1
    for (int c = 0; c < kSub / 8; ++c) {
      uint32_t v[16];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        double sn, cs;
        sincos((double)d * a.thetas[j0 + 8 * c + jj], &sn, &cs);
        v[2 * jj] = __float_as_uint((float)cs);
        v[2 * jj + 1] = __float_as_uint((float)sn);
      }
      tmem_st16(tmem + lane_base + kColPh + 16 * c, v);
    }
    tmem_wait_st();
    const uint64_t* kw = a.kpool + (size_t)s * a.kstride;
    const float* qs = a.q + (size_t)s * G * 128;
    float* ps = a.ps + (((size_t)s * per + part) * a.n) * G;
    auto load_window = [&](long long tbase, int nvalid, uint64_t& x0, uint64_t& x1, uint64_t& x2,
                           uint32_t& off) {
      const long long i = tbase + (d < nvalid ? d : 0);
      const unsigned long long bit = ((unsigned long long)i * (2 * a.R) + 2 * r0) * 6ull;
      const unsigned long long w = bit >> 6;
      off = (uint32_t)(bit & 63u);
      x0 = __ldg(kw + w);
      x1 = __ldg(kw + w + 1);
      x2 = __ldg(kw + w + 2);
    };
    // epilogue of tile kk: K = D_a + i D_b, RoPE phase, G query-head dots
    auto epilogue = [&](int kk) {
      const long long ti = i0 + (long long)kk * kTcTile;
      const int valid = (int)min((long long)kTcTile, i1 - ti);
      const int db = kk & 1;
      mbar_wait(dfull + db, (kk >> 1) & 1);
      tc_fence_after();
      asm volatile("bar.sync 1, 128;" ::: "memory");  // w' of tile kk (written by warp 0)
      const float2* wk = wq + (kk % 3) * kSub * G;
      float acc[G];
#pragma unroll
      for (int h = 0; h < G; ++h) acc[h] = 0.f;
      const uint32_t dcol = db * 128;
#pragma unroll 1
      for (int c = 0; c < kSub / 8; ++c) {
        uint32_t va[16], vb[16], vp[16];
        tmem_ld16(tmem + lane_base + dcol + 16 * c, va);
        tmem_ld16(tmem + lane_base + dcol + 64 + 16 * c, vb);
        tmem_ld16(tmem + lane_base + kColPh + 16 * c, vp);
        tmem_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const float kx = __uint_as_float(va[2 * jj]) - __uint_as_float(vb[2 * jj + 1]);
          const float ky = __uint_as_float(va[2 * jj + 1]) + __uint_as_float(vb[2 * jj]);
          const float px = __uint_as_float(vp[2 * jj]), py = __uint_as_float(vp[2 * jj + 1]);
          const float rx = px * kx - py * ky, ry = px * ky + py * kx;
          const float2* w = wk + (8 * c + jj) * G;
#pragma unroll
          for (int h = 0; h < G; ++h) acc[h] += w[h].x * rx - w[h].y * ry;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dempty + db);
      if (d < valid) {
#pragma unroll
        for (int h = 0; h < G; ++h) ps[(ti + d) * G + h] = acc[h];
      }
    };
    uint64_t wn0 = 0, wn1 = 0, wn2 = 0;
    uint32_t woff = 0;
    uint32_t g = 0;  // global one-hot step counter (stage = g % kTcStages)
    constexpr int kGroup = 4;  // one-hot steps per proxy fence
    for (int k = 0; k < ntiles; ++k) {
      const long long ti = i0 + (long long)k * kTcTile;
      const int valid = (int)min((long long)kTcTile, i1 - ti);
      if (k == 0) load_window(ti, valid, wn0, wn1, wn2, woff);
      const uint64_t w0 = wn0, w1 = wn1, w2 = wn2;
      const uint32_t off0 = woff;
      // query folded with this tile's phase base (triple-buffered by tile)
      if (d < kSub) {
        float2* wk = wq + (k % 3) * kSub * G;
        const float2 pb = phase_neg(a.t - (a.pos0 + ti), a.thetas[j0 + d]);
        const int j = j0 + d;
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const float qx = qs[h * 128 + 2 * j] * 0.08838834764831845f;
          const float qy = -qs[h * 128 + 2 * j + 1] * 0.08838834764831845f;
          wk[d * G + h] = make_float2(qx * pb.x - qy * pb.y, qx * pb.y + qy * pb.x);
        }
      }
      // one-hot stages: (round r, side) steps, a then b, fenced in groups
#pragma unroll
      for (int s0 = 0; s0 < 2 * kTcRR; s0 += kGroup) {
        if (s0 < 2 * rr) {
#pragma unroll
          for (int i = 0; i < kGroup; ++i) {
            const int step = s0 + i;
            if (step < 2 * kTcRR && step < 2 * rr) {
              const uint32_t bit = off0 + 6u * step;
              const uint32_t wi = bit >> 6, sh = bit & 63u;
              const uint64_t lo = wi == 0 ? w0 : (wi == 1 ? w1 : w2);
              const uint64_t hi = wi == 0 ? w1 : w2;
              uint64_t v = lo >> sh;
              if (sh > 58u) v |= hi << (64u - sh);
              const int code = (int)(v & 63u);
              const uint32_t gg = g + i;
              const uint32_t st = gg % kTcStages, n_use = gg / kTcStages;
              if (n_use > 0) mbar_wait(empty + st, (n_use - 1) & 1);  // MMA done with it
              unsigned char* A = As + st * 16384;
              const uint32_t old = lastoff[st * 128 + d];
              if (old != 0xffffu) *reinterpret_cast<uint16_t*>(A + 2 * old) = 0;
              const uint32_t off = kmaj_off(d, code);
              *reinterpret_cast<uint16_t*>(A + off) = 0x3C00;  // fp16 1.0
              lastoff[st * 128 + d] = (uint16_t)(off >> 1);
            }
          }
          fence_async_smem();
          __syncwarp();
          const int nstep = min(kGroup, 2 * rr - s0);
          if (lane < nstep) mbar_arrive(full + (g + lane) % kTcStages);  // one per warp each
          g += nstep;
        }
      }
      // prefetch the next tile's code window only now: the proxy fences above
      // wait for all of this thread's outstanding memory operations
      if (k + 1 < ntiles) {
        const long long tn = ti + kTcTile;
        load_window(tn, (int)min((long long)kTcTile, i1 - tn), wn0, wn1, wn2, woff);
      }
      // the epilogue trails by one tile so the MMA never waits for it
      if (k > 0) epilogue(k - 1);
    }
    epilogue(ntiles - 1);
  } else if (tid == 128) {
    // ================= single-thread tcgen05.mma issuer ==================
    constexpr uint32_t idesc = (1u << 4) | ((kNB >> 3) << 17) | (8u << 24);  // f16->f32, M128 N64
    const uint32_t a_base = su32(As), b_base = su32(Bs);
    uint32_t g = 0;
    for (int k = 0; k < ntiles; ++k) {
      const int db = k & 1;
      if (k >= 2) {  // epilogue of tile k-2 released this D buffer
        mbar_wait(dempty + db, ((k - 2) >> 1) & 1);
        tc_fence_after();
      }
      for (int step = 0; step < 2 * rr; ++step, ++g) {
        const uint32_t st = g % kTcStages, u = g / kTcStages;
        mbar_wait(full + st, u & 1);
        tc_fence_after();
        const int r = step >> 1;
        const uint32_t dcol = db * 128 + ((step & 1) ? 64 : 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // K = 64 levels as 4 x K16
          const uint64_t ad = sdesc(a_base + st * 16384 + kk * 4096, 2048, 128);
          const uint64_t bd = sdesc(b_base + r * kBBytes + kk * 2048, 1024, 128);
          umma_f16(tmem + dcol, ad, bd, idesc, (r > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(empty + st);
      }
      tc_commit(dfull + db);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 4)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
}

}  // namespace

size_t tc_smem_bytes(int G) {
  return (size_t)kTcRR * kBBytes + kTcStages * 16384 + 3 * kSub * G * sizeof(float2) +
         kTcStages * 128 * 2 + (2 * kTcStages + 4) * 8 + 16;
}

// partial-score blocks per stream: round blocks x 2 subspace halves
int tc_blocks(int R) { return 2 * ((R + kTcRR - 1) / kTcRR); }

// Host-side B layout for one slot: [R][half][K-major 64 x 64 fp16] with
// n = 2(j - 32 half) + {0: x, 1: y}, l = level; core matrix (kc = l/8,
// g = n/8) at (kc*8 + g)*128 B.
void tc_build_codebook(int R, int L, int subs, const double* xy, uint16_t* out,
                       uint16_t (*to_half)(double)) {
  for (int r = 0; r < R; ++r)
    for (int j = 0; j < subs; ++j)
      for (int l = 0; l < L; ++l)
        for (int c = 0; c < 2; ++c) {
          const int hf = j / kSub, n = 2 * (j % kSub) + c;
          const size_t off = ((((size_t)(l >> 3) * 8 + (n >> 3)) << 7) + ((n & 7) << 4) +
                              ((l & 7) << 1)) / 2;
          out[((size_t)r * 2 + hf) * (kBBytes / 2) + off] =
              to_half(xy[(((size_t)r * subs + j) * L + l) * 2 + c]);
        }
}

cudaError_t run_tc_score(const AttnJob& job, const float* q, float* ps, int chunk,
                         cudaStream_t st) {
  const Geom& g = job.geo;
  TcArgs a{};
  a.kpool = job.kpool;
  a.kstride = job.kstride;
  a.cbtc = job.cb_key_tc;
  a.n_slots = job.n_slots;
  a.q = q;
  a.thetas = job.thetas;
  a.t = job.t;
  a.pos0 = job.pos0;
  a.n = job.n;
  a.chunk = chunk;
  a.R = g.R;
  a.nblk = tc_blocks(g.R) / 2;
  a.ps = ps;
  const size_t sm = tc_smem_bytes(g.G);
  dim3 grid((unsigned)((job.n + chunk - 1) / chunk), job.S * a.nblk * 2);
  cudaError_t e;
  if (g.G == 4) {
    static size_t done = 0;
    if (sm > done) {
      e = cudaFuncSetAttribute(k_tc_score<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      done = sm;
    }
    k_tc_score<4><<<grid, kTcThreads, sm, st>>>(a);
  } else {
    static size_t done = 0;
    if (sm > done) {
      e = cudaFuncSetAttribute(k_tc_score<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      done = sm;
    }
    k_tc_score<1><<<grid, kTcThreads, sm, st>>>(a);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace cvq
