// attn_tc.cu -- tcgen05 (5th-gen tensor core) score kernel for the head
// presets: the key decode K_j(i) = sum_r U[r,j,a_r] + i U[r,j,b_r] as a
// one-hot GEMM, laid out so each MMA is full width:
//
//   D^T[n, t] += A_{r,s}[n, l] * B_{r,s}[t, l]     (M = 128, N = 256, K = 64)
//
// * n = 2j + {x, y} indexes the 128 reals of a key, t the 256 tokens of a
//   tile.  For side a, A = U_r (A[2j+c, l] = U[r,j,l].c); for side b, A is
//   the ROTATED codebook (A[2j, l] = -U[r,j,l].y, A[2j+1, l] = U[r,j,l].x),
//   so both sides accumulate into one D that holds (Re K, Im K) directly.
// * B_{r,s} = one-hot of the tile tokens' side-s codes (fp16 1.0 at
//   l = code), written into a K-major smem stage by 4 producer warps that
//   only set and clear the 1.0 entries.  The A slice (16 KiB fp16, built
//   once per codebook in the MMA's core-matrix layout) arrives in the same
//   stage by one cp.async.bulk; a stage is 48 KiB, 4 stages deep.
// * Measured on B200 (profiles/r01_umma_issue_bench.txt) a single issuer's
//   tcgen05.mma costs >= ~125 clk whatever N <= 256, so N = 256 (128 clk of
//   tensor work) is the only shape that is not issue-bound; D (256 fp32
//   columns) is double-buffered in TMEM (all 512 columns) so the epilogue of
//   tile k overlaps the MMAs of tile k+1.
// * epilogue (16 warps; thread = real n = TMEM lane; warp (quarter, slot)
//   owns 64 tokens of the tile and frees D right after its two TMEM loads):
//   partner shuffle for the other component, the RoPE phase by a
//   per-subspace fp32 recurrence from an fp64-reduced base per tile; for
//   G = 4 each lane of a (x, y) pair forms the full complex product for two
//   of the heads, so the cross-lane reduction runs over 16 lanes; a 4-warp
//   sum in smem -> partial scores.
//
// Persistent CTAs (one per SM) walk (stream, chunk) work items.  Warp roles
// (640 threads): 0-15 epilogue, 16-17 one-hot producers, 18 TMEM allocator +
// MMA issuer (elected lane), 19 codebook loader.  mbarriers: full[stage]
// (2 producer warps + loader with tx bytes), empty[stage] and d_full[buf]
// (tcgen05.commit), d_empty[buf] (16 epilogue warps).
//
// Codebook precision fp16 (as CVQ_CACHE_KEYS_FP16), accumulation fp32.
#include <cstdlib>

#include "cvq_internal.cuh"


namespace cvq {

namespace {

constexpr int kTok = 256;                 // tokens per tile (MMA N)
constexpr int kEpiWarps = 16;             // 4 per TMEM lane quarter
constexpr int kEpiSlots = kEpiWarps / 4;  // slot s takes tile tokens [64 s, 64 s + 64)
constexpr int kProdWarps = 2;             // thread p owns tile tokens p + 64 i
constexpr int kMmaWarp = kEpiWarps + kProdWarps;
constexpr int kLoadWarp = kMmaWarp + 1;
constexpr int kThreads = (kLoadWarp + 1) * 32;
constexpr int kStages = 4;
constexpr int kPGroup = 2;                // producer steps per proxy fence
constexpr int kABytes = 128 * 64 * 2;     // 16 KiB codebook slice
constexpr int kBBytes = kTok * 64 * 2;    // 32 KiB one-hot
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kChunk = kTok / kEpiSlots;  // epilogue tokens per warp per tile
constexpr uint32_t kTmemCols = 512;

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
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(su32(bar)),
      "r"(bytes)
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
// for waiters off the critical path: back off so the spin does not take
// issue slots from the epilogue warps
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) __nanosleep(64);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
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
// between row-adjacent ones; descriptor version 1 at bit 46.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

// packed fp32x2 arithmetic (FMUL2 / FFMA2 on sm_100a); the scalar operand is
// broadcast to both halves
__device__ __forceinline__ float2 fmul2(float2 a, float b) {
  uint64_t d;
  asm("{.reg .b64 a, b;\n\tmov.b64 a, {%1, %2};\n\tmov.b64 b, {%3, %3};\n\t"
      "mul.rn.f32x2 %0, a, b;}"
      : "=l"(d)
      : "f"(a.x), "f"(a.y), "f"(b));
  return make_float2(__uint_as_float((uint32_t)d), __uint_as_float((uint32_t)(d >> 32)));
}
__device__ __forceinline__ float2 ffma2(float2 a, float b, float2 c) {
  uint64_t d;
  asm("{.reg .b64 a, b, c;\n\tmov.b64 a, {%1, %2};\n\tmov.b64 b, {%3, %3};\n\t"
      "mov.b64 c, {%4, %5};\n\tfma.rn.f32x2 %0, a, b, c;}"
      : "=l"(d)
      : "f"(a.x), "f"(a.y), "f"(b), "f"(c.x), "f"(c.y));
  return make_float2(__uint_as_float((uint32_t)d), __uint_as_float((uint32_t)(d >> 32)));
}

// Byte offset of (row t, level l) in a K-major, no-swizzle ROWS x 64 fp16
// operand: core matrix (kc = l/8, g = t/8) at (kc*ROWS/8 + g)*128.
template <int ROWS>
__host__ __device__ __forceinline__ uint32_t kmaj(int t, int l) {
  return (uint32_t)((((l >> 3) * (ROWS / 8) + (t >> 3)) << 7) + ((t & 7) << 4) + ((l & 7) << 1));
}

struct TcArgs {
  const uint64_t* kpool;
  uint64_t kstride;
  const uint16_t* cbtc;  // slot s at cbtc + s * slot_elems: [R][2][8192] fp16 A operand
  size_t slot_elems;
  int n_slots;
  const float* q;        // [S][G][128]
  const double* thetas;
  long long t, pos0, n;
  int chunk;             // tokens per work item (multiple of kTok)
  int cps;               // work items per stream
  int n_items;
  float* ps;             // [S][n][G]
};

// Iterate this CTA's tiles in order: (stream, first token, valid tokens).
struct TileIter {
  int item, s;
  long long ti, hi;
  __device__ bool first(const TcArgs& a) {
    item = blockIdx.x;
    return setup(a);
  }
  __device__ bool setup(const TcArgs& a) {
    while (item < a.n_items) {
      s = item / a.cps;
      ti = (long long)(item % a.cps) * a.chunk;
      hi = min(a.n, ti + a.chunk);
      if (ti < hi) return true;
      item += gridDim.x;
    }
    return false;
  }
  __device__ bool next(const TcArgs& a) {
    ti += kTok;
    if (ti < hi) return true;
    item += gridDim.x;
    return setup(a);
  }
  __device__ int valid() const { return (int)min((long long)kTok, hi - ti); }
};

template <int R, int G>
__global__ void __launch_bounds__(kThreads, 1) k_tc_score(TcArgs a) {
  static_assert(32 % G == 0, "G must divide the warp");
  constexpr int NSTEP = 2 * R;  // (round, side) steps per tile
  constexpr int NW = (NSTEP * 6 + 60 + 63) / 64 + 1;  // code window words (+1 for the shift)
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* stages = smem;                                                // [kStages][A|B]
  float* red = reinterpret_cast<float*>(stages + kStages * kStageBytes);  // [slot][4][kChunk][G]
  // raw key-code windows of the NEXT tile, prefetched by the producers with
  // cp.async while the current tile is produced: [kTok][NW] words
  uint64_t* wbuf = reinterpret_cast<uint64_t*>(red + kEpiSlots * 4 * kChunk * G);
  uint64_t* bars = wbuf + (size_t)kTok * NW;
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* dfull = bars + 2 * kStages;
  uint64_t* dempty = dfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(full + i, kProdWarps + 1);
      mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(dfull + i, 1);
      mbar_init(dempty + i, kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int st = 0; st < kStages; ++st) {
    uint4* bz = reinterpret_cast<uint4*>(stages + st * kStageBytes + kABytes);
    for (int e = tid; e < kBBytes / 16; e += kThreads) bz[e] = make_uint4(0, 0, 0, 0);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kEpiWarps) {
    // ============ epilogue: thread = real n (TMEM lane); warp (quarter,
    // slot) takes the tile's 64 tokens [64 slot, 64 slot + 64)
    const int quarter = warp & 3, eslot = warp >> 2;
    const int n = quarter * 32 + lane;
    const int j = n >> 1, c = n & 1;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const double theta = a.thetas[j];
    // lane c = 0 owns Z.x = ph.x K.x - ph.y K.y, lane c = 1 owns
    // Z.y = ph.x K.y + ph.y K.x.  With the partner's component ko and
    // phs = (ph.x, sgn ph.y): own Z.c = phs.x kc + phs.y ko and other
    // Z.(1-c) = phs.x ko - phs.y kc, for both lanes.  The recurrence
    // phs <- phs * e^{i theta} keeps that form with sgn folded into the
    // step's imaginary part.
    const float sgn = c ? 1.f : -1.f;
    float2 stepm;
    {
      double sn, cs;
      sincos(theta, &sn, &cs);  // e^{+i theta}: one token later
      stepm = make_float2((float)cs, sgn * (float)sn);
    }
    float* rb = red + eslot * (4 * kChunk * G);  // [quarter][token][head]
    const int hsw = (lane >> 4) & 1;
    TileIter it;
    int k = 0;
    for (bool ok = it.first(a); ok; ok = it.next(a), ++k) {
      const int db = k & 1;
      const int valid = it.valid();
      const long long t0 = it.ti + eslot * kChunk;
      // G = 4: lane (j, c) forms the full Re(conj(q_h) Z_j) / sqrt(d) for
      // heads 2c + (hb ^ hsw), hb = 0, 1: (qa, qb) = (q.c, q.(1-c)).
      // G = 1: lane c forms q.c Z.c / sqrt(d).
      const float sc = 0.08838834764831845f;
      const float* qs = a.q + (size_t)it.s * G * 128;
      float2 qa, qb;
      if constexpr (G == 4) {
        const int h0 = 2 * c + hsw, h1 = 2 * c + (1 ^ hsw);
        qa = make_float2(__ldg(qs + h0 * 128 + 2 * j + c) * sc, __ldg(qs + h1 * 128 + 2 * j + c) * sc);
        qb = make_float2(__ldg(qs + h0 * 128 + 2 * j + 1 - c) * sc,
                         __ldg(qs + h1 * 128 + 2 * j + 1 - c) * sc);
      } else {
        qa = make_float2(__ldg(qs + n) * sc, 0.f);
        qb = make_float2(0.f, 0.f);
      }
      float2 ph = phase_neg(a.t - (a.pos0 + t0), theta);
      ph.y *= sgn;
      mbar_wait_sleep(dfull + db, (k >> 1) & 1);
      tc_fence_after();
      uint32_t v[kChunk];
      tmem_ld32(tmem + lane_base + db * kTok + eslot * kChunk, v);
      tmem_ld32(tmem + lane_base + db * kTok + eslot * kChunk + 32, v + 32);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dempty + db);  // D[db] is in registers: free it
      if constexpr (G == 4) {
        // acc_h = qa_h A + qb_h B with A = phs.x kc + phs.y ko and
        // B = phs.x ko - phs.y kc equals al_h kc + be_h ko where
        // al_h + i be_h = (qa_h + i qb_h)(phs.x + i phs.y); (al, be) follow the
        // same per-token rotation as the phase.  Both heads of the lane ride
        // in packed fp32x2 (FMUL2 / FFMA2 with scalar-broadcast operands).
        float2 al = make_float2(qa.x * ph.x - qb.x * ph.y, qa.y * ph.x - qb.y * ph.y);
        float2 be = make_float2(qa.x * ph.y + qb.x * ph.x, qa.y * ph.y + qb.y * ph.x);
        const float nsy = -stepm.y;
#pragma unroll
        for (int grp = 0; grp < kChunk / 8; ++grp) {
          float acc[16];  // position hb * 8 + token
#pragma unroll
          for (int tt = 0; tt < 8; ++tt) {
            const float kc = __uint_as_float(v[grp * 8 + tt]);
            const float ko = __shfl_xor_sync(0xffffffffu, kc, 1);
            const float2 r = ffma2(be, ko, fmul2(al, kc));
            acc[tt] = r.x;
            acc[8 + tt] = r.y;
            const float2 nal = ffma2(al, stepm.x, fmul2(be, nsy));
            be = ffma2(al, stepm.y, fmul2(be, stepm.x));
            al = nal;
          }
          // over the 16 same-c lanes: head level select-free (lanes with
          // bit 4 hold the heads swapped), then reduce-scatter of the tokens
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i + 8], 16);
#pragma unroll
          for (int o = 8; o >= 2; o >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < o / 2; ++i) {
              const float send = up ? acc[i] : acc[i + o / 2];
              const float keep = up ? acc[i + o / 2] : acc[i];
              acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          // lane holds head 2c + hsw, token grp*8 + ((lane >> 1) & 7)
          rb[(quarter * kChunk + grp * 8 + ((lane >> 1) & 7)) * 4 + 2 * c + hsw] = acc[0];
        }
      } else {
#pragma unroll
        for (int grp = 0; grp < kChunk / 16; ++grp) {
          float acc[16];
#pragma unroll
          for (int tt = 0; tt < 16; ++tt) {
            const float kc = __uint_as_float(v[grp * 16 + tt]);
            const float ko = __shfl_xor_sync(0xffffffffu, kc, 1);
            acc[tt] = qa.x * fmaf(ph.x, kc, ph.y * ko);
            const float nx = fmaf(ph.x, stepm.x, -ph.y * stepm.y);
            ph.y = fmaf(ph.x, stepm.y, ph.y * stepm.x);
            ph.x = nx;
          }
          // pair (x, y) first, then the tokens over lanes xor 16, 8, 4, 2
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 1);
#pragma unroll
          for (int o = 16; o >= 2; o >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < o / 2; ++i) {
              const float send = up ? acc[i] : acc[i + o / 2];
              const float keep = up ? acc[i + o / 2] : acc[i];
              acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          if (c == 0) rb[quarter * kChunk + grp * 16 + (lane >> 1)] = acc[0];
        }
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + eslot) : "memory");
#pragma unroll
      for (int e = quarter * 32 + lane; e < kChunk * G; e += 128) {  // (token, head)
        const int tt = e / G;
        if (eslot * kChunk + tt < valid)
          a.ps[((size_t)it.s * a.n + t0 + tt) * G + (e % G)] =
              (rb[e] + rb[kChunk * G + e]) + (rb[2 * kChunk * G + e] + rb[3 * kChunk * G + e]);
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + eslot) : "memory");
    }
  } else if (warp < kEpiWarps + kProdWarps) {
    // ============ one-hot producers: thread p owns tile tokens p + 128 i ====
    // A stage's previous user was the same thread 4 steps earlier (same token
    // slot), so the entry to clear is recomputed from the code windows (this
    // tile's, or the previous tile's for the first kStages steps).  The next
    // tile's code words are prefetched into smem during this tile.
    constexpr int TPT = kTok / (kProdWarps * 32);  // tokens per producer thread
    const int p = tid - kEpiWarps * 32;
    uint64_t w[TPT][NW], wp[TPT][NW];  // code windows (current, previous tile)
    // the raw words of this thread's tokens of a tile -> wbuf (cp.async; a
    // token past the end reads token 0's record, as the epilogue ignores it)
    auto issue = [&](int s, long long ti, int valid) {
      const uint64_t* kw = a.kpool + (size_t)s * a.kstride;
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const int t = p + kProdWarps * 32 * u;
        const long long tok = ti + (t < valid ? t : 0);
        const unsigned long long w0 = ((unsigned long long)tok * (NSTEP * 6)) >> 6;
#pragma unroll
        for (int i = 0; i < NW; ++i)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(wbuf + t * NW + i)),
                       "l"(kw + w0 + i)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // windows shifted so a token's code q sits at bit 6q
    auto fetch = [&](long long ti, int valid, int u, uint64_t* wv) {
      const int t = p + kProdWarps * 32 * u;
      const long long tok = ti + (t < valid ? t : 0);
      const uint32_t off = (uint32_t)(((unsigned long long)tok * (NSTEP * 6)) & 63u);
      uint64_t raw[NW];
#pragma unroll
      for (int i = 0; i < NW; ++i) raw[i] = wbuf[t * NW + i];
#pragma unroll
      for (int i = 0; i + 1 < NW; ++i)
        wv[i] = off ? (raw[i] >> off) | (raw[i + 1] << (64u - off)) : raw[i];
    };
    auto code_at = [](const uint64_t* wv, int q) -> int {  // q is a compile-time constant
      const int b0 = 6 * q, wi = b0 >> 6, sh = b0 & 63;
      return (int)((wv[wi] >> sh) | (sh > 58 ? wv[wi + 1] << (64 - sh) : 0)) & 63;
    };
#pragma unroll
    for (int u = 0; u < TPT; ++u)
#pragma unroll
      for (int i = 0; i < NW; ++i) w[u][i] = 0;
    TileIter it;
    uint32_t g = 0;
    bool have_prev = false;
    bool ok = it.first(a);
    if (ok) issue(it.s, it.ti, it.valid());
    while (ok) {
      const int valid = it.valid();
      asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's words of this tile
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
#pragma unroll
        for (int i = 0; i < NW; ++i) wp[u][i] = w[u][i];
        fetch(it.ti, valid, u, w[u]);
      }
      TileIter nx = it;  // prefetch the next tile's words behind this tile's steps
      const bool okn = nx.next(a);
      if (okn) issue(nx.s, nx.ti, nx.valid());
      // kPGroup steps per proxy fence + arrival round (NSTEP is even)
#pragma unroll
      for (int q0 = 0; q0 < NSTEP; q0 += kPGroup) {
#pragma unroll
        for (int q = q0; q < q0 + kPGroup; ++q) {
          const uint32_t gq = g + (q - q0);
          const uint32_t st = gq % kStages, use = gq / kStages;
          if (use > 0) mbar_wait_sleep(empty + st, (use - 1) & 1);
          uint16_t* B = reinterpret_cast<uint16_t*>(stages + st * kStageBytes + kABytes);
#pragma unroll
          for (int u = 0; u < TPT; ++u) {
            const int t = p + kProdWarps * 32 * u;
            if (q >= kStages)
              B[kmaj<kTok>(t, code_at(w[u], q - kStages)) >> 1] = 0;
            else if (have_prev)
              B[kmaj<kTok>(t, code_at(wp[u], q - kStages + NSTEP)) >> 1] = 0;
            B[kmaj<kTok>(t, code_at(w[u], q)) >> 1] = 0x3C00;  // fp16 1.0
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane < kPGroup) mbar_arrive(full + (g + lane) % kStages);
        g += kPGroup;
      }
      have_prev = true;
      it = nx;
      ok = okn;
    }
  } else if (warp == kMmaWarp) {
    // ============ tcgen05.mma issuer: the whole warp walks the schedule (so
    // descriptors stay warp-uniform), one elected lane issues ===============
    // f16 x f16 -> f32; A and B K-major in smem; M128 N256
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(kTok >> 3) << 17) | (8u << 24);
    const uint64_t adesc0 = sdesc(su32(stages), 2048, 128);
    const uint64_t bdesc0 = sdesc(su32(stages) + kABytes, 4096, 128);
    TileIter it;
    uint32_t g = 0;
    int k = 0;
    for (bool ok = it.first(a); ok; ok = it.next(a), ++k) {
      const int db = k & 1;
      if (k >= 2) {  // D buffer db was read by the epilogue of tile k-2
        mbar_wait(dempty + db, ((k - 2) >> 1) & 1);
        tc_fence_after();
      }
      for (int q = 0; q < NSTEP; ++q, ++g) {
        const uint32_t st = g % kStages, use = g / kStages;
        mbar_wait(full + st, use & 1);
        tc_fence_after();
        // descriptor start addresses advance in 16-B units
        const uint64_t ad = adesc0 + (uint64_t)(st * (kStageBytes >> 4));
        const uint64_t bd = bdesc0 + (uint64_t)(st * (kStageBytes >> 4));
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // K = 64 levels as 4 x K16
            umma_ss(tmem + db * kTok, ad + (uint64_t)(kk * (4096 >> 4)),
                    bd + (uint64_t)(kk * (8192 >> 4)), idesc, (q > 0 || kk > 0) ? 1u : 0u);
          tc_commit(empty + st);
        }
        __syncwarp();
      }
      if (elect_one()) tc_commit(dfull + db);
      __syncwarp();
    }
  } else if (tid == kLoadWarp * 32) {
    // ============ codebook loader: one 16-KiB bulk copy per step ===========
    TileIter it;
    uint32_t g = 0;
    for (bool ok = it.first(a); ok; ok = it.next(a)) {
      const uint16_t* src = a.cbtc + (size_t)(it.s % a.n_slots) * a.slot_elems;
      for (int q = 0; q < NSTEP; ++q, ++g) {
        const uint32_t st = g % kStages, use = g / kStages;
        if (use > 0) mbar_wait_sleep(empty + st, (use - 1) & 1);
        mbar_arrive_tx(full + st, kABytes);
        bulk_g2s(stages + st * kStageBytes, src + (size_t)q * (kABytes / 2), kABytes, full + st);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
}

template <int R, int G>
cudaError_t launch_tc(const TcArgs& a, cudaStream_t st) {
  const size_t sm = tc_smem_bytes(G, R);
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(k_tc_score<R, G>), sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.n_items < sms ? a.n_items : sms;
  k_tc_score<R, G><<<grid, kThreads, sm, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

size_t tc_smem_bytes(int G, int R) {
  const int nw = (2 * R * 6 + 60 + 63) / 64 + 1;  // = NW of k_tc_score<R, G>
  return (size_t)kStages * kStageBytes + kEpiSlots * 4 * kChunk * G * 4 + (size_t)kTok * nw * 8 +
         (2 * kStages + 4) * 8 + 16;
}

// the 2:4-sparse kernel is used where it applies unless the cache selected
// the dense one (CVQ_VARIANT_TC_DENSE)
static bool tc_use_sparse(const AttnJob& job) {
  return sp_supported(job.geo.R) && !(job.variant & kVarTcDense);
}

// partial-score slices per stream written by the tcgen05 score kernel (the
// sparse kernel keeps <= 11 rounds resident, so R = 21 runs as 2 parts)
int tc_blocks(const AttnJob& job) { return tc_use_sparse(job) ? sp_parts(job.geo.R) : 1; }

bool tc_half_scores(const AttnJob& job) {
  return job.cb_key_tc && tc_use_sparse(job) && !(job.variant & kVarF32W) &&
         sp_parts(job.geo.R) == 1 && job.geo.d == 128 &&
         job.geo.L == 64 && job.geo.subs == 64;
}

// per slot: the dense layout [R][2][8192], then (R = 11) the sparse kernel's
// [R][X | Y][64] blocks (attn_sp.cu)
size_t tc_codebook_elems(int R) { return (size_t)R * 2 * (kABytes / 2) + sp_codebook_elems(R); }

void tc_build_codebook(int R, const double* xy, uint16_t* out, uint16_t (*to_half)(double)) {
  // xy: [R][64 subs][64 levels][2] (rope-commutative atoms, x then y)
  for (int r = 0; r < R; ++r)
    for (int side = 0; side < 2; ++side) {
      uint16_t* o = out + ((size_t)r * 2 + side) * (kABytes / 2);
      for (int j = 0; j < 64; ++j)
        for (int l = 0; l < 64; ++l) {
          const double x = xy[(((size_t)r * 64 + j) * 64 + l) * 2];
          const double y = xy[(((size_t)r * 64 + j) * 64 + l) * 2 + 1];
          // side a: (x, y); side b: i * (x + iy) = (-y, x)
          o[kmaj<128>(2 * j, l) >> 1] = to_half(side ? -y : x);
          o[kmaj<128>(2 * j + 1, l) >> 1] = to_half(side ? x : y);
        }
    }
  if (sp_supported(R)) sp_build_codebook(R, xy, out + (size_t)R * 2 * (kABytes / 2), to_half);
}

cudaError_t run_tc_score(const AttnJob& job, const float* q, float* ps, int chunk,
                         cudaStream_t st, const HalfOut* ho) {
  const Geom& g = job.geo;
  if (!job.cb_key_tc || g.d != 128 || g.L != 64 || g.subs != 64) return cudaErrorInvalidValue;
  const size_t slot_elems = tc_codebook_elems(g.R);
  // 2:4-sparse kernel where it applies (CVQ_VARIANT_TC_DENSE keeps the dense one)
  if (tc_use_sparse(job))
    return run_sp_score(job, job.cb_key_tc + (size_t)g.R * 2 * (kABytes / 2), slot_elems, q, ps,
                        chunk, st, ho);
  if (ho) return cudaErrorInvalidValue;
  TcArgs a{};
  a.kpool = job.kpool;
  a.kstride = job.kstride;
  a.cbtc = job.cb_key_tc;
  a.slot_elems = slot_elems;
  a.n_slots = job.n_slots;
  a.q = q;
  a.thetas = job.thetas;
  a.t = job.t;
  a.pos0 = job.pos0;
  a.n = job.n;
  a.chunk = (chunk + kTok - 1) / kTok * kTok;
  a.cps = (int)((job.n + a.chunk - 1) / a.chunk);
  a.n_items = job.S * a.cps;
  a.ps = ps;
  if (g.R == 11) return g.G == 4 ? launch_tc<11, 4>(a, st) : launch_tc<11, 1>(a, st);
  if (g.R == 21) return g.G == 4 ? launch_tc<21, 4>(a, st) : launch_tc<21, 1>(a, st);
  return cudaErrorInvalidValue;
}

}  // namespace cvq
