// attn_sp.cu -- 2:4-sparse tcgen05 score kernel for the 1-bit head preset
// (R = 11 rounds, 64 levels, d = 128, one key group).  The key decode is the
// same one-hot GEMM as attn_tc.cu, turned so the one-hot is the A operand:
//
//   D[t, n] += A_{r,s}[t, l] * B_r[n, l]     (M = 128 tokens, N = 64, K = 64)
//
// A one-hot row has a single non-zero per 64 levels, so it is 2:4 sparse and
// runs on tcgen05.mma.sp (K = 32 logical per instruction, half the physical
// MACs of a dense K = 32).  Measured on B200 (profiles/r01_umma_sparse_*):
// sparse M128 x N64 with A in TMEM issues every 32 clk from ONE thread with
// warp-uniform operands, twice the dense rate, and a 64-row B slice (4 KiB
// per K = 32) is exactly the 128 B/clk the tensor core reads from smem.
//
// * B_r = the round-r codebook as two 64-row blocks, X (rows j: U[r,j,l].x)
//   and Y (rows 64 + j: U[r,j,l].y), K-major fp16 -- 16 KiB per round, all
//   11 rounds RESIDENT in smem (176 KiB; reloaded only when a CTA's stream
//   changes codebook slot).  Nothing is re-streamed per tile.
// * D = [Re K | Im K] (2 x 64 fp32 columns).  Side a adds X into Re and Y
//   into Im; side b (K += i U[b]) adds -Y into Re (instruction-descriptor
//   negate-A) and X into Im: 4 MMAs (N = 64) per (round, side, K-half).
// * A = compressed one-hot in TMEM (lane = token): per K = 32 half, 8
//   columns of fp16 pairs, group g = (c & 31) / 4 holds 1.0 in slot c & 1;
//   the metadata column selects index pair (0,1) or (2,3) from bit 1 of c
//   -- one column per (round, side); its lane L = m0 + 8 k1 + 16 m2 holds
//   K-half k1 of rows m0 + 16 m2 (low 16 bits) and m0 + 8 + 16 m2 (high).
//   16 producer warps, 4 per TMEM lane quarter (thread = token), take the
//   rounds by global round index g = sub (mod 4); 6 round stages (both
//   sides: 32 + 2 metadata columns).  A producer publishes a stage with a
//   hardware named barrier (bar.arrive, ids 5-10), not an mbarrier: every
//   shared-memory access of the issuer waits behind the tensor core's B
//   reads (~100-200 clk), a named barrier does not.
// * Two issuer warps take alternate global rounds (one's stage wait overlaps
//   the other's MMAs).  Each round is ONE predicated asm block of 8 .ws.sp
//   MMAs + the commit that frees its stage (sp_issue_round).  The round-0
//   issuer of a tile zeroes D and releases the other through a named barrier.
// * D double-buffered (TMEM columns 0-255); epilogue = 8 warps, warp
//   (quarter, e2) owns tokens [32 quarter, +32) x subspaces [32 e2, +32) in
//   two 16-subspace passes: z = E[lane][j] K_j with the per-lane phase table
//   E = e^{+i lane theta_j}, score_h += Re(w_hj z) where w_hj = conj(q_hj)
//   e^{-i(t - p0 - 32 quarter) theta_j} / sqrt(d) is per warp (fp64-based at a
//   work item's first tile, advanced by e^{+i 128 theta_j} per tile); a
//   2-warp smem sum per quarter.  Output: fp32 partial scores per round part
//   (R = 21 runs as 2 parts), or -- one part, the default -- fp16 weights
//   exp(s - m32) with the max m32 of each 32-token group per head
//   (k_fast_value<PH> rescales them; half the bytes of fp32 scores).
//   Round-2 measurements of these choices: DESIGN.md section 4 and
//   profiles/r02_*.
//
// * CTA pairs (CVQ_VARIANT_TC_PAIR, experimental, off by default): clusters of 2
//   with tcgen05 cta_group::2 -- one MMA covers 256 tokens x N = 128. Each
//   CTA keeps half of B: rank 0 P = X, Q = Y; rank 1 P = Y, Q = -X, so side a
//   is [X ; Y] over the P halves and side b is -[Y ; -X] over the Q halves
//   (negate-A).  Producers of both CTAs arrive on the leader's stage
//   mbarriers, the leader's commits multicast to both; one issuer.  Exact
//   (same parity tests), but slower than the single-CTA kernel at C3
//   (DESIGN.md section 4).
//
// Codebook precision fp16 (as CVQ_CACHE_KEYS_FP16), accumulation fp32.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "cvq_internal.cuh"

namespace cvq {

namespace {

#ifdef SP_TRACE
// clock64 trace of CTA 0 over tiles [kTrK0, kTrK0 + 4) (tools/sp_trace.py)
__device__ long long g_sptr[8192];
#ifndef SP_TRACE_K0
#define SP_TRACE_K0 20
#endif
constexpr int kTrK0 = SP_TRACE_K0;
#define SPTR(idx) \
  do { if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) g_sptr[(idx)] = clock64(); } while (0)
#define TRK(k) ((k) >= kTrK0 && (k) < kTrK0 + 4)
// layout: MMA afull wait begin/end [tile][round]: 0 / 64; dempty begin/end
// [tile]: 128 / 136; dfull commit 144; producer (quarter, sub) wait
// begin/end/arrive [q][tile][round]: 256 / 512 / 768 (q*64 + tile*16 + r);
// epilogue warp w: dfull wait begin/end, release, end [w][tile]: 1024 + w*16 + 4*f + tile
#else
#define SPTR(idx) do {} while (0)
#define TRK(k) false
#endif
#ifdef CVQ_DEVICE_CHECKS
// Debug build (CVQ_NVCC_EXTRA=-DCVQ_DEVICE_CHECKS): the stage / D-buffer
// protocol is checked with sequence tags in shared memory and every global
// access is bounds-checked; a violation traps (the launch fails with
// cudaErrorLaunchFailure).  Stands in for compute-sanitizer racecheck, which
// this GPU pool does not offer.
#define SP_CHECK(cond) \
  do { if (!(cond)) asm volatile("trap;"); } while (0)
#else
#define SP_CHECK(cond) do {} while (0)
#endif
constexpr int kTok = 128;                 // tokens per tile (MMA M)
constexpr int kEpiWarps = 8;              // warp (quarter, e2): subspaces [32 e2, +32) in 2 passes
constexpr int kProdWarps = 16;            // 4 per lane quarter, global rounds g = sub (mod 4)
constexpr int kProdPerQ = 4;
constexpr int kEpiPerQ = kEpiWarps / 4;    // epilogue warps per lane quarter
constexpr int kSubsPerEpi = 64 / kEpiPerQ; // subspaces per epilogue warp
constexpr int kMmaWarp = kEpiWarps + kProdWarps;  // MMA issuer + codebook loader
#ifndef CVQ_SP_ISSUERS
#define CVQ_SP_ISSUERS 2
#endif
constexpr int kIssuers = CVQ_SP_ISSUERS;  // warps kMmaWarp, kMmaWarp + 1 issue alternate rounds
// 1 issuer: C3 score kernel 11.38 ms vs 10.69 with 2 (same-box A/B).  More
// than 2 would let an issuer sync a stage / zero named barrier of a later
// generation while another still owes the current one (measured: hangs).
static_assert(kIssuers == 1 || kIssuers == 2, "issuer warps");
constexpr int kThreads = (kMmaWarp + kIssuers) * 32;
// named barriers (bar.sync ids): 1-4 the epilogue's per-quarter reduction,
// 5-10 the A stages (producers arrive, the round's issuer syncs), 11-12 the
// "D zeroed" handoff between the issuers per D buffer, 13 codebook reloaded
constexpr int kBarStage0 = 5, kBarZero0 = 11, kBarCodebook = 13;
constexpr int kAStages = 6;               // round stages: both sides of one round (32 + 4 metadata columns)
constexpr uint32_t kACol0 = 256;          // round stage st: side s at columns 256 + 32 st + 16 s
constexpr uint32_t kMetaCol0 = kACol0 + 32 * kAStages;  // its metadata: column kMetaCol0 + 4 st + 2 s
constexpr int kRoundBytes = 128 * 64 * 2;  // 16 KiB [X; Y] x 64 levels
constexpr int kRPart = 11;                // rounds resident per CTA (176 KiB); 2-bit = 2 parts
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
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
#ifdef CVQ_SP_SUSPEND
  // try_wait with a suspend-time hint: the warp is parked by the hardware
  // until the phase completes (or the hint expires) instead of re-issuing a
  // poll + nanosleep loop that competes for issue slots
  uint32_t ok;
  do {
    asm volatile(
        "{.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;}"
        : "=r"(ok)
        : "r"(su32(bar)), "r"(parity), "r"((uint32_t)CVQ_SP_SUSPEND)
        : "memory");
  } while (!ok);
#else
  while (!mbar_try(bar, parity)) __nanosleep(64);
#endif
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
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// D[tmem] (+)= A[a_tmem] (2:4 compressed, metadata at e_tmem) x B[b_desc]
__device__ __forceinline__ void umma_sp_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                           uint32_t accum, uint32_t e) {
  asm volatile(
      "{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(accum), "r"(e));
}
// arrive on the mbarrier at the same smem offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];}" ::"r"(su32(bar)),
      "r"(cta)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// CTA-pair MMA (M = 256: 128 token rows of A in each CTA's TMEM, half of the
// N rows of B in each CTA's smem), issued by the leader CTA only
__device__ __forceinline__ void umma_sp_ts_pair(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                                uint32_t accum, uint32_t e) {
  asm volatile(
      "{.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [%1], %2, [%5], %3, p;}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(accum), "r"(e));
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {  // arrives in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(su32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ float2 ffma2(float2 a, float b, float2 c) {
  uint64_t d;
  asm("{.reg .b64 a, b, c;\n\tmov.b64 a, {%1, %2};\n\tmov.b64 b, {%3, %3};\n\t"
      "mov.b64 c, {%4, %5};\n\tfma.rn.f32x2 %0, a, b, c;}"
      : "=l"(d)
      : "f"(a.x), "f"(a.y), "f"(b), "f"(c.x), "f"(c.y));
  return make_float2(__uint_as_float((uint32_t)d), __uint_as_float((uint32_t)(d >> 32)));
}

// One round of the resident-codebook schedule as ONE asm block: elect.sync,
// 8 predicated sparse MMAs (sides a/b x K halves x Re/Im blocks) and the
// commit that frees the round's A stage.  No branch, so ptxas emits
// @UP-predicated UTCHMMAs with no BSSY/BSYNC reconvergence (a BSYNC waits on
// the UTCHMMA scoreboards, i.e. drains the MMA queue, ~200 clk per region;
// tools/umma_pred_bench.cu).  The MMAs are weight-stationary (.ws) with B
// collector buffers: a round reads only 4 distinct B slices (X_h, Y_h per K
// half h) and each is read from smem once (fill on side a, lastuse on side
// b) instead of twice -- half of the smem bandwidth the B operand took
// (bit-identical to plain .sp, tools/umma_ws_probe.cu).
//   side a: Re += X (rows 0-63), Im += Y (rows 64-127)
//   side b: Re -= Y (negate-A), Im += X;  K half h at +8 A columns, +4 x 2048 B
__device__ __forceinline__ void sp_issue_round(uint32_t d, uint32_t a, uint32_t e, uint64_t br,
                                               uint32_t idesc, uint32_t accum, uint64_t* bar) {
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
      "@q tcgen05.mma.ws.sp.cta_group::1.kind::f16.collector::b2::lastuse [d1], [a3], b2, [e1], %4, t;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];}" ::"r"(d),
      "r"(a), "r"(e), "l"(br), "r"(idesc), "r"(accum), "r"(idesc | (1u << 13)), "r"(su32(bar))
      : "memory");
}
// commit to `bar` from one elected lane, branch-free
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(su32(bar))
      : "memory");
}

// Byte offset of (row, level) in the K-major no-swizzle 128 x 64 fp16 round
// block: core matrix (level / 8, row / 8) at ((level / 8) * 16 + row / 8) * 128.
__host__ __device__ __forceinline__ uint32_t kmaj128(int row, int l) {
  return (uint32_t)((((l >> 3) * 16 + (row >> 3)) << 7) + ((row & 7) << 4) + ((l & 7) << 1));
}

struct SpArgs {
  const uint64_t* kpool;
  uint64_t kstride;
  const uint16_t* cb;    // slot s: cb + s * slot_elems = [R][128 x 64] fp16 B blocks
  size_t slot_elems;
  int n_slots;
  const float* q;        // [S][G][128]
  const double* thetas;
  long long t, pos0, n;
  int chunk;             // tokens per work item (multiple of 2 kTok)
  int cps;               // work items per (stream, round part)
  int n_items;
  int rtot;              // rounds of the preset (11, 21)
  int js;                // round parts of <= RP rounds (scores are linear in K)
  float* ps;             // [S][js][n][G] partial scores
  size_t ps_elems;       // its extent (device bounds checks)
  // half-weight mode (js == 1): ph[S][nps][G] = fp16 exp(s - m32) and
  // m32[S][nps / 32][G] per 32-token group instead of ps
  __half* ph;
  float* m32;
  long long nps;
};

// This CTA's tiles in order; each CTA owns a contiguous range of work items
// (so consecutive items mostly share a stream and its codebook slot).
template <bool PAIR>
struct SpIter {
  // a CTA pair walks 256-token pair tiles; CTA `rank` takes tokens
  // [ti + 128 rank, +128) of each
  static constexpr int kStep = PAIR ? 2 * kTok : kTok;
  int item, end, s, part, r0, nr;  // stream, round part, its first round and round count
  long long ti, hi;
  bool item_start;
  int rank;
  __device__ bool first(const SpArgs& a) {
    rank = PAIR ? (int)(blockIdx.x & 1) : 0;
    const int units = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
    const int per = a.n_items / units, rem = a.n_items % units;
    const int b = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
    item = b * per + min(b, rem);
    end = item + per + (b < rem ? 1 : 0);
    return setup(a);
  }
  __device__ bool setup(const SpArgs& a) {
    while (item < end) {
      s = item / (a.cps * a.js);
      part = (item / a.cps) % a.js;
      r0 = part * kRPart;
      nr = min(kRPart, a.rtot - r0);
      ti = (long long)(item % a.cps) * a.chunk;
      hi = min(a.n, ti + a.chunk);
      item_start = true;
      if (ti < hi) return true;
      ++item;
    }
    return false;
  }
  __device__ bool next(const SpArgs& a) {
    ti += kStep;
    item_start = false;
    if (ti < hi) return true;
    ++item;
    return setup(a);
  }
  __device__ long long base() const { return ti + (long long)rank * kTok; }
  // tokens of this CTA in the tile (0 for the second CTA of a short last tile)
  __device__ int valid() const { return (int)max(0ll, min((long long)kTok, hi - base())); }
};

// PAIR: CTA pairs (cluster of 2) with tcgen05 cta_group::2 -- one MMA covers
// 256 tokens and N = 128 ([Re | Im] in one instruction per side), each CTA
// holding half of the B rows (attn_sp.cu header, "CTA pairs").
template <int R, int G, bool PAIR>  // R = rounds per part (kRPart)
__global__ void __launch_bounds__(kThreads, 1) k_sp_score(SpArgs a) {
  static_assert(G == 1 || G == 4, "heads per KV stream");
  static_assert(kMetaCol0 + 4 * kAStages <= kTmemCols, "TMEM columns");
  constexpr int NSTEP = 2 * R;
  constexpr int NW = (NSTEP * 6 + 63 + 63) / 64;  // raw words covering a token's record
  // the value kernel (launched with programmatic stream serialization) may
  // be scheduled onto SMs this persistent grid frees; it waits for our writes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* cbs = smem;                                             // [R][16 KiB]
  float2* etab = reinterpret_cast<float2*>(cbs + R * kRoundBytes);         // [64 j][32 lanes]
  float* wtab = reinterpret_cast<float*>(etab + 64 * 32);                 // [warp][16 j][2G]
  float* red = wtab + kEpiWarps * kSubsPerEpi * 2 * G;                     // [2][4 q][4 e][32][G]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * 16 * 32 * G);
  uint64_t* afull = bars;
  uint64_t* aempty = bars + kAStages;
  uint64_t* dfull = bars + 2 * kAStages;
  uint64_t* dempty = dfull + 2;
  uint64_t* cbfull = dempty + 2;
  uint64_t* cbempty = cbfull + 1;
  uint64_t* cbpeer = cbempty + 1;  // PAIR: the second CTA's codebook half is in
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cbpeer + 1);
  // protocol tags (CVQ_DEVICE_CHECKS): producers' round per (stage, quarter),
  // the issued round per stage, the tile per D buffer
  uint32_t* stag = tmem_slot + 4;       // [kAStages][4]
  uint32_t* itag = stag + 4 * kAStages;  // [kAStages]
  uint32_t* dtag = itag + kAStages;      // [2]
  const uint32_t rank = PAIR ? cluster_rank() : 0u;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == kMmaWarp) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (tid == 0) {
    for (int i = 0; i < kAStages; ++i) {
      mbar_init(afull + i, PAIR ? 8 : 4);  // one producer warp per lane quarter (per CTA)
      mbar_init(aempty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(dfull + i, PAIR ? 1 : kIssuers);
      mbar_init(dempty + i, PAIR ? 2 * kEpiWarps : kEpiWarps);
    }
    for (int i = 0; i < 5 * kAStages + 2; ++i) stag[i] = 0xFFFFFFFFu;
    mbar_init(cbfull, 1);
    mbar_init(cbempty, PAIR ? 1 : kIssuers);
    mbar_init(cbpeer, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // per-lane phase table e^{+i lane theta_j}
  for (int e = tid; e < 64 * 32; e += kThreads) {
    const int j = e >> 5, ln = e & 31;
    double sn, cs;
    sincos((double)ln * a.thetas[j], &sn, &cs);
    etab[e] = make_float2((float)cs, (float)sn);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all();  // barriers of both CTAs initialised
  else __syncthreads();
  tc_fence_after();
  // launched with programmatic stream serialization: the prologue above (TMEM,
  // barriers, the fp64 phase table) overlapped the previous kernel; the codes,
  // queries and codebooks it may have written are read only from here on
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef CVQ_SP_TMEM0
  // the CTA owns all 512 TMEM columns, so the allocation starts at lane 0,
  // column 0: a compile-time base keeps every TMEM operand address uniform
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tmem = 0u;
#else
  const uint32_t tmem = *tmem_slot;
#endif

  if (warp < kEpiWarps) {
    // ============ epilogue: lane = token 32 quarter + lane of the tile,
    // warp slot e2 = subspaces [32 e2, 32 e2 + 32) in two passes =========
    const int quarter = warp & 3, eslot = warp >> 2;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    // lane keeps the phase of subspace 32 e2 + lane and produces w for all
    // 4 heads (G = 4) or the one head (G = 1)
    const int jl = eslot * 32 + lane;
    const double theta = a.thetas[jl];
    float2 step;
    {
      double sn, cs;
      sincos((double)SpIter<PAIR>::kStep * theta, &sn, &cs);  // e^{+i step theta}: one tile later
      step = make_float2((float)cs, (float)sn);
    }
    float* wt = wtab + warp * (kSubsPerEpi * 2 * G);
    const float sc = 0.08838834764831845f;  // 1 / sqrt(128)
    float2 ph = make_float2(1.f, 0.f);
    float2 qv[G];  // this lane's subspace of every head's query, / sqrt(d)
#pragma unroll
    for (int u = 0; u < G; ++u) qv[u] = make_float2(0.f, 0.f);
    SpIter<PAIR> it;
    int k = 0;
    for (bool ok = it.first(a); ok; ok = it.next(a), ++k) {
      const int db = k & 1;
      if (it.item_start) {
        ph = phase_neg(a.t - (a.pos0 + it.base() + 32 * quarter), theta);
        const float* qs = a.q + (size_t)it.s * G * 128;
#pragma unroll
        for (int h = 0; h < G; ++h)
          qv[h] = make_float2(__ldg(qs + h * 128 + 2 * jl) * sc, __ldg(qs + h * 128 + 2 * jl + 1) * sc);
      } else {
        ph = make_float2(ph.x * step.x - ph.y * step.y, ph.x * step.y + ph.y * step.x);
      }
      // w = conj(q) ph; stored as (w.x, -w.y) so Re(w z) = w.x z.x + (-w.y) z.y
      {
        float o[2 * G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
          o[u] = qv[u].x * ph.x + qv[u].y * ph.y;
          o[G + u] = -(qv[u].x * ph.y - qv[u].y * ph.x);
        }
        if constexpr (G == 4) {  // [j][h pair]: (wx_h0, wx_h1, -wy_h0, -wy_h1), (.. h2, h3)
          reinterpret_cast<float4*>(wt)[lane * 2] = make_float4(o[0], o[1], o[4], o[5]);
          reinterpret_cast<float4*>(wt)[lane * 2 + 1] = make_float4(o[2], o[3], o[6], o[7]);
        } else {
          reinterpret_cast<float2*>(wt)[lane] = make_float2(o[0], o[1]);
        }
      }
      __syncwarp();
      if (TRK(k)) SPTR(1024 + warp * 16 + 0 + (k - kTrK0));
      mbar_wait_sleep(dfull + db, (k >> 1) & 1);
      if (!PAIR) SP_CHECK(*(volatile uint32_t*)(dtag + db) == (uint32_t)k);
      if (TRK(k)) SPTR(1024 + warp * 16 + 4 + (k - kTrK0));
      tc_fence_after();
      {
      float* rb = red + (size_t)((db * 4 + quarter) * 2) * 32 * G;  // [e2][lane][G]
      float2 acc01 = make_float2(0.f, 0.f), acc23 = make_float2(0.f, 0.f);
      float acc1 = 0.f;
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        uint32_t re[16], im[16];
        tmem_ld16(tmem + lane_base + db * 128 + eslot * 32 + pass * 16, re);
        tmem_ld16(tmem + lane_base + db * 128 + 64 + eslot * 32 + pass * 16, im);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (pass == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {  // D[db] is in registers: free it
            if constexpr (PAIR) mbar_arrive_cluster(dempty + db, 0);
            else mbar_arrive(dempty + db);
          }
        }
        const float2* E = etab + (eslot * 32 + pass * 16) * 32 + lane;
        const float* wp = wt + pass * 16 * 2 * G;
#pragma unroll
#ifdef CVQ_DIAG_NOEPI  // diagnostic only (wrong scores): no epilogue math
        if (false)
#endif
        for (int jj = 0; jj < 16; ++jj) {
#ifdef CVQ_DIAG_NOSMEM  // diagnostic only (wrong scores): no E / w table loads
          const float2 ej = make_float2(__int_as_float(lane + jj), 0.5f);
#else
          const float2 ej = E[jj * 32];
#endif
          const float kr = __uint_as_float(re[jj]), ki = __uint_as_float(im[jj]);
          const float zx = ej.x * kr - ej.y * ki;
          const float zy = ej.x * ki + ej.y * kr;
          if constexpr (G == 4) {
#ifdef CVQ_DIAG_NOSMEM
            const float4 w01 = make_float4(0.1f * jj, 0.2f, 0.3f, 0.4f);
            const float4 w23 = make_float4(0.5f, 0.6f * jj, 0.7f, 0.8f);
#else
            const float4 w01 = reinterpret_cast<const float4*>(wp)[jj * 2];
            const float4 w23 = reinterpret_cast<const float4*>(wp)[jj * 2 + 1];
#endif
            acc01 = ffma2(make_float2(w01.x, w01.y), zx, acc01);
            acc01 = ffma2(make_float2(w01.z, w01.w), zy, acc01);
            acc23 = ffma2(make_float2(w23.x, w23.y), zx, acc23);
            acc23 = ffma2(make_float2(w23.z, w23.w), zy, acc23);
          } else {
            const float2 w = reinterpret_cast<const float2*>(wp)[jj];
            acc1 = fmaf(w.x, zx, acc1);
            acc1 = fmaf(w.y, zy, acc1);
          }
        }
      }
      if constexpr (G == 4)
        reinterpret_cast<float4*>(rb)[eslot * 32 + lane] = make_float4(acc01.x, acc01.y, acc23.x, acc23.y);
      else
        rb[eslot * 32 + lane] = acc1;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
      // warp e2 writes heads 2 e2, 2 e2 + 1 (G = 4) / e2 = 0 the head (G = 1)
      if (a.ph) {
        // half weights: per head the max m over this quarter's 32 tokens,
        // fp16 exp(s - m) per token (k_fast_value<PH> rescales by group)
        const int tok = 32 * quarter + lane;
        const bool valid = tok < it.valid();
        if (G == 4 || eslot == 0) {
          float pw[2] = {0.f, 0.f};
#pragma unroll
          for (int hq = 0; hq < (G == 4 ? 2 : 1); ++hq) {
            const int h = (G == 4) ? 2 * eslot + hq : 0;
            const float v = valid ? rb[(0 * 32 + lane) * G + h] + rb[(1 * 32 + lane) * G + h]
                                  : -INFINITY;
            float m = v;
#pragma unroll
            for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            pw[hq] = valid ? __expf(v - m) : 0.f;
            if (lane == 0 && m != -INFINITY) {
              const size_t gi = ((size_t)it.s * (a.nps >> 5) + ((it.base() + 32 * quarter) >> 5)) * G + h;
              SP_CHECK(gi < a.ps_elems / 32);
              a.m32[gi] = m;
            }
          }
          if (valid) {
            const size_t pi = ((size_t)it.s * a.nps + it.base() + tok) * G;
            SP_CHECK(pi + G <= a.ps_elems);
            if constexpr (G == 4)
              *reinterpret_cast<__half2*>(a.ph + pi + 2 * eslot) = __floats2half2_rn(pw[0], pw[1]);
            else
              a.ph[pi] = __float2half_rn(pw[0]);
          }
        }
      } else {
        const int tok = 32 * quarter + lane;
        if (tok < it.valid()) {
#pragma unroll
          for (int hq = 0; hq < (G == 4 ? 2 : 1); ++hq) {
            const int h = (G == 4) ? 2 * eslot + hq : 0;
            if (G == 1 && eslot != 0) break;
            const float v = rb[(0 * 32 + lane) * G + h] + rb[(1 * 32 + lane) * G + h];
            const size_t pi = (((size_t)it.s * a.js + it.part) * a.n + it.base() + tok) * G + h;
            SP_CHECK(pi < a.ps_elems);
            a.ps[pi] = v;
          }
        }
      }
      if (TRK(k)) SPTR(1024 + warp * 16 + 12 + (k - kTrK0));
      }
    }
  } else if (warp < kEpiWarps + kProdWarps) {
    // ============ one-hot producers: thread = token 32 quarter + lane; warp
    // sub = 0..3 takes the rounds with global index g = sub (mod 4) (both
    // sides), so four chains of tcgen05.st -> wait::st per lane quarter run
    // concurrently; a warp's rounds are 4 apart, fewer than the 6 stages, so
    // the aempty parity waits stay unambiguous ==========================
    const int p = warp - kEpiWarps, quarter = p & 3, sub = p >> 2;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const int t = quarter * 32 + lane;
    auto load_raw = [&](const SpIter<PAIR>& x, uint64_t* raw, uint32_t& off) {
      const uint64_t* kw = a.kpool + (size_t)x.s * a.kstride;
      // rows past the end reuse a valid token's record (the epilogue skips them)
      const int v = x.valid();
      const long long tok = v > 0 ? x.base() + (t < v ? t : 0) : x.ti;
      // this part's fields start 12 r0 bits into the token's 12 rtot-bit record
      const unsigned long long b0 = (unsigned long long)tok * (12u * a.rtot) + 12u * x.r0;
      off = (uint32_t)(b0 & 63u);
#pragma unroll
      SP_CHECK((b0 >> 6) + NW <= a.kstride);
      for (int i = 0; i < NW; ++i) raw[i] = __ldg(kw + (b0 >> 6) + i);
    };
    uint64_t raw[NW], nraw[NW];
    uint32_t off = 0, noff = 0;
    SpIter<PAIR> it;
    uint32_t gbase = 0;  // rounds of the previous tiles (stage accounting)
    bool ok = it.first(a);
    if (ok) load_raw(it, raw, off);
    const int src = (lane & 7) | (lane & 16);
    int kk = 0;
    while (ok) {
      uint64_t w[NW];  // token record at bit 0
#pragma unroll
      for (int i = 0; i < NW; ++i)
        w[i] = off ? (raw[i] >> off) | (i + 1 < NW ? raw[i + 1] << (64u - off) : 0ull) : raw[i];
      SpIter<PAIR> nx = it;
      const bool okn = nx.next(a);
      if (okn) load_raw(nx, nraw, noff);
      // this warp's rounds r = sub, sub + 2, ...: their 12-bit (a, b) fields
      // packed back to back into (pk0, pk1)
      uint64_t pk0 = 0, pk1 = 0;
      // rounds by GLOBAL round index: this warp takes g = gbase + r with
      // g % kProdPerQ == sub, so its rounds are evenly spaced across tiles
      const int rfirst = (int)((uint32_t)(sub + kProdPerQ - (int)(gbase % kProdPerQ)) % kProdPerQ);
      static_assert(kProdPerQ == 4 && R <= 12, "at most 3 rounds per producer warp and tile");
#pragma unroll
      for (int j = 0; j < 3; ++j) {  // rounds rfirst + 4 j: runtime bit offsets, no skipped rounds
        const int bit = 12 * (rfirst + 4 * j), wi = bit >> 6, sh = bit & 63;
        const uint64_t lo = wi == 0 ? w[0] : (wi == 1 ? w[1] : w[2]);
        const uint64_t hi = wi == 0 ? w[1] : (wi == 1 ? w[2] : w[3]);
        const uint64_t f = ((lo >> sh) | (sh > 52 ? hi << (64 - sh) : 0ull)) & 0xFFFull;
        pk0 |= f << (12 * j);
      }
#pragma unroll 1
      for (int r = rfirst; r < it.nr; r += kProdPerQ) {
        const uint32_t fld = (uint32_t)pk0 & 0xFFFu;
        pk0 = (pk0 >> 12) | (pk1 << 48);
        pk1 >>= 12;
        // round stage of this CTA's global round g
        const uint32_t g = gbase + (uint32_t)r, st = g % kAStages, use = g / kAStages;
        if (use > 0) {
          if (TRK(kk)) SPTR(256 + quarter * 64 + (kk - kTrK0) * 16 + r);
          mbar_wait_sleep(aempty + st, (use - 1) & 1u);  // back off: spinning takes issue slots from the MMA warp
          if (!PAIR) SP_CHECK(*(volatile uint32_t*)(itag + st) == g - kAStages);
          if (TRK(kk)) SPTR(512 + quarter * 64 + (kk - kTrK0) * 16 + r);
          tc_fence_after();
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
#ifdef CVQ_DIAG_NOPROD  // diagnostic only (wrong scores): constant codes
          const uint32_t c = (uint32_t)s2 * 5u + 7u;
#else
          const uint32_t c = (fld >> (6 * s2)) & 63u;
#endif
          uint32_t v[16];
          const uint32_t col = ((c >> 5) << 3) | ((c & 31) >> 2);
          // word col holds fp16 1.0 in slot c & 1; one compare per word pair
          const uint32_t one = (c & 1) ? 0x3C000000u : 0x00003C00u;
          const uint32_t onee = (col & 1) ? 0u : one, oneo = (col & 1) ? one : 0u;
          const uint32_t hp = col >> 1;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool hit = hp == (uint32_t)i;
            v[2 * i] = hit ? onee : 0u;
            v[2 * i + 1] = hit ? oneo : 0u;
          }
          // metadata word of TMEM lane L = m0 + 8 k1 + 16 m2 (measured,
          // profiles/r01_umma_sparse_lanemap.txt): bits [16 m1, 16 m1 + 16)
          // are the 4 group nibbles of K-half k1 for row m0 + 8 m1 + 16 m2.
          // Every group of a row uses pair (2,3) / (0,1) from bit 1 of c.
          const uint32_t hb = (c >> 1) & 1u;
          const uint32_t ba = __shfl_sync(0xffffffffu, hb, src);
          const uint32_t bb = __shfl_sync(0xffffffffu, hb, src | 8);
          const uint32_t meta =
              (ba ? 0x0000EEEEu : 0x00004444u) | (bb ? 0xEEEE0000u : 0x44440000u);
          tmem_st16(tmem + lane_base + kACol0 + 32 * st + 16 * s2, v);
          tmem_st1(tmem + lane_base + kMetaCol0 + 4 * st + 2 * s2, meta);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        // hardware named barrier per stage (ids 5..10): one warp per lane
        // quarter arrives, the MMA warp syncs -- no shared-memory round trip
        // on the issuer's critical path
        if constexpr (!PAIR) {
#ifdef CVQ_DEVICE_CHECKS
          if (lane == 0) *(volatile uint32_t*)(stag + st * 4 + quarter) = g;
#endif
          asm volatile("bar.arrive %0, 160;" ::"r"(kBarStage0 + (int)st) : "memory");
        } else
        if (lane == 0) {  // (PAIR: the leader's barrier counts both CTAs' rows)
          if constexpr (PAIR) mbar_arrive_cluster(afull + st, 0);
          else mbar_arrive(afull + st);
        }
        if (TRK(kk)) SPTR(768 + quarter * 64 + (kk - kTrK0) * 16 + r);
      }
#pragma unroll
      for (int i = 0; i < NW; ++i) raw[i] = nraw[i];
      off = noff;
      gbase += (uint32_t)it.nr;
      ++kk;
      it = nx;
      ok = okn;
    }
  }
  else if (!PAIR && warp >= kMmaWarp) {
    // ============ two issuer warps: warp kMmaWarp + w issues the rounds
    // with global round index g = w (mod 2), so one warp's wait for its
    // next stage overlaps the other's MMAs.  The round-0 issuer of a tile
    // zeroes D (accumulate = 0) and releases the other warp through named
    // barrier 11 + db; both commit dfull (count 2) and cbempty (count 2);
    // warp kMmaWarp reloads the codebook, releasing the other through
    // barrier 13.
    constexpr uint32_t idesc = (1u << 2) | (1u << 4) | ((64u >> 3) << 17) | (8u << 24);
    const int me = warp - kMmaWarp;
    const uint64_t bdesc0 = sdesc(su32(cbs), 2048, 128);
    SpIter<PAIR> it;
    uint32_t nload = 0, gbase = 0;
    int k = 0, prev_slot = -1;
    for (bool ok = it.first(a); ok; ok = it.next(a), ++k) {
      const int db = k & 1;
      if (it.item_start) {
        const int slot = (it.s % a.n_slots) * a.js + it.part;
        if (slot != prev_slot) {
          if (nload > 0) {
            tc_commit_elect(cbempty);  // every MMA of this warp reading the old codebook
            if (me == 0) mbar_wait(cbempty, (nload - 1) & 1);
          }
          if (me == 0) {
            if (elect_one()) {
              const uint16_t* src = a.cb + (size_t)(it.s % a.n_slots) * a.slot_elems +
                                    (size_t)it.r0 * (kRoundBytes / 2);
              mbar_arrive_tx(cbfull, (uint32_t)it.nr * kRoundBytes);
              for (int r = 0; r < it.nr; ++r)
                bulk_g2s(cbs + r * kRoundBytes, src + (size_t)r * (kRoundBytes / 2), kRoundBytes,
                         cbfull);
            }
            __syncwarp();
            mbar_wait(cbfull, nload & 1);
            if (kIssuers > 1)
              asm volatile("bar.arrive %0, %1;" ::"r"(kBarCodebook), "r"(32 * kIssuers) : "memory");
          } else {
            asm volatile("bar.sync %0, %1;" ::"r"(kBarCodebook), "r"(32 * kIssuers) : "memory");
          }
          ++nload;
          prev_slot = slot;
        }
      }
      const int w0 = (int)(gbase % (uint32_t)kIssuers);  // issuer of round 0 of this tile
      const uint32_t dcol = tmem + (uint32_t)db * 128u;
      if (me == w0 && k >= 2) {  // D buffer db was read by the epilogue of tile k-2
        if (TRK(k)) SPTR(128 + (k - kTrK0));
        mbar_wait(dempty + db, ((k - 2) >> 1) & 1);
        if (TRK(k)) SPTR(136 + (k - kTrK0));
        tc_fence_after();
      }
#pragma unroll 1
      const int rme = (me - w0 + kIssuers) % kIssuers;  // this warp's first round
      for (int r = rme; r < it.nr; r += kIssuers) {
        const uint32_t g = gbase + (uint32_t)r, st = g % kAStages;
        if (kIssuers > 1 && r == rme && r > 0)  // D zeroed by round 0's issue
          asm volatile("bar.sync %0, %1;" ::"r"(kBarZero0 + db), "r"(32 * kIssuers) : "memory");
        if (TRK(k)) SPTR(0 + (k - kTrK0) * 16 + r);
        asm volatile("bar.sync %0, 160;" ::"r"(kBarStage0 + (int)st) : "memory");  // stage full
        if (TRK(k)) SPTR(64 + (k - kTrK0) * 16 + r);
#ifdef CVQ_DEVICE_CHECKS
        for (int q2 = 0; q2 < 4; ++q2) SP_CHECK(*(volatile uint32_t*)(stag + st * 4 + q2) == g);
        if (r == 0 && lane == 0) *(volatile uint32_t*)(dtag + db) = (uint32_t)k;
        if (lane == 0) *(volatile uint32_t*)(itag + st) = g;
        __threadfence_block();
#endif
        tc_fence_after();
        sp_issue_round(dcol, tmem + kACol0 + 32 * st, tmem + kMetaCol0 + 4 * st,
                                      bdesc0 + (uint64_t)((r * kRoundBytes) >> 4), idesc,
                                      r > 0 ? 1u : 0u, aempty + st);
        if (TRK(k)) SPTR(192 + (k - kTrK0) * 16 + r);
        if (kIssuers > 1 && r == 0)
          asm volatile("bar.arrive %0, %1;" ::"r"(kBarZero0 + db), "r"(32 * kIssuers) : "memory");
      }
      tc_commit_elect(dfull + db);
      if (TRK(k)) SPTR(144 + (k - kTrK0) + 4 * me);
      gbase += (uint32_t)it.nr;
    }
  }
  else if (PAIR && warp == kMmaWarp) {
    // ============ CTA-pair issuer (cta_group::2, leader CTA issues) ======
    // ============ tcgen05.mma.sp issuer (warp-uniform walk, elected lane) ==
    // f16 x f16 -> f32, sparse A from TMEM, B K-major in smem; M128 N64
    constexpr uint32_t idesc = (1u << 2) | (1u << 4) | ((64u >> 3) << 17) | (8u << 24);
    constexpr uint32_t kNegA = 1u << 13;
    const uint64_t bdesc0 = sdesc(su32(cbs), 2048, 128);
    SpIter<PAIR> it;
    uint32_t nload = 0, gst = 0, gph = 0;  // stage / parity of the next round
    int k = 0, prev_slot = -1;
    for (bool ok = it.first(a); ok; ok = it.next(a), ++k) {
      const int db = k & 1;
      if (it.item_start) {
        const int slot = (it.s % a.n_slots) * a.js + it.part;  // (codebook slot, round part)
        if (slot != prev_slot) {
          // (re)load the resident codebook: once every MMA reading the old
          // one has completed (rare: work items are contiguous per CTA)
          if (nload > 0) {
            // PAIR: the leader's commit arrives in both CTAs
            if (rank == 0 && elect_one()) {
              if constexpr (PAIR) tc_commit_pair(cbempty);
              else tc_commit(cbempty);
            }
            __syncwarp();
            mbar_wait(cbempty, (nload - 1) & 1);
          }
          if (elect_one()) {
            // PAIR: this CTA's half, [P | Q] per round (sp2 layout)
            const uint16_t* src = a.cb + (size_t)(it.s % a.n_slots) * a.slot_elems +
                                  (size_t)it.r0 * (PAIR ? kRoundBytes : kRoundBytes / 2);
            mbar_arrive_tx(cbfull, (uint32_t)it.nr * kRoundBytes);
            for (int r = 0; r < it.nr; ++r)
              bulk_g2s(cbs + r * kRoundBytes,
                       src + (PAIR ? (size_t)r * kRoundBytes + rank * (kRoundBytes / 2)
                                   : (size_t)r * (kRoundBytes / 2)),
                       kRoundBytes, cbfull);
          }
          __syncwarp();
          mbar_wait(cbfull, nload & 1);
          if constexpr (PAIR) {
            if (rank == 1) {
              if (lane == 0) mbar_arrive_cluster(cbpeer, 0);
            } else {
              mbar_wait(cbpeer, nload & 1);
            }
          }
          ++nload;
          prev_slot = slot;
        }
      }
      if constexpr (PAIR) {
        if (rank != 0) continue;  // the peer CTA only loads its codebook half
        if (TRK(k)) SPTR(128 + (k - kTrK0));
        if (k >= 2) {  // D buffer db was read by both CTAs' epilogues of tile k-2
          mbar_wait(dempty + db, ((k - 2) >> 1) & 1);
          tc_fence_after();
        }
        if (TRK(k)) SPTR(136 + (k - kTrK0));
        // M = 256 (both CTAs' tokens), N = 128: side a = [X ; Y] (P halves),
        // side b = -[Y ; -X] (Q halves, negate-A) -> [Re | Im] of every token
        constexpr uint32_t idesc2 = (1u << 2) | (1u << 4) | ((128u >> 3) << 17) | (16u << 24);
        const uint64_t pdesc0 = sdesc(su32(cbs), 1024, 128);
        const uint32_t dcol = tmem + (uint32_t)db * 128u;
#pragma unroll 1
        for (int r = 0; r < it.nr; r += 2) {
          const bool two = r + 1 < it.nr;
          const uint32_t st0 = gst, ph0 = gph;
          uint32_t st1 = gst + 1, ph1 = gph;
          if (st1 == kAStages) {
            st1 = 0;
            ph1 ^= 1u;
          }
          if (TRK(k)) SPTR(0 + (k - kTrK0) * 16 + r);
          mbar_wait(afull + st0, ph0);
          if (TRK(k)) SPTR(64 + (k - kTrK0) * 16 + r);
          if (two) mbar_wait(afull + st1, ph1);
          if (TRK(k) && two) SPTR(64 + (k - kTrK0) * 16 + r + 1);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (u == 1 && !two) break;
              const uint32_t st = u ? st1 : st0;
              const uint64_t pr = pdesc0 + (uint64_t)(((r + u) * kRoundBytes) >> 4);
#pragma unroll
              for (int s2 = 0; s2 < 2; ++s2) {
                const uint32_t a_tm = tmem + kACol0 + 32 * st + 16 * s2;
                const uint32_t e_tm = tmem + kMetaCol0 + 4 * st + 2 * s2;
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  umma_sp_ts_pair(dcol, a_tm + h * 8,
                                  pr + (uint64_t)((s2 * (kRoundBytes / 2) + h * 4 * 1024) >> 4),
                                  idesc2 | (s2 ? kNegA : 0u),
                                  (u > 0 || s2 > 0 || h > 0 || r > 0) ? 1u : 0u, e_tm);
              }
              tc_commit_pair(aempty + st);
            }
          }
          __syncwarp();
          gst += two ? 2u : 1u;
          if (gst >= kAStages) {
            gst -= kAStages;
            gph ^= 1u;
          }
        }
        if (elect_one()) tc_commit_pair(dfull + db);
        __syncwarp();
        if (TRK(k)) SPTR(144 + (k - kTrK0));
      }
    }
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all();  // the leader's MMAs into this CTA's TMEM are done
  else __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) {
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(kTmemCols));
  }
}

size_t sp_smem(int G, int R) {
  return (size_t)R * kRoundBytes + 64 * 32 * 8 + (size_t)kEpiWarps * kSubsPerEpi * 2 * G * 4 +
         (size_t)2 * 16 * 32 * G * 4 + (2 * kAStages + 7) * 8 + 16 + (5 * kAStages + 2) * 4;
}

template <int R, int G, bool PAIR>
cudaError_t launch_sp(const SpArgs& a, cudaStream_t st) {
  const size_t sm = sp_smem(G, R);
  const void* fn = reinterpret_cast<const void*>(k_sp_score<R, G, PAIR>);
  cudaError_t e = ensure_dyn_smem(fn, sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if constexpr (PAIR) {
    // clusters of 2 CTAs (an SM pair each); one work-item range per pair
    const int pairs = a.n_items < sms / 2 ? a.n_items : sms / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_sp_score<R, G, PAIR>, a);
  } else {
    const int grid = a.n_items < sms ? a.n_items : sms;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_sp_score<R, G, PAIR>, a);
  }
  count_launch();
  return e;
}

}  // namespace

#ifdef SP_TRACE
}  // namespace cvq
extern "C" __attribute__((visibility("default"))) int cvq_debug_sp_trace(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, cvq::g_sptr, sizeof(long long) * (size_t)n);
}
namespace cvq {
#endif
bool sp_supported(int R) { return R == 11 || R == 21; }

int sp_parts(int R) { return (R + kRPart - 1) / kRPart; }

// per slot: the single-CTA layout [R][X | Y][64] (R x 8192 fp16), then the
// CTA-pair layout [R][rank][P | Q][64 rows x 64 levels] (R x 16384 fp16):
// rank 0 holds P = X, Q = Y; rank 1 holds P = Y, Q = -X, so the pair MMA over
// the P halves is [X ; Y] and, negated, over the Q halves [-Y ; X].
size_t sp_codebook_elems(int R) {
  return sp_supported(R) ? (size_t)R * (kRoundBytes / 2) + (size_t)R * kRoundBytes : 0;
}

// (row, level) of a K-major no-swizzle 64 x 64 fp16 block
static uint32_t kmaj64(int row, int l) {
  return (uint32_t)((((l >> 3) * 8 + (row >> 3)) << 7) + ((row & 7) << 4) + ((l & 7) << 1));
}

void sp_build_codebook(int R, const double* xy, uint16_t* out, uint16_t (*to_half)(double)) {
  // xy: [R][64 subs][64 levels][2]; out: [R][X rows 0-63 | Y rows 64-127][64 levels]
  uint16_t* pair = out + (size_t)R * (kRoundBytes / 2);
  for (int r = 0; r < R; ++r) {
    uint16_t* o = out + (size_t)r * (kRoundBytes / 2);
    uint16_t* p0 = pair + (size_t)r * kRoundBytes;  // rank 0: P, Q
    uint16_t* p1 = p0 + kRoundBytes / 2;            // rank 1: P, Q
    for (int j = 0; j < 64; ++j)
      for (int l = 0; l < 64; ++l) {
        const double x = xy[(((size_t)r * 64 + j) * 64 + l) * 2];
        const double y = xy[(((size_t)r * 64 + j) * 64 + l) * 2 + 1];
        o[kmaj128(j, l) >> 1] = to_half(x);
        o[kmaj128(64 + j, l) >> 1] = to_half(y);
        p0[kmaj64(j, l) >> 1] = to_half(x);
        p0[4096 + (kmaj64(j, l) >> 1)] = to_half(y);
        p1[kmaj64(j, l) >> 1] = to_half(y);
        p1[4096 + (kmaj64(j, l) >> 1)] = to_half(-x);
      }
  }
}


cudaError_t run_sp_score(const AttnJob& job, const uint16_t* cb, size_t slot_elems,
                         const float* q, float* ps, int chunk, cudaStream_t st,
                         const HalfOut* ho) {
  // cb: slot 0's single-CTA layout; the pair layout follows it (sp_build_codebook)
  const bool pair = (job.variant & kVarTcPair) != 0;
  const Geom& g = job.geo;
  if (!cb || g.d != 128 || g.L != 64 || g.subs != 64 || !sp_supported(g.R))
    return cudaErrorInvalidValue;
  SpArgs a{};
  a.kpool = job.kpool;
  a.kstride = job.kstride;
  a.cb = pair ? cb + (size_t)job.geo.R * (kRoundBytes / 2) : cb;
  a.slot_elems = slot_elems;
  a.n_slots = job.n_slots;
  a.q = q;
  a.thetas = job.thetas;
  a.t = job.t;
  a.pos0 = job.pos0;
  a.n = job.n;
  // work items: up to 64 tiles (8192 tokens), fewer when the job is small so
  // every SM gets >= 4 items (load balance within one item); a CTA's items
  // are contiguous, so small items add no codebook reloads
  (void)chunk;
  {
    const long long step = pair ? 2 * kTok : kTok;
    const long long tiles = (long long)job.S * sp_parts(g.R) * ((job.n + step - 1) / step);
    const long long units = pair ? 74 : 148;
    const long long ct = std::max(1ll, std::min(64ll, tiles / (4 * units)));
    a.chunk = (int)(ct * step);
  }
  a.cps = (int)((job.n + a.chunk - 1) / a.chunk);
  a.rtot = g.R;
  a.js = sp_parts(g.R);
  a.n_items = job.S * a.js * a.cps;
  a.ps = ps;
  a.ps_elems = (size_t)job.S * sp_parts(g.R) * (size_t)job.n * g.G;
  if (ho) {
    if (a.js != 1 || ho->nps < job.n || ho->nps % kTok) return cudaErrorInvalidValue;
    a.ph = static_cast<__half*>(ho->ph);
    a.m32 = ho->m32;
    a.nps = ho->nps;
    a.ps_elems = (size_t)job.S * ho->nps * g.G;
  }
  if (pair) {
    if (g.G == 4) return launch_sp<kRPart, 4, true>(a, st);
    if (g.G == 1) return launch_sp<kRPart, 1, true>(a, st);
  } else {
    if (g.G == 4) return launch_sp<kRPart, 4, false>(a, st);
    if (g.G == 1) return launch_sp<kRPart, 1, false>(a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace cvq
