/*
 * cvq.h -- C-ABI of the B200-native CommVQ decode hot path (libcvq_b200.so).
 *
 * Drop-in boundary for the reference library commvq_core
 * (/root/reference/proj/core).  The reference has no FFI of its own; its
 * public C++ entry points for this path are
 *
 *   fused_attention(const AttnInput&, RopeTable&)          attn.hpp:62
 *   naive_quantized_attention(...)                          attn.hpp:56
 *   encode_keys(const Mat&, const KeyCodebook&, AssignSearch) keyquant.hpp:135-136
 *   encoder_forward(const Vec&, const ValueEncoder&, infer)   valquant.hpp:62-64
 *   pack_key_codes / unpack_key_codes / pack_value_codes /
 *   unpack_value_codes                                      cache.hpp:36-41
 *   QuantizedKVCache::{prefill, append, decode_step, save, load}
 *                                                           cache.hpp:63-96
 *   predicted_flops_fused / predicted_flops_naive           attn.hpp:66-71
 *
 * Every function below replaces one of those (cited per function).  Plain C
 * types only: no torch, no C++ in the signatures.  Errors are status codes
 * mirroring the reference's exception classes (error.hpp:11-20,
 * std::invalid_argument, std::out_of_range); the message is retrievable with
 * cvq_last_error() on the calling thread.  There is no CPU fallback: every
 * numeric entry point runs sm_100a kernels and fails with CVQ_ECUDA when no
 * B200 is usable.
 *
 * Layouts (all little-endian, identical to the reference in-memory / CVQC
 * on-disk forms so callers can switch without re-encoding):
 *   key atoms   : R x (d/2) x L (x, y) pairs in atom_index order
 *                 (keyquant.hpp:37-39), fp64 like KeyCodebook::atoms
 *   key codes   : a[], b[] uint16 in KeyCodes::idx order (keyquant.hpp:57-59)
 *   value bits  : one byte per (token, code), ValueCodes::bits (valquant.hpp:36-48)
 *   packed words: BitBuffer LE bit stream, bit k at bit (k%64) of word k/64
 *                 (cache.hpp:16-31); key record per token = rounds outer,
 *                 groups inner, a then b, log2(L) bits each (cache.cpp:90-106);
 *                 value record = n_codes bits ascending (cache.cpp:137-143)
 */
#ifndef CVQ_H
#define CVQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
#define CVQ_API extern "C" __attribute__((visibility("default")))
#else
#define CVQ_API __attribute__((visibility("default")))
#endif

typedef enum cvq_status {
  CVQ_OK = 0,
  CVQ_EINVAL = 1,    /* std::invalid_argument                         */
  CVQ_ETRAINING = 2, /* commvq::TrainingError (non-finite activations) */
  CVQ_ERANGE = 3,    /* std::out_of_range                             */
  CVQ_EIO = 4,       /* commvq::IoError                               */
  CVQ_ECUDA = 5,     /* device / driver failure (no CPU fallback)     */
  CVQ_ENOMEM = 6,    /* device allocation failed                      */
  CVQ_ENCCL = 7      /* NCCL missing or a collective failed (mgpu)    */
} cvq_status;

/* KeyQuantConfig (keyquant.hpp:16-28). */
typedef struct cvq_key_config {
  uint32_t d;          /* head dim, even                   */
  uint32_t group_size; /* subspaces per code group         */
  uint32_t n_levels;   /* L, power of two, <= 65536        */
  uint32_t rounds;     /* R residual rounds                */
} cvq_key_config;

/* FlopReport (attn.hpp:16-27) counters; the GPU path reports the formula
 * values of the reference fused pathway so JSON reports match. */
typedef struct cvq_flop_report {
  uint64_t predicted_mults;
  uint64_t measured_mults;
} cvq_flop_report;

typedef struct cvq_context cvq_context;
typedef struct cvq_cache cvq_cache;

enum { CVQ_F32 = 0, CVQ_F64 = 1 };    /* element type of K/V inputs      */
enum { CVQ_DEVICE = 0, CVQ_HOST = 1 }; /* where a caller buffer lives     */

/* ------------------------------------------------------------ general */
CVQ_API const char* cvq_last_error(void);
CVQ_API int cvq_abi_version(void);
/* Number of kernel launches issued by this process so far (all contexts).
 * Used by bench.py to report gpu_launches. */
CVQ_API uint64_t cvq_launch_count(void);

/* One context = one device + one CUDA stream (cudaStream_t, may be NULL for
 * a private stream).  Calls on a context are externally serialised
 * (SURVEY.md 8b "Threading"); contexts on different devices run
 * concurrently. */
CVQ_API cvq_status cvq_context_create(int device, void* cuda_stream,
                                      cvq_context** out);
CVQ_API cvq_status cvq_context_destroy(cvq_context* ctx);
CVQ_API cvq_status cvq_context_synchronize(cvq_context* ctx);
/* The context's cudaStream_t (callers order their own streams against it). */
CVQ_API cvq_status cvq_context_stream(cvq_context* ctx, void** stream);
/* Live timing of the dominant attention kernel: when enabled, every
 * attention call brackets its main (score/decode) kernel with CUDA events on
 * the context stream; _read synchronises, returns the summed milliseconds
 * and the number of bracketed launches since the last read, and resets. */
CVQ_API cvq_status cvq_context_profile(cvq_context* ctx, int enable);
CVQ_API cvq_status cvq_context_profile_read(cvq_context* ctx, double* ms,
                                            uint64_t* launches);

/* attn.hpp:66-71 cost models (0 on invalid input, as the reference throws). */
CVQ_API uint64_t cvq_predicted_flops_fused(uint64_t n_tokens, uint64_t d,
                                           uint64_t n_codes, uint64_t rounds,
                                           uint64_t n_levels);
CVQ_API uint64_t cvq_predicted_flops_naive(uint64_t n_tokens, uint64_t d,
                                           uint64_t n_codes);
CVQ_API uint32_t cvq_bits_per_token(const cvq_key_config* kc);

/* ------------------------------------- single-stream reference mirrors */
/* All buffers are HOST memory; the call uploads, runs the sm_100a kernels
 * and downloads.  Semantics and preconditions are those of the cited
 * reference function, including the exceptions it raises. */

/* fused_attention (attn.cpp:164-263): pre-RoPE query q[d] at position t
 * against n_tokens cached tokens.  scores_out (optional, may be NULL)
 * receives the n_tokens pre-softmax scores (attn.cpp:233). */
CVQ_API cvq_status cvq_fused_attention(
    cvq_context* ctx, const cvq_key_config* kc, uint32_t n_codes,
    const double* key_atoms_xy, const uint16_t* a, const uint16_t* b,
    uint64_t n_tokens, const uint8_t* value_bits, const double* value_rows,
    const double* q, uint64_t t, double rope_base, double* out,
    double* scores_out, cvq_flop_report* flops);

/* naive_quantized_attention (attn.cpp:130-162): decode-then-attend. */
CVQ_API cvq_status cvq_naive_attention(
    cvq_context* ctx, const cvq_key_config* kc, uint32_t n_codes,
    const double* key_atoms_xy, const uint16_t* a, const uint16_t* b,
    uint64_t n_tokens, const uint8_t* value_bits, const double* value_rows,
    const double* q, uint64_t t, double rope_base, double* out,
    cvq_flop_report* flops);

/* encode_keys, brute-force semantics (keyquant.cpp:705-739 + 180-200):
 * codes are bit-identical to the reference (ties -> smallest a*L+b). */
CVQ_API cvq_status cvq_encode_keys(cvq_context* ctx, const cvq_key_config* kc,
                                   const double* key_atoms_xy,
                                   const double* keys, uint64_t n_tokens,
                                   uint16_t* a, uint16_t* b);

/* decode_keys (keyquant.hpp:137, keyquant.cpp:741-768): out[n][d] = the sum
 * over rounds of each token's cluster centres, in the reference's order
 * (fp64, no FMA; bit-identical).  a, b as cvq_encode_keys returns them.
 * CVQ_EINVAL "decode_keys: code out of range" for a code >= n_levels. */
CVQ_API cvq_status cvq_decode_keys(cvq_context* ctx, const cvq_key_config* kc,
                                   const double* key_atoms_xy, const uint16_t* a,
                                   const uint16_t* b, uint64_t n_tokens, double* out);
/* decode_values (valquant.hpp:67, valquant.cpp:115-128): out[n][d] = the sum
 * of the codebook rows whose bit is set, ascending code order (fp64;
 * bit-identical).  bits: [n][n_codes] bytes, 0 / 1; rows: [n_codes][d]. */
CVQ_API cvq_status cvq_decode_values(cvq_context* ctx, uint32_t n_codes, uint32_t d,
                                     const double* rows, const uint8_t* bits, uint64_t n_tokens,
                                     double* out);

/* encode_keys with the AssignSearch argument (keyquant.hpp:135-136):
 * search 0 = brute_force (as cvq_encode_keys), 1 = factorized -- the
 * reference's assign_factorized ranking base - 2 pu - 2 pv (keyquant.cpp:
 * 204-224) in its fp64 operation order, so codes equal the reference's for
 * that search, near-ties included (the two searches may differ there). */
CVQ_API cvq_status cvq_encode_keys_search(cvq_context* ctx, const cvq_key_config* kc,
                                          const double* key_atoms_xy, const double* keys,
                                          uint64_t n_tokens, int32_t search, uint16_t* a,
                                          uint16_t* b);

/* EmConfig (keyquant.hpp:71-80).  search: 0 = brute_force (default),
 * 1 = factorized. */
typedef struct cvq_em_config {
  uint64_t soft_iters;      /* 30 */
  uint64_t hard_iters_max;  /* 100 */
  double t0;                /* 0 = auto temperature */
  double decay;             /* 0.9 */
  double tol;               /* 1e-6 */
  double ridge;             /* -1 = auto */
  uint64_t seed;            /* 1 */
  int32_t search;
} cvq_em_config;

/* train_key_codebook (keyquant.cpp:641-703) on the GPU: the reference's
 * soft-to-hard EM schedule per (round, group), E-steps and moments on the
 * device, refit (Cholesky) on the host.  calib [n][d] fp64 host rows.
 * atoms_out [R][d/2][L][2] (CVQK order); objective_len[R * groups] receives
 * each group's hard-objective trace length and objective_out (capacity
 * objective_cap, may be NULL) the traces concatenated round-major;
 * mse_out[R] the per-round reconstruction MSE.  Errors: CVQ_EINVAL (fewer
 * than L^2 rows, non-finite input), CVQ_ETRAINING (all-zero calibration,
 * singular refit). */
CVQ_API cvq_status cvq_train_key_codebook(cvq_context* ctx, const cvq_key_config* kc,
                                          const double* calib, uint64_t n_rows,
                                          const cvq_em_config* em, double* atoms_out,
                                          double* objective_out, uint64_t objective_cap,
                                          uint64_t* objective_len, double* mse_out);

/* ValTrainConfig (valquant.hpp:76-86). */
typedef struct cvq_val_train_config {
  uint64_t steps;            /* 10000 */
  uint64_t batch;            /* 256 */
  double step_size;          /* 1e-3 */
  double gumbel_t_start;     /* 1.0 */
  double gumbel_t_end;       /* 0.1 */
  uint64_t hidden;           /* 0 -> 2 * n_codes */
  uint64_t seed;             /* 1 */
  uint64_t checkpoint_every; /* 100 */
  int32_t freeze_codebook;
} cvq_val_train_config;

/* train_value_quantizer (valquant.cpp:172-383) on the GPU: SGD with
 * straight-through Gumbel-sigmoid gradients on the reference's random
 * stream; reductions in the reference order.  calib [n][d] fp64 host rows;
 * init_codebook [n_codes][d] or NULL.  Outputs: w1 [d][H], b1 [H],
 * w2 [H][n_codes], b2 [n_codes], codebook [n_codes][d] with
 * H = hidden ? hidden : 2 n_codes; loss_curve[steps] (curve_len entries
 * written), diverged, steps_run.  Errors: CVQ_EINVAL (valquant.cpp:175-200). */
CVQ_API cvq_status cvq_train_value_quantizer(cvq_context* ctx, const double* calib,
                                             uint64_t n_rows, uint32_t d, uint32_t n_codes,
                                             const cvq_val_train_config* cfg,
                                             const double* init_codebook, double* w1, double* b1,
                                             double* w2, double* b2, double* codebook,
                                             double* loss_curve, uint64_t* curve_len,
                                             int32_t* diverged, uint64_t* steps_run);

/* encoder_forward in infer mode (valquant.cpp:50-101), batched over tokens:
 * values[n][d] -> bits[n][n_codes] (logit > 0), logits optional. */
CVQ_API cvq_status cvq_encoder_forward_infer(
    cvq_context* ctx, uint32_t d, uint32_t hidden, uint32_t n_codes,
    const double* w1, const double* b1, const double* w2, const double* b2,
    const double* values, uint64_t n_tokens, uint8_t* bits, double* logits);

/* cache.cpp:90-155 bit packing; word counts are ceil(n*bits/64). */
CVQ_API cvq_status cvq_pack_key_codes(cvq_context* ctx,
                                      const cvq_key_config* kc,
                                      const uint16_t* a, const uint16_t* b,
                                      uint64_t n_tokens, uint64_t* words);
CVQ_API cvq_status cvq_unpack_key_codes(cvq_context* ctx,
                                        const cvq_key_config* kc,
                                        const uint64_t* words, uint64_t n_words,
                                        uint64_t n_tokens, uint16_t* a,
                                        uint16_t* b);
CVQ_API cvq_status cvq_pack_value_codes(cvq_context* ctx, uint32_t n_codes,
                                        const uint8_t* bits, uint64_t n_tokens,
                                        uint64_t* words);
CVQ_API cvq_status cvq_unpack_value_codes(cvq_context* ctx, uint32_t n_codes,
                                          const uint64_t* words,
                                          uint64_t n_words, uint64_t n_tokens,
                                          uint8_t* bits);

/* ------------------------------- device-resident multi-stream cache */
/* QuantizedKVCache (cache.hpp:63-113) for a whole model: one code stream per
 * (seq, layer, kv_head), codebooks per (layer, kv_head), each stream served
 * to q_per_kv query heads (GQA).  Packed words live in HBM in the exact
 * BitBuffer layout.  position_offset is the global position of this
 * cache's first token (context sharding across GPUs). */
typedef struct cvq_cache_desc {
  cvq_key_config key;
  uint32_t n_codes;    /* value bits per token (N_c)        */
  uint32_t hidden;     /* value-encoder hidden width        */
  uint32_t n_seqs;     /* batch                             */
  uint32_t n_layers;
  uint32_t n_kv_heads;
  uint32_t q_per_kv;   /* query heads per KV stream (GQA)   */
  uint64_t capacity;   /* initial reservation (tokens/stream) */
  uint64_t position_offset;
  double rope_base;    /* RopeParams::base (rope.hpp:17)    */
  uint32_t flags;      /* CVQ_CACHE_* below                 */
} cvq_cache_desc;

/* Keep the on-chip copy of the key codebook as fp16 (x, y) pairs with fp32
 * accumulation: half the shared-memory traffic of the score kernel, output
 * error ~1e-5 at the bench's codebook scale ("precision modes").
 * Default (0): fp32 codebook. */
#define CVQ_CACHE_KEYS_FP16 1u
/* Score with the tcgen05 tensor-core kernel: the key decode as a one-hot
 * GEMM (fp16 codebook operand, fp32 accumulators in TMEM); the fastest mode
 * on B200 (bench.py default).  Same precision class as CVQ_CACHE_KEYS_FP16,
 * guarded per codebook (cvq_cache_key_mode).  Head presets (d=128, g=64,
 * L=64, R in {11, 21}, 1 or 4 query heads per KV head); other shapes run the
 * CUDA-core kernels.  Both presets use the 2:4-sparse kernel (one-hot as the
 * sparse operand); CVQ_VARIANT_TC_DENSE selects the dense kernel instead. */
#define CVQ_CACHE_KEYS_TC 2u

/* Kernel variants (cvq_cache_set_variant): cross-check and experimental
 * kernels next to the defaults.  Selected per cache by the caller (never by
 * the environment); 0 = the defaults the bench runs. */
#define CVQ_VARIANT_GENERIC 1u  /* generic kernels for every shape (no specialisation) */
#define CVQ_VARIANT_TC_DENSE 2u /* tcgen05: dense one-hot MMA instead of 2:4 sparse   */
#define CVQ_VARIANT_TC_PAIR 4u  /* tcgen05: CTA-pair (cta_group::2) sparse kernel     */
#define CVQ_VARIANT_FUSED 8u    /* fp16 codebook: one fused score+value kernel        */
/* The sparse tcgen05 kernel (R = 11) hands the value kernel fp16 softmax
 * weights exp(s - m) with one fp32 max per 32-token group per head (half the
 * bytes of fp32 scores; relative weight error <= 2^-11, output within the
 * 1e-3 bar); this bit keeps the fp32 score hand-off instead. */
#define CVQ_VARIANT_F32_WEIGHTS 16u

CVQ_API cvq_status cvq_cache_create(cvq_context* ctx, const cvq_cache_desc* d,
                                    cvq_cache** out);
CVQ_API cvq_status cvq_cache_destroy(cvq_cache* c);
/* Tokens per stream (QuantizedKVCache::size, cache.hpp:83).  Synchronises when
 * appends are unchecked, so deferred encoder errors surface here. */
CVQ_API cvq_status cvq_cache_length(const cvq_cache* c, uint64_t* n_tokens);
/* desc.capacity is an initial reservation, not a limit: appends, imports and
 * set_length grow the pools (x1.5, whole 128-token tiles) like the reference
 * cache grows its vectors (cache.cpp:256-285).  Growth moves the pools
 * (cvq_cache_pools pointers are invalidated). */
CVQ_API cvq_status cvq_cache_reserve(cvq_cache* c, uint64_t n_tokens);
CVQ_API cvq_status cvq_cache_capacity(const cvq_cache* c, uint64_t* n_tokens);
/* Appends never wait for the device: an encoder failure (non-finite logits,
 * valquant.cpp:86-87) is recorded on the device, later appends are skipped,
 * and the next synchronising call on the cache (this one, cvq_cache_length,
 * export, any host-buffer attention / decode step) returns CVQ_ETRAINING
 * with the length rolled back to the failed append -- the state the
 * reference's throwing append leaves.  Prefill checks before returning. */
CVQ_API cvq_status cvq_cache_synchronize(cvq_cache* c);
/* CVQ_VARIANT_* bits; takes effect from the next attention call. */
CVQ_API cvq_status cvq_cache_set_variant(cvq_cache* c, uint32_t variant);
/* Effective key-codebook mode (CVQ_CACHE_KEYS_* bits actually in use).  A
 * CVQ_CACHE_KEYS_TC cache whose key codebook fails the fp16 guard (an atom
 * outside the fp16 range, or sum_r max|U| > 96: the output error of the
 * fp16 operand approaches the 1e-3 bar) runs the fp32 CUDA-core kernels and
 * reports the bit cleared. */
CVQ_API cvq_status cvq_cache_key_mode(const cvq_cache* c, uint32_t* flags);

/* Codebooks for slot (layer, head); host fp64 in reference order.
 * key: R*(d/2)*L*2 doubles.  value quantizer: w1[d][hidden], b1[hidden],
 * w2[hidden][n_codes], b2[n_codes], rows[n_codes][d] (CVQV order
 * valquant.cpp:450-454).  w1..b2 may be NULL when the cache only attends
 * (codes imported), rows may not. */
CVQ_API cvq_status cvq_cache_set_key_codebook(cvq_cache* c, uint32_t layer,
                                              uint32_t head,
                                              const double* atoms_xy);
CVQ_API cvq_status cvq_cache_set_value_quantizer(
    cvq_cache* c, uint32_t layer, uint32_t head, const double* w1,
    const double* b1, const double* w2, const double* b2, const double* rows);

/* QuantizedKVCache::prefill (cache.cpp:213-254) for every stream at once:
 * K, V are [n_seqs][n_layers][n_kv_heads][n_tokens][d] of dtype CVQ_F32 or
 * CVQ_F64 in host or device memory.  Appends after the current length
 * (prefill on an empty cache == the reference prefill; on a non-empty
 * cache == sequential appends, word-identical per test_cache.cpp:155-180). */
CVQ_API cvq_status cvq_cache_prefill(cvq_cache* c, const void* K,
                                     const void* V, uint64_t n_tokens,
                                     int dtype, int where);

/* QuantizedKVCache::append (cache.cpp:256-285): one token per stream,
 * k, v are [n_seqs][n_layers][n_kv_heads][d]. */
CVQ_API cvq_status cvq_cache_append(cvq_cache* c, const void* k, const void* v,
                                    int dtype, int where);

/* Attention for every (seq, layer, q head) at query position t (global),
 * q/out are fp32 [n_seqs][n_layers][n_kv_heads*q_per_kv][d].  Requires
 * t + 1 >= position_offset + length (attn.cpp:97-98). */
CVQ_API cvq_status cvq_cache_attention(cvq_cache* c, const float* q,
                                       uint64_t t, float* out, int where);

/* naive_quantized_attention (attn.cpp:130-162) for every row: decode-then-
 * attend -- the whole cache dequantised to dense fp16 K (RoPE applied) and V
 * (512 B per token and stream at d = 128), then dense flash-decoding over
 * it.  The baseline the fused path is measured against (Table 4);
 * scratch grows to S x N x d x 4 bytes. */
CVQ_API cvq_status cvq_cache_attention_naive(cvq_cache* c, const float* q, uint64_t t,
                                             float* out, int where);

/* Split-K partial for context sharding: per row (seq, layer, q head) the
 * running max m, sum l and normalised o[d] over this cache's tokens
 * (device buffers). */
CVQ_API cvq_status cvq_cache_attention_partial(cvq_cache* c, const float* q,
                                               uint64_t t, float* m, float* l,
                                               float* o);

/* Log-sum-exp merge of n_parts partials (device buffers, part-major):
 * m,l [n_parts][rows], o [n_parts][rows][d] -> out [rows][d]. */
CVQ_API cvq_status cvq_lse_combine(cvq_context* ctx, const float* m,
                                   const float* l, const float* o,
                                   uint32_t n_parts, uint64_t rows, uint32_t d,
                                   float* out);

/* Same merge over packed per-part blocks [m (rows) | l (rows) | o (rows x d)]
 * at parts + p * rows * (d + 2): one all-gather of such blocks (the layout
 * cvq_cache_attention_partial writes when m, l, o point into one buffer)
 * feeds it directly. */
CVQ_API cvq_status cvq_lse_combine_packed(cvq_context* ctx, const float* parts,
                                          uint32_t n_parts, uint64_t rows, uint32_t d,
                                          float* out);

/* Same merge with part p's packed block at parts[p] + offset (floats), parts
 * a DEVICE array of device pointers.  The pointers may address peer GPUs'
 * memory (symmetric / IPC buffers mapped over NVLink): the combine kernel
 * then gathers the partials itself, with no separate collective. */
CVQ_API cvq_status cvq_lse_combine_ptrs(cvq_context* ctx, const float* const* parts,
                                        uint64_t offset, uint32_t n_parts, uint64_t rows,
                                        uint32_t d, float* out);

/* QuantizedKVCache::decode_step (cache.cpp:287-296): append k, v then attend
 * q at the new last position.  All buffers in `where`. */
CVQ_API cvq_status cvq_cache_decode_step(cvq_cache* c, const void* k,
                                         const void* v, int kv_dtype,
                                         const float* q, float* out, int where);

/* Shape of a cache (from its descriptor) and the context it runs on. */
typedef struct cvq_cache_shape {
  uint32_t n_seqs, n_layers, n_kv_heads, q_per_kv, d, n_codes;
  uint64_t position_offset;
} cvq_cache_shape;
CVQ_API cvq_status cvq_cache_shape_of(const cvq_cache* c, cvq_cache_shape* out);
CVQ_API cvq_context* cvq_cache_context(const cvq_cache* c);

/* ----------------------------- context sharding across GPUs */
/* Contiguous per-rank token ranges: bounds[2r], bounds[2r+1] = [lo, hi) of
 * rank r, boundaries on `align`-token tiles (128 keeps packed tiles 32-B
 * aligned); trailing ranks may be empty.  Host-only (no device needed). */
CVQ_API cvq_status cvq_shard_plan(uint64_t n_tokens, uint32_t world, uint32_t align,
                                  uint64_t* bounds);

/* One rank of a context-sharded cache: `shard` holds this rank's tokens of
 * every stream (position_offset = its first global position).  Attention =
 * partial on the shard written as one packed [m | l | o] block (520 B per
 * row at d = 128), ONE ncclAllGather of the blocks on the context stream,
 * then the LSE combine kernel.  NCCL is loaded at run time (libnccl.so.2;
 * in a torch process the copy torch loaded).  Errors: CVQ_ENCCL.
 *   cvq_mgpu_init       an initialised ncclComm_t (passed as void*) that
 *                       spans the ranks; the caller keeps ownership;
 *   cvq_mgpu_init_rank  the library creates the communicator from a unique
 *                       id (cvq_mgpu_unique_id on one rank, 128 bytes,
 *                       broadcast by the caller's bootstrap). */
typedef struct cvq_mgpu cvq_mgpu;
CVQ_API cvq_status cvq_mgpu_unique_id(void* id_out /* 128 bytes */);
CVQ_API cvq_status cvq_mgpu_init(cvq_cache* shard, void* nccl_comm, cvq_mgpu** out);
CVQ_API cvq_status cvq_mgpu_init_rank(cvq_cache* shard, const void* unique_id, int rank,
                                      int world, cvq_mgpu** out);
CVQ_API cvq_status cvq_mgpu_destroy(cvq_mgpu* g);
/* Global tokens per stream (the last shard's end). */
CVQ_API cvq_status cvq_mgpu_length(const cvq_mgpu* g, uint64_t* n_tokens);
/* Collective: every rank calls it with the same q and t; out gets the merged
 * attention of all ranks' tokens.  q/out in `where` (host: one sync). */
CVQ_API cvq_status cvq_mgpu_attention(cvq_mgpu* g, const float* q, uint64_t t, float* out,
                                      int where);
/* QuantizedKVCache::decode_step across the group (cache.cpp:287-296): the
 * last rank appends (k, v) to its shard (other ranks ignore k, v, which may
 * be NULL there), then every rank attends q at the new global position. */
CVQ_API cvq_status cvq_mgpu_decode_step(cvq_mgpu* g, const void* k, const void* v, int kv_dtype,
                                        const float* q, float* out, int where);

/* Packed-word import/export of one stream (CVQC payload, cache.cpp:310-373).
 * Import sets the stream's words for tokens [0, n_tokens); all streams must
 * be imported with the same n_tokens before attending (the cache length is
 * the last imported n_tokens).  Buffers in `where`. */
CVQ_API cvq_status cvq_cache_import_stream(cvq_cache* c, uint32_t seq,
                                           uint32_t layer, uint32_t head,
                                           const uint64_t* key_words,
                                           const uint64_t* value_words,
                                           uint64_t n_tokens, int where);
CVQ_API cvq_status cvq_cache_export_stream(const cvq_cache* c, uint32_t seq,
                                           uint32_t layer, uint32_t head,
                                           uint64_t* key_words,
                                           uint64_t* value_words, int where);

/* Raw device pools (stream-major, fixed stride in words) and length setter,
 * for callers that fill codes on the device (synthetic benchmarks, CVQC
 * bulk loads).  Streams are ordered (seq, layer, kv_head).  set_length grows
 * the pools when needed (then re-query the pointers). */
CVQ_API cvq_status cvq_cache_pools(cvq_cache* c, uint64_t** key_words,
                                   uint64_t* key_stride_words,
                                   uint64_t** value_words,
                                   uint64_t* value_stride_words);
CVQ_API cvq_status cvq_cache_set_length(cvq_cache* c, uint64_t n_tokens);

#endif /* CVQ_H */
