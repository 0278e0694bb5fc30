/*
 * cvq_oracle.h -- CPU restatement of the CommVQ decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product (paper_2506_18879_b200/, libcvq_b200.so) never
 * links, imports or falls back to it.
 *
 * Every function restates one reference function, in the reference's exact
 * fp64 operation order (no FMA contraction: build with -ffp-contract=off),
 * and cites the file:line it follows under /root/reference/proj/core/.
 * Pinned against the compiled reference (oracle/_ref) and the reference's
 * own known-answer tests by tests/test_oracle_pins.py.
 */
#ifndef CVQ_ORACLE_H
#define CVQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:13-56 : mt19937_64 + hand-written distributions ---------- */
typedef struct {
  uint64_t mt[312];
  int idx;
  int has_spare;
  double spare;
} cvqo_rng;

void cvqo_rng_seed(cvqo_rng* r, uint64_t seed);
uint64_t cvqo_rng_next_u64(cvqo_rng* r);
double cvqo_rng_uniform01(cvqo_rng* r);
double cvqo_rng_normal(cvqo_rng* r);
uint64_t cvqo_rng_index(cvqo_rng* r, uint64_t n);
/* bulk helpers (ctypes friendly) */
cvqo_rng* cvqo_rng_new(uint64_t seed);
void cvqo_rng_free(cvqo_rng* r);
void cvqo_rng_fill_normal(cvqo_rng* r, double* out, size_t n, double scale);
void cvqo_rng_fill_index_u16(cvqo_rng* r, uint16_t* out, size_t n, uint64_t bound);
void cvqo_rng_fill_bit_u8(cvqo_rng* r, uint8_t* out, size_t n);
void cvqo_rng_fill_u64(cvqo_rng* r, uint64_t* out, size_t n);

/* ---- keyquant.hpp:16-28 KeyQuantConfig -------------------------------- */
typedef struct {
  size_t d, group_size, n_levels, rounds;
} cvqo_kq;

size_t cvqo_level_bits(const cvqo_kq* c);     /* keyquant.cpp:40 */
size_t cvqo_bits_per_token(const cvqo_kq* c); /* keyquant.cpp:42-44 */
int cvqo_validate(const cvqo_kq* c);          /* keyquant.cpp:46-60; 0 = ok */

/* Status codes (mirror the reference's exception classes). */
#define CVQO_OK 0
#define CVQO_EINVAL 1   /* std::invalid_argument */
#define CVQO_ETRAIN 2   /* commvq::TrainingError */
#define CVQO_ERANGE 3   /* std::out_of_range */
const char* cvqo_last_error(void);

/* ---- rope.cpp:8-25 ---------------------------------------------------- */
double cvqo_theta(size_t i, size_t d, double base);

/* ---- linalg.cpp:63-75 softmax_row (in place into out) ------------------ */
int cvqo_softmax_row(const double* v, size_t n, double* out);

/* ---- attn.cpp:125-128 reference_attention ----------------------------- */
int cvqo_reference_attention(const double* q, const double* K, const double* V,
                             size_t n, size_t d, double base, size_t t,
                             double* out);

/* Attention inputs restated from attn.hpp:31-39 (AttnInput).  Atoms are
 * interleaved (x, y) pairs in atom_index order keyquant.hpp:37-39; key codes
 * a/b in KeyCodes::idx order keyquant.hpp:57-59; value bits one byte per
 * (token, code) as ValueCodes::bits valquant.hpp:36-48; value rows
 * n_codes x d row-major. */
typedef struct {
  const cvqo_kq* kq;
  size_t n_codes;
  const double* atoms_xy;
  const uint16_t* a;
  const uint16_t* b;
  const uint8_t* bits;
  size_t n_tokens;
  const double* value_rows;
  const double* q;
  size_t t;
  double rope_base;
} cvqo_attn_in;

/* attn.cpp:164-263 fused_attention (+ FlopReport counts attn.cpp:176-261) */
int cvqo_fused_attention(const cvqo_attn_in* in, double* out,
                         uint64_t* predicted, uint64_t* measured);
/* same, additionally exporting the pre-softmax scores (attn.cpp:233) */
int cvqo_fused_scores(const cvqo_attn_in* in, double* scores);
/* attn.cpp:130-162 naive_quantized_attention */
int cvqo_naive_attention(const cvqo_attn_in* in, double* out,
                         uint64_t* predicted, uint64_t* measured);
/* attn.cpp:265-280 cost models (0 on invalid input) */
uint64_t cvqo_predicted_flops_naive(size_t n, size_t d, size_t n_codes);
uint64_t cvqo_predicted_flops_fused(size_t n, size_t d, size_t n_codes,
                                    size_t rounds, size_t n_levels);

/* ---- keyquant.cpp:705-739 encode_keys (brute force, 180-200) ---------- */
int cvqo_encode_keys(const cvqo_kq* kq, const double* atoms_xy,
                     const double* keys, size_t n, uint16_t* a, uint16_t* b);
/* keyquant.cpp:204-224 factorized search variant (ranking oracle) */
int cvqo_encode_keys_factorized(const cvqo_kq* kq, const double* atoms_xy,
                                const double* keys, size_t n, uint16_t* a,
                                uint16_t* b);
/* keyquant.cpp:741-768 decode_keys */
int cvqo_decode_keys(const cvqo_kq* kq, const double* atoms_xy,
                     const uint16_t* a, const uint16_t* b, size_t n,
                     double* out);

/* ---- valquant.cpp:50-101 encoder_forward, infer mode, batched --------- */
int cvqo_encoder_forward_infer(size_t d, size_t hidden, size_t n_codes,
                               const double* w1, const double* b1,
                               const double* w2, const double* b2,
                               const double* values, size_t n, uint8_t* bits,
                               double* logits /* may be NULL */);
/* valquant.cpp:115-128 decode_values */
int cvqo_decode_values(size_t n_codes, size_t d, const double* rows,
                       const uint8_t* bits, size_t n, double* out);

/* ---- cache.cpp:54-155 bit packing ------------------------------------- */
size_t cvqo_words_for_bits(uint64_t bits);
int cvqo_pack_key_codes(const cvqo_kq* kq, const uint16_t* a, const uint16_t* b,
                        size_t n, uint64_t* words /* words_for_bits(n*bpt) */);
int cvqo_unpack_key_codes(const cvqo_kq* kq, const uint64_t* words,
                          size_t n_words, size_t n, uint16_t* a, uint16_t* b);
int cvqo_pack_value_codes(size_t n_codes, const uint8_t* bits, size_t n,
                          uint64_t* words);
int cvqo_unpack_value_codes(size_t n_codes, const uint64_t* words,
                            size_t n_words, size_t n, uint8_t* bits);

/* ---- ctf.cpp:97-144 gen_synth (synthetic low-rank K/V) ---------------- */
int cvqo_gen_synth(size_t n, size_t d, size_t rank, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
