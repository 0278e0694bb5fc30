// ref_shim.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled against the reference headers and
// sources where they lie under /root/reference/proj/core (oracle/Makefile),
// output into oracle/_ref/libcvq_ref.so.  Used to pin the C restatement
// (oracle/cvq_oracle.c), to generate tests/golden fixtures, and as the
// reference arm / cpu_baseline of bench.py.  The argument lists mirror
// cvq_oracle.h so tests can run both side by side.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "commvq/attn.hpp"
#include "commvq/cache.hpp"
#include "commvq/ctf.hpp"
#include "commvq/error.hpp"
#include "commvq/keyquant.hpp"
#include "commvq/linalg.hpp"
#include "commvq/rng.hpp"
#include "commvq/rope.hpp"
#include "commvq/valquant.hpp"

using namespace commvq;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const TrainingError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

KeyQuantConfig kqc(size_t d, size_t g, size_t L, size_t R) {
  KeyQuantConfig c;
  c.d = d;
  c.group_size = g;
  c.n_levels = L;
  c.rounds = R;
  return c;
}

KeyCodebook make_kcb(const KeyQuantConfig& c, const double* xy) {
  KeyCodebook cb = KeyCodebook::zeros(c);
  for (size_t i = 0; i < cb.atoms.size(); ++i)
    cb.atoms[i] = CommMat{xy[2 * i], xy[2 * i + 1]};
  return cb;
}

KeyCodes make_kc(const KeyQuantConfig& c, const uint16_t* a, const uint16_t* b,
                 size_t n) {
  KeyCodes kc = KeyCodes::empty(c, n);
  std::memcpy(kc.a.data(), a, kc.a.size() * 2);
  std::memcpy(kc.b.data(), b, kc.b.size() * 2);
  return kc;
}

ValueCodes make_vc(size_t n_codes, const uint8_t* bits, size_t n) {
  ValueCodes vc = ValueCodes::empty(n_codes, n);
  std::memcpy(vc.bits.data(), bits, vc.bits.size());
  return vc;
}

ValueCodebook make_vcb(size_t n_codes, size_t d, const double* rows) {
  ValueCodebook cb = ValueCodebook::zeros(n_codes, d);
  std::memcpy(cb.rows.data.data(), rows, n_codes * d * sizeof(double));
  return cb;
}

Mat make_mat(size_t r, size_t c, const double* p) {
  Mat m(r, c);
  std::memcpy(m.data.data(), p, r * c * sizeof(double));
  return m;
}

ValueEncoder make_enc(size_t d, size_t hidden, size_t n_codes,
                      const double* w1, const double* b1, const double* w2,
                      const double* b2) {
  ValueEncoder e = ValueEncoder::zeros(d, hidden, n_codes);
  std::memcpy(e.w1.data.data(), w1, d * hidden * 8);
  std::memcpy(e.b1.data(), b1, hidden * 8);
  std::memcpy(e.w2.data.data(), w2, hidden * n_codes * 8);
  std::memcpy(e.b2.data(), b2, n_codes * 8);
  return e;
}
}  // namespace

extern "C" {

const char* cvqr_last_error() { return g_err.c_str(); }

// ---- rng.hpp ------------------------------------------------------------
void* cvqr_rng_new(uint64_t seed) { return new Rng(seed); }
void cvqr_rng_free(void* r) { delete static_cast<Rng*>(r); }
void cvqr_rng_fill_normal(void* r, double* out, size_t n, double scale) {
  for (size_t i = 0; i < n; ++i) out[i] = scale * static_cast<Rng*>(r)->normal();
}
void cvqr_rng_fill_index_u16(void* r, uint16_t* out, size_t n, uint64_t bound) {
  for (size_t i = 0; i < n; ++i)
    out[i] = static_cast<uint16_t>(static_cast<Rng*>(r)->index(bound));
}
void cvqr_rng_fill_bit_u8(void* r, uint8_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i)
    out[i] = static_cast<uint8_t>(static_cast<Rng*>(r)->next_u64() & 1);
}
void cvqr_rng_fill_u64(void* r, uint64_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = static_cast<Rng*>(r)->next_u64();
}
double cvqr_rng_uniform01(void* r) { return static_cast<Rng*>(r)->uniform01(); }

// ---- attention ----------------------------------------------------------
int cvqr_fused_attention(size_t d, size_t g, size_t L, size_t R, size_t n_codes,
                         const double* atoms, const uint16_t* a,
                         const uint16_t* b, const uint8_t* bits, size_t n,
                         const double* vrows, const double* q, size_t t,
                         double base, double* out, uint64_t* predicted,
                         uint64_t* measured) {
  return guard([&] {
    KeyQuantConfig c = kqc(d, g, L, R);
    KeyCodebook kcb = make_kcb(c, atoms);
    KeyCodes kc = make_kc(c, a, b, n);
    ValueCodes vc = make_vc(n_codes, bits, n);
    ValueCodebook vcb = make_vcb(n_codes, d, vrows);
    Vec qv(q, q + d);
    RopeParams rope = RopeParams::make(d, base);
    AttnInput in{qv, t, kc, vc, kcb, vcb, rope};
    RopeTable table(rope);
    AttnResult res = fused_attention(in, table);
    std::memcpy(out, res.out.data(), d * sizeof(double));
    if (predicted) *predicted = res.flops.predicted_mults;
    if (measured) *measured = res.flops.measured_mults;
  });
}

int cvqr_naive_attention(size_t d, size_t g, size_t L, size_t R, size_t n_codes,
                         const double* atoms, const uint16_t* a,
                         const uint16_t* b, const uint8_t* bits, size_t n,
                         const double* vrows, const double* q, size_t t,
                         double base, double* out, uint64_t* predicted,
                         uint64_t* measured) {
  return guard([&] {
    KeyQuantConfig c = kqc(d, g, L, R);
    KeyCodebook kcb = make_kcb(c, atoms);
    KeyCodes kc = make_kc(c, a, b, n);
    ValueCodes vc = make_vc(n_codes, bits, n);
    ValueCodebook vcb = make_vcb(n_codes, d, vrows);
    Vec qv(q, q + d);
    RopeParams rope = RopeParams::make(d, base);
    AttnInput in{qv, t, kc, vc, kcb, vcb, rope};
    RopeTable table(rope);
    AttnResult res = naive_quantized_attention(in, table);
    std::memcpy(out, res.out.data(), d * sizeof(double));
    if (predicted) *predicted = res.flops.predicted_mults;
    if (measured) *measured = res.flops.measured_mults;
  });
}

int cvqr_reference_attention(const double* q, const double* K, const double* V,
                             size_t n, size_t d, double base, size_t t,
                             double* out) {
  return guard([&] {
    Vec qv(q, q + d);
    Vec o = reference_attention(qv, make_mat(n, d, K), make_mat(n, d, V),
                                RopeParams::make(d, base), t);
    std::memcpy(out, o.data(), d * sizeof(double));
  });
}

uint64_t cvqr_predicted_flops_fused(size_t n, size_t d, size_t nc, size_t R,
                                   size_t L) {
  uint64_t v = 0;
  if (guard([&] { v = predicted_flops_fused(n, d, nc, R, L); })) return 0;
  return v;
}
uint64_t cvqr_predicted_flops_naive(size_t n, size_t d, size_t nc) {
  uint64_t v = 0;
  if (guard([&] { v = predicted_flops_naive(n, d, nc); })) return 0;
  return v;
}

int cvqr_softmax_row(const double* v, size_t n, double* out) {
  return guard([&] {
    Vec o = softmax_row(std::span<const double>(v, n));
    std::memcpy(out, o.data(), n * sizeof(double));
  });
}

// ---- keyquant -------------------------------------------------------------
int cvqr_encode_keys(size_t d, size_t g, size_t L, size_t R,
                     const double* atoms, const double* keys, size_t n,
                     int factorized, uint16_t* a, uint16_t* b) {
  return guard([&] {
    KeyQuantConfig c = kqc(d, g, L, R);
    KeyCodebook kcb = make_kcb(c, atoms);
    KeyCodes kc = encode_keys(make_mat(n, d, keys), kcb,
                              factorized ? AssignSearch::factorized
                                         : AssignSearch::brute_force);
    std::memcpy(a, kc.a.data(), kc.a.size() * 2);
    std::memcpy(b, kc.b.data(), kc.b.size() * 2);
  });
}

int cvqr_decode_keys(size_t d, size_t g, size_t L, size_t R,
                     const double* atoms, const uint16_t* a, const uint16_t* b,
                     size_t n, double* out) {
  return guard([&] {
    KeyQuantConfig c = kqc(d, g, L, R);
    Mat m = decode_keys(make_kc(c, a, b, n), make_kcb(c, atoms));
    std::memcpy(out, m.data.data(), n * d * sizeof(double));
  });
}

// train_key_codebook (keyquant.cpp:641-703).  atoms_out: [R][d/2][L][2];
// obj_out: the hard-objective traces, round-major then group, concatenated
// (obj_len[r * groups + grp] entries each, at most obj_cap in total);
// mse_out[R]: reconstruction MSE after each round.
int cvqr_decode_values(size_t n_codes, size_t d, const double* rows, const uint8_t* bits,
                       size_t n, double* out) {
  return guard([&] {
    Mat m = decode_values(make_vc(n_codes, bits, n), make_vcb(n_codes, d, rows));
    std::memcpy(out, m.data.data(), n * d * sizeof(double));
  });
}

int cvqr_train_key_codebook(size_t d, size_t g, size_t L, size_t R, const double* calib,
                            size_t n, size_t soft_iters, size_t hard_iters_max, double t0,
                            double decay, double tol, double ridge, uint64_t seed,
                            int factorized, double* atoms_out, double* obj_out,
                            size_t obj_cap, size_t* obj_len, double* mse_out) {
  return guard([&] {
    KeyQuantConfig c = kqc(d, g, L, R);
    EmConfig em;
    em.soft_iters = soft_iters;
    em.hard_iters_max = hard_iters_max;
    em.t0 = t0;
    em.decay = decay;
    em.tol = tol;
    em.ridge = ridge;
    em.seed = seed;
    em.search = factorized ? AssignSearch::factorized : AssignSearch::brute_force;
    KeyTrainResult res = train_key_codebook(make_mat(n, d, calib), c, em);
    for (size_t i = 0; i < res.codebook.atoms.size(); ++i) {
      atoms_out[2 * i] = res.codebook.atoms[i].x;
      atoms_out[2 * i + 1] = res.codebook.atoms[i].y;
    }
    size_t k = 0;
    for (size_t r = 0; r < R; ++r) {
      const auto& rr = res.report.rounds[r];
      for (size_t grp = 0; grp < rr.hard_objective.size(); ++grp) {
        const auto& tr = rr.hard_objective[grp];
        obj_len[r * rr.hard_objective.size() + grp] = tr.size();
        for (double v : tr)
          if (k < obj_cap) obj_out[k++] = v;
      }
      mse_out[r] = rr.reconstruction_mse;
    }
  });
}

// train_value_quantizer (valquant.cpp:172-383).  Outputs as the reference's
// ValueTrainResult: w1 [d][H], b1 [H], w2 [H][C], b2 [C], cb [C][d],
// loss_curve (curve_len entries), diverged, steps_run.
int cvqr_train_value_quantizer(const double* calib, size_t n, size_t d, size_t n_codes,
                               size_t steps, size_t batch, double step_size, double t_start,
                               double t_end, size_t hidden, uint64_t seed,
                               size_t checkpoint_every, int freeze, const double* init_cb,
                               double* w1, double* b1, double* w2, double* b2, double* cb,
                               double* loss_curve, size_t* curve_len, int* diverged,
                               size_t* steps_run) {
  return guard([&] {
    ValTrainConfig cfg;
    cfg.steps = steps;
    cfg.batch = batch;
    cfg.step_size = step_size;
    cfg.gumbel_t_start = t_start;
    cfg.gumbel_t_end = t_end;
    cfg.hidden = hidden;
    cfg.seed = seed;
    cfg.checkpoint_every = checkpoint_every;
    cfg.freeze_codebook = freeze != 0;
    ValueCodebook init;
    if (init_cb) init = make_vcb(n_codes, d, init_cb);
    ValueTrainResult r =
        train_value_quantizer(make_mat(n, d, calib), n_codes, cfg, init_cb ? &init : nullptr);
    std::memcpy(w1, r.encoder.w1.data.data(), r.encoder.w1.data.size() * 8);
    std::memcpy(b1, r.encoder.b1.data(), r.encoder.b1.size() * 8);
    std::memcpy(w2, r.encoder.w2.data.data(), r.encoder.w2.data.size() * 8);
    std::memcpy(b2, r.encoder.b2.data(), r.encoder.b2.size() * 8);
    std::memcpy(cb, r.codebook.rows.data.data(), r.codebook.rows.data.size() * 8);
    std::memcpy(loss_curve, r.loss_curve.data(), r.loss_curve.size() * 8);
    *curve_len = r.loss_curve.size();
    *diverged = r.diverged ? 1 : 0;
    *steps_run = r.steps_run;
  });
}

size_t cvqr_bits_per_token(size_t d, size_t g, size_t L, size_t R) {
  return kqc(d, g, L, R).bits_per_token();
}

// ---- valquant -------------------------------------------------------------
int cvqr_encoder_forward_infer(size_t d, size_t hidden, size_t n_codes,
                               const double* w1, const double* b1,
                               const double* w2, const double* b2,
                               const double* values, size_t n, uint8_t* bits,
                               double* logits) {
  return guard([&] {
    ValueEncoder e = make_enc(d, hidden, n_codes, w1, b1, w2, b2);
    for (size_t p = 0; p < n; ++p) {
      Vec t(values + p * d, values + (p + 1) * d);
      EncoderOut o = encoder_forward(t, e, EncoderMode::infer, 1.0);
      for (size_t k = 0; k < n_codes; ++k) {
        bits[p * n_codes + k] = o.bits[k];
        if (logits) logits[p * n_codes + k] = o.logits[k];
      }
    }
  });
}

// ---- cache ----------------------------------------------------------------
int cvqr_pack_key_codes(size_t d, size_t g, size_t L, size_t R,
                        const uint16_t* a, const uint16_t* b, size_t n,
                        uint64_t* words, size_t* n_words) {
  return guard([&] {
    KeyQuantConfig c = kqc(d, g, L, R);
    std::vector<uint64_t> w = pack_key_codes(make_kc(c, a, b, n));
    std::memcpy(words, w.data(), w.size() * 8);
    *n_words = w.size();
  });
}
int cvqr_pack_value_codes(size_t n_codes, const uint8_t* bits, size_t n,
                          uint64_t* words, size_t* n_words) {
  return guard([&] {
    std::vector<uint64_t> w = pack_value_codes(make_vc(n_codes, bits, n));
    std::memcpy(words, w.data(), w.size() * 8);
    *n_words = w.size();
  });
}
int cvqr_unpack_key_codes(size_t d, size_t g, size_t L, size_t R,
                          const uint64_t* words, size_t n_words, size_t n,
                          uint16_t* a, uint16_t* b) {
  return guard([&] {
    KeyCodes kc = unpack_key_codes(
        std::vector<uint64_t>(words, words + n_words), n, kqc(d, g, L, R));
    std::memcpy(a, kc.a.data(), kc.a.size() * 2);
    std::memcpy(b, kc.b.data(), kc.b.size() * 2);
  });
}
int cvqr_unpack_value_codes(size_t n_codes, const uint64_t* words,
                            size_t n_words, size_t n, uint8_t* bits) {
  return guard([&] {
    ValueCodes vc = unpack_value_codes(
        std::vector<uint64_t>(words, words + n_words), n, n_codes);
    std::memcpy(bits, vc.bits.data(), vc.bits.size());
  });
}

// QuantizedKVCache driven token by token (cache.cpp:213-296): prefill or
// appends, then decode_step outputs.  out_steps: n_steps x d.
struct RefCache {
  std::shared_ptr<const KeyCodebook> kcb;
  std::shared_ptr<const ValueCodebook> vcb;
  std::shared_ptr<const ValueEncoder> enc;
  std::unique_ptr<QuantizedKVCache> cache;
};

void* cvqr_cache_new(size_t d, size_t g, size_t L, size_t R, size_t n_codes,
                     size_t hidden, const double* atoms, const double* vrows,
                     const double* w1, const double* b1, const double* w2,
                     const double* b2) {
  RefCache* rc = new RefCache;
  int st = guard([&] {
    KeyQuantConfig c = kqc(d, g, L, R);
    rc->kcb = std::make_shared<KeyCodebook>(make_kcb(c, atoms));
    rc->vcb = std::make_shared<ValueCodebook>(make_vcb(n_codes, d, vrows));
    rc->enc = std::make_shared<ValueEncoder>(
        make_enc(d, hidden, n_codes, w1, b1, w2, b2));
    rc->cache = std::make_unique<QuantizedKVCache>(rc->kcb, rc->vcb, rc->enc);
  });
  if (st) {
    delete rc;
    return nullptr;
  }
  return rc;
}
void cvqr_cache_free(void* c) { delete static_cast<RefCache*>(c); }
int cvqr_cache_prefill(void* c, const double* K, const double* V, size_t n) {
  // QuantizedKVCache::prefill (cache.cpp:213-254) replaces the cache.
  return guard([&] {
    RefCache* rc = static_cast<RefCache*>(c);
    size_t d = rc->kcb->config.d;
    rc->cache = std::make_unique<QuantizedKVCache>(QuantizedKVCache::prefill(
        make_mat(n, d, K), make_mat(n, d, V), rc->kcb, rc->vcb, rc->enc));
  });
}
int cvqr_cache_append(void* c, const double* k, const double* v) {
  return guard([&] {
    RefCache* rc = static_cast<RefCache*>(c);
    size_t d = rc->kcb->config.d;
    rc->cache->append(Vec(k, k + d), Vec(v, v + d));
  });
}
int cvqr_cache_decode_step(void* c, const double* k, const double* v,
                           const double* q, double* out) {
  return guard([&] {
    RefCache* rc = static_cast<RefCache*>(c);
    size_t d = rc->cache->key_codebook().config.d;
    Vec o = rc->cache->decode_step(Vec(k, k + d), Vec(v, v + d), Vec(q, q + d));
    std::memcpy(out, o.data(), d * sizeof(double));
  });
}
size_t cvqr_cache_size(void* c) { return static_cast<RefCache*>(c)->cache->size(); }
size_t cvqr_cache_key_words(void* c, uint64_t* out) {
  const auto& w = static_cast<RefCache*>(c)->cache->packed_keys().words();
  if (out) std::memcpy(out, w.data(), w.size() * 8);
  return w.size();
}
size_t cvqr_cache_value_words(void* c, uint64_t* out) {
  const auto& w = static_cast<RefCache*>(c)->cache->packed_values().words();
  if (out) std::memcpy(out, w.data(), w.size() * 8);
  return w.size();
}

// ---- ctf ------------------------------------------------------------------
int cvqr_gen_synth(size_t n, size_t d, size_t rank, uint64_t seed, double* out) {
  return guard([&] {
    Mat m = gen_synth(n, d, rank, seed);
    std::memcpy(out, m.data.data(), n * d * sizeof(double));
  });
}

// ---- CPU baseline: fused_attention over independent q-head calls ----------
// Builds n_streams random streams of n tokens (codes as acceptance.cpp:77-100,
// atoms 0.3*N(0,1), value rows N(0,1)/16) and times n_calls fused_attention
// calls (q-head calls; call c reads stream c / q_per_stream) spread over
// n_threads std::threads sharing one pre-grown RopeTable (read-only).
// Returns wall seconds of the timed region in *seconds.
int cvqr_bench_fused(size_t d, size_t g, size_t L, size_t R, size_t n_codes,
                     size_t n, size_t n_streams, size_t q_per_stream,
                     size_t n_calls, size_t n_threads, uint64_t seed,
                     double* seconds, double* checksum) {
  return guard([&] {
    KeyQuantConfig c = kqc(d, g, L, R);
    Rng rng(seed);
    KeyCodebook kcb = KeyCodebook::zeros(c);
    for (CommMat& m : kcb.atoms) m = comm_mat(0.3 * rng.normal(), 0.3 * rng.normal());
    ValueCodebook vcb = ValueCodebook::zeros(n_codes, d);
    for (double& v : vcb.rows.data) v = rng.normal() / 16.0;
    std::vector<KeyCodes> kcs;
    std::vector<ValueCodes> vcs;
    for (size_t s = 0; s < n_streams; ++s) {
      KeyCodes kc = KeyCodes::empty(c, n);
      for (auto& v : kc.a) v = static_cast<uint16_t>(rng.index(L));
      for (auto& v : kc.b) v = static_cast<uint16_t>(rng.index(L));
      ValueCodes vc = ValueCodes::empty(n_codes, n);
      for (auto& bb : vc.bits) bb = rng.next_u64() & 1;
      kcs.push_back(std::move(kc));
      vcs.push_back(std::move(vc));
    }
    std::vector<Vec> qs(n_calls, Vec(d));
    for (auto& q : qs)
      for (double& v : q) v = rng.normal();
    RopeParams rope = RopeParams::make(d);
    RopeTable table(rope);
    table.ensure(n);
    std::vector<double> sums(n_threads, 0.0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (size_t w = 0; w < n_threads; ++w) {
      th.emplace_back([&, w] {
        for (size_t call = w; call < n_calls; call += n_threads) {
          size_t s = (call / q_per_stream) % n_streams;
          AttnInput in{qs[call], n - 1, kcs[s], vcs[s], kcb, vcb, rope};
          AttnResult r = fused_attention(in, table);
          sums[w] += r.out[0];
        }
      });
    }
    for (auto& t : th) t.join();
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    double cs = 0.0;
    for (double s : sums) cs += s;
    *checksum = cs;
  });
}

// Prefill (encode + pack) baseline: n tokens of gen_synth K/V for n_streams
// streams over n_threads threads.  Returns wall seconds.
int cvqr_bench_prefill(size_t d, size_t g, size_t L, size_t R, size_t n_codes,
                       size_t hidden, size_t n, size_t n_streams,
                       size_t n_threads, uint64_t seed, double* seconds) {
  return guard([&] {
    KeyQuantConfig c = kqc(d, g, L, R);
    Rng rng(seed);
    auto kcb = std::make_shared<KeyCodebook>(KeyCodebook::zeros(c));
    for (CommMat& m : kcb->atoms) m = comm_mat(0.3 * rng.normal(), 0.3 * rng.normal());
    auto vcb = std::make_shared<ValueCodebook>(ValueCodebook::zeros(n_codes, d));
    for (double& v : vcb->rows.data) v = rng.normal() / 16.0;
    auto enc = std::make_shared<ValueEncoder>(ValueEncoder::zeros(d, hidden, n_codes));
    for (double& v : enc->w1.data) v = 0.1 * rng.normal();
    for (double& v : enc->w2.data) v = 0.1 * rng.normal();
    std::vector<Mat> ks, vs;
    for (size_t s = 0; s < n_streams; ++s) {
      ks.push_back(gen_synth(n, d, 32, seed + 2 * s + 1));
      vs.push_back(gen_synth(n, d, 32, seed + 2 * s + 2));
    }
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (size_t w = 0; w < n_threads; ++w)
      th.emplace_back([&, w] {
        for (size_t s = w; s < n_streams; s += n_threads)
          QuantizedKVCache::prefill(ks[s], vs[s], kcb, vcb, enc);
      });
    for (auto& t : th) t.join();
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

}  // extern "C"
