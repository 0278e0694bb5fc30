// commvq_gpu.hpp -- C++ drop-in adapter over libcvq_b200.so (include/cvq.h).
//
// Callers of the reference library commvq_core switch by namespace:
//
//   commvq::fused_attention(in, table)       ->  commvq::gpu::fused_attention(in, table)
//   commvq::naive_quantized_attention(...)   ->  commvq::gpu::naive_quantized_attention(...)
//   commvq::encode_keys(keys, cb)            ->  commvq::gpu::encode_keys(keys, cb)
//   commvq::encoder_forward(t, enc, infer,.) ->  commvq::gpu::encoder_forward(...)
//   commvq::pack_key_codes(...) & friends    ->  commvq::gpu::pack_key_codes(...)
//   commvq::QuantizedKVCache                 ->  commvq::gpu::QuantizedKVCache
//
// Types are the reference's own public types (attn.hpp, keyquant.hpp,
// valquant.hpp, cache.hpp), so this header is compiled with the reference's
// include directory on the path; it adds no symbols to commvq_core and the
// two can be linked into one binary (tests/cpp/parity.cpp does exactly that).
// Preconditions and exception types mirror the reference functions cited
// below; numerics run on the B200 (no CPU fallback).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "commvq/attn.hpp"
#include "commvq/cache.hpp"
#include "commvq/error.hpp"
#include "commvq/keyquant.hpp"
#include "commvq/valquant.hpp"
#include "cvq.h"

namespace commvq {
namespace gpu {

inline void check(cvq_status s) {
  if (s == CVQ_OK) return;
  const std::string msg = cvq_last_error();
  switch (s) {
    case CVQ_EINVAL: throw std::invalid_argument(msg);
    case CVQ_ETRAINING: throw TrainingError(msg);
    case CVQ_ERANGE: throw std::out_of_range(msg);
    case CVQ_EIO: throw IoError(msg);
    default: throw std::runtime_error("libcvq_b200: " + msg);
  }
}

// One context per thread on device 0 (calls on a context are serialised).
inline cvq_context* context() {
  struct Holder {
    cvq_context* c = nullptr;
    ~Holder() { cvq_context_destroy(c); }
  };
  thread_local Holder h;
  if (!h.c) check(cvq_context_create(0, nullptr, &h.c));
  return h.c;
}

inline cvq_key_config key_config(const KeyQuantConfig& c) {
  return cvq_key_config{static_cast<uint32_t>(c.d), static_cast<uint32_t>(c.group_size),
                        static_cast<uint32_t>(c.n_levels), static_cast<uint32_t>(c.rounds)};
}

inline std::vector<double> atoms_xy(const KeyCodebook& cb) {
  std::vector<double> xy(2 * cb.atoms.size());
  for (size_t i = 0; i < cb.atoms.size(); ++i) {
    xy[2 * i] = cb.atoms[i].x;
    xy[2 * i + 1] = cb.atoms[i].y;
  }
  return xy;
}

// validate_input (attn.cpp:91-110), including the RopeTable check.
inline void validate(const AttnInput& in, const RopeTable& table) {
  const KeyQuantConfig& kc = in.key_codebook.config;
  const size_t n = in.key_codes.tokens;
  if (n == 0) throw std::invalid_argument("attention: empty cache");
  if (in.value_codes.tokens != n)
    throw std::invalid_argument("attention: key/value token counts differ");
  if (in.t + 1 < n) throw std::invalid_argument("attention: query position precedes cache");
  if (in.q.size() != kc.d || in.value_codebook.d != kc.d || in.rope.d != kc.d)
    throw std::invalid_argument("attention: dimension mismatch");
  if (in.value_codes.n_codes != in.value_codebook.n_codes)
    throw std::invalid_argument("attention: value codes/codebook mismatch");
  if (in.key_codes.rounds != kc.rounds || in.key_codes.groups != kc.groups() ||
      in.key_codes.n_levels != kc.n_levels)
    throw std::invalid_argument("attention: key codes/codebook mismatch");
  if (table.params().d != kc.d)
    throw std::invalid_argument("attention: rope table dimension mismatch");
}

inline AttnResult attend(const AttnInput& in, RopeTable& table, bool naive) {
  validate(in, table);
  const KeyQuantConfig& kc = in.key_codebook.config;
  const cvq_key_config ck = key_config(kc);
  const std::vector<double> xy = atoms_xy(in.key_codebook);
  AttnResult r;
  r.out.assign(kc.d, 0.0);
  cvq_flop_report fl{};
  const uint32_t nc = static_cast<uint32_t>(in.value_codebook.n_codes);
  if (naive)
    check(cvq_naive_attention(context(), &ck, nc, xy.data(), in.key_codes.a.data(),
                              in.key_codes.b.data(), in.key_codes.tokens,
                              in.value_codes.bits.data(), in.value_codebook.rows.data.data(),
                              in.q.data(), in.t, in.rope.base, r.out.data(), &fl));
  else
    check(cvq_fused_attention(context(), &ck, nc, xy.data(), in.key_codes.a.data(),
                              in.key_codes.b.data(), in.key_codes.tokens,
                              in.value_codes.bits.data(), in.value_codebook.rows.data.data(),
                              in.q.data(), in.t, in.rope.base, r.out.data(), nullptr, &fl));
  r.flops.pathway = naive ? "naive" : "fused";
  r.flops.tokens = in.key_codes.tokens;
  r.flops.d = kc.d;
  r.flops.n_codes = in.value_codebook.n_codes;
  r.flops.rounds = kc.rounds;
  r.flops.n_levels = kc.n_levels;
  r.flops.predicted_mults = fl.predicted_mults;
  r.flops.measured_mults = fl.measured_mults;
  return r;
}

// attn.hpp:62 / attn.cpp:164-263.  The RopeTable is not read (phases are
// formed on the device from fp64-reduced angles) but its dimension is
// checked as the reference does.
inline AttnResult fused_attention(const AttnInput& in, RopeTable& table) {
  return attend(in, table, false);
}

// attn.hpp:56 / attn.cpp:130-162.
inline AttnResult naive_quantized_attention(const AttnInput& in, RopeTable& table) {
  return attend(in, table, true);
}

// keyquant.hpp:135-136 / keyquant.cpp:705-739.  Each AssignSearch value
// reproduces the reference's own search bit for bit: brute_force the exact
// sequential distances (180-200), factorized the base - 2 pu - 2 pv ranking
// (204-224) -- they can pick differently on fp64 near-ties, as the
// reference's do.
inline KeyCodes encode_keys(const Mat& keys, const KeyCodebook& cb,
                            AssignSearch search = AssignSearch::brute_force) {
  cb.config.validate();
  if (keys.cols != cb.config.d) throw std::invalid_argument("encode_keys: keys width != d");
  KeyCodes codes = KeyCodes::empty(cb.config, keys.rows);
  if (keys.rows == 0) return codes;
  const cvq_key_config ck = key_config(cb.config);
  const std::vector<double> xy = atoms_xy(cb);
  check(cvq_encode_keys_search(context(), &ck, xy.data(), keys.data.data(), keys.rows,
                               search == AssignSearch::factorized ? 1 : 0, codes.a.data(),
                               codes.b.data()));
  return codes;
}

// keyquant.hpp:137 / keyquant.cpp:741-768: dense keys, bit-identical.
inline Mat decode_keys(const KeyCodes& codes, const KeyCodebook& cb) {
  const KeyQuantConfig& cfg = cb.config;
  if (codes.rounds != cfg.rounds || codes.groups != cfg.groups() ||
      codes.n_levels != cfg.n_levels)
    throw std::invalid_argument("decode_keys: codes do not match codebook");
  Mat out(codes.tokens, cfg.d);
  if (codes.tokens == 0) return out;
  const cvq_key_config ck = key_config(cfg);
  const std::vector<double> xy = atoms_xy(cb);
  check(cvq_decode_keys(context(), &ck, xy.data(), codes.a.data(), codes.b.data(), codes.tokens,
                        out.data.data()));
  return out;
}

// valquant.hpp:67 / valquant.cpp:115-128: dense values, bit-identical.
inline Mat decode_values(const ValueCodes& codes, const ValueCodebook& cb) {
  if (codes.n_codes != cb.n_codes)
    throw std::invalid_argument("decode_values: codes do not match codebook");
  Mat out(codes.tokens, cb.d);
  if (codes.tokens == 0 || cb.d == 0) return out;
  check(cvq_decode_values(context(), (uint32_t)cb.n_codes, (uint32_t)cb.d, cb.rows.data.data(),
                          codes.bits.data(), codes.tokens, out.data.data()));
  return out;
}

// keyquant.hpp:131-133: the soft-to-hard EM schedule with device E-steps
// (train.cu); bit-identical to the reference on the golden cases.
inline KeyTrainResult train_key_codebook(const Mat& calib_keys, const KeyQuantConfig& config,
                                         const EmConfig& em = {}) {
  config.validate();
  if (calib_keys.cols != config.d)
    throw std::invalid_argument("train_key_codebook: calib width != d");
  const cvq_key_config ck = key_config(config);
  cvq_em_config ce{em.soft_iters, em.hard_iters_max, em.t0, em.decay, em.tol, em.ridge, em.seed,
                   em.search == AssignSearch::factorized ? 1 : 0};
  const size_t groups = config.groups();
  std::vector<double> xy(config.rounds * (config.d / 2) * config.n_levels * 2);
  std::vector<double> obj(config.rounds * groups * (em.hard_iters_max + 2));
  std::vector<uint64_t> olen(config.rounds * groups);
  std::vector<double> mse(config.rounds);
  check(cvq_train_key_codebook(context(), &ck, calib_keys.data.data(), calib_keys.rows, &ce,
                               xy.data(), obj.data(), obj.size(), olen.data(), mse.data()));
  KeyTrainResult res{KeyCodebook::zeros(config), {}};
  for (size_t i = 0; i < res.codebook.atoms.size(); ++i)
    res.codebook.atoms[i] = CommMat{xy[2 * i], xy[2 * i + 1]};
  res.report.rounds.resize(config.rounds);
  size_t k = 0;
  for (size_t r = 0; r < config.rounds; ++r) {
    res.report.rounds[r].hard_objective.resize(groups);
    for (size_t grp = 0; grp < groups; ++grp) {
      const size_t len = static_cast<size_t>(olen[r * groups + grp]);
      res.report.rounds[r].hard_objective[grp].assign(obj.begin() + k, obj.begin() + k + len);
      k += len;
    }
    res.report.rounds[r].reconstruction_mse = mse[r];
  }
  return res;
}

// valquant.hpp:96-104: SGD on the reference's random stream (train_value.cu).
inline ValueTrainResult train_value_quantizer(const Mat& calib, size_t n_codes,
                                              const ValTrainConfig& cfg = {},
                                              const ValueCodebook* init_codebook = nullptr) {
  if (init_codebook && (init_codebook->n_codes != n_codes || init_codebook->d != calib.cols))
    throw std::invalid_argument("train_value_quantizer: init codebook shape mismatch");
  const size_t d = calib.cols, H = cfg.hidden ? cfg.hidden : 2 * n_codes;
  cvq_val_train_config c{cfg.steps,  cfg.batch, cfg.step_size, cfg.gumbel_t_start,
                         cfg.gumbel_t_end, cfg.hidden, cfg.seed, cfg.checkpoint_every,
                         cfg.freeze_codebook ? 1 : 0};
  ValueTrainResult res;
  res.encoder = ValueEncoder::zeros(d, H, n_codes);
  res.codebook = ValueCodebook::zeros(n_codes, d);
  std::vector<double> curve(cfg.steps ? cfg.steps : 1);
  uint64_t len = 0, steps_run = 0;
  int32_t diverged = 0;
  check(cvq_train_value_quantizer(
      context(), calib.data.data(), calib.rows, static_cast<uint32_t>(d),
      static_cast<uint32_t>(n_codes), &c, init_codebook ? init_codebook->rows.data.data() : nullptr,
      res.encoder.w1.data.data(), res.encoder.b1.data(), res.encoder.w2.data.data(),
      res.encoder.b2.data(), res.codebook.rows.data.data(), curve.data(), &len, &diverged,
      &steps_run));
  res.loss_curve.assign(curve.begin(), curve.begin() + static_cast<long>(len));
  res.diverged = diverged != 0;
  res.steps_run = static_cast<size_t>(steps_run);
  return res;
}

// valquant.hpp:62-64, infer mode on the device (train mode draws Gumbel
// noise from the caller's CPU Rng and is calibration, not the decode path).
inline EncoderOut encoder_forward(const Vec& t, const ValueEncoder& enc, EncoderMode mode,
                                  double temperature, Rng* = nullptr) {
  if (t.size() != enc.d) throw std::invalid_argument("encoder_forward: input size != d");
  if (!(temperature > 0.0)) throw std::invalid_argument("encoder_forward: temperature must be > 0");
  if (mode != EncoderMode::infer)
    throw std::invalid_argument("gpu::encoder_forward: only infer mode runs on the device");
  EncoderOut out;
  out.bits.resize(enc.n_codes);
  out.logits.resize(enc.n_codes);
  out.soft.resize(enc.n_codes);
  check(cvq_encoder_forward_infer(context(), static_cast<uint32_t>(enc.d),
                                  static_cast<uint32_t>(enc.hidden),
                                  static_cast<uint32_t>(enc.n_codes), enc.w1.data.data(),
                                  enc.b1.data(), enc.w2.data.data(), enc.b2.data(), t.data(), 1,
                                  out.bits.data(), out.logits.data()));
  for (size_t k = 0; k < enc.n_codes; ++k)  // valquant.cpp:96 (sigmoid of the raw logit)
    out.soft[k] = 1.0 / (1.0 + std::exp(-(out.logits[k] / temperature)));
  return out;
}

// cache.hpp:36-41.
inline std::vector<uint64_t> pack_key_codes(const KeyCodes& codes) {
  KeyQuantConfig c;
  c.d = codes.groups ? 2 * codes.groups : 2;
  c.group_size = 1;
  c.n_levels = codes.n_levels;
  c.rounds = codes.rounds;
  const cvq_key_config ck = key_config(c);
  const uint32_t bpt = cvq_bits_per_token(&ck);
  if (bpt == 0) throw std::invalid_argument("pack_key_codes: n_levels not a power of two");
  std::vector<uint64_t> w((codes.tokens * bpt + 63) / 64);
  if (codes.tokens)
    check(cvq_pack_key_codes(context(), &ck, codes.a.data(), codes.b.data(), codes.tokens,
                             w.data()));
  return w;
}

inline KeyCodes unpack_key_codes(const std::vector<uint64_t>& words, size_t tokens,
                                 const KeyQuantConfig& config) {
  config.validate();
  KeyCodes codes = KeyCodes::empty(config, tokens);
  const cvq_key_config ck = key_config(config);
  check(cvq_unpack_key_codes(context(), &ck, words.data(), words.size(), tokens,
                             codes.a.data(), codes.b.data()));
  return codes;
}

inline std::vector<uint64_t> pack_value_codes(const ValueCodes& codes) {
  std::vector<uint64_t> w((codes.tokens * codes.n_codes + 63) / 64);
  if (codes.tokens)
    check(cvq_pack_value_codes(context(), static_cast<uint32_t>(codes.n_codes),
                               codes.bits.data(), codes.tokens, w.data()));
  return w;
}

inline ValueCodes unpack_value_codes(const std::vector<uint64_t>& words, size_t tokens,
                                     size_t n_codes) {
  ValueCodes codes = ValueCodes::empty(n_codes, tokens);
  check(cvq_unpack_value_codes(context(), static_cast<uint32_t>(n_codes), words.data(),
                               words.size(), tokens, codes.bits.data()));
  return codes;
}

// CacheStats / compute_cache_stats (cache.hpp:43-58, cache.cpp:157-186):
// closed-form bookkeeping, restated so the gpu namespace is complete.
inline CacheStats compute_cache_stats(const KeyQuantConfig& key_config, size_t n_codes,
                                      size_t tokens) {
  key_config.validate();
  if (n_codes == 0) throw std::invalid_argument("cache stats: n_codes must be positive");
  CacheStats s;
  if (tokens == 0) return s;
  const size_t d = key_config.d;
  const uint64_t key_bits = static_cast<uint64_t>(tokens) * key_config.bits_per_token();
  const uint64_t value_bits = static_cast<uint64_t>(tokens) * n_codes;
  s.tokens = tokens;
  s.fp16_equivalent_bytes = static_cast<uint64_t>(tokens) * d * 2 * 2;
  s.quantized_payload_bits = key_bits + value_bits;
  s.quantized_payload_bytes = static_cast<double>(s.quantized_payload_bits) / 8.0;
  s.codebook_bytes = key_codebook_bytes(key_config) + value_codebook_bytes(n_codes, d);
  const double scalars = static_cast<double>(tokens) * d * 2;
  s.avg_bit_effective = static_cast<double>(s.quantized_payload_bits) / scalars;
  s.avg_bit_amortized = (static_cast<double>(s.quantized_payload_bits) +
                         8.0 * static_cast<double>(s.codebook_bytes)) / scalars;
  s.avg_bit_key_side = static_cast<double>(key_bits) / (static_cast<double>(tokens) * d);
  s.avg_bit_value_side = static_cast<double>(value_bits) / (static_cast<double>(tokens) * d);
  return s;
}

// Device options of the GPU cache (not in the reference API: defaulted, so
// reference call sites compile unchanged).
struct CacheOptions {
  size_t reserve = 1024;       // initial device reservation in tokens; grows on demand
  bool tensor_cores = false;   // CVQ_CACHE_KEYS_TC: tcgen05 score kernel, fp16 codebook
                               // operand (guarded, cvq_cache_key_mode), fp32 accumulate
};

// QuantizedKVCache (cache.hpp:62-113): same constructors, by-value
// prefill / load, accessors and save format as the reference; the packed
// words live in HBM (one stream) and the pools grow like the reference's
// vectors.  Accessors that return references (key_codes, value_codes,
// packed_keys, packed_values) materialise host mirrors from the device words
// on first use after a change, so the decode loop itself never copies back.
// Copyable (deep copy on the device) and movable.
class QuantizedKVCache {
 public:
  QuantizedKVCache(std::shared_ptr<const KeyCodebook> key_codebook,
                   std::shared_ptr<const ValueCodebook> value_codebook,
                   std::shared_ptr<const ValueEncoder> encoder, CacheOptions opt = {})
      : kcb_(std::move(key_codebook)), vcb_(std::move(value_codebook)), enc_(std::move(encoder)),
        opt_(opt) {
    // cache.cpp:189-212 (rope_for throws first on a null key codebook)
    if (!kcb_) throw std::invalid_argument("cache: key codebook is null");
    if (!vcb_) throw std::invalid_argument("cache: value codebook is null");
    if (!enc_) throw std::invalid_argument("cache: encoder is null");
    kcb_->config.validate();
    if (vcb_->d != kcb_->config.d) throw std::invalid_argument("cache: key/value dimension mismatch");
    if (enc_->d != kcb_->config.d || enc_->n_codes != vcb_->n_codes)
      throw std::invalid_argument("cache: encoder does not match value codebook");
    create();
  }
  ~QuantizedKVCache() {
    if (c_) cvq_cache_destroy(c_);
  }
  QuantizedKVCache(const QuantizedKVCache& o)
      : kcb_(o.kcb_), vcb_(o.vcb_), enc_(o.enc_), opt_(o.opt_) {
    create();
    const size_t n = o.size();
    if (n) {
      auto [kw, vw] = o.export_words();
      check(cvq_cache_import_stream(c_, 0, 0, 0, kw.data(), vw.data(), n, CVQ_HOST));
    }
  }
  QuantizedKVCache& operator=(const QuantizedKVCache& o) {
    if (this != &o) {
      QuantizedKVCache tmp(o);
      swap(tmp);
    }
    return *this;
  }
  QuantizedKVCache(QuantizedKVCache&& o) noexcept { swap(o); }
  QuantizedKVCache& operator=(QuantizedKVCache&& o) noexcept {
    swap(o);
    return *this;
  }

  // cache.cpp:213-254.
  static QuantizedKVCache prefill(const Mat& keys, const Mat& values,
                                  std::shared_ptr<const KeyCodebook> key_codebook,
                                  std::shared_ptr<const ValueCodebook> value_codebook,
                                  std::shared_ptr<const ValueEncoder> encoder,
                                  CacheOptions opt = {}) {
    if (keys.rows > opt.reserve) opt.reserve = keys.rows;
    QuantizedKVCache c(std::move(key_codebook), std::move(value_codebook), std::move(encoder), opt);
    if (keys.rows != values.rows)
      throw std::invalid_argument("prefill: key/value token count mismatch");
    const size_t d = c.kcb_->config.d;
    if (keys.rows > 0 && (keys.cols != d || values.cols != d))
      throw std::invalid_argument("prefill: wrong dimension");
    if (keys.rows)
      check(cvq_cache_prefill(c.c_, keys.data.data(), values.data.data(), keys.rows, CVQ_F64,
                              CVQ_HOST));
    return c;
  }

  size_t size() const {
    uint64_t n = 0;
    check(cvq_cache_length(c_, &n));
    return n;
  }

  // cache.cpp:256-285 (an encoder failure throws TrainingError at the next
  // synchronising call -- size(), decode_step, accessors -- with the cache
  // rolled back to the failed append).
  void append(const Vec& key, const Vec& value) {
    const size_t d = kcb_->config.d;
    if (key.size() != d || value.size() != d) throw std::invalid_argument("append: wrong dimension");
    check(cvq_cache_append(c_, key.data(), value.data(), CVQ_F64, CVQ_HOST));
    ++version_;
  }

  // cache.cpp:287-296.
  Vec decode_step(const Vec& key, const Vec& value, const Vec& q, FlopReport* flops = nullptr) {
    const size_t d = kcb_->config.d;
    if (q.size() != d) throw std::invalid_argument("attention: dimension mismatch");
    append(key, value);
    const size_t n = size();  // surfaces an append error before attending
    std::vector<float> qf(q.begin(), q.end()), of(d);
    check(cvq_cache_attention(c_, qf.data(), n - 1, of.data(), CVQ_HOST));
    if (flops) {  // FlopReport of the fused pathway (attn.cpp:176-178, 258-261)
      const KeyQuantConfig& kc = kcb_->config;
      flops->pathway = "fused";
      flops->tokens = n;
      flops->d = d;
      flops->n_codes = vcb_->n_codes;
      flops->rounds = kc.rounds;
      flops->n_levels = kc.n_levels;
      flops->predicted_mults = predicted_flops_fused(n, d, vcb_->n_codes, kc.rounds, kc.n_levels);
      flops->measured_mults = 2 * d + 2 * d * kc.rounds * kc.n_levels +
                              n * (kc.rounds * d + 1) + vcb_->n_codes * d;
    }
    return Vec(of.begin(), of.end());
  }

  // cache.hpp:84-89.
  const KeyCodes& key_codes() const {
    refresh();
    return key_codes_;
  }
  const ValueCodes& value_codes() const {
    refresh();
    return value_codes_;
  }
  const BitBuffer& packed_keys() const {
    refresh();
    return key_bits_;
  }
  const BitBuffer& packed_values() const {
    refresh();
    return value_bits_;
  }
  const KeyCodebook& key_codebook() const { return *kcb_; }
  const ValueCodebook& value_codebook() const { return *vcb_; }

  // cache.cpp:298-308.
  CacheStats stats() const {
    const size_t n = size();
    CacheStats s = gpu::compute_cache_stats(kcb_->config, vcb_->n_codes, n);
    if (n > 0) {
      const uint64_t actual = packed_keys().bit_size() + packed_values().bit_size();
      if (actual != s.quantized_payload_bits)
        throw std::logic_error("cache stats: payload size drifted from formula");
    }
    return s;
  }

  // GPU extras: the device words, the C handle, the effective key mode.
  std::vector<uint64_t> packed_key_words() const { return export_words().first; }
  std::vector<uint64_t> packed_value_words() const { return export_words().second; }
  cvq_cache* handle() const { return c_; }
  bool uses_tensor_cores() const {
    uint32_t f = 0;
    check(cvq_cache_key_mode(c_, &f));
    return (f & CVQ_CACHE_KEYS_TC) != 0;
  }

  // CVQC v1 (cache.cpp:310-327): magic, version, d, g, L, R, N_c, tokens,
  // key words, value words, all little-endian.
  void save(const std::string& path) const {
    auto [kw, vw] = export_words();
    const size_t n = size();
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) throw IoError("cannot open for write: " + path);
    const KeyQuantConfig& c = kcb_->config;
    put32(os, 0x43515643u);
    put32(os, 1);
    put32(os, static_cast<uint32_t>(c.d));
    put32(os, static_cast<uint32_t>(c.group_size));
    put32(os, static_cast<uint32_t>(c.n_levels));
    put32(os, static_cast<uint32_t>(c.rounds));
    put32(os, static_cast<uint32_t>(vcb_->n_codes));
    put64(os, n);
    put64(os, kw.size());
    for (uint64_t w : kw) put64(os, w);
    put64(os, vw.size());
    for (uint64_t w : vw) put64(os, w);
    if (!os) throw IoError("write failed: " + path);
  }

  // cache.cpp:329-373.
  static QuantizedKVCache load(const std::string& path, std::shared_ptr<const KeyCodebook> kcb,
                               std::shared_ptr<const ValueCodebook> vcb,
                               std::shared_ptr<const ValueEncoder> enc, CacheOptions opt = {}) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw IoError("cannot open: " + path);
    if (get32(is) != 0x43515643u) throw IoError("not a cache file: " + path);
    if (get32(is) != 1) throw IoError("unsupported cache version: " + path);
    QuantizedKVCache c(std::move(kcb), std::move(vcb), std::move(enc), opt);
    const KeyQuantConfig& cfg = c.kcb_->config;
    const uint32_t d = get32(is), g = get32(is), L = get32(is), r = get32(is), nc = get32(is);
    if (d != cfg.d || g != cfg.group_size || L != cfg.n_levels || r != cfg.rounds ||
        nc != c.vcb_->n_codes)
      throw IoError("cache config does not match provided codebooks: " + path);
    const uint64_t tokens = get64(is);
    const uint64_t nkw = get64(is);
    if (nkw != (tokens * cfg.bits_per_token() + 63) / 64)
      throw IoError("cache key payload size mismatch: " + path);
    std::vector<uint64_t> kw(nkw);
    for (auto& w : kw) w = get64(is);
    const uint64_t nvw = get64(is);
    if (nvw != (tokens * nc + 63) / 64) throw IoError("cache value payload size mismatch: " + path);
    std::vector<uint64_t> vw(nvw);
    for (auto& w : vw) w = get64(is);
    is.peek();
    if (!is.eof()) throw IoError("trailing bytes in cache file: " + path);
    try {  // BitBuffer::from_words padding check (cache.cpp:78-88)
      gpu::unpack_key_codes(kw, tokens, cfg);
      gpu::unpack_value_codes(vw, tokens, nc);
    } catch (const std::invalid_argument& e) {
      throw IoError(std::string("corrupt cache payload: ") + e.what());
    }
    if (tokens) check(cvq_cache_import_stream(c.c_, 0, 0, 0, kw.data(), vw.data(), tokens, CVQ_HOST));
    return c;
  }

 private:
  void create() {
    cvq_cache_desc d{};
    d.key = key_config(kcb_->config);
    d.n_codes = static_cast<uint32_t>(vcb_->n_codes);
    d.hidden = static_cast<uint32_t>(enc_->hidden);
    d.n_seqs = d.n_layers = d.n_kv_heads = d.q_per_kv = 1;
    d.capacity = opt_.reserve ? opt_.reserve : 1;
    d.rope_base = 10000.0;  // RopeParams::make default base (cache.cpp:47-50)
    d.flags = opt_.tensor_cores ? CVQ_CACHE_KEYS_TC : 0u;
    check(cvq_cache_create(context(), &d, &c_));
    const std::vector<double> xy = atoms_xy(*kcb_);
    check(cvq_cache_set_key_codebook(c_, 0, 0, xy.data()));
    check(cvq_cache_set_value_quantizer(c_, 0, 0, enc_->w1.data.data(), enc_->b1.data(),
                                        enc_->w2.data.data(), enc_->b2.data(),
                                        vcb_->rows.data.data()));
  }
  void swap(QuantizedKVCache& o) noexcept {
    std::swap(kcb_, o.kcb_);
    std::swap(vcb_, o.vcb_);
    std::swap(enc_, o.enc_);
    std::swap(opt_, o.opt_);
    std::swap(c_, o.c_);
    std::swap(version_, o.version_);
    std::swap(mirror_version_, o.mirror_version_);
    std::swap(n_mirrored_, o.n_mirrored_);
    std::swap(key_codes_, o.key_codes_);
    std::swap(value_codes_, o.value_codes_);
    std::swap(key_bits_, o.key_bits_);
    std::swap(value_bits_, o.value_bits_);
  }
  // host mirrors (cache.hpp:107-112) rebuilt from the device words when stale
  void refresh() const {
    const size_t n = size();
    if (mirror_version_ == version_ && key_codes_.tokens == n && n_mirrored_ == n) return;
    auto [kw, vw] = export_words();
    const KeyQuantConfig& cfg = kcb_->config;
    key_codes_ = gpu::unpack_key_codes(kw, n, cfg);
    value_codes_ = gpu::unpack_value_codes(vw, n, vcb_->n_codes);
    key_bits_ = BitBuffer::from_words(std::move(kw), n * cfg.bits_per_token());
    value_bits_ = BitBuffer::from_words(std::move(vw), n * vcb_->n_codes);
    mirror_version_ = version_;
    n_mirrored_ = n;
  }
  std::pair<std::vector<uint64_t>, std::vector<uint64_t>> export_words() const {
    const size_t n = size();
    std::vector<uint64_t> kw((n * kcb_->config.bits_per_token() + 63) / 64);
    std::vector<uint64_t> vw((n * vcb_->n_codes + 63) / 64);
    if (n) check(cvq_cache_export_stream(c_, 0, 0, 0, kw.data(), vw.data(), CVQ_HOST));
    return {std::move(kw), std::move(vw)};
  }
  static void put32(std::ostream& os, uint32_t v) {
    unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                          static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
    os.write(reinterpret_cast<const char*>(b), 4);
  }
  static void put64(std::ostream& os, uint64_t v) {
    put32(os, static_cast<uint32_t>(v));
    put32(os, static_cast<uint32_t>(v >> 32));
  }
  static uint32_t get32(std::istream& is) {
    unsigned char b[4];
    is.read(reinterpret_cast<char*>(b), 4);
    if (!is) throw IoError("cache file: truncated read");
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
  }
  static uint64_t get64(std::istream& is) {
    const uint64_t lo = get32(is);
    return lo | (uint64_t(get32(is)) << 32);
  }

  std::shared_ptr<const KeyCodebook> kcb_;
  std::shared_ptr<const ValueCodebook> vcb_;
  std::shared_ptr<const ValueEncoder> enc_;
  CacheOptions opt_;
  cvq_cache* c_ = nullptr;
  uint64_t version_ = 0;
  mutable uint64_t mirror_version_ = ~0ull;
  mutable size_t n_mirrored_ = ~size_t(0);
  mutable KeyCodes key_codes_;
  mutable ValueCodes value_codes_;
  mutable BitBuffer key_bits_;
  mutable BitBuffer value_bits_;
};

}  // namespace gpu
}  // namespace commvq
