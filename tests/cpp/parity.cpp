// parity.cpp -- the drop-in claim, tested from C++: one binary links the
// UNMODIFIED reference library (oracle/_ref/libcvq_ref.so, built from
// /root/reference sources) and libcvq_b200.so through include/commvq_gpu.hpp,
// and runs the reference's pinned scenarios through both namespaces side by
// side (test_attn.cpp, test_keyquant.cpp, test_valquant.cpp, test_cache.cpp).
// Needs a B200.  Prints one [PASS]/[FAIL] line per check; exit code = #fails.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <memory>
#include <string>

#include "commvq/attn.hpp"
#include "commvq/cache.hpp"
#include "commvq/keyquant.hpp"
#include "commvq/rng.hpp"
#include "commvq/valquant.hpp"
#include "commvq/ctf.hpp"
#include "commvq_gpu.hpp"

using namespace commvq;

static int g_fail = 0;
static void report(bool ok, const std::string& name, const std::string& detail = "") {
  std::printf("[%s] %s %s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.c_str());
  if (!ok) ++g_fail;
}

static double rel_err(const Vec& a, const Vec& b) {  // test_attn.cpp:87-94
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / std::max(den, 1e-300));
}

static KeyCodebook rand_kcb(const KeyQuantConfig& c, Rng& r, double s = 1.0) {
  KeyCodebook cb = KeyCodebook::zeros(c);
  for (CommMat& m : cb.atoms) m = comm_mat(s * r.normal(), s * r.normal());
  return cb;
}

struct CacheFixture {  // test_cache.cpp:18-36
  KeyQuantConfig cfg{8, 2, 4, 2};
  std::shared_ptr<KeyCodebook> kcb;
  std::shared_ptr<ValueCodebook> vcb;
  std::shared_ptr<ValueEncoder> enc;
  explicit CacheFixture(uint64_t seed = 51) {
    kcb = std::make_shared<KeyCodebook>(KeyCodebook::zeros(cfg));
    Rng rng(seed);
    for (CommMat& m : kcb->atoms) m = comm_mat(rng.normal(), rng.normal());
    vcb = std::make_shared<ValueCodebook>(ValueCodebook::zeros(8, 8));
    for (double& v : vcb->rows.data) v = 0.5 * rng.normal();
    enc = std::make_shared<ValueEncoder>(ValueEncoder::zeros(8, 16, 8));
    for (double& v : enc->w1.data) v = 0.4 * rng.normal();
    for (double& v : enc->b1) v = 0.1 * rng.normal();
    for (double& v : enc->w2.data) v = 0.4 * rng.normal();
    for (double& v : enc->b2) v = 0.1 * rng.normal();
  }
};

static Mat rmat(size_t r, size_t c, uint64_t seed) {  // oracles.hpp random_mat
  Mat m(r, c);
  Rng rng(seed);
  for (double& v : m.data) v = rng.normal();
  return m;
}

struct CacheRun {
  std::vector<uint64_t> kw_pre, vw_pre, kw_inc, kw_loaded, kw_long, vw_long;
  std::vector<uint16_t> a, b, a_loaded;
  std::vector<uint8_t> bits;
  std::vector<Vec> outs;
  Vec out_long;
  CacheStats stats;
  size_t n_loaded = 0, n_long = 0;
  bool threw_dim = false, flop_tokens_ok = true, copy_ok = false;
};

// One body, any cache type with the reference's API (cache.hpp:62-113).
template <class Cache>
static CacheRun run_cache_body(const CacheFixture& fx, const std::string& tag) {
  CacheRun r;
  Mat keys = rmat(24, 8, 81), values = rmat(24, 8, 82);
  Cache pre = Cache::prefill(keys, values, fx.kcb, fx.vcb, fx.enc);
  Cache inc(fx.kcb, fx.vcb, fx.enc);
  for (size_t t = 0; t < 24; ++t)
    inc.append(Vec(keys.row(t).begin(), keys.row(t).end()),
               Vec(values.row(t).begin(), values.row(t).end()));
  r.kw_pre = pre.packed_keys().words();
  r.vw_pre = pre.packed_values().words();
  r.kw_inc = inc.packed_keys().words();
  r.a = pre.key_codes().a;
  r.b = pre.key_codes().b;
  r.bits = pre.value_codes().bits;
  try {
    inc.append(Vec(7), Vec(8));
  } catch (const std::invalid_argument&) {
    r.threw_dim = true;
  }
  Mat qk = rmat(16, 8, 91), qv = rmat(16, 8, 92), qq = rmat(16, 8, 93);
  Cache dec(fx.kcb, fx.vcb, fx.enc);
  for (size_t t = 0; t < 16; ++t) {
    FlopReport fl;
    r.outs.push_back(dec.decode_step(Vec(qk.row(t).begin(), qk.row(t).end()),
                                     Vec(qv.row(t).begin(), qv.row(t).end()),
                                     Vec(qq.row(t).begin(), qq.row(t).end()), &fl));
    r.flop_tokens_ok = r.flop_tokens_ok && fl.tokens == t + 1 && dec.size() == t + 1;
  }
  Mat sk = rmat(10, 8, 95), sv = rmat(10, 8, 96);
  r.stats = Cache::prefill(sk, sv, fx.kcb, fx.vcb, fx.enc).stats();
  const std::string path =
      (std::filesystem::temp_directory_path() / ("parity_" + tag + ".cvqc")).string();
  pre.save(path);
  Cache back = Cache::load(path, fx.kcb, fx.vcb, fx.enc);
  r.kw_loaded = back.packed_keys().words();
  r.a_loaded = back.key_codes().a;
  r.n_loaded = back.size();
  std::filesystem::remove(path);
  // copy is deep, move keeps the contents
  Cache cp = pre;
  cp.append(Vec(8, 0.25), Vec(8, -0.5));
  Cache mv = std::move(cp);
  r.copy_ok = pre.size() == 24 && mv.size() == 25 && mv.packed_keys().words().size() >= r.kw_pre.size();
  // 70,000 appends (past any initial device reservation), then one decode step
  Mat lk = rmat(70000, 8, 201), lv = rmat(70000, 8, 202);
  Cache lng(fx.kcb, fx.vcb, fx.enc);
  for (size_t t = 0; t < 70000; ++t)
    lng.append(Vec(lk.row(t).begin(), lk.row(t).end()), Vec(lv.row(t).begin(), lv.row(t).end()));
  r.n_long = lng.size();
  r.kw_long = lng.packed_keys().words();
  r.vw_long = lng.packed_values().words();
  r.out_long = lng.decode_step(Vec(8, 0.3), Vec(8, -0.2), Vec(qq.row(0).begin(), qq.row(0).end()));
  return r;
}

int main() {
  // 1. fused attention: reference vs GPU, incl. preset head shapes
  {
    Rng rng(303);
    struct S { size_t d, g, L, R, n, nc; double sc; };
    const S shapes[] = {{8, 2, 4, 2, 1024, 8, 1.0},  {64, 16, 64, 3, 4096, 32, 1.0},
                        {128, 64, 64, 11, 8192, 128, 0.3}, {128, 64, 64, 21, 4096, 256, 0.3},
                        {128, 64, 2048, 21, 64, 32, 1.0}};
    double worst = 0;
    for (const S& s : shapes) {
      KeyQuantConfig cfg{s.d, s.g, s.L, s.R};
      KeyCodebook kcb = rand_kcb(cfg, rng, s.sc);
      KeyCodes kc = KeyCodes::empty(cfg, s.n);
      for (auto& v : kc.a) v = static_cast<uint16_t>(rng.index(s.L));
      for (auto& v : kc.b) v = static_cast<uint16_t>(rng.index(s.L));
      ValueCodes vc = ValueCodes::empty(s.nc, s.n);
      for (auto& b : vc.bits) b = rng.next_u64() & 1;
      ValueCodebook vcb = ValueCodebook::zeros(s.nc, s.d);
      for (double& v : vcb.rows.data) v = rng.normal() * (s.sc < 1 ? 1.0 / 16 : 1.0);
      Vec q(s.d);
      for (double& v : q) v = rng.normal();
      RopeParams rope = RopeParams::make(s.d);
      AttnInput in{q, s.n - 1, kc, vc, kcb, vcb, rope};
      RopeTable t1(rope), t2(rope);
      AttnResult ref = commvq::fused_attention(in, t1);
      AttnResult gpu = commvq::gpu::fused_attention(in, t2);
      worst = std::max(worst, rel_err(gpu.out, ref.out));
      report(gpu.flops.to_json() == ref.flops.to_json(), "flop report json d=" + std::to_string(s.d));
    }
    report(worst <= 1e-4, "fused_attention gpu vs reference", "worst rel_err " + std::to_string(worst));
  }
  // 2. encoders bit-exact
  {
    KeyQuantConfig cfg{128, 64, 64, 11};
    Rng rng(7);
    KeyCodebook kcb = rand_kcb(cfg, rng, 0.3);
    Mat keys(200, 128);
    for (double& v : keys.data) v = rng.normal() * 0.5;
    KeyCodes ref = commvq::encode_keys(keys, kcb);
    KeyCodes gpu = commvq::gpu::encode_keys(keys, kcb);
    report(ref.a == gpu.a && ref.b == gpu.b, "encode_keys bit-exact (1bit preset, 200 tokens)");
    ValueEncoder enc = ValueEncoder::zeros(128, 256, 128);
    for (double& v : enc.w1.data) v = 0.1 * rng.normal();
    for (double& v : enc.w2.data) v = 0.1 * rng.normal();
    bool same = true;
    for (size_t i = 0; i < 50; ++i) {
      Vec t(keys.row(i).begin(), keys.row(i).end());
      EncoderOut a = commvq::encoder_forward(t, enc, EncoderMode::infer, 1.0);
      EncoderOut b = commvq::gpu::encoder_forward(t, enc, EncoderMode::infer, 1.0);
      same = same && a.bits == b.bits && a.logits == b.logits;
    }
    report(same, "encoder_forward infer bits+logits exact");
    report(commvq::pack_key_codes(ref) == commvq::gpu::pack_key_codes(gpu), "pack_key_codes words");
    report(commvq::decode_keys(ref, kcb).data == commvq::gpu::decode_keys(gpu, kcb).data,
           "decode_keys dense rows bit-exact");
    ValueCodebook vcb = ValueCodebook::zeros(128, 128);
    for (double& v : vcb.rows.data) v = rng.normal() / 16;
    ValueCodes vc = ValueCodes::empty(128, 50);
    for (uint8_t& bt : vc.bits) bt = rng.normal() > 0 ? 1 : 0;
    report(commvq::decode_values(vc, vcb).data == commvq::gpu::decode_values(vc, vcb).data,
           "decode_values dense rows bit-exact");
  }
  // 3. cache: prefill / decode_step / CVQC interop both ways
  {
    KeyQuantConfig cfg{16, 2, 16, 2};
    Rng rng(808);
    auto kcb = std::make_shared<KeyCodebook>(rand_kcb(cfg, rng));
    auto vcb = std::make_shared<ValueCodebook>(ValueCodebook::zeros(16, 16));
    for (double& v : vcb->rows.data) v = 0.5 * rng.normal();
    auto enc = std::make_shared<ValueEncoder>(ValueEncoder::zeros(16, 32, 16));
    for (double& v : enc->w1.data) v = 0.4 * rng.normal();
    for (double& v : enc->w2.data) v = 0.4 * rng.normal();
    for (double& v : enc->b1) v = 0.1 * rng.normal();
    for (double& v : enc->b2) v = 0.1 * rng.normal();
    const size_t n = 512;
    Mat keys(n, 16), values(n, 16), qs(n, 16);
    for (double& v : keys.data) v = rng.normal();
    for (double& v : values.data) v = rng.normal();
    for (double& v : qs.data) v = rng.normal();
    QuantizedKVCache ref(kcb, vcb, enc);
    gpu::QuantizedKVCache gc(kcb, vcb, enc);
    double worst = 0;
    for (size_t t = 0; t < n; ++t) {
      Vec k(keys.row(t).begin(), keys.row(t).end()), v(values.row(t).begin(), values.row(t).end());
      Vec q(qs.row(t).begin(), qs.row(t).end());
      Vec a = ref.decode_step(k, v, q);
      Vec b = gc.decode_step(k, v, q);
      worst = std::max(worst, rel_err(b, a));
    }
    report(worst <= 1e-4, "decode_step incremental gpu vs reference", std::to_string(worst));
    report(gc.packed_key_words() == ref.packed_keys().words() &&
               gc.packed_value_words() == ref.packed_values().words(),
           "incremental packed words identical");
    gpu::QuantizedKVCache pre = gpu::QuantizedKVCache::prefill(keys, values, kcb, vcb, enc);
    report(pre.packed_key_words() == ref.packed_keys().words(), "gpu prefill == reference appends");
    const auto dir = std::filesystem::temp_directory_path();
    const std::string p1 = (dir / "cvq_gpu.cvqc").string(), p2 = (dir / "cvq_ref.cvqc").string();
    gc.save(p1);
    QuantizedKVCache back = QuantizedKVCache::load(p1, kcb, vcb, enc);
    report(back.packed_keys().words() == ref.packed_keys().words(), "reference loads GPU CVQC");
    ref.save(p2);
    gpu::QuantizedKVCache gback = gpu::QuantizedKVCache::load(p2, kcb, vcb, enc);
    report(gback.packed_key_words() == ref.packed_keys().words() && gback.size() == n,
           "GPU loads reference CVQC");
    bool threw = false;
    try {
      gpu::QuantizedKVCache::load(p2 + ".missing", kcb, vcb, enc);
    } catch (const IoError&) {
      threw = true;
    }
    report(threw, "missing file -> IoError");
    std::filesystem::remove(p1);
    std::filesystem::remove(p2);
  }
  // 4. exceptions mirror the reference
  {
    KeyQuantConfig cfg{8, 2, 4, 1};
    KeyCodebook kcb = KeyCodebook::zeros(cfg);
    KeyCodes kc = KeyCodes::empty(cfg, 4);
    ValueCodes vc = ValueCodes::empty(8, 4);
    ValueCodebook vcb = ValueCodebook::zeros(8, 8);
    Vec q(8, 0.1);
    RopeParams rope = RopeParams::make(8);
    RopeTable table(rope);
    AttnInput early{q, 2, kc, vc, kcb, vcb, rope};
    bool threw = false;
    try {
      gpu::fused_attention(early, table);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    report(threw, "query before cache -> invalid_argument");
  }
  // 5. train_key_codebook: drop-in for keyquant.hpp:131-133
  {
    KeyQuantConfig cfg{8, 2, 4, 2};
    Mat calib = gen_synth(128, 8, 3, 21);
    EmConfig em;
    em.soft_iters = 5;
    em.hard_iters_max = 20;
    KeyTrainResult ref = train_key_codebook(calib, cfg, em);
    KeyTrainResult dev = gpu::train_key_codebook(calib, cfg, em);
    double worst = 0.0, scale = 0.0;
    for (size_t i = 0; i < ref.codebook.atoms.size(); ++i) {
      const CommMat& x = ref.codebook.atoms[i];
      const CommMat& y = dev.codebook.atoms[i];
      worst = std::max({worst, std::abs(x.x - y.x), std::abs(x.y - y.y)});
      scale = std::max({scale, std::abs(x.x), std::abs(x.y)});
    }
    bool same_len = ref.report.rounds.size() == dev.report.rounds.size();
    for (size_t r = 0; same_len && r < ref.report.rounds.size(); ++r)
      for (size_t g2 = 0; g2 < ref.report.rounds[r].hard_objective.size(); ++g2)
        same_len = same_len && ref.report.rounds[r].hard_objective[g2].size() ==
                                   dev.report.rounds[r].hard_objective[g2].size();
    report(worst <= 1e-9 * scale && same_len, "train_key_codebook",
           "max |d atom| / max |atom| = " + std::to_string(worst / scale));
    bool threw = false;
    try {
      gpu::train_key_codebook(Mat(4, 8), cfg, em);  // fewer than L^2 rows
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    report(threw, "train: too few rows -> invalid_argument");
  }
  // 6. train_value_quantizer: drop-in for valquant.hpp:96-104
  {
    Mat calib = gen_synth(96, 8, 3, 22);
    ValTrainConfig cfg;
    cfg.steps = 150;
    cfg.batch = 16;
    cfg.step_size = 1e-2;
    ValueTrainResult ref = train_value_quantizer(calib, 8, cfg);
    ValueTrainResult dev = gpu::train_value_quantizer(calib, 8, cfg);
    double worst = 0.0, scale = 0.0;
    auto cmp = [&](const std::vector<double>& a, const std::vector<double>& b) {
      for (size_t i = 0; i < a.size(); ++i) {
        worst = std::max(worst, std::abs(a[i] - b[i]));
        scale = std::max(scale, std::abs(a[i]));
      }
    };
    cmp(ref.encoder.w1.data, dev.encoder.w1.data);
    cmp(ref.encoder.w2.data, dev.encoder.w2.data);
    cmp(ref.codebook.rows.data, dev.codebook.rows.data);
    const bool same = ref.steps_run == dev.steps_run && ref.diverged == dev.diverged &&
                      ref.loss_curve.size() == dev.loss_curve.size();
    report(same && worst <= 1e-9 * scale, "train_value_quantizer",
           "max |d param| / max |param| = " + std::to_string(worst / scale));
  }
  // 7. the reference's cache test bodies (test_cache.cpp:155-276) written
  // once against a Cache type and instantiated with commvq::QuantizedKVCache
  // and commvq::gpu::QuantizedKVCache -- only the namespace differs
  {
    CacheFixture fx;
    const CacheRun ref = run_cache_body<QuantizedKVCache>(fx, "ref");
    const CacheRun dev = run_cache_body<gpu::QuantizedKVCache>(fx, "gpu");
    report(dev.kw_pre == ref.kw_pre && dev.vw_pre == ref.vw_pre && dev.kw_inc == ref.kw_inc,
           "cache body: prefill / appends words (by-value prefill)");
    report(dev.a == ref.a && dev.b == ref.b && dev.bits == ref.bits,
           "cache body: key_codes() / value_codes() accessors");
    report(dev.threw_dim && ref.threw_dim, "cache body: append(Vec(7), Vec(8)) -> invalid_argument");
    double worst = 0;
    for (size_t i = 0; i < ref.outs.size(); ++i) worst = std::max(worst, rel_err(dev.outs[i], ref.outs[i]));
    report(worst <= 1e-5 && dev.flop_tokens_ok && ref.flop_tokens_ok,
           "cache body: decode_step + FlopReport", std::to_string(worst));
    report(dev.stats.tokens == ref.stats.tokens &&
               dev.stats.quantized_payload_bits == ref.stats.quantized_payload_bits &&
               dev.stats.fp16_equivalent_bytes == ref.stats.fp16_equivalent_bytes &&
               dev.stats.codebook_bytes == ref.stats.codebook_bytes &&
               dev.stats.avg_bit_effective == ref.stats.avg_bit_effective &&
               dev.stats.avg_bit_amortized == ref.stats.avg_bit_amortized,
           "cache body: stats() == compute_cache_stats");
    const CacheStats z1 = compute_cache_stats(fx.cfg, 8, 131072),
                     z2 = gpu::compute_cache_stats(fx.cfg, 8, 131072);
    report(z1.quantized_payload_bits == z2.quantized_payload_bits &&
               z1.avg_bit_amortized == z2.avg_bit_amortized,
           "compute_cache_stats closed form");
    report(dev.kw_loaded == ref.kw_loaded && dev.n_loaded == ref.n_loaded &&
               dev.a_loaded == ref.a_loaded,
           "cache body: save / load by value");
    report(dev.kw_long == ref.kw_long && dev.vw_long == ref.vw_long && dev.n_long == 70000 &&
               ref.n_long == 70000,
           "cache body: 70,000 appends past the initial reservation (words identical)");
    report(rel_err(dev.out_long, ref.out_long) <= 1e-5, "decode_step at 70,001 tokens",
           std::to_string(rel_err(dev.out_long, ref.out_long)));
    report(dev.copy_ok && ref.copy_ok, "cache body: copy is deep, move keeps contents");
  }
  // 8. encode_keys honours AssignSearch (keyquant.cpp:724-730): both searches
  // bit-exact against the reference's, on constructed near-ties where the two
  // searches may disagree
  {
    KeyQuantConfig cfg{16, 4, 16, 3};
    Rng rng(99);
    KeyCodebook kcb = rand_kcb(cfg, rng);
    Mat keys(300, 16);
    for (double& v : keys.data) v = rng.normal();
    for (size_t p = 0; p < 60; ++p) {  // midpoints of two centers of round 0, group 0..3
      const size_t a1 = rng.index(16), b1 = rng.index(16), a2 = rng.index(16), b2 = rng.index(16);
      for (size_t j = 0; j < 8; ++j) {
        const CommMat& u1 = kcb.atoms[kcb.atom_index(0, j, a1)];
        const CommMat& v1 = kcb.atoms[kcb.atom_index(0, j, b1)];
        const CommMat& u2 = kcb.atoms[kcb.atom_index(0, j, a2)];
        const CommMat& v2 = kcb.atoms[kcb.atom_index(0, j, b2)];
        keys(p, 2 * j) = 0.5 * ((u1.x - v1.y) + (u2.x - v2.y));
        keys(p, 2 * j + 1) = 0.5 * ((u1.y + v1.x) + (u2.y + v2.x));
      }
    }
    bool ok = true;
    size_t differ = 0;
    for (AssignSearch sch : {AssignSearch::brute_force, AssignSearch::factorized}) {
      KeyCodes r = commvq::encode_keys(keys, kcb, sch);
      KeyCodes g2 = gpu::encode_keys(keys, kcb, sch);
      ok = ok && r.a == g2.a && r.b == g2.b;
    }
    KeyCodes rb = commvq::encode_keys(keys, kcb, AssignSearch::brute_force);
    KeyCodes rf = commvq::encode_keys(keys, kcb, AssignSearch::factorized);
    for (size_t i = 0; i < rb.a.size(); ++i) differ += rb.a[i] != rf.a[i] || rb.b[i] != rf.b[i];
    report(ok, "encode_keys brute_force and factorized bit-exact",
           "(reference searches differ on " + std::to_string(differ) + " codes)");
  }
  std::printf("%d failure(s)\n", g_fail);
  return g_fail;
}
