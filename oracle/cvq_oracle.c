/*
 * cvq_oracle.c -- CPU restatement of the CommVQ decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see cvq_oracle.h).  Plain C99, fp64, in the
 * reference's exact operation order.  Build with -ffp-contract=off so no
 * multiply-add is fused (the reference build has none: x86-64 baseline ISA,
 * SURVEY.md section 2 "build" row).  File:line citations are relative to
 * /root/reference/proj/core/.
 */
#include "cvq_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
const char* cvqo_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------ rng */
/* std::mt19937_64 (rng.hpp:53 member gen_), standard parameters. */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x000000007FFFFFFFULL

void cvqo_rng_seed(cvqo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

uint64_t cvqo_rng_next_u64(cvqo_rng* r) { /* rng.hpp:17 */
  if (r->idx >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (r->mt[i] & MT_UM) | (r->mt[(i + 1) % MT_N] & MT_LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= MT_A;
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

double cvqo_rng_uniform01(cvqo_rng* r) { /* rng.hpp:20-22 */
  return (double)(cvqo_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

double cvqo_rng_normal(cvqo_rng* r) { /* rng.hpp:25-38 Box-Muller */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = ((double)(cvqo_rng_next_u64(r) >> 11) + 1.0) * 0x1.0p-53;
  double u2 = cvqo_rng_uniform01(r);
  double rad = sqrt(-2.0 * log(u1));
  double a = 6.283185307179586476925286766559 * u2;
  r->spare = rad * sin(a);
  r->has_spare = 1;
  return rad * cos(a);
}

uint64_t cvqo_rng_index(cvqo_rng* r, uint64_t n) { /* rng.hpp:47-50 */
  return (uint64_t)(((unsigned __int128)cvqo_rng_next_u64(r) * n) >> 64);
}

cvqo_rng* cvqo_rng_new(uint64_t seed) {
  cvqo_rng* r = (cvqo_rng*)malloc(sizeof(cvqo_rng));
  if (r) cvqo_rng_seed(r, seed);
  return r;
}
void cvqo_rng_free(cvqo_rng* r) { free(r); }
void cvqo_rng_fill_normal(cvqo_rng* r, double* out, size_t n, double scale) {
  for (size_t i = 0; i < n; ++i) out[i] = scale * cvqo_rng_normal(r);
}
void cvqo_rng_fill_index_u16(cvqo_rng* r, uint16_t* out, size_t n,
                             uint64_t bound) {
  for (size_t i = 0; i < n; ++i) out[i] = (uint16_t)cvqo_rng_index(r, bound);
}
void cvqo_rng_fill_bit_u8(cvqo_rng* r, uint8_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = (uint8_t)(cvqo_rng_next_u64(r) & 1);
}
void cvqo_rng_fill_u64(cvqo_rng* r, uint64_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = cvqo_rng_next_u64(r);
}

/* ------------------------------------------------------------ keyquant */
static size_t ilog2_ceil(size_t v) { /* keyquant.cpp:19-23 */
  size_t b = 0;
  while (((size_t)1 << b) < v) ++b;
  return b;
}
size_t cvqo_level_bits(const cvqo_kq* c) { return ilog2_ceil(c->n_levels); }
size_t cvqo_bits_per_token(const cvqo_kq* c) {
  return c->rounds * ((c->d / 2) / c->group_size) * 2 * cvqo_level_bits(c);
}

int cvqo_validate(const cvqo_kq* c) { /* keyquant.cpp:46-60 */
  if (c->d == 0 || c->d % 2 != 0)
    return fail(CVQO_EINVAL, "KeyQuantConfig: d must be positive and even");
  if (c->group_size == 0)
    return fail(CVQO_EINVAL, "KeyQuantConfig: group_size must be positive");
  if ((c->d / 2) % c->group_size != 0)
    return fail(CVQO_EINVAL, "KeyQuantConfig: group_size must divide d/2 evenly");
  if (c->n_levels == 0 || (c->n_levels & (c->n_levels - 1)) != 0)
    return fail(CVQO_EINVAL, "KeyQuantConfig: n_levels must be a power of two");
  if (c->n_levels > 65536)
    return fail(CVQO_EINVAL, "KeyQuantConfig: n_levels too large");
  if (c->rounds == 0)
    return fail(CVQO_EINVAL, "KeyQuantConfig: rounds must be positive");
  return CVQO_OK;
}

/* ---------------------------------------------------------------- rope */
double cvqo_theta(size_t i, size_t d, double base) { /* rope.cpp:8-14 */
  double exponent = -2.0 * (double)(i - 1) / (double)d;
  return pow(base, exponent);
}

static double* make_thetas(size_t d, double base) { /* rope.cpp:16-25 */
  size_t s = d / 2;
  double* th = (double*)malloc(s * sizeof(double));
  for (size_t j = 0; j < s; ++j) th[j] = cvqo_theta(j + 1, d, base);
  return th;
}

/* --------------------------------------------------------------- linalg */
int cvqo_softmax_row(const double* v, size_t n, double* out) { /* linalg.cpp:63-75 */
  if (n == 0) return fail(CVQO_EINVAL, "softmax_row: empty input");
  double mx = v[0];
  for (size_t i = 0; i < n; ++i) mx = (mx < v[i]) ? v[i] : mx; /* std::max */
  double sum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    out[i] = exp(v[i] - mx);
    sum += out[i];
  }
  for (size_t i = 0; i < n; ++i) out[i] /= sum;
  return CVQO_OK;
}

/* ----------------------------------------------------------- attention */
/* attn.cpp:24-89 attention_core; cos/sin of m*theta_j as RopeTable
 * (rope.cpp:84-98) or libm -- both evaluate the same expressions. */
static int attention_core(const double* q, const double* keys,
                          const double* values, size_t n, size_t d,
                          const double* thetas, size_t t, double* out,
                          uint64_t* mults) {
  size_t subs = d / 2;
  if (n == 0) return fail(CVQO_EINVAL, "attention: empty cache");
  if (t + 1 < n)
    return fail(CVQO_EINVAL, "attention: query position precedes cache");
  double* qr = (double*)malloc(d * sizeof(double));
  for (size_t j = 0; j < subs; ++j) {
    double a = (double)t * thetas[j];
    double c = cos(a), s = sin(a);
    double x = q[2 * j], y = q[2 * j + 1];
    qr[2 * j] = x * c - y * s;
    qr[2 * j + 1] = x * s + y * c;
  }
  if (mults) *mults += 2 * d;
  double* scores = (double*)malloc(n * sizeof(double));
  double inv_sqrt_d = 1.0 / sqrt((double)d);
  for (size_t i = 0; i < n; ++i) {
    const double* krow = keys + i * d;
    double acc = 0.0;
    for (size_t j = 0; j < subs; ++j) {
      double a = (double)i * thetas[j];
      double c = cos(a), s = sin(a);
      double x = krow[2 * j], y = krow[2 * j + 1];
      double rx = x * c - y * s;
      double ry = x * s + y * c;
      acc += qr[2 * j] * rx + qr[2 * j + 1] * ry;
    }
    scores[i] = acc * inv_sqrt_d;
  }
  if (mults) *mults += (2 * d + d + 1) * (uint64_t)n;
  double* w = (double*)malloc(n * sizeof(double));
  cvqo_softmax_row(scores, n, w);
  for (size_t j = 0; j < d; ++j) out[j] = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double wi = w[i];
    const double* vrow = values + i * d;
    for (size_t j = 0; j < d; ++j) out[j] += wi * vrow[j];
  }
  if (mults) *mults += (uint64_t)n * d;
  free(qr);
  free(scores);
  free(w);
  return CVQO_OK;
}

int cvqo_reference_attention(const double* q, const double* K, const double* V,
                             size_t n, size_t d, double base, size_t t,
                             double* out) { /* attn.cpp:125-128 */
  if (d == 0 || d % 2) return fail(CVQO_EINVAL, "RopeParams: d must be positive and even");
  double* th = make_thetas(d, base);
  int rc = attention_core(q, K, V, n, d, th, t, out, NULL);
  free(th);
  return rc;
}

static int validate_input(const cvqo_attn_in* in) { /* attn.cpp:91-110 */
  int rc = cvqo_validate(in->kq);
  if (rc) return rc;
  if (in->n_tokens == 0) return fail(CVQO_EINVAL, "attention: empty cache");
  if (in->t + 1 < in->n_tokens)
    return fail(CVQO_EINVAL, "attention: query position precedes cache");
  if (in->n_codes == 0)
    return fail(CVQO_EINVAL, "attention: value codes/codebook mismatch");
  return CVQO_OK;
}

uint64_t cvqo_predicted_flops_naive(size_t n, size_t d, size_t n_codes) {
  if (n == 0 || d == 0 || n_codes == 0) return 0; /* attn.cpp:265-270 */
  return (2 * (uint64_t)d + 1) * n + 2 * (uint64_t)d * n_codes * n;
}
uint64_t cvqo_predicted_flops_fused(size_t n, size_t d, size_t n_codes,
                                    size_t rounds, size_t n_levels) {
  if (n == 0 || d == 0 || n_codes == 0 || rounds == 0 || n_levels == 0)
    return 0; /* attn.cpp:272-280 */
  return ((uint64_t)rounds * d + n_codes + 1) * n +
         (uint64_t)d * (n_codes + (uint64_t)rounds * n_levels);
}

/* attn.cpp:164-235: rotate q, fold through atoms, per-token alpha. */
static int fused_scores_impl(const cvqo_attn_in* in, double* scores,
                             uint64_t* mults) {
  const cvqo_kq* kc = in->kq;
  size_t n = in->n_tokens, d = kc->d, subs = d / 2, g = kc->group_size;
  size_t rounds = kc->rounds, levels = kc->n_levels, groups = subs / g;
  double* th = make_thetas(d, in->rope_base);
  double* qr = (double*)malloc(d * sizeof(double));
  for (size_t j = 0; j < subs; ++j) { /* attn.cpp:181-190 */
    double a = (double)in->t * th[j];
    double c = cos(a), s = sin(a);
    double x = in->q[2 * j], y = in->q[2 * j + 1];
    qr[2 * j] = x * c - y * s;
    qr[2 * j + 1] = x * s + y * c;
  }
  *mults += 2 * d;
  size_t np = rounds * subs * levels; /* attn.cpp:192-207 */
  double* px = (double*)malloc(np * sizeof(double));
  double* py = (double*)malloc(np * sizeof(double));
  for (size_t r = 0; r < rounds; ++r)
    for (size_t j = 0; j < subs; ++j) {
      double qx = qr[2 * j], qy = qr[2 * j + 1];
      size_t base = (r * subs + j) * levels;
      for (size_t l = 0; l < levels; ++l) {
        double mx = in->atoms_xy[2 * (base + l)];
        double my = in->atoms_xy[2 * (base + l) + 1];
        px[base + l] = qx * mx + qy * my;
        py[base + l] = qy * mx - qx * my;
      }
    }
  *mults += (uint64_t)2 * d * rounds * levels;
  double inv_sqrt_d = 1.0 / sqrt((double)d);
  double* crow = (double*)malloc(subs * sizeof(double));
  double* srow = (double*)malloc(subs * sizeof(double));
  int rc = CVQO_OK;
  for (size_t i = 0; i < n && rc == CVQO_OK; ++i) { /* attn.cpp:215-234 */
    for (size_t j = 0; j < subs; ++j) {
      double a = (double)i * th[j];
      crow[j] = cos(a);
      srow[j] = sin(a);
    }
    double alpha = 0.0;
    for (size_t r = 0; r < rounds; ++r)
      for (size_t grp = 0; grp < groups; ++grp) {
        size_t idx = (i * rounds + r) * groups + grp;
        size_t a = in->a[idx], b = in->b[idx];
        if (a >= levels || b >= levels) {
          rc = fail(CVQO_EINVAL, "fused_attention: code out of range");
          break;
        }
        for (size_t s = 0; s < g; ++s) {
          size_t j = grp * g + s;
          size_t base = (r * subs + j) * levels;
          alpha += crow[j] * (px[base + a] + py[base + b]) +
                   srow[j] * (py[base + a] - px[base + b]);
        }
      }
    scores[i] = alpha * inv_sqrt_d;
  }
  *mults += (uint64_t)n * (rounds * d + 1);
  free(th); free(qr); free(px); free(py); free(crow); free(srow);
  return rc;
}

int cvqo_fused_scores(const cvqo_attn_in* in, double* scores) {
  int rc = validate_input(in);
  if (rc) return rc;
  uint64_t m = 0;
  return fused_scores_impl(in, scores, &m);
}

int cvqo_fused_attention(const cvqo_attn_in* in, double* out,
                         uint64_t* predicted, uint64_t* measured) {
  int rc = validate_input(in);
  if (rc) return rc;
  size_t n = in->n_tokens, d = in->kq->d, n_codes = in->n_codes;
  uint64_t mults = 0;
  double* scores = (double*)malloc(n * sizeof(double));
  rc = fused_scores_impl(in, scores, &mults);
  if (rc) { free(scores); return rc; }
  double* w = (double*)malloc(n * sizeof(double));
  cvqo_softmax_row(scores, n, w); /* attn.cpp:237 */
  double* z = (double*)calloc(n_codes, sizeof(double));
  for (size_t i = 0; i < n; ++i) { /* attn.cpp:240-247 */
    double wi = w[i];
    const uint8_t* bits = in->bits + i * n_codes;
    for (size_t k = 0; k < n_codes; ++k)
      if (bits[k]) z[k] += wi;
  }
  for (size_t j = 0; j < d; ++j) out[j] = 0.0;
  for (size_t k = 0; k < n_codes; ++k) { /* attn.cpp:250-255 */
    double zk = z[k];
    const double* cr = in->value_rows + k * d;
    for (size_t j = 0; j < d; ++j) out[j] += zk * cr[j];
  }
  mults += (uint64_t)n_codes * d;
  if (predicted)
    *predicted = cvqo_predicted_flops_fused(n, d, n_codes, in->kq->rounds,
                                            in->kq->n_levels);
  if (measured) *measured = mults;
  free(scores); free(w); free(z);
  return CVQO_OK;
}

int cvqo_decode_keys(const cvqo_kq* kq, const double* atoms_xy,
                     const uint16_t* a, const uint16_t* b, size_t n,
                     double* out) { /* keyquant.cpp:741-768 */
  int rc = cvqo_validate(kq);
  if (rc) return rc;
  size_t d = kq->d, subs = d / 2, g = kq->group_size, L = kq->n_levels;
  size_t groups = subs / g, w = 2 * g;
  memset(out, 0, n * d * sizeof(double));
  for (size_t r = 0; r < kq->rounds; ++r)
    for (size_t grp = 0; grp < groups; ++grp) {
      const double* slice = atoms_xy + 2 * ((r * subs + grp * g) * L);
      for (size_t p = 0; p < n; ++p) {
        size_t idx = (p * kq->rounds + r) * groups + grp;
        size_t aa = a[idx], bb = b[idx];
        if (aa >= L || bb >= L)
          return fail(CVQO_EINVAL, "decode_keys: code out of range");
        double* row = out + p * d + grp * w;
        for (size_t s = 0; s < g; ++s) {
          const double* ma = slice + 2 * (s * L + aa);
          const double* mb = slice + 2 * (s * L + bb);
          row[2 * s] += ma[0] - mb[1];
          row[2 * s + 1] += ma[1] + mb[0];
        }
      }
    }
  return CVQO_OK;
}

int cvqo_decode_values(size_t n_codes, size_t d, const double* rows,
                       const uint8_t* bits, size_t n, double* out) {
  memset(out, 0, n * d * sizeof(double)); /* valquant.cpp:115-128 */
  for (size_t p = 0; p < n; ++p) {
    double* orow = out + p * d;
    for (size_t k = 0; k < n_codes; ++k) {
      if (!bits[p * n_codes + k]) continue;
      const double* row = rows + k * d;
      for (size_t j = 0; j < d; ++j) orow[j] += row[j];
    }
  }
  return CVQO_OK;
}

int cvqo_naive_attention(const cvqo_attn_in* in, double* out,
                         uint64_t* predicted, uint64_t* measured) {
  int rc = validate_input(in); /* attn.cpp:130-162 */
  if (rc) return rc;
  size_t n = in->n_tokens, d = in->kq->d, n_codes = in->n_codes;
  uint64_t mults = 0;
  double* keys = (double*)malloc(n * d * sizeof(double));
  rc = cvqo_decode_keys(in->kq, in->atoms_xy, in->a, in->b, n, keys);
  if (rc) { free(keys); return rc; }
  double* values = (double*)calloc(n * d, sizeof(double));
  for (size_t i = 0; i < n; ++i) { /* attn.cpp:146-154 */
    double* vrow = values + i * d;
    for (size_t k = 0; k < n_codes; ++k) {
      double bit = (double)in->bits[i * n_codes + k];
      const double* crow = in->value_rows + k * d;
      for (size_t j = 0; j < d; ++j) vrow[j] += bit * crow[j];
    }
  }
  mults += (uint64_t)n * n_codes * d;
  double* th = make_thetas(d, in->rope_base);
  rc = attention_core(in->q, keys, values, n, d, th, in->t, out, &mults);
  if (predicted) *predicted = cvqo_predicted_flops_naive(n, d, n_codes);
  if (measured) *measured = mults;
  free(th); free(keys); free(values);
  return rc;
}

/* keyquant.cpp:121-225 CenterCache for one (round, group) slice. */
typedef struct {
  size_t g, L;
  double *u, *v, *base, *centers;
} center_cache;

static void cc_init(center_cache* cc, const double* atoms_xy, size_t g,
                    size_t L, int want_base) {
  size_t w = 2 * g;
  cc->g = g;
  cc->L = L;
  cc->u = (double*)calloc(L * w, sizeof(double));
  cc->v = (double*)calloc(L * w, sizeof(double));
  for (size_t l = 0; l < L; ++l)
    for (size_t s = 0; s < g; ++s) {
      double mx = atoms_xy[2 * (s * L + l)], my = atoms_xy[2 * (s * L + l) + 1];
      cc->u[l * w + 2 * s] = mx;
      cc->u[l * w + 2 * s + 1] = my;
      cc->v[l * w + 2 * s] = -my;
      cc->v[l * w + 2 * s + 1] = mx;
    }
  cc->base = NULL;
  if (want_base) {
    double* un = (double*)malloc(L * sizeof(double));
    double* vn = (double*)malloc(L * sizeof(double));
    for (size_t l = 0; l < L; ++l) {
      double su = 0.0, sv = 0.0;
      for (size_t i = 0; i < w; ++i) su += cc->u[l * w + i] * cc->u[l * w + i];
      for (size_t i = 0; i < w; ++i) sv += cc->v[l * w + i] * cc->v[l * w + i];
      un[l] = su;
      vn[l] = sv;
    }
    cc->base = (double*)malloc(L * L * sizeof(double));
    for (size_t a = 0; a < L; ++a)
      for (size_t b = 0; b < L; ++b) {
        double uv = 0.0;
        for (size_t i = 0; i < w; ++i) uv += cc->u[a * w + i] * cc->v[b * w + i];
        cc->base[a * L + b] = un[a] + vn[b] + 2.0 * uv;
      }
    free(un);
    free(vn);
  }
  cc->centers = (double*)malloc(L * L * w * sizeof(double));
  for (size_t a = 0; a < L; ++a)
    for (size_t b = 0; b < L; ++b)
      for (size_t i = 0; i < w; ++i)
        cc->centers[(a * L + b) * w + i] = cc->u[a * w + i] + cc->v[b * w + i];
}

static void cc_free(center_cache* cc) {
  free(cc->u); free(cc->v); free(cc->base); free(cc->centers);
}

static size_t assign_brute(const center_cache* cc, const double* p) {
  size_t w = 2 * cc->g, nc = cc->L * cc->L; /* keyquant.cpp:180-200 */
  double best = INFINITY;
  size_t best_c = 0;
  for (size_t c = 0; c < nc; ++c) {
    const double* cr = cc->centers + c * w;
    double s = 0.0;
    for (size_t i = 0; i < w; ++i) {
      double dif = p[i] - cr[i];
      s += dif * dif;
    }
    if (s < best) {
      best = s;
      best_c = c;
    }
  }
  return best_c;
}

static size_t assign_factorized(const center_cache* cc, const double* p) {
  size_t w = 2 * cc->g, L = cc->L; /* keyquant.cpp:163-176, 204-224 */
  double* pu = (double*)malloc(L * sizeof(double));
  double* pv = (double*)malloc(L * sizeof(double));
  for (size_t l = 0; l < L; ++l) {
    double su = 0.0, sv = 0.0;
    for (size_t i = 0; i < w; ++i) {
      su += p[i] * cc->u[l * w + i];
      sv += p[i] * cc->v[l * w + i];
    }
    pu[l] = su;
    pv[l] = sv;
  }
  double best = INFINITY;
  size_t best_c = 0;
  for (size_t a = 0; a < L; ++a) {
    double pa2 = 2.0 * pu[a];
    for (size_t b = 0; b < L; ++b) {
      double s = cc->base[a * L + b] - pa2 - 2.0 * pv[b];
      if (s < best) {
        best = s;
        best_c = a * L + b;
      }
    }
  }
  free(pu);
  free(pv);
  return best_c;
}

static int encode_impl(const cvqo_kq* kq, const double* atoms_xy,
                       const double* keys, size_t n, uint16_t* a, uint16_t* b,
                       int factorized) { /* keyquant.cpp:705-739 */
  int rc = cvqo_validate(kq);
  if (rc) return rc;
  size_t d = kq->d, subs = d / 2, g = kq->group_size, L = kq->n_levels;
  size_t groups = subs / g, w = 2 * g;
  double* res = (double*)malloc(n * d * sizeof(double));
  memcpy(res, keys, n * d * sizeof(double));
  for (size_t r = 0; r < kq->rounds; ++r)
    for (size_t grp = 0; grp < groups; ++grp) {
      center_cache cc;
      cc_init(&cc, atoms_xy + 2 * ((r * subs + grp * g) * L), g, L, factorized);
      for (size_t p = 0; p < n; ++p) {
        double* row = res + p * d + grp * w;
        size_t c = factorized ? assign_factorized(&cc, row) : assign_brute(&cc, row);
        size_t idx = (p * kq->rounds + r) * groups + grp;
        a[idx] = (uint16_t)(c / L);
        b[idx] = (uint16_t)(c % L);
        const double* cr = cc.centers + c * w;
        for (size_t i = 0; i < w; ++i) row[i] -= cr[i];
      }
      cc_free(&cc);
    }
  free(res);
  return CVQO_OK;
}

int cvqo_encode_keys(const cvqo_kq* kq, const double* atoms_xy,
                     const double* keys, size_t n, uint16_t* a, uint16_t* b) {
  return encode_impl(kq, atoms_xy, keys, n, a, b, 0);
}
int cvqo_encode_keys_factorized(const cvqo_kq* kq, const double* atoms_xy,
                                const double* keys, size_t n, uint16_t* a,
                                uint16_t* b) {
  return encode_impl(kq, atoms_xy, keys, n, a, b, 1);
}

/* ------------------------------------------------------------- valquant */
int cvqo_encoder_forward_infer(size_t d, size_t hidden, size_t n_codes,
                               const double* w1, const double* b1,
                               const double* w2, const double* b2,
                               const double* values, size_t n, uint8_t* bits,
                               double* logits_out) {
  if (d == 0 || hidden == 0 || n_codes == 0)
    return fail(CVQO_EINVAL, "ValueEncoder: zero dimension");
  double* h = (double*)malloc(hidden * sizeof(double));
  double* lg = (double*)malloc(n_codes * sizeof(double));
  int rc = CVQO_OK;
  for (size_t p = 0; p < n && rc == CVQO_OK; ++p) {
    const double* t = values + p * d;
    for (size_t j = 0; j < hidden; ++j) h[j] = 0.0; /* valquant.cpp:50-70 */
    for (size_t i = 0; i < d; ++i) {
      double ti = t[i];
      if (ti == 0.0) continue;
      const double* wrow = w1 + i * hidden;
      for (size_t j = 0; j < hidden; ++j) h[j] += ti * wrow[j];
    }
    for (size_t j = 0; j < hidden; ++j) {
      h[j] += b1[j];
      if (h[j] < 0.0) h[j] = 0.0;
    }
    for (size_t k = 0; k < n_codes; ++k) lg[k] = 0.0;
    for (size_t j = 0; j < hidden; ++j) {
      double hj = h[j];
      if (hj == 0.0) continue;
      const double* wrow = w2 + j * n_codes;
      for (size_t k = 0; k < n_codes; ++k) lg[k] += hj * wrow[k];
    }
    for (size_t k = 0; k < n_codes; ++k) lg[k] += b2[k];
    for (size_t k = 0; k < n_codes; ++k) /* valquant.cpp:86-87 */
      if (!isfinite(lg[k])) {
        rc = fail(CVQO_ETRAIN, "encoder_forward: non-finite activations");
        break;
      }
    for (size_t k = 0; k < n_codes; ++k) { /* valquant.cpp:98 */
      bits[p * n_codes + k] = lg[k] > 0.0 ? 1 : 0;
      if (logits_out) logits_out[p * n_codes + k] = lg[k];
    }
  }
  free(h);
  free(lg);
  return rc;
}

/* ---------------------------------------------------------------- cache */
size_t cvqo_words_for_bits(uint64_t bits) { return (size_t)((bits + 63) / 64); }

/* BitBuffer::append cache.cpp:54-64 */
static void bb_append(uint64_t* words, uint64_t* pos, uint64_t value,
                      unsigned nbits) {
  if (nbits == 0) return;
  if (nbits < 64) value &= ((uint64_t)1 << nbits) - 1;
  uint64_t word = *pos / 64;
  unsigned off = (unsigned)(*pos % 64);
  *pos += nbits;
  words[word] |= value << off;
  if (off + nbits > 64) words[word + 1] |= value >> (64 - off);
}
/* BitBuffer::read cache.cpp:66-76 */
static uint64_t bb_read(const uint64_t* words, uint64_t pos, unsigned nbits) {
  if (nbits == 0) return 0;
  uint64_t word = pos / 64;
  unsigned off = (unsigned)(pos % 64);
  uint64_t v = words[word] >> off;
  if (off + nbits > 64) v |= words[word + 1] << (64 - off);
  if (nbits < 64) v &= ((uint64_t)1 << nbits) - 1;
  return v;
}

int cvqo_pack_key_codes(const cvqo_kq* kq, const uint16_t* a, const uint16_t* b,
                        size_t n, uint64_t* words) { /* cache.cpp:90-106 */
  int rc = cvqo_validate(kq);
  if (rc) return rc;
  unsigned lb = (unsigned)cvqo_level_bits(kq);
  size_t groups = (kq->d / 2) / kq->group_size;
  uint64_t total = (uint64_t)n * cvqo_bits_per_token(kq);
  memset(words, 0, cvqo_words_for_bits(total) * sizeof(uint64_t));
  uint64_t pos = 0;
  for (size_t t = 0; t < n; ++t)
    for (size_t r = 0; r < kq->rounds; ++r)
      for (size_t g = 0; g < groups; ++g) {
        size_t i = (t * kq->rounds + r) * groups + g;
        bb_append(words, &pos, a[i], lb);
        bb_append(words, &pos, b[i], lb);
      }
  return CVQO_OK;
}

int cvqo_unpack_key_codes(const cvqo_kq* kq, const uint64_t* words,
                          size_t n_words, size_t n, uint16_t* a, uint16_t* b) {
  int rc = cvqo_validate(kq); /* cache.cpp:108-135 + from_words 78-88 */
  if (rc) return rc;
  uint64_t total = (uint64_t)n * cvqo_bits_per_token(kq);
  if (n_words != cvqo_words_for_bits(total))
    return fail(CVQO_EINVAL, "BitBuffer: word count mismatch");
  unsigned tail = (unsigned)(total % 64);
  if (tail != 0 && (words[n_words - 1] >> tail) != 0)
    return fail(CVQO_EINVAL, "BitBuffer: nonzero padding bits");
  unsigned lb = (unsigned)cvqo_level_bits(kq);
  size_t groups = (kq->d / 2) / kq->group_size;
  uint64_t pos = 0;
  for (size_t t = 0; t < n; ++t)
    for (size_t r = 0; r < kq->rounds; ++r)
      for (size_t g = 0; g < groups; ++g) {
        size_t i = (t * kq->rounds + r) * groups + g;
        a[i] = (uint16_t)bb_read(words, pos, lb);
        pos += lb;
        b[i] = (uint16_t)bb_read(words, pos, lb);
        pos += lb;
      }
  return CVQO_OK;
}

int cvqo_pack_value_codes(size_t n_codes, const uint8_t* bits, size_t n,
                          uint64_t* words) { /* cache.cpp:137-143 */
  uint64_t total = (uint64_t)n * n_codes;
  memset(words, 0, cvqo_words_for_bits(total) * sizeof(uint64_t));
  uint64_t pos = 0;
  for (size_t t = 0; t < n; ++t)
    for (size_t k = 0; k < n_codes; ++k)
      bb_append(words, &pos, bits[t * n_codes + k], 1);
  return CVQO_OK;
}

int cvqo_unpack_value_codes(size_t n_codes, const uint64_t* words,
                            size_t n_words, size_t n, uint8_t* bits) {
  uint64_t total = (uint64_t)n * n_codes; /* cache.cpp:145-155 */
  if (n_words != cvqo_words_for_bits(total))
    return fail(CVQO_EINVAL, "BitBuffer: word count mismatch");
  unsigned tail = (unsigned)(total % 64);
  if (tail != 0 && (words[n_words - 1] >> tail) != 0)
    return fail(CVQO_EINVAL, "BitBuffer: nonzero padding bits");
  uint64_t pos = 0;
  for (size_t t = 0; t < n; ++t)
    for (size_t k = 0; k < n_codes; ++k)
      bits[t * n_codes + k] = (uint8_t)bb_read(words, pos++, 1);
  return CVQO_OK;
}

/* ------------------------------------------------------------------ ctf */
int cvqo_gen_synth(size_t n, size_t d, size_t rank, uint64_t seed,
                   double* x) { /* ctf.cpp:97-144 */
  if (d == 0 || n == 0) return fail(CVQO_EINVAL, "gen_synth: empty shape");
  if (rank < 1 || rank > d)
    return fail(CVQO_EINVAL, "gen_synth: rank must be in [1, d]");
  cvqo_rng rng;
  cvqo_rng_seed(&rng, seed);
  double* a = (double*)malloc(rank * d * sizeof(double));
  for (size_t i = 0; i < rank * d; ++i) a[i] = cvqo_rng_normal(&rng);
  for (size_t i = 0; i < rank; ++i) {
    double* ri = a + i * d;
    for (size_t j = 0; j < i; ++j) {
      double* rj = a + j * d;
      double proj = 0.0;
      for (size_t k = 0; k < d; ++k) proj += ri[k] * rj[k];
      for (size_t k = 0; k < d; ++k) ri[k] -= proj * rj[k];
    }
    double nn = 0.0;
    for (size_t k = 0; k < d; ++k) nn += ri[k] * ri[k];
    double norm = sqrt(nn);
    while (norm < 1e-8) {
      for (size_t k = 0; k < d; ++k) ri[k] = cvqo_rng_normal(&rng);
      for (size_t j = 0; j < i; ++j) {
        double* rj = a + j * d;
        double proj = 0.0;
        for (size_t k = 0; k < d; ++k) proj += ri[k] * rj[k];
        for (size_t k = 0; k < d; ++k) ri[k] -= proj * rj[k];
      }
      nn = 0.0;
      for (size_t k = 0; k < d; ++k) nn += ri[k] * ri[k];
      norm = sqrt(nn);
    }
    for (size_t k = 0; k < d; ++k) ri[k] /= norm;
  }
  double sigma_noise = 0.01 * sqrt((double)rank / (double)d);
  double* z = (double*)malloc(rank * sizeof(double));
  for (size_t t = 0; t < n; ++t) {
    for (size_t j = 0; j < rank; ++j) z[j] = cvqo_rng_normal(&rng);
    double* row = x + t * d;
    for (size_t k = 0; k < d; ++k) {
      double acc = 0.0;
      for (size_t j = 0; j < rank; ++j) acc += z[j] * a[j * d + k];
      acc += sigma_noise * cvqo_rng_normal(&rng);
      row[k] = (double)(float)acc;
    }
  }
  free(a);
  free(z);
  return CVQO_OK;
}
