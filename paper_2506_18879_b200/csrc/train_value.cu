// train_value.cu -- value-quantizer training on the GPU (SURVEY.md 8f
// rank 4): train_value_quantizer (valquant.cpp:172-383), plain SGD on
// straight-through Gumbel-sigmoid gradients, batch-parallel on sm_100a.
//
// Faithfulness.  The random stream is the reference's own: the host draws
// the mt19937_64 words in the reference order (init normals / row indices,
// then per step and sample one row index and 2 n_codes Gumbel words) and the
// device turns them into row indices (exact Lemire multiply-shift) and
// Gumbel noise.  Every reduction runs in the reference's order -- per
// output element, sequentially over the reduced index, zero-skips kept, no
// FMA -- and the per-sample gradient sums run sequentially over the batch,
// so the trajectory matches the reference to the last bits of exp/log
// (device vs libm), far inside the 1e-9 parity bar.  Divergence handling
// (loss not finite or > 100x the first loss) and checkpoints happen on the
// device, so steps run without host round trips.
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "cvq_internal.cuh"

namespace cvq {

namespace {

struct VtDims {
  int d, H, C, B;
  long long n;
};

// Row indices and Gumbel differences from the raw words of one step:
// words [B][1 + 2C] (index, then (g1, g0) per code, rng.hpp:42-52).
__global__ void k_vt_noise(const uint64_t* __restrict__ raw, VtDims m, int* __restrict__ idx,
                           double* __restrict__ dg) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int per = 1 + 2 * m.C;
  if (e >= m.B * m.C) return;
  const int s = e / m.C, k = e % m.C;
  const uint64_t* w = raw + (size_t)s * per;
  if (k == 0) idx[s] = (int)__umul64hi(w[0], (unsigned long long)m.n);
  auto gumbel = [](uint64_t x) {
    const double u = __dmul_rn(__dadd_rn((double)(x >> 11), 0.5), 0x1.0p-53);
    return -log(-log(u));
  };
  const double g1 = gumbel(w[1 + 2 * k]), g0 = gumbel(w[2 + 2 * k]);
  dg[e] = __dsub_rn(g1, g0);
}

// h[s][j] = relu(sum_i t_i w1[i][j] + b1[j]), i ascending, t_i == 0 skipped
// (valquant.cpp:260-269).
__global__ void k_vt_hidden(const double* __restrict__ calib, const int* __restrict__ idx,
                            const double* __restrict__ w1, const double* __restrict__ b1, VtDims m,
                            double* __restrict__ h) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.B * m.H) return;
  const int s = e / m.H, j = e % m.H;
  const double* t = calib + (size_t)idx[s] * m.d;
  double acc = 0.0;
#pragma unroll 8
  for (int i = 0; i < m.d; ++i) {
    const double ti = t[i], w = w1[(size_t)i * m.H + j];
    if (ti != 0.0) acc = __dadd_rn(acc, __dmul_rn(ti, w));
  }
  acc = __dadd_rn(acc, b1[j]);
  h[e] = acc < 0.0 ? 0.0 : acc;
}

// logits, u = logit + b2 + (g1 - g0), soft = sigmoid(u / tau), bit = u > 0
// (valquant.cpp:270-283).
__global__ void k_vt_logits(const double* __restrict__ h, const double* __restrict__ w2,
                            const double* __restrict__ b2, const double* __restrict__ dg, double tau,
                            VtDims m, double* __restrict__ soft, uint8_t* __restrict__ bits) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.B * m.C) return;
  const int s = e / m.C, k = e % m.C;
  const double* hs = h + (size_t)s * m.H;
  double lg = 0.0;
#pragma unroll 8
  for (int j = 0; j < m.H; ++j) {
    const double hj = hs[j], w = w2[(size_t)j * m.C + k];
    if (hj != 0.0) lg = __dadd_rn(lg, __dmul_rn(hj, w));
  }
  const double u = __dadd_rn(__dadd_rn(lg, b2[k]), dg[e]);
  soft[e] = 1.0 / (1.0 + exp(-(u / tau)));
  bits[e] = u > 0.0 ? 1 : 0;
}

// t_hat = sum of set codebook rows (k ascending); dl/dt_hat = 2 (t_hat - t)
// and the per-sample squared error (valquant.cpp:285-300).
__global__ void k_vt_recon(const double* __restrict__ calib, const int* __restrict__ idx,
                           const uint8_t* __restrict__ bits, const double* __restrict__ cb, VtDims m,
                           double* __restrict__ dthat, double* __restrict__ diff2) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.B * m.d) return;
  const int s = e / m.d, j = e % m.d;
  const uint8_t* bs = bits + (size_t)s * m.C;
  double th = 0.0;
#pragma unroll 8
  for (int k = 0; k < m.C; ++k) {
    const double c = cb[(size_t)k * m.d + j];
    if (bs[k]) th = __dadd_rn(th, c);
  }
  const double diff = __dsub_rn(th, calib[(size_t)idx[s] * m.d + j]);
  diff2[e] = __dmul_rn(diff, diff);
  dthat[e] = __dmul_rn(2.0, diff);
}

// dl/dz[s][k] = (c_k . dl/dt_hat) * soft (1 - soft) / tau (valquant.cpp:310-318).
__global__ void k_vt_dz(const double* __restrict__ cb, const double* __restrict__ dthat,
                        const double* __restrict__ soft, double tau, VtDims m,
                        double* __restrict__ dz) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.B * m.C) return;
  const int s = e / m.C, k = e % m.C;
  double g = 0.0;
#pragma unroll 8
  for (int j = 0; j < m.d; ++j)
    g = __dadd_rn(g, __dmul_rn(cb[(size_t)k * m.d + j], dthat[(size_t)s * m.d + j]));
  const double sf = soft[e];
  const double slope = __ddiv_rn(__dmul_rn(sf, __dsub_rn(1.0, sf)), tau);
  dz[e] = __dmul_rn(g, slope);
}

// dl/dh[s][j] = [h > 0] sum_k w2[j][k] dl/dz[k] (valquant.cpp:327-334).
__global__ void k_vt_dh(const double* __restrict__ h, const double* __restrict__ w2,
                        const double* __restrict__ dz, VtDims m, double* __restrict__ dh) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.B * m.H) return;
  const int s = e / m.H, j = e % m.H;
  double acc = 0.0;
  if (h[e] > 0.0)
#pragma unroll 8
    for (int k = 0; k < m.C; ++k)
      acc = __dadd_rn(acc, __dmul_rn(w2[(size_t)j * m.C + k], dz[(size_t)s * m.C + k]));
  dh[e] = acc;
}

struct VtState {  // one copy of the trainable parameters
  double *w1, *b1, *w2, *b2, *cb;
};

// Per-element gradient sums over the batch in sample order, then the SGD
// update p -= (step / B) g (valquant.cpp:302-309, 320-341, 360-369).  One
// thread per parameter; all parameters in one launch.
__global__ void k_vt_grad_update(const double* __restrict__ calib, const int* __restrict__ idx,
                                 const double* __restrict__ h, const uint8_t* __restrict__ bits,
                                 const double* __restrict__ dthat, const double* __restrict__ dz,
                                 const double* __restrict__ dh, VtDims m, VtState st, double scale,
                                 int freeze_cb, const int* __restrict__ flags) {
  if (flags[0]) return;  // stopped (diverged): the state was restored
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n1 = (long long)m.d * m.H, n2 = (long long)m.H * m.C, nc = (long long)m.C * m.d;
  const long long o_b1 = n1, o_w2 = o_b1 + m.H, o_b2 = o_w2 + n2, o_cb = o_b2 + m.C,
                  end = o_cb + nc;
  if (e >= end) return;
  double g = 0.0;
  if (e < o_b1) {  // gw1[i][j] += t_i dl/dh_j (t_i != 0)
    const int i = (int)(e / m.H), j = (int)(e % m.H);
#pragma unroll 8
    for (int s = 0; s < m.B; ++s) {
      const double ti = calib[(size_t)idx[s] * m.d + i], v = dh[(size_t)s * m.H + j];
      if (ti != 0.0) g = __dadd_rn(g, __dmul_rn(ti, v));
    }
    st.w1[e] = __dsub_rn(st.w1[e], __dmul_rn(scale, g));
  } else if (e < o_w2) {  // gb1
    const int j = (int)(e - o_b1);
#pragma unroll 8
    for (int s = 0; s < m.B; ++s) g = __dadd_rn(g, dh[(size_t)s * m.H + j]);
    st.b1[j] = __dsub_rn(st.b1[j], __dmul_rn(scale, g));
  } else if (e < o_b2) {  // gw2[j][k] += h_j dl/dz_k (h_j != 0)
    const long long f = e - o_w2;
    const int j = (int)(f / m.C), k = (int)(f % m.C);
#pragma unroll 8
    for (int s = 0; s < m.B; ++s) {
      const double hj = h[(size_t)s * m.H + j], v = dz[(size_t)s * m.C + k];
      if (hj != 0.0) g = __dadd_rn(g, __dmul_rn(hj, v));
    }
    st.w2[f] = __dsub_rn(st.w2[f], __dmul_rn(scale, g));
  } else if (e < o_cb) {  // gb2
    const int k = (int)(e - o_b2);
#pragma unroll 8
    for (int s = 0; s < m.B; ++s) g = __dadd_rn(g, dz[(size_t)s * m.C + k]);
    st.b2[k] = __dsub_rn(st.b2[k], __dmul_rn(scale, g));
  } else if (!freeze_cb) {  // gcb[k][j] += dl/dt_hat_j for set bits
    const long long f = e - o_cb;
    const int k = (int)(f / m.d), j = (int)(f % m.d);
#pragma unroll 8
    for (int s = 0; s < m.B; ++s) {
      const double v = dthat[(size_t)s * m.d + j];
      if (bits[(size_t)s * m.C + k]) g = __dadd_rn(g, v);
    }
    st.cb[f] = __dsub_rn(st.cb[f], __dmul_rn(scale, g));
  }
}

// Batch loss (per-element MSE, sample order), divergence test against the
// first loss (valquant.cpp:343-357).  flags: [0] stopped, [1] diverged,
// [2] steps_done; lossv: [0] initial loss.
__global__ void k_vt_loss(const double* __restrict__ diff2, VtDims m, int step,
                          double* __restrict__ curve, double* __restrict__ lossv,
                          int* __restrict__ flags) {
  extern __shared__ double persample[];  // [B]: sq / d, one thread per sample
  if (flags[0]) return;
  for (int s = threadIdx.x; s < m.B; s += blockDim.x) {
    double sq = 0.0;
    for (int j = 0; j < m.d; ++j) sq = __dadd_rn(sq, diff2[(size_t)s * m.d + j]);
    persample[s] = __ddiv_rn(sq, (double)m.d);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double bl = 0.0;
  for (int s = 0; s < m.B; ++s) bl = __dadd_rn(bl, persample[s]);  // sample order
  bl = __ddiv_rn(bl, (double)m.B);
  curve[step] = bl;
  if (lossv[0] < 0.0) lossv[0] = bl;
  const double init = lossv[0];
  const bool bad = !isfinite(bl) || (init > 0.0 && bl > 100.0 * init);
  if (bad) {
    flags[0] = 1;
    flags[1] = 1;
    flags[3] = step + 1;  // curve length
  } else {
    flags[2] = step + 1;
    flags[3] = step + 1;
  }
}

// Checkpoint (every N steps) / restore-on-divergence copies.
__global__ void k_vt_copy(const double* __restrict__ src, double* __restrict__ dst, long long n,
                          const int* __restrict__ flags, int mode, int* __restrict__ ckpt_step) {
  // mode 0: checkpoint if not stopped; mode 1: restore if just stopped
  if (mode == 0 && flags[0]) return;
  if (mode == 1 && !flags[0]) return;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[e];
  if (e == 0 && mode == 0 && ckpt_step) *ckpt_step = flags[2];
}

unsigned nb(long long n, int t) { return (unsigned)((n + t - 1) / t); }

struct RefRngV {  // commvq::Rng (rng.hpp), host
  std::mt19937_64 gen;
  bool has_spare = false;
  double spare = 0.0;
  explicit RefRngV(uint64_t seed) : gen(seed) {}
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = (static_cast<double>(gen() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    has_spare = true;
    return r * std::cos(a);
  }
  size_t index(size_t n) {
    return static_cast<size_t>((static_cast<unsigned __int128>(gen()) * n) >> 64);
  }
};

#define VCU(x)                                  \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) {                    \
      *err = cudaGetErrorString(e_);            \
      for (void* p : owned) cudaFree(p);        \
      if (pinned) cudaFreeHost(pinned);         \
      return 3;                                 \
    }                                           \
  } while (0)

}  // namespace

int train_value_quantizer_gpu(const double* calib, long long n, int d, int n_codes,
                              const ValTrainCfg& cfg, const double* init_cb, double* w1,
                              double* b1, double* w2, double* b2, double* cb, double* loss_curve,
                              int* diverged, long long* steps_run, long long* curve_len,
                              std::string* err, cudaStream_t st) {
  // argument checks (valquant.cpp:175-200)
  if (n == 0 || d == 0) return *err = "train_value_quantizer: empty calibration", 1;
  if (n_codes == 0) return *err = "train_value_quantizer: n_codes == 0", 1;
  for (long long i = 0; i < n * d; ++i)
    if (!std::isfinite(calib[i])) return *err = "train_value_quantizer: calib not finite", 1;
  if (cfg.steps == 0 || cfg.batch == 0)
    return *err = "train_value_quantizer: steps/batch == 0", 1;
  if ((size_t)n < cfg.batch) return *err = "train_value_quantizer: fewer rows than batch", 1;
  if (!(cfg.step_size > 0.0)) return *err = "train_value_quantizer: step_size <= 0", 1;
  if (!(cfg.t_start > 0.0) || !(cfg.t_end > 0.0))
    return *err = "train_value_quantizer: temperatures <= 0", 1;
  if (cfg.t_start < cfg.t_end) return *err = "train_value_quantizer: temperature must not rise", 1;
  const int H = cfg.hidden ? (int)cfg.hidden : 2 * n_codes;
  const int C = n_codes, B = (int)cfg.batch;
  VtDims m{d, H, C, B, n};

  // ---- host: initial state from the reference stream (valquant.cpp:206-226)
  RefRngV rng(cfg.seed);
  std::vector<double> hw1((size_t)d * H, 0.0), hb1(H, 0.0), hw2((size_t)H * C, 0.0), hb2(C, 0.0),
      hcb((size_t)C * d, 0.0);
  const double s1 = std::sqrt(2.0 / static_cast<double>(d));
  for (double& w : hw1) w = s1 * rng.normal();
  const double s2 = 1.0 / std::sqrt(static_cast<double>(H));
  for (double& w : hw2) w = s2 * rng.normal();
  if (init_cb) {
    std::memcpy(hcb.data(), init_cb, hcb.size() * 8);
  } else {
    const double sc = 2.0 / static_cast<double>(C);
    for (int k = 0; k < C; ++k) {
      const double* src = calib + rng.index((size_t)n) * d;
      for (int j = 0; j < d; ++j) hcb[(size_t)k * d + j] = sc * src[j];
    }
  }

  // ---- device buffers
  std::vector<void*> owned;
  uint64_t* pinned = nullptr;
  auto dalloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes ? bytes : 8) != cudaSuccess) return nullptr;
    owned.push_back(p);
    return p;
  };
  const long long nparam = (long long)d * H + H + (long long)H * C + C + (long long)C * d;
  double* dcal = static_cast<double*>(dalloc((size_t)n * d * 8));
  double* state = static_cast<double*>(dalloc((size_t)nparam * 8));
  double* ckpt = static_cast<double*>(dalloc((size_t)nparam * 8));
  const int per = 1 + 2 * C;
  const int kSlots = 2;  // double-buffered raw words: host fills k+1 while k runs
  uint64_t* draw = static_cast<uint64_t*>(dalloc((size_t)kSlots * B * per * 8));
  int* didx = static_cast<int*>(dalloc((size_t)B * 4));
  double* dg = static_cast<double*>(dalloc((size_t)B * C * 8));
  double* hb = static_cast<double*>(dalloc((size_t)B * H * 8));
  double* soft = static_cast<double*>(dalloc((size_t)B * C * 8));
  uint8_t* bits = static_cast<uint8_t*>(dalloc((size_t)B * C));
  double* dthat = static_cast<double*>(dalloc((size_t)B * d * 8));
  double* diff2 = static_cast<double*>(dalloc((size_t)B * d * 8));
  double* dz = static_cast<double*>(dalloc((size_t)B * C * 8));
  double* dh = static_cast<double*>(dalloc((size_t)B * H * 8));
  double* curve = static_cast<double*>(dalloc((size_t)cfg.steps * 8));
  double* lossv = static_cast<double*>(dalloc(8));
  int* flags = static_cast<int*>(dalloc(16));
  int* ckstep = static_cast<int*>(dalloc(4));
  for (void* p : owned)
    if (!p) {
      for (void* q : owned) cudaFree(q);
      return *err = "train_value_quantizer: device allocation failed", 3;
    }
  VCU(cudaMallocHost(&pinned, (size_t)kSlots * B * per * 8));
  VtState sv{state, state + (size_t)d * H, state + (size_t)d * H + H,
             state + (size_t)d * H + H + (size_t)H * C,
             state + (size_t)d * H + H + (size_t)H * C + C};
  VCU(cudaMemcpyAsync(dcal, calib, (size_t)n * d * 8, cudaMemcpyHostToDevice, st));
  VCU(cudaMemcpyAsync(sv.w1, hw1.data(), hw1.size() * 8, cudaMemcpyHostToDevice, st));
  VCU(cudaMemcpyAsync(sv.b1, hb1.data(), hb1.size() * 8, cudaMemcpyHostToDevice, st));
  VCU(cudaMemcpyAsync(sv.w2, hw2.data(), hw2.size() * 8, cudaMemcpyHostToDevice, st));
  VCU(cudaMemcpyAsync(sv.b2, hb2.data(), hb2.size() * 8, cudaMemcpyHostToDevice, st));
  VCU(cudaMemcpyAsync(sv.cb, hcb.data(), hcb.size() * 8, cudaMemcpyHostToDevice, st));
  VCU(cudaMemcpyAsync(ckpt, state, (size_t)nparam * 8, cudaMemcpyDeviceToDevice, st));
  VCU(cudaMemsetAsync(flags, 0, 16, st));
  VCU(cudaMemsetAsync(ckstep, 0, 4, st));
  const double neg1 = -1.0;
  VCU(cudaMemcpyAsync(lossv, &neg1, 8, cudaMemcpyHostToDevice, st));
  std::vector<cudaEvent_t> slot_free(kSlots);
  for (auto& ev : slot_free) VCU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));

  const double scale = cfg.step_size / static_cast<double>(B);
  const size_t words = (size_t)B * per;
  int hflags[4] = {0, 0, 0, 0};
  for (size_t step = 0; step < cfg.steps; ++step) {
    const int slot = (int)(step % kSlots);
    if (step >= (size_t)kSlots) VCU(cudaEventSynchronize(slot_free[slot]));
    uint64_t* hw = pinned + (size_t)slot * words;
    for (size_t w = 0; w < words; ++w) hw[w] = rng.gen();  // index, then (g1, g0) per code
    VCU(cudaMemcpyAsync(draw + (size_t)slot * words, hw, words * 8, cudaMemcpyHostToDevice, st));
    const double frac =
        cfg.steps > 1 ? static_cast<double>(step) / static_cast<double>(cfg.steps - 1) : 0.0;
    const double tau = cfg.t_start + (cfg.t_end - cfg.t_start) * frac;
    k_vt_noise<<<nb((long long)B * C, 256), 256, 0, st>>>(draw + (size_t)slot * words, m, didx, dg);
    VCU(cudaEventRecord(slot_free[slot], st));
    k_vt_hidden<<<nb((long long)B * H, 128), 128, 0, st>>>(dcal, didx, sv.w1, sv.b1, m, hb);
    k_vt_logits<<<nb((long long)B * C, 128), 128, 0, st>>>(hb, sv.w2, sv.b2, dg, tau, m, soft, bits);
    k_vt_recon<<<nb((long long)B * d, 128), 128, 0, st>>>(dcal, didx, bits, sv.cb, m, dthat, diff2);
    k_vt_dz<<<nb((long long)B * C, 128), 128, 0, st>>>(sv.cb, dthat, soft, tau, m, dz);
    k_vt_dh<<<nb((long long)B * H, 128), 128, 0, st>>>(hb, sv.w2, dz, m, dh);
    k_vt_loss<<<1, 256, (size_t)B * 8, st>>>(diff2, m, (int)step, curve, lossv, flags);
    k_vt_copy<<<nb(nparam, 256), 256, 0, st>>>(ckpt, state, nparam, flags, 1, nullptr);
    k_vt_grad_update<<<nb(nparam, 128), 128, 0, st>>>(dcal, didx, hb, bits, dthat, dz, dh, m, sv,
                                                      scale, cfg.freeze_codebook ? 1 : 0, flags);
    count_launch(9);
    if (cfg.checkpoint_every && (step + 1) % cfg.checkpoint_every == 0) {
      k_vt_copy<<<nb(nparam, 256), 256, 0, st>>>(state, ckpt, nparam, flags, 0, ckstep);
      count_launch();
    }
    VCU(cudaGetLastError());
    if ((step + 1) % 64 == 0 || step + 1 == cfg.steps) {  // stop early once diverged
      VCU(cudaMemcpyAsync(hflags, flags, 16, cudaMemcpyDeviceToHost, st));
      VCU(cudaStreamSynchronize(st));
      if (hflags[0]) break;
    }
  }
  VCU(cudaMemcpyAsync(hflags, flags, 16, cudaMemcpyDeviceToHost, st));
  int hck = 0;
  VCU(cudaMemcpyAsync(&hck, ckstep, 4, cudaMemcpyDeviceToHost, st));
  VCU(cudaMemcpyAsync(w1, sv.w1, (size_t)d * H * 8, cudaMemcpyDeviceToHost, st));
  VCU(cudaMemcpyAsync(b1, sv.b1, (size_t)H * 8, cudaMemcpyDeviceToHost, st));
  VCU(cudaMemcpyAsync(w2, sv.w2, (size_t)H * C * 8, cudaMemcpyDeviceToHost, st));
  VCU(cudaMemcpyAsync(b2, sv.b2, (size_t)C * 8, cudaMemcpyDeviceToHost, st));
  VCU(cudaMemcpyAsync(cb, sv.cb, (size_t)C * d * 8, cudaMemcpyDeviceToHost, st));
  VCU(cudaStreamSynchronize(st));
  *curve_len = hflags[3];
  VCU(cudaMemcpy(loss_curve, curve, (size_t)hflags[3] * 8, cudaMemcpyDeviceToHost));
  *diverged = hflags[1];
  *steps_run = hflags[1] ? hck : hflags[2];
  for (auto& ev : slot_free) cudaEventDestroy(ev);
  for (void* p : owned) cudaFree(p);
  cudaFreeHost(pinned);
  return 0;
}

}  // namespace cvq
