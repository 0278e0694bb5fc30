// decode.cu -- dense reconstruction of key / value codes on sm_100a
// (decode_keys keyquant.cpp:741-768, decode_values valquant.cpp:115-128).
//
// Thread = one output element of one token.  Each element is accumulated
// in the reference's order -- over rounds (keys) or ascending codes with a
// set bit (values), starting from +0.0, fp64 without FMA -- so the dense
// rows are bit-identical to the reference's Mat.
#include "cvq_internal.cuh"

namespace cvq {
namespace {

__global__ void k_decode_keys(Geom g, const double2* __restrict__ atoms,
                              const uint16_t* __restrict__ a, const uint16_t* __restrict__ b,
                              long long n, double* __restrict__ out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * g.d) return;
  const long long p = e / g.d;
  const int j = (int)(e % g.d), w = 2 * g.g;
  const int grp = j / w, s = (j % w) >> 1, im = j & 1;
  double v = 0.0;
  for (int r = 0; r < g.R; ++r) {
    const size_t idx = ((size_t)p * g.R + r) * g.groups + grp;
    const double2* slice = atoms + ((size_t)r * g.subs + (size_t)grp * g.g) * g.L;
    const double2 ua = slice[(size_t)s * g.L + a[idx]], ub = slice[(size_t)s * g.L + b[idx]];
    // row[2s] += x_a - y_b; row[2s+1] += y_a + x_b (keyquant.cpp:762-763)
    v = __dadd_rn(v, im ? __dadd_rn(ua.y, ub.x) : __dsub_rn(ua.x, ub.y));
  }
  out[e] = v;
}

__global__ void k_decode_values(int n_codes, int d, const double* __restrict__ rows,
                                const uint8_t* __restrict__ bits, long long n,
                                double* __restrict__ out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * d) return;
  const long long p = e / d;
  const int j = (int)(e % d);
  const uint8_t* bp = bits + (size_t)p * n_codes;
  double v = 0.0;
  for (int k = 0; k < n_codes; ++k)
    if (bp[k]) v = __dadd_rn(v, rows[(size_t)k * d + j]);  // valquant.cpp:121-125
  out[e] = v;
}

}  // namespace

cudaError_t run_decode_keys(const Geom& g, const double* atoms, const uint16_t* a,
                            const uint16_t* b, long long n, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long tot = n * g.d;
  k_decode_keys<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
      g, reinterpret_cast<const double2*>(atoms), a, b, n, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t run_decode_values(int n_codes, int d, const double* rows, const uint8_t* bits,
                              long long n, double* out, cudaStream_t st) {
  if (n <= 0 || d <= 0) return cudaSuccess;
  const long long tot = n * d;
  k_decode_values<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(n_codes, d, rows, bits, n, out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace cvq
