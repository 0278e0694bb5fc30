// pack.cu -- BitBuffer packing on sm_100a (cache.cpp:54-155).
//
// A packed key stream is a plain sequence of lb-bit fields (token-major,
// then rounds, then groups, a before b: cache.cpp:96-103); a value stream is
// a sequence of 1-bit fields (token-major, codes ascending: cache.cpp:
// 139-141).  Packing is therefore "one thread per output word": word w
// gathers the fields overlapping bits [64w, 64w+64), so appends at any
// token offset need no atomics; boundary words keep their bits outside the
// written range (tail padding stays zero as BitBuffer requires).
#include "cvq_internal.cuh"

namespace cvq {

// Key codes a/b laid out [s][n][R*groups] (KeyCodes::idx order per stream).
struct KeyFieldSrc {
  const uint16_t* a;
  const uint16_t* b;
  unsigned long long fields_per_stream;  // n * fpt
  __device__ __forceinline__ unsigned operator()(int s, unsigned long long f) const {
    const unsigned long long pair = (s * fields_per_stream + f) >> 1;
    return (f & 1) ? b[pair] : a[pair];
  }
};

// Value bits laid out [s][n][n_codes], one byte each (ValueCodes::bits).
struct BitFieldSrc {
  const uint8_t* bits;
  unsigned long long fields_per_stream;  // n * n_codes
  __device__ __forceinline__ unsigned operator()(int s, unsigned long long f) const {
    return bits[s * fields_per_stream + f];
  }
};

// Writes batch fields [0, nf) of stream s at stream field offset f0.
template <class Src>
__global__ void k_pack(Src src, int lb, unsigned long long f0, unsigned long long nf,
                       uint64_t* __restrict__ pool, uint64_t stride,
                       const unsigned long long* __restrict__ errpos, unsigned long long tok0) {
  if (errpos && *errpos <= tok0) return;  // this append (or an earlier one) failed
  const int s = blockIdx.y;
  const unsigned long long bit0 = f0 * lb, bit1 = (f0 + nf) * lb;  // [bit0, bit1)
  const unsigned long long w0 = bit0 >> 6, w1 = (bit1 + 63) >> 6;
  const unsigned long long w = w0 + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= w1) return;
  const unsigned long long lo = w << 6, hi = lo + 64;
  const unsigned long long b_lo = lo > bit0 ? lo : bit0;
  const unsigned long long b_hi = hi < bit1 ? hi : bit1;
  const unsigned long long fa = b_lo / lb, fb = (b_hi - 1) / lb;
  const uint64_t mask = lb >= 64 ? ~0ull : ((1ull << lb) - 1ull);
  uint64_t v = 0;
  for (unsigned long long f = fa; f <= fb; ++f) {
    const uint64_t val = (uint64_t)src(s, f - f0) & mask;  // BitBuffer::append masks
    const long long sh = (long long)(f * lb) - (long long)lo;
    v |= sh >= 0 ? (val << sh) : (val >> (-sh));
  }
  uint64_t keep = 0;
  if (b_lo > lo) keep |= (1ull << (b_lo - lo)) - 1ull;
  if (b_hi < hi) keep |= ~((1ull << (b_hi - lo)) - 1ull);
  uint64_t* dst = pool + (size_t)s * stride + w;
  *dst = keep ? ((*dst & keep) | (v & ~keep)) : v;
}

template <class Src>
static cudaError_t launch_pack(Src src, int S, int lb, unsigned long long f0,
                               unsigned long long nf, uint64_t* pool, uint64_t stride,
                               cudaStream_t st, const unsigned long long* errpos,
                               unsigned long long tok0) {
  // lb = 0 (n_levels = 1): zero-width fields, nothing to write (BitBuffer
  // appends of 0 bits, cache.cpp:60-75)
  if (nf == 0 || S == 0 || lb == 0) return cudaSuccess;
  const unsigned long long w0 = (f0 * lb) >> 6, w1 = ((f0 + nf) * lb + 63) >> 6;
  const unsigned long long nw = w1 - w0;
  dim3 grid((unsigned)((nw + 255) / 256), S);
  k_pack<Src><<<grid, 256, 0, st>>>(src, lb, f0, nf, pool, stride, errpos, tok0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t run_pack_keys(const Geom& g, int S, const uint16_t* a, const uint16_t* b,
                          long long n, long long tok0, uint64_t* kpool, uint64_t kstride,
                          cudaStream_t st, const unsigned long long* errpos) {
  KeyFieldSrc src{a, b, (unsigned long long)n * g.fpt};
  return launch_pack(src, S, g.lb, (unsigned long long)tok0 * g.fpt,
                     (unsigned long long)n * g.fpt, kpool, kstride, st, errpos,
                     (unsigned long long)tok0);
}

cudaError_t run_pack_values(const Geom& g, int S, const uint8_t* bits, long long n,
                            long long tok0, uint64_t* vpool, uint64_t vstride, cudaStream_t st,
                            const unsigned long long* errpos) {
  BitFieldSrc src{bits, (unsigned long long)n * g.n_codes};
  return launch_pack(src, S, 1, (unsigned long long)tok0 * g.n_codes,
                     (unsigned long long)n * g.n_codes, vpool, vstride, st, errpos,
                     (unsigned long long)tok0);
}

// ---- unpack (cache.cpp:108-135, 145-155): one thread per field ----------
__global__ void k_unpack_keys(const uint64_t* __restrict__ w, int lb, unsigned long long nf,
                              uint16_t* __restrict__ a, uint16_t* __restrict__ b) {
  const unsigned long long f = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const unsigned v = read_field(w, f * lb, lb);
  if (f & 1)
    b[f >> 1] = (uint16_t)v;
  else
    a[f >> 1] = (uint16_t)v;
}

__global__ void k_unpack_bits(const uint64_t* __restrict__ w, unsigned long long nf,
                              uint8_t* __restrict__ bits) {
  const unsigned long long f = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  bits[f] = (uint8_t)((__ldg(w + (f >> 6)) >> (f & 63)) & 1ull);
}

cudaError_t run_unpack_keys(const Geom& g, const uint64_t* words, long long n, uint16_t* a,
                            uint16_t* b, cudaStream_t st) {
  const unsigned long long nf = (unsigned long long)n * g.fpt;
  if (nf == 0) return cudaSuccess;
  if (g.lb == 0) {  // n_levels = 1: every code is 0 (cache.cpp:108-135)
    cudaError_t e = cudaMemsetAsync(a, 0, (nf / 2) * sizeof(uint16_t), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(b, 0, (nf / 2) * sizeof(uint16_t), st);
    return e;
  }
  k_unpack_keys<<<(unsigned)((nf + 255) / 256), 256, 0, st>>>(words, g.lb, nf, a, b);
  count_launch();
  return cudaGetLastError();
}

cudaError_t run_unpack_values(const Geom& g, const uint64_t* words, long long n, uint8_t* bits,
                              cudaStream_t st) {
  const unsigned long long nf = (unsigned long long)n * g.n_codes;
  if (nf == 0) return cudaSuccess;
  k_unpack_bits<<<(unsigned)((nf + 255) / 256), 256, 0, st>>>(words, nf, bits);
  count_launch();
  return cudaGetLastError();
}

}  // namespace cvq
