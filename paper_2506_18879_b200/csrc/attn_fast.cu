// attn_fast.cu -- specialised decode-attention path (filled in below).
#include "cvq_internal.cuh"

namespace cvq {

bool fast_path_applies(const AttnJob&) { return false; }
size_t fast_scratch_bytes(const AttnJob&, int* n_chunks) {
  *n_chunks = 0;
  return 0;
}
cudaError_t run_attention_fast(const AttnJob&, const float*, float*, float*, float*, int, void*,
                               cudaStream_t, cudaEvent_t*) {
  return cudaErrorNotSupported;
}

}  // namespace cvq
