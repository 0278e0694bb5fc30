// mgpu.cu -- context sharding across GPUs inside the C-ABI (SURVEY.md 8e,
// 8b "cvq_mgpu_init(ncclComm_t) / cvq_mgpu_merge").
//
// Rank r holds tokens [lo_r, hi_r) of every stream in its own cache (global
// positions through position_offset).  One attention step per rank:
//   1. cvq_cache_attention_partial on the local shard, written straight into
//      one packed block [m (rows) | l (rows) | o (rows x d)] (520 B per row);
//   2. ONE ncclAllGather of the blocks on the context stream (NVLink);
//   3. the LSE combine kernel (k_combine) over the gathered blocks.
// A decode step appends the new token to the LAST shard only, then every
// rank attends at the new global position.  NCCL is resolved at run time
// (dlopen of libnccl.so.2: the copy torch already loaded, or the system's),
// so libcvq_b200.so has no link-time NCCL dependency; callers either pass an
// initialised ncclComm_t or let the library create one from a unique id they
// broadcast with any bootstrap.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/cvq.h"
#include "cvq_internal.cuh"

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("mgpu: cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.comm_count = reinterpret_cast<decltype(api.comm_count)>(sym("ncclCommCount"));
    api.comm_user_rank = reinterpret_cast<decltype(api.comm_user_rank)>(sym("ncclCommUserRank"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_count &&
             api.comm_user_rank && api.all_gather && api.error_string;
    if (!api.ok) api.why = "mgpu: libnccl.so.2 lacks a required symbol";
  });
  return api;
}

}  // namespace

// ------------------------------------------------------------ shard plan
// Contiguous ranges, boundaries on `align`-token tiles (packed records stay
// 32-B aligned), covering [0, n); trailing ranks may be empty.
CVQ_API cvq_status cvq_shard_plan(uint64_t n_tokens, uint32_t world, uint32_t align,
                                  uint64_t* bounds) {
  if (world == 0 || align == 0 || !bounds) return CVQ_EINVAL;
  uint64_t per = (n_tokens + world - 1) / world;
  per = (per + align - 1) / align * align;
  for (uint32_t r = 0; r < world; ++r) {
    const uint64_t lo = std::min<uint64_t>(n_tokens, (uint64_t)r * per);
    const uint64_t hi = std::min<uint64_t>(n_tokens, (uint64_t)(r + 1) * per);
    bounds[2 * r] = lo;
    bounds[2 * r + 1] = hi;
  }
  return CVQ_OK;
}

// ------------------------------------------------------------- the group
struct cvq_mgpu {
  cvq_cache* shard = nullptr;
  cvq_context* ctx = nullptr;
  ncclComm_t comm = nullptr;
  bool own_comm = false;
  int rank = 0, world = 1;
  uint64_t total = 0;  // global tokens per stream (the last shard's end)
  long long rows = 0;
  int d = 0;
  float* block = nullptr;     // [rows * (d + 2)]
  float* gathered = nullptr;  // [world][rows * (d + 2)]
  float* qstage = nullptr;
  float* ostage = nullptr;
  uint64_t* tot_dev = nullptr;
};

namespace {

cvq_status mfail(cvq_status s, const std::string& m) { return cvq::set_error(s, m); }

#define MCU(x)                                                                 \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) return mfail(CVQ_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define MNC(x)                                                                  \
  do {                                                                          \
    ncclResult_t r_ = (x);                                                      \
    if (r_ != ncclSuccess) return mfail(CVQ_ENCCL, std::string(#x) + ": " + nccl().error_string(r_)); \
  } while (0)

cvq_status finish_create(cvq_mgpu* g, cvq_mgpu** out) {
  const NcclApi& api = nccl();
  MNC(api.comm_count(g->comm, &g->world));
  MNC(api.comm_user_rank(g->comm, &g->rank));
  cvq_cache_shape sh{};
  cvq_status s = cvq_cache_shape_of(g->shard, &sh);
  if (s != CVQ_OK) return s;
  g->rows = (long long)sh.n_seqs * sh.n_layers * sh.n_kv_heads * sh.q_per_kv;
  g->d = (int)sh.d;
  void* st_v = nullptr;
  cvq_context_stream(g->ctx, &st_v);
  cudaStream_t st = static_cast<cudaStream_t>(st_v);
  const size_t blk = (size_t)g->rows * (g->d + 2);
  MCU(cudaMalloc(&g->block, blk * sizeof(float)));
  MCU(cudaMalloc(&g->gathered, blk * g->world * sizeof(float)));
  MCU(cudaMalloc(&g->qstage, (size_t)g->rows * g->d * sizeof(float) * 2));
  g->ostage = g->qstage + (size_t)g->rows * g->d;
  MCU(cudaMalloc(&g->tot_dev, sizeof(uint64_t) * (g->world + 1)));
  // the global length: every rank contributes the end of its shard, the
  // maximum is the last shard's end (an all-gather, once)
  uint64_t n = 0;
  s = cvq_cache_length(g->shard, &n);
  if (s != CVQ_OK) return s;
  const uint64_t end = n ? sh.position_offset + n : 0;
  MCU(cudaMemcpyAsync(g->tot_dev + g->world, &end, sizeof(end), cudaMemcpyHostToDevice, st));
  MNC(api.all_gather(g->tot_dev + g->world, g->tot_dev, 1, ncclUint64, g->comm, st));
  std::vector<uint64_t> ends(g->world);
  MCU(cudaMemcpyAsync(ends.data(), g->tot_dev, g->world * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                      st));
  MCU(cudaStreamSynchronize(st));
  g->total = 0;
  for (uint64_t e : ends) g->total = std::max(g->total, e);
  *out = g;
  return CVQ_OK;
}

void release(cvq_mgpu* g) {
  if (!g) return;
  for (void* p : {(void*)g->block, (void*)g->gathered, (void*)g->qstage, (void*)g->tot_dev})
    if (p) cudaFree(p);
  if (g->own_comm && g->comm && nccl().ok) nccl().comm_destroy(g->comm);
  delete g;
}

}  // namespace

CVQ_API cvq_status cvq_mgpu_unique_id(void* id_out /* 128 bytes */) {
  const NcclApi& api = nccl();
  if (!api.ok) return mfail(CVQ_ENCCL, api.why);
  if (!id_out) return mfail(CVQ_EINVAL, "null argument");
  ncclUniqueId id;
  MNC(api.get_unique_id(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return CVQ_OK;
}

CVQ_API cvq_status cvq_mgpu_init(cvq_cache* shard, void* nccl_comm, cvq_mgpu** out) {
  const NcclApi& api = nccl();
  if (!api.ok) return mfail(CVQ_ENCCL, api.why);
  if (!shard || !nccl_comm || !out) return mfail(CVQ_EINVAL, "null argument");
  cvq_mgpu* g = new cvq_mgpu;
  g->shard = shard;
  g->ctx = cvq_cache_context(shard);
  g->comm = static_cast<ncclComm_t>(nccl_comm);
  cvq_status s = finish_create(g, out);
  if (s != CVQ_OK) release(g);
  return s;
}

CVQ_API cvq_status cvq_mgpu_init_rank(cvq_cache* shard, const void* unique_id, int rank,
                                      int world, cvq_mgpu** out) {
  const NcclApi& api = nccl();
  if (!api.ok) return mfail(CVQ_ENCCL, api.why);
  if (!shard || !unique_id || !out || world < 1 || rank < 0 || rank >= world)
    return mfail(CVQ_EINVAL, "mgpu: bad argument");
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  cvq_mgpu* g = new cvq_mgpu;
  g->shard = shard;
  g->ctx = cvq_cache_context(shard);
  g->own_comm = true;
  ncclResult_t r = api.comm_init_rank(&g->comm, world, id, rank);
  if (r != ncclSuccess) {
    release(g);
    return mfail(CVQ_ENCCL, std::string("ncclCommInitRank: ") + api.error_string(r));
  }
  cvq_status s = finish_create(g, out);
  if (s != CVQ_OK) release(g);
  return s;
}

CVQ_API cvq_status cvq_mgpu_destroy(cvq_mgpu* g) {
  release(g);
  return CVQ_OK;
}

CVQ_API cvq_status cvq_mgpu_length(const cvq_mgpu* g, uint64_t* n_tokens) {
  if (!g || !n_tokens) return mfail(CVQ_EINVAL, "null argument");
  *n_tokens = g->total;
  return CVQ_OK;
}

// partial on the local shard -> all-gather -> combine.  q / out in `where`.
CVQ_API cvq_status cvq_mgpu_attention(cvq_mgpu* g, const float* q, uint64_t t, float* out,
                                      int where) {
  if (!g || !q || !out) return mfail(CVQ_EINVAL, "null argument");
  void* st_v = nullptr;
  cvq_context_stream(g->ctx, &st_v);
  cudaStream_t st = static_cast<cudaStream_t>(st_v);
  const size_t qbytes = (size_t)g->rows * g->d * sizeof(float);
  const float* qd = q;
  if (where == CVQ_HOST) {
    MCU(cudaMemcpyAsync(g->qstage, q, qbytes, cudaMemcpyHostToDevice, st));
    qd = g->qstage;
  }
  uint64_t n = 0;
  cvq_status s = cvq_cache_length(g->shard, &n);
  if (s != CVQ_OK) return s;
  const size_t blk = (size_t)g->rows * (g->d + 2);
  if (n == 0) {  // an empty shard contributes l = 0 (skipped by the combine)
    MCU(cudaMemsetAsync(g->block, 0, blk * sizeof(float), st));
  } else {
    s = cvq_cache_attention_partial(g->shard, qd, t, g->block, g->block + g->rows,
                                    g->block + 2 * g->rows);
    if (s != CVQ_OK) return s;
  }
  MNC(nccl().all_gather(g->block, g->gathered, blk, ncclFloat, g->comm, st));
  float* od = where == CVQ_HOST ? g->ostage : out;
  s = cvq_lse_combine_packed(g->ctx, g->gathered, (uint32_t)g->world, (uint64_t)g->rows,
                             (uint32_t)g->d, od);
  if (s != CVQ_OK) return s;
  if (where == CVQ_HOST) {
    MCU(cudaMemcpyAsync(out, od, qbytes, cudaMemcpyDeviceToHost, st));
    return cvq_cache_synchronize(g->shard);  // one sync; surfaces append errors
  }
  return CVQ_OK;
}

// cache.cpp:287-296 across the group: the new token goes to the last shard,
// every rank attends at the new last global position.
CVQ_API cvq_status cvq_mgpu_decode_step(cvq_mgpu* g, const void* k, const void* v, int kv_dtype,
                                        const float* q, float* out, int where) {
  if (!g) return mfail(CVQ_EINVAL, "null argument");
  if (g->rank == g->world - 1) {
    cvq_status s = cvq_cache_append(g->shard, k, v, kv_dtype, where);
    if (s != CVQ_OK) return s;
  }
  g->total += 1;
  return cvq_mgpu_attention(g, q, g->total - 1, out, where);
}
