// dist.cu -- the exchange step of the sharded store and the
// kernels around it.
//
// Store rows are independent, so a sharded call is: the local scan on this
// rank's slots (the unchanged single-GPU kernels, ids offset to global) ->
// ONE all-gather of a packed per-rank payload -> a merge on every rank, so
// outputs are replicated and bit-identical to the unsharded store (a row's
// score does not depend on the rank that computes it; ties break by global id,
// SURVEY §8(c) c9).
//
// Transports (fmoe_dist_config.transport):
//  * NCCL: ncclAllGather on the caller's stream (asynchronous, CUDA-graph
//    capturable; NVLink / NVSwitch between B200s).  libnccl.so.2 is loaded at
//    run time (the one the process already has, e.g. PyTorch's), so the
//    library has no link-time NCCL dependency.
//  * HOST: a caller-supplied all-gather over host buffers (e.g. gloo, MPI, or
//    two processes sharing one GPU in tests, where NCCL refuses duplicate
//    devices).  The payload is copied D2H, the stream synchronised, the
//    callback called, the result copied H2D: synchronous, not capturable.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include <nccl.h>

#include "common.cuh"
#include "kernels.cuh"

namespace fmoe {

// ------------------------------------------------------------------ NCCL, loaded at run time
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

static const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the process's NCCL if one is loaded (PyTorch), else the system's
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.error_string;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

bool nccl_unique_id(void* out, std::string* err) {
  const NcclApi& n = nccl();
  if (!n.ok) { *err = n.why; return false; }
  ncclUniqueId id;
  const ncclResult_t r = n.get_unique_id(&id);
  if (r != ncclSuccess) { *err = std::string("ncclGetUniqueId: ") + n.error_string(r); return false; }
  std::memcpy(out, &id, sizeof(id));
  return true;
}

bool Comm::init(int rank_, int world_, int transport_, const void* uid, AllGatherFn fn, void* user, std::string* err) {
  rank = rank_;
  world = world_;
  transport = transport_;
  host_fn = fn;
  host_user = user;
  if (transport == kTransportHost) {
    if (!fn) { *err = "HOST transport needs an allgather callback"; return false; }
    return true;
  }
  const NcclApi& n = nccl();
  if (!n.ok) { *err = n.why; return false; }
  if (!uid) { *err = "NCCL transport needs the unique id"; return false; }
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t c = nullptr;
  const ncclResult_t r = n.comm_init_rank(&c, world, id, rank);
  if (r != ncclSuccess) { *err = std::string("ncclCommInitRank: ") + n.error_string(r); return false; }
  comm = c;
  return true;
}

void Comm::destroy() {
  if (comm) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
  comm = nullptr;
  if (h_send) cudaFreeHost(h_send);
  if (h_recv) cudaFreeHost(h_recv);
  h_send = h_recv = nullptr;
  h_bytes = 0;
}

// recv [world][bytes] <- every rank's send [bytes], rank order
bool Comm::allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s, std::string* err) {
  if (world == 1 && transport == kTransportHost) {
    if (cudaMemcpyAsync(drecv, dsend, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
      *err = "allgather copy";
      return false;
    }
    return true;
  }
  if (transport == kTransportNccl) {
    const ncclResult_t r = nccl().all_gather(dsend, drecv, bytes, ncclUint8, static_cast<ncclComm_t>(comm), s);
    if (r != ncclSuccess) { *err = std::string("ncclAllGather: ") + nccl().error_string(r); return false; }
    return true;
  }
  // HOST: pinned staging, synchronous callback
  if (h_bytes < bytes) {
    if (h_send) cudaFreeHost(h_send);
    if (h_recv) cudaFreeHost(h_recv);
    h_send = h_recv = nullptr;
    h_bytes = 0;
    if (cudaMallocHost(&h_send, bytes) != cudaSuccess || cudaMallocHost(&h_recv, bytes * world) != cudaSuccess) {
      *err = "pinned staging for the HOST transport";
      return false;
    }
    h_bytes = bytes;
  }
  if (cudaMemcpyAsync(h_send, dsend, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {
    *err = "HOST transport D2H";
    return false;
  }
  if (host_fn(h_send, h_recv, int64_t(bytes), host_user) != 0) {
    *err = "HOST transport allgather callback failed";
    return false;
  }
  if (cudaMemcpyAsync(drecv, h_recv, bytes * world, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {    // the pinned buffer is reused by the next call
    *err = "HOST transport H2D";
    return false;
  }
  return true;
}

// ------------------------------------------------------------------ payload kernels
// Local top-k (score, id) [B][k] -> payload [B*k keys | B flags]: key 0 for an
// empty entry (id -1); flag 0 when the query is invalid here (NaN score: zero
// norm, R3), else 1.
__global__ void pack_topk_kernel(int B, int k, const float* __restrict__ sc, const int64_t* __restrict__ id,
                                 uint64_t* payload) {
  pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < B * k) {
    const int64_t i = id[t];
    payload[t] = i < 0 ? 0ull : pack_key(sc[t], uint32_t(i));
  }
  if (t < B) payload[int64_t(B) * k + t] = sc[int64_t(t) * k] != sc[int64_t(t) * k] ? 0ull : 1ull;
}

// Gathered payloads [G][B*k_in + B] -> the global top k per query, (score
// desc, global id asc); a query any rank flags invalid gets (NaN, -1).
template <int KPL>
__global__ void __launch_bounds__(32) merge_gathered_kernel(int G, int B, int k_in, int k,
                                                            const uint64_t* __restrict__ g, float* out_score,
                                                            int64_t* out_id, uint64_t* out_keys) {
  pdl_wait();
  const int x = blockIdx.x, lane = threadIdx.x;
  const int64_t stride = int64_t(B) * (k_in + 1);
  WarpTopK<KPL> m;
  m.init();
  bool valid = true;
  for (int r = 0; r < G; ++r) {
    const uint64_t* src = g + r * stride;
    valid = valid && src[int64_t(B) * k_in + x] != 0ull;
    for (int j0 = 0; j0 < k_in; j0 += 32) m.offer(j0 + lane < k_in ? src[int64_t(x) * k_in + j0 + lane] : 0ull, k);
  }
#pragma unroll
  for (int s = 0; s < KPL; ++s) {
    const int j = s * 32 + lane;
    if (j < k) {
      const uint64_t key = valid ? m.v[s] : 0ull;
      const int64_t o = int64_t(x) * k + j;
      if (out_keys) out_keys[o] = key;
      if (out_score) out_score[o] = valid ? key_score(key) : __int_as_float(0x7fc00000);
      if (out_id) out_id[o] = valid ? key_id(key) : -1;
    }
  }
}

// Selection payloads [G][2][n] (masks, counts): exactly one rank -- the owner
// of the matched map -- contributes a non-zero entry; OR / sum combines them.
__global__ void combine_select_kernel(int G, int n, const uint64_t* __restrict__ g, uint64_t* out_mask,
                                      int32_t* out_count) {
  pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint64_t m = 0ull, c = 0ull;
  for (int r = 0; r < G; ++r) {
    m |= g[int64_t(r) * 2 * n + t];
    c += g[int64_t(r) * 2 * n + n + t];
  }
  out_mask[t] = m;
  out_count[t] = int32_t(c);
}

__global__ void pack_select_kernel(int n, const uint64_t* __restrict__ mask, const int32_t* __restrict__ count,
                                   uint64_t* payload) {
  pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  payload[t] = mask[t];
  payload[n + t] = uint64_t(uint32_t(count[t]));
}

cudaError_t launch_pack_topk(int B, int k, const float* sc, const int64_t* id, uint64_t* payload, cudaStream_t s) {
  const int n = B * k > B ? B * k : B;
  count_launch();
  return launch_pdl(pack_topk_kernel, dim3((n + 255) / 256), dim3(256), 0, s, B, k, sc, id, payload);
}

cudaError_t launch_merge_gathered(int G, int B, int k_in, int k, const uint64_t* g, float* out_score,
                                  int64_t* out_id, uint64_t* out_keys, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  count_launch();
  if (k <= 32)
    return launch_pdl(merge_gathered_kernel<1>, dim3(B), dim3(32), 0, s, G, B, k_in, k, g, out_score, out_id,
                      out_keys);
  return launch_pdl(merge_gathered_kernel<2>, dim3(B), dim3(32), 0, s, G, B, k_in, k, g, out_score, out_id,
                    out_keys);
}

cudaError_t launch_pack_select(int n, const uint64_t* mask, const int32_t* count, uint64_t* payload,
                               cudaStream_t s) {
  count_launch();
  return launch_pdl(pack_select_kernel, dim3((n + 255) / 256), dim3(256), 0, s, n, mask, count, payload);
}

cudaError_t launch_combine_select(int G, int n, const uint64_t* g, uint64_t* out_mask, int32_t* out_count,
                                  cudaStream_t s) {
  count_launch();
  return launch_pdl(combine_select_kernel, dim3((n + 255) / 256), dim3(256), 0, s, G, n, g, out_mask, out_count);
}

}  // namespace fmoe
