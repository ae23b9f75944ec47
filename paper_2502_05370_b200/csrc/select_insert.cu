// select_insert.cu -- K4 top-k merge, K5 expert selection, K6 row writes and
// the victim resolution of the RDY insert.
#include <atomic>
#include <cstdlib>
#include "common.cuh"
#include "kernels.cuh"
#include "select.cuh"

namespace fmoe {

static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(); }

// ------------------------------------------------------------------ K4 merge
// One CTA per query: 8 warps stream a strided share of the candidate keys
// through their own WarpTopK with 4 loads in flight per lane, then warp 0
// merges the 8 lists.
constexpr int kMergeWarps = 8;
constexpr int kMergeUnroll = 4;

template <int KPL>
__global__ void __launch_bounds__(kMergeWarps * 32) merge_keys_kernel(int n_lists, int k_in, const uint64_t* __restrict__ keys,
                                                        int k, const float* __restrict__ valid_q,
                                                        float* out_score, int64_t* out_id, uint64_t* out_keys,
                                                        const int* gate) {
  __shared__ uint64_t sk[kMergeWarps][KPL * 32];
  pdl_wait();
  if (gate && *gate == 0) return;
  const int q = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpTopK<KPL> m;
  m.init();
  const int64_t total = int64_t(n_lists) * k_in;
  const uint64_t* src = keys + int64_t(q) * total;
  constexpr int64_t kStep = int64_t(kMergeWarps) * kMergeUnroll * 32;
  for (int64_t j0 = int64_t(warp) * kMergeUnroll * 32; j0 < total; j0 += kStep) {
    uint64_t v[kMergeUnroll];
#pragma unroll
    for (int u = 0; u < kMergeUnroll; ++u) {
      const int64_t j = j0 + u * 32 + lane;
      v[u] = j < total ? __ldcs(src + j) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kMergeUnroll; ++u) m.offer(v[u], k);
  }
  m.store(sk[warp], k);
  __syncthreads();
  if (warp != 0) return;
  WarpTopK<KPL> f;
  f.init();
  for (int w = 0; w < kMergeWarps; ++w)
#pragma unroll
    for (int s = 0; s < KPL; ++s) {
      const int j = s * 32 + lane;
      f.offer(j < k ? sk[w][j] : 0ull, k);
    }
  const bool valid = valid_q ? valid_q[q] != 0.f : true;
#pragma unroll
  for (int s = 0; s < KPL; ++s) {
    const int j = s * 32 + lane;
    if (j < k) {
      const uint64_t key = f.v[s];
      if (out_keys) out_keys[int64_t(q) * k + j] = valid ? key : 0ull;
      if (out_score) out_score[int64_t(q) * k + j] = valid ? key_score(key) : __int_as_float(0x7fc00000);
      if (out_id) out_id[int64_t(q) * k + j] = valid ? key_id(key) : -1;
    }
  }
}

// Alternative merge for n_lists * k_in <= 2048 keys per query (opt-in,
// FMOE_MERGE_SORT=1): one block per query sorts the padded keys descending in
// shared memory (bitonic network, 256 threads) and writes the first k.
// Measured slower than the warp lists below: 32 vs 17 us per 64-query merge
// of 148 x 8 keys into 32 (C3 session step, profiles/r02n_merge_sort.md) --
// the 66 block barriers cost more than the warps' dependent inserts.  Keys are
// unique (a row lives in one list) and empty slots are key 0, so the order is
// the (score desc, id asc) order of the warp lists.
constexpr int kSortMax = 2048;
__global__ void __launch_bounds__(256) merge_sort_kernel(int total, int n_pow2, const uint64_t* __restrict__ keys, int k,
                                                         const float* __restrict__ valid_q, float* out_score,
                                                         int64_t* out_id, uint64_t* out_keys, const int* gate) {
  __shared__ uint64_t sk[kSortMax];
  pdl_wait();
  if (gate && *gate == 0) return;
  const int q = blockIdx.x, tid = threadIdx.x;
  const uint64_t* src = keys + int64_t(q) * total;
  for (int i = tid; i < n_pow2; i += 256) sk[i] = i < total ? __ldcs(src + i) : 0ull;
  __syncthreads();
  for (int size = 2; size <= n_pow2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < n_pow2 / 2; i += 256) {
        const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
        const bool up = (lo & size) == 0;          // this block sorts descending (else ascending)
        const uint64_t a = sk[lo], b = sk[hi];
        if ((a < b) == up) { sk[lo] = b; sk[hi] = a; }
      }
      __syncthreads();
    }
  const bool valid = valid_q ? valid_q[q] != 0.f : true;
  for (int j = tid; j < k; j += 256) {
    const uint64_t key = j < n_pow2 ? sk[j] : 0ull;
    if (out_keys) out_keys[int64_t(q) * k + j] = valid ? key : 0ull;
    if (out_score) out_score[int64_t(q) * k + j] = valid ? key_score(key) : __int_as_float(0x7fc00000);
    if (out_id) out_id[int64_t(q) * k + j] = valid ? key_id(key) : -1;
  }
}

cudaError_t launch_merge_keys(int B, int n_lists, int k_in, const uint64_t* keys, int k, const float* valid,
                              float* out_score, int64_t* out_id, uint64_t* out_keys, cudaStream_t s,
                              const int* gate) {
  if (B <= 0) return cudaSuccess;
  const int64_t total = int64_t(n_lists) * k_in;
  static const bool sort = getenv("FMOE_MERGE_SORT") && atoi(getenv("FMOE_MERGE_SORT")) == 1;   // knob
  if (total >= 1 && total <= kSortMax && sort) {
    int n2 = 64;
    while (n2 < total) n2 <<= 1;
    count_launch();
    return launch_pdl(merge_sort_kernel, dim3(B), dim3(256), 0, s, int(total), n2, keys, k, valid, out_score, out_id,
                      out_keys, gate);
  }
  if (k <= 32)
    return count_launch(), launch_pdl(merge_keys_kernel<1>, dim3(B), dim3(kMergeWarps * 32), 0, s, n_lists, k_in, keys, k, valid, out_score, out_id, out_keys, gate);
  else
    return count_launch(), launch_pdl(merge_keys_kernel<2>, dim3(B), dim3(kMergeWarps * 32), 0, s, n_lists, k_in, keys, k, valid, out_score, out_id, out_keys, gate);
  count_launch();
  return cudaGetLastError();
}

// (score, id) lists of an all-gather: [n_lists][B][k_in]
template <int KPL>
__global__ void __launch_bounds__(32) merge_lists_kernel(int B, int n_lists, int k_in, const float* __restrict__ scores,
                                                         const int64_t* __restrict__ ids, int k, float* out_score,
                                                         int64_t* out_id) {
  pdl_wait();
  const int q = blockIdx.x, lane = threadIdx.x;
  WarpTopK<KPL> m;
  m.init();
  bool bad = false;
  for (int r = 0; r < n_lists; ++r) {
    const int64_t base = (int64_t(r) * B + q) * k_in;
    for (int j0 = 0; j0 < k_in; j0 += 32) {
      uint64_t key = 0ull;
      if (j0 + lane < k_in) {
        const float sc = scores[base + j0 + lane];
        const int64_t id = ids[base + j0 + lane];
        bad |= (sc != sc);
        if (id >= 0) key = pack_key(sc, uint32_t(id));
      }
      m.offer(key, k);
    }
  }
  bad = __any_sync(0xffffffffu, bad);
#pragma unroll
  for (int s = 0; s < KPL; ++s) {
    const int j = s * 32 + lane;
    if (j < k) {
      out_score[int64_t(q) * k + j] = bad ? __int_as_float(0x7fc00000) : key_score(m.v[s]);
      out_id[int64_t(q) * k + j] = bad ? -1 : key_id(m.v[s]);
    }
  }
}

cudaError_t launch_merge_lists(int B, int n_lists, int k_in, const float* scores, const int64_t* ids, int k,
                               float* out_score, int64_t* out_id, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  if (k <= 32)
    return count_launch(), launch_pdl(merge_lists_kernel<1>, dim3(B), dim3(32), 0, s, B, n_lists, k_in, scores, ids, k, out_score, out_id);
  else
    return count_launch(), launch_pdl(merge_lists_kernel<2>, dim3(B), dim3(32), 0, s, B, n_lists, k_in, scores, ids, k, out_score, out_id);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K5 select (Eq. 4-6): kernel
// (the per-warp selection, warp_select, is in select.cuh)
template <class Tag>
__global__ void __launch_bounds__(kSelWarps * 32) select_kernel(StoreView st, int B, const int64_t* __restrict__ map_id,
                                                                const float* __restrict__ score, float delta, int K,
                                                                int lb, int T, int64_t id_offset, int64_t n_rows,
                                                                uint64_t* out_mask, int32_t* out_count, int stride,
                                                                int layer_step) {
  pdl_wait();
  __shared__ float sp[kSelWarps][kMaxE];
  __shared__ int si[kSelWarps][kMaxE];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = int64_t(blockIdx.x) * kSelWarps + warp;
  if (gw >= int64_t(B) * T) return;
  const int q = int(gw / T), tt = int(gw % T), t = lb + tt + q * layer_step;
  const int64_t id = map_id[int64_t(q) * stride];
  const int64_t loc = id - id_offset;
  const int64_t o = int64_t(q) * T + tt;
  if (id < 0 || loc < 0 || loc >= n_rows || t >= st.L) {
    if (lane == 0) { out_mask[o] = 0ull; out_count[o] = 0; }
    return;
  }
  const double dl = selection_delta(delta, score ? score[int64_t(q) * stride] : 0.f);
  uint64_t mask;
  int m;
  warp_select<Tag>(st, t, loc, dl, K, sp[warp], si[warp], &mask, &m);
  if (lane == 0) {
    out_mask[o] = mask;
    out_count[o] = m;
  }
}

cudaError_t launch_select(const StoreView& st, int B, const int64_t* map_id, const float* score, float delta, int K,
                          int layer_begin, int layer_end, int64_t id_offset, int64_t n_rows, uint64_t* out_mask,
                          int32_t* out_count, cudaStream_t s, int stride, int layer_step) {
  const int T = layer_end - layer_begin;
  const int64_t warps = int64_t(B) * T;
  if (warps <= 0) return cudaSuccess;
  const int grid = int((warps + kSelWarps - 1) / kSelWarps);
  if (st.bf16)
    return count_launch(), launch_pdl(select_kernel<Bf16Tag>, dim3(grid), dim3(kSelWarps * 32), 0, s, st, B, map_id, score,
                                      delta, K, layer_begin, T, id_offset, n_rows, out_mask, out_count, stride, layer_step);
  else
    return count_launch(), launch_pdl(select_kernel<F32Tag>, dim3(grid), dim3(kSelWarps * 32), 0, s, st, B, map_id, score,
                                      delta, K, layer_begin, T, id_offset, n_rows, out_mask, out_count, stride, layer_step);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K6 write rows
// One warp per new row: quantise (RNE), write the embedding row, its inverse
// norm (float64 accumulation of the quantised values), the map row into each
// layer slab and the prefix squared-norm table.
__device__ __forceinline__ double warp_sum_dbl(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One block per new row (rows are independent).  The embedding row is
// quantised and its squared norm reduced in float64 (fixed order: per-thread
// strided partials, then warp and block trees); each warp quantises whole
// layers of the map, reduces each layer's squared norm, and one thread forms
// the prefix sums -- deterministic, so r_e / psq are bit-reproducible.
constexpr int kWriteThreads = 256;

template <class Tag>
__global__ void __launch_bounds__(kWriteThreads) write_rows_kernel(WriteArgs w) {
  pdl_wait();
  using T = typename StoreT<Tag>::T;
  __shared__ double red[kWriteThreads / 32];
  __shared__ double lsum[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t x = blockIdx.x;
  const int64_t slot = w.slots ? w.slots[x] - w.slot_offset : w.first_slot + x;
  if (slot < 0 || slot >= w.slot_limit) return;
  T* emb = static_cast<T*>(w.emb);
  T* maps = static_cast<T*>(w.maps);
  double acc = 0.0;
  for (int e = tid; e < w.Dp; e += kWriteThreads) {
    const float v = e < w.D ? to_store_value(w.in_emb[x * w.D + e], Tag()) : 0.f;
    if constexpr (sizeof(T) == 2) emb[slot * w.Dp + e] = __float2bfloat16_rn(v);
    else emb[slot * w.Dp + e] = v;
    acc += double(v) * double(v);
  }
  acc = warp_sum_dbl(acc);
  if (lane == 0) red[warp] = acc;
  for (int l = warp; l < w.L; l += kWriteThreads / 32) {
    double a = 0.0;
    for (int j = lane; j < w.Ep; j += 32) {
      const float v = j < w.E ? to_store_value(w.in_maps[(x * w.L + l) * w.E + j], Tag()) : 0.f;
      const int64_t o = (int64_t(l) * w.cap + slot) * w.Ep + j;
      if constexpr (sizeof(T) == 2) maps[o] = __float2bfloat16_rn(v);
      else maps[o] = v;
      a += double(v) * double(v);
    }
    a = warp_sum_dbl(a);
    if (lane == 0) lsum[l] = a;
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int i = 0; i < kWriteThreads / 32; ++i) t += red[i];
    w.r_e[slot] = t > 0.0 ? float(1.0 / sqrt(t)) : 0.f;
    double cum = 0.0;
    for (int l = 0; l < w.L; ++l) {
      cum += lsum[l];
      w.psq[int64_t(l) * w.cap + slot] = float(cum);
    }
  }
}

cudaError_t launch_write_rows(const WriteArgs& w, cudaStream_t s) {
  if (w.B <= 0) return cudaSuccess;
  if (w.L > 256) return cudaErrorInvalidValue;
  count_launch();
  if (w.bf16) return launch_pdl(write_rows_kernel<Bf16Tag>, dim3(w.B), dim3(kWriteThreads), 0, s, w);
  return launch_pdl(write_rows_kernel<F32Tag>, dim3(w.B), dim3(kWriteThreads), 0, s, w);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ victim resolution (R8)
// Single warp.  Row j (batch order) takes the best-ranked candidate whose slot
// is not claimed by an earlier row.  keys hold LOCAL slots (scan id_offset 0).
__global__ void __launch_bounds__(32) resolve_kernel(int nrep, int kk, const uint64_t* __restrict__ keys,
                                                     uint32_t id_offset, int64_t* slots_all, int x0,
                                                     int64_t first_append_slot, int64_t* out_slot,
                                                     int64_t* out_replaced, int* need_full, int k_full,
                                                     const int* gate, int mark_append) {
  pdl_wait();
  if (gate && *gate == 0) return;
  __shared__ uint64_t ks[kMaxK * kMaxK];   // the candidate lists, staged once (independent, coalesced loads)
  const int lane = threadIdx.x;
  bool need = false;
  for (int i = lane; i < nrep * kk; i += 32) ks[i] = keys[i];
  __syncwarp();
  for (int x = lane; x < mark_append; x += 32) {
    slots_all[x] = first_append_slot + x;
    if (out_slot) out_slot[x] = int64_t(id_offset) + first_append_slot + x;
    if (out_replaced) out_replaced[x] = -1;
  }
  // the victims claimed so far live in registers: row i's in lane i % 32,
  // slot i / 32 (nrep <= 64); a candidate is checked against all of them by
  // one vote.  Row j walks its list in order (best first) and takes the first
  // candidate no earlier row claimed -- usually the first, so a row costs a
  // few votes instead of a j-long scan per lane.
  int64_t cl0 = -3, cl1 = -3;
  for (int j = 0; j < nrep; ++j) {
    int64_t best = -1;
    for (int c = 0; c < kk; ++c) {
      const uint64_t key = ks[j * kk + c];
      if (key == 0ull) continue;
      const int64_t loc = key_id(key);
      if (!__any_sync(0xffffffffu, cl0 == loc || cl1 == loc)) {
        best = loc;
        break;
      }
    }
    // exhausted while the list was full: the victim may lie beyond the kk keys
    if (best < 0 && k_full > kk && ks[j * kk + kk - 1] != 0ull) need = true;
    const int64_t claim = best >= 0 ? best : -2;
    if (lane == (j & 31)) {
      if (j < 32) cl0 = claim;
      else cl1 = claim;
    }
    if (lane == 0) {
      slots_all[x0 + j] = best;
      if (out_slot) out_slot[x0 + j] = best >= 0 ? int64_t(id_offset) + best : -1;
      if (out_replaced) out_replaced[x0 + j] = best >= 0 ? int64_t(id_offset) + best : -1;
    }
  }
  if (need_full && lane == 0) *need_full = need ? 1 : 0;
}

cudaError_t launch_resolve(int nrep, int kk, const uint64_t* keys, uint32_t id_offset, int64_t* slots_all, int x0,
                           int64_t first_append_slot, int64_t* out_slot, int64_t* out_replaced, cudaStream_t s,
                           int* need_full, int k_full, const int* gate, int mark_append) {
  count_launch();
  return launch_pdl(resolve_kernel, dim3(1), dim3(32), 0, s, nrep, kk, keys, id_offset, slots_all, x0,
                    first_append_slot, out_slot, out_replaced, need_full, k_full, gate,
                    mark_append < 0 ? x0 : mark_append);
  count_launch();
  return cudaGetLastError();
}

__global__ void excl_kernel(uint32_t* excl, const int64_t* __restrict__ slots, int n, int64_t offset, int64_t limit,
                            int set) {
  pdl_wait();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int64_t v = slots[x] - offset;
  if (slots[x] < 0 || v < 0 || v >= limit) return;
  const uint32_t bit = 1u << (v & 31);
  if (set) atomicOr(excl + (v >> 5), bit);
  else atomicAnd(excl + (v >> 5), ~bit);
}

cudaError_t launch_excl(uint32_t* excl, const int64_t* slots, int n, int64_t offset, int64_t limit, int set,
                        cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  return launch_pdl(excl_kernel, dim3((n + 127) / 128), dim3(128), 0, s, excl, slots, n, offset, limit, set);
}

__global__ void __launch_bounds__(32) resolve_ids_kernel(int B, int k, const int64_t* __restrict__ ids,
                                                         int64_t* out_victim) {
  pdl_wait();
  const int lane = threadIdx.x;
  // claims in registers (row i in lane i % 32, slot i / 32; B <= 64), one vote per candidate (as resolve_kernel)
  int64_t cl0 = -3, cl1 = -3;
  for (int j = 0; j < B; ++j) {
    int64_t best = -1;
    for (int c = 0; c < k; ++c) {
      const int64_t id = ids[int64_t(j) * k + c];
      if (id < 0) continue;
      if (!__any_sync(0xffffffffu, cl0 == id || cl1 == id)) {
        best = id;
        break;
      }
    }
    const int64_t claim = best >= 0 ? best : -2;
    if (lane == (j & 31)) {
      if (j < 32) cl0 = claim;
      else cl1 = claim;
    }
    if (lane == 0) out_victim[j] = best;
  }
}

cudaError_t launch_resolve_ids(int B, int k, const int64_t* ids, int64_t* out_victim, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  count_launch();
  return launch_pdl(resolve_ids_kernel, dim3(1), dim3(32), 0, s, B, k, ids, out_victim);
}

__global__ void append_ids_kernel(int n, int64_t first_slot, uint32_t id_offset, int64_t* out_slot,
                                  int64_t* out_replaced) {
  pdl_wait();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  if (out_slot) out_slot[x] = int64_t(id_offset) + first_slot + x;
  if (out_replaced) out_replaced[x] = -1;
}

cudaError_t launch_append_ids(int n, int64_t first_slot, uint32_t id_offset, int64_t* out_slot, int64_t* out_replaced,
                              cudaStream_t s) {
  if (n <= 0 || (!out_slot && !out_replaced)) return cudaSuccess;
  count_launch();
  return launch_pdl(append_ids_kernel, dim3((n + 255) / 256), dim3(256), 0, s, n, first_slot, id_offset, out_slot,
                    out_replaced);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ read back
template <class Tag>
__global__ void read_rows_kernel(StoreView st, int64_t slot0, int64_t count, float* out_emb, float* out_maps) {
  pdl_wait();
  using T = typename StoreT<Tag>::T;
  const T* emb = static_cast<const T*>(st.emb);
  const T* maps = static_cast<const T*>(st.maps);
  const int64_t ne = out_emb ? count * st.D : 0;
  const int64_t nm = out_maps ? count * st.L * st.E : 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < ne + nm; i += int64_t(gridDim.x) * blockDim.x) {
    if (i < ne) {
      const int64_t r = i / st.D, e = i % st.D;
      out_emb[i] = float(emb[(slot0 + r) * st.Dp + e]);
    } else {
      const int64_t k = i - ne;
      const int64_t r = k / (int64_t(st.L) * st.E), rem = k % (int64_t(st.L) * st.E);
      const int l = int(rem / st.E), j = int(rem % st.E);
      out_maps[k] = float(maps[(int64_t(l) * st.cap + slot0 + r) * st.Ep + j]);
    }
  }
}

cudaError_t launch_read_rows(const StoreView& st, int64_t slot0, int64_t count, float* out_emb, float* out_maps,
                             cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int grid = 592;
  if (st.bf16) read_rows_kernel<Bf16Tag><<<grid, 256, 0, s>>>(st, slot0, count, out_emb, out_maps);
  else read_rows_kernel<F32Tag><<<grid, 256, 0, s>>>(st, slot0, count, out_emb, out_maps);
  count_launch();
  return cudaGetLastError();
}

}  // namespace fmoe

// ------------------------------------------------------------------ debug: phase tracer
namespace fmoe {
static unsigned long long* g_trace_buf = nullptr;
unsigned long long* trace_buffer() { return g_trace_buf; }
}  // namespace fmoe

// enable > 0: allocate + zero the buffer and trace subsequent scans; enable == 0:
// stop tracing; enable < 0: leave as is.  out (host, [max_blocks][8] u64), if
// given, receives the buffer (device-synchronous).  Not part of the product ABI.
extern "C" int fmoe_debug_trace(int enable, unsigned long long* out, int max_blocks) {
  using namespace fmoe;
  const size_t bytes = size_t(kTraceBlocks) * kTracePhases * 8;
  if (enable > 0) {
    if (!g_trace_buf && cudaMalloc(&g_trace_buf, bytes) != cudaSuccess) return -1;
    if (cudaMemset(g_trace_buf, 0, bytes) != cudaSuccess) return -1;
  }
  if (out && g_trace_buf) {
    const int nb = max_blocks < kTraceBlocks ? max_blocks : kTraceBlocks;
    if (cudaMemcpy(out, g_trace_buf, size_t(nb) * kTracePhases * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  }
  if (enable == 0 && g_trace_buf) {
    cudaDeviceSynchronize();
    cudaFree(g_trace_buf);
    g_trace_buf = nullptr;
  }
  return 0;
}

// ------------------------------------------------------------------ expert-cache priorities
namespace fmoe {

struct PlanJob {
  double pri;
  int tie;      // ascending secondary order (prefetch: layer*64 + expert; eviction: cache index)
};

__device__ __forceinline__ bool job_before(const PlanJob& a, const PlanJob& b) {
  return a.pri > b.pri || (a.pri == b.pri && a.tie < b.tie);
}

// block-wide bitonic sort of n2 (a power of two) entries into "before" order
__device__ void bitonic_sort(PlanJob* v, int n2) {
  for (int size = 2; size <= n2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const PlanJob a = v[lo], b = v[hi];
        if (up ? job_before(b, a) : job_before(a, b)) {
          v[lo] = b;
          v[hi] = a;
        }
      }
    }
  __syncthreads();
}

constexpr int kPlanThreads = 256;
constexpr int kPlanMax = 2048;

// One CTA per query: the Eq. 4-6 sets of the target layers (warp per layer,
// warp_select), PRI^prefetch = p / (t - l_now) in float64, one bitonic sort.
template <class Tag>
__global__ void __launch_bounds__(kPlanThreads) plan_kernel(StoreView st, const int64_t* __restrict__ map_id,
                                                            const float* __restrict__ score, float delta, int K,
                                                            int l_now, int lb, int T, int64_t id_offset,
                                                            int64_t n_rows, int max_jobs, int32_t* out_layer,
                                                            int32_t* out_expert, double* out_pri, int32_t* out_njobs) {
  pdl_wait();
  __shared__ PlanJob jobs[kPlanMax];
  __shared__ float sp[kPlanThreads / 32][kMaxE];
  __shared__ int si[kPlanThreads / 32][kMaxE];
  __shared__ int nj_sh;
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = st.E, n = T * E;
  int n2 = 2;
  while (n2 < n) n2 <<= 1;
  for (int i = tid; i < n2; i += kPlanThreads) jobs[i] = PlanJob{-__longlong_as_double(0x7ff0000000000000ll), (1 << 30) + i};
  if (tid == 0) nj_sh = 0;
  __syncthreads();
  const int64_t id = map_id[q], loc = id - id_offset;
  if (id >= 0 && loc >= 0 && loc < n_rows) {
    const double dl = selection_delta(delta, score ? score[q] : 0.f);
    for (int tt = warp; tt < T; tt += kPlanThreads / 32) {
      const int t = lb + tt;
      uint64_t mask;
      int m;
      warp_select<Tag>(st, t, loc, dl, K, sp[warp], si[warp], &mask, &m);
      for (int r = lane; r < m; r += 32) {
        const int j = si[warp][r];
        jobs[tt * E + j] = PlanJob{double(sp[warp][r]) / double(t - l_now), t * 64 + j};
      }
      if (lane == 0) atomicAdd(&nj_sh, m);
      __syncwarp();
    }
  }
  bitonic_sort(jobs, n2);
  const int nj = nj_sh < max_jobs ? nj_sh : max_jobs;
  for (int i = tid; i < max_jobs; i += kPlanThreads) {
    const bool ok = i < nj;
    out_layer[int64_t(q) * max_jobs + i] = ok ? (jobs[i].tie >> 6) : -1;
    out_expert[int64_t(q) * max_jobs + i] = ok ? (jobs[i].tie & 63) : -1;
    out_pri[int64_t(q) * max_jobs + i] = ok ? jobs[i].pri : 0.0;
  }
  if (tid == 0) out_njobs[q] = nj;
}

cudaError_t launch_prefetch_plan(const StoreView& st, int B, const int64_t* map_id, const float* score, float delta,
                                 int K, int l_now, int lb, int le, int64_t id_offset, int64_t n_rows, int max_jobs,
                                 int32_t* out_layer, int32_t* out_expert, double* out_pri, int32_t* out_njobs,
                                 cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  count_launch();
  if (st.bf16)
    return launch_pdl(plan_kernel<Bf16Tag>, dim3(B), dim3(kPlanThreads), 0, s, st, map_id, score, delta, K, l_now, lb,
                      le - lb, id_offset, n_rows, max_jobs, out_layer, out_expert, out_pri, out_njobs);
  return launch_pdl(plan_kernel<F32Tag>, dim3(B), dim3(kPlanThreads), 0, s, st, map_id, score, delta, K, l_now, lb,
                    le - lb, id_offset, n_rows, max_jobs, out_layer, out_expert, out_pri, out_njobs);
}

constexpr int kEvictThreads = 1024;

// One CTA: PRI^evict = 1 / (max(p, eps) * freq) in float64 and the eviction order.
__global__ void __launch_bounds__(kEvictThreads) evict_kernel(int n, const float* __restrict__ p,
                                                              const float* __restrict__ freq, float eps,
                                                              double* out_pri, int32_t* out_order) {
  pdl_wait();
  extern __shared__ PlanJob v[];
  int n2 = 2;
  while (n2 < n) n2 <<= 1;
  for (int i = threadIdx.x; i < n2; i += kEvictThreads) {
    if (i < n) {
      const double pp = double(p[i]) > double(eps) ? double(p[i]) : double(eps);
      const double pri = 1.0 / (pp * double(freq[i]));
      out_pri[i] = pri;
      v[i] = PlanJob{pri, i};
    } else {
      v[i] = PlanJob{-__longlong_as_double(0x7ff0000000000000ll), (1 << 30) + i};
    }
  }
  bitonic_sort(v, n2);
  for (int i = threadIdx.x; i < n; i += kEvictThreads) out_order[i] = v[i].tie;
}

cudaError_t launch_eviction_order(int n, const float* p, const float* freq, float eps, double* out_pri,
                                  int32_t* out_order, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int n2 = 2;
  while (n2 < n) n2 <<= 1;
  const size_t smem = size_t(n2) * sizeof(PlanJob);
  cudaError_t e = cudaFuncSetAttribute(evict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  count_launch();
  return launch_pdl(evict_kernel, dim3(1), dim3(kEvictThreads), smem, s, n, p, freq, eps, out_pri, out_order);
}

// ------------------------------------------------------------------ expert hits
// One warp per (query, layer) row of the observed gate: the K activated experts
// are the ranks < K under (p desc, index asc) -- the rank computation of
// warp_select -- collected with two ballots; hits = popcount(active & prefetched).
__global__ void __launch_bounds__(kSelWarps * 32) hits_kernel(int64_t rows, int E, int K, const float* __restrict__ gate,
                                                              const uint64_t* __restrict__ pmask,
                                                              uint64_t* __restrict__ out_active,
                                                              int32_t* __restrict__ out_hits) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * kSelWarps + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float* g = gate + r * E;
  const float NEG = -__int_as_float(0x7f800000);
  const float p0 = lane < E ? __ldg(g + lane) : NEG;
  const float p1 = lane + 32 < E ? __ldg(g + lane + 32) : NEG;
  int r0 = 0, r1 = 0;
  for (int j = 0; j < E; ++j) {
    const float a = __shfl_sync(0xffffffffu, p0, j & 31);
    const float b = __shfl_sync(0xffffffffu, p1, j & 31);
    const float pj = j < 32 ? a : b;
    r0 += (pj > p0) || (pj == p0 && j < lane);
    r1 += (pj > p1) || (pj == p1 && j < lane + 32);
  }
  const uint32_t lo = __ballot_sync(0xffffffffu, lane < E && r0 < K);
  const uint32_t hi = __ballot_sync(0xffffffffu, lane + 32 < E && r1 < K);
  if (lane == 0) {
    const uint64_t act = (uint64_t(hi) << 32) | lo;
    if (out_active) out_active[r] = act;
    out_hits[r] = __popcll(act & pmask[r]);
  }
  pdl_trigger();
}

cudaError_t launch_expert_hits(int64_t rows, int E, int K, const float* gate, const uint64_t* pmask,
                               uint64_t* out_active, int32_t* out_hits, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  count_launch();
  const unsigned grid = unsigned((rows + kSelWarps - 1) / kSelWarps);
  return launch_pdl(hits_kernel, dim3(grid), dim3(kSelWarps * 32), 0, s, rows, E, K, gate, pmask, out_active,
                    out_hits);
}

}  // namespace fmoe
