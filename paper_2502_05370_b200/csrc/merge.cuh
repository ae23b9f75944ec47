// merge.cuh -- the tail shared by every scan kernel: block merge of the warps'
// top-k lists, then a grid merge by the last block to finish (ticket counter),
// which writes the call's outputs.  No extra launch, no host round trip.
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace fmoe {

// All NW*32 threads of the block call this.  sk: shared scratch of at least
// NW*NQ*k u64 keys.  s_valid[q]: query q has non-zero norms.
template <int NQ, int KPL, int NW>
__device__ __forceinline__ void finish_topk(WarpTopK<KPL> (&lists)[NQ], uint64_t* sk, const ScanArgs& a,
                                            const int* s_valid, int* s_last) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = a.k;
  if (k == 1) {
    // argmax: warp bests -> block best -> one atomicMax per query; the last
    // block converts the winning key (4 dependent memory ops instead of a
    // grid-wide list merge)
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint64_t b = lists[q].get(0);
      if (lane == 0) sk[warp * NQ + q] = b;
    }
    __syncthreads();
    if (tid < a.nq) {
      uint64_t b = 0ull;
      for (int w2 = 0; w2 < NW; ++w2) b = b > sk[w2 * NQ + tid] ? b : sk[w2 * NQ + tid];
      if (b) atomicMax(a.best + a.q0 + tid, static_cast<unsigned long long>(b));
    }
    __threadfence();
    __syncthreads();
    trace_mark(a.trace, 4);
    if (tid == 0) *s_last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!*s_last) return;
    trace_mark(a.trace, 5);
    __threadfence();
    if (tid < a.nq) {
      const int q = tid;
      const uint64_t key = __ldcg(a.best + a.q0 + q);
      a.best[a.q0 + q] = 0ull;
      const bool valid = !a.check_valid || s_valid[q];
      const int64_t ob = int64_t(a.q0 + q);
      if (a.out_keys) a.out_keys[ob] = valid ? key : 0ull;
      if (a.out_score) a.out_score[ob] = valid ? key_score(key) : __int_as_float(0x7fc00000);
      if (a.out_id) a.out_id[ob] = valid ? key_id(key) : -1;
    }
    if (tid == 0) *a.counter = 0u;
    trace_mark(a.trace, 6);
    return;
  }
  if constexpr (KPL > 0) {
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NQ; ++q) lists[q].store(sk + (warp * NQ + q) * k, k);
  __syncthreads();
  // block merge: warp q merges query q over the NW warps
  if (warp < a.nq) {
    const int q = warp;
    WarpTopK<KPL> m;
#pragma unroll
    for (int s = 0; s < KPL; ++s) {
      const int j = s * 32 + lane;
      m.v[s] = j < k ? sk[q * k + j] : 0ull;
    }
    for (int w2 = 1; w2 < NW; ++w2)
      for (int j0 = 0; j0 < k; j0 += 32) {
        const uint64_t key = (j0 + lane < k) ? sk[(w2 * NQ + q) * k + j0 + lane] : 0ull;
        m.offer(key, k);
      }
    m.store(a.cand + (int64_t(a.q0 + q) * a.grid + blockIdx.x) * k, k);
  }
  // grid merge: the last block to finish merges every block's lists
  __threadfence();
  __syncthreads();
  trace_mark(a.trace, 4);
  if (tid == 0) *s_last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!*s_last) return;
  trace_mark(a.trace, 5);
  __threadfence();
  constexpr int WPQ = NW / NQ;   // warps per query
  const int q = warp / WPQ, wpart = warp % WPQ;
  WarpTopK<KPL> m;
  m.init();
  if (q < a.nq) {
    const uint64_t* src = a.cand + int64_t(a.q0 + q) * a.grid * k;
    const int64_t total = int64_t(a.grid) * k;
    const int64_t j = int64_t(wpart) * 32 + lane;
    uint64_t nxt = j < total ? __ldcg(reinterpret_cast<const unsigned long long*>(src + j)) : 0ull;
    for (int64_t j0 = int64_t(wpart) * 32; j0 < total; j0 += WPQ * 32) {
      const uint64_t cur = nxt;
      const int64_t jn = j0 + WPQ * 32 + lane;
      nxt = jn < total ? __ldcg(reinterpret_cast<const unsigned long long*>(src + jn)) : 0ull;
      m.offer(cur, k);
    }
  }
  if (warp < WPQ * NQ) m.store(sk + warp * k, k);
  __syncthreads();
  if (q < a.nq && wpart == 0) {
    for (int p2 = 1; p2 < WPQ; ++p2)
      for (int j0 = 0; j0 < k; j0 += 32) {
        const uint64_t key = (j0 + lane < k) ? sk[(warp + p2) * k + j0 + lane] : 0ull;
        m.offer(key, k);
      }
    const bool valid = !a.check_valid || s_valid[q];
    const int64_t ob = int64_t(a.q0 + q) * k;
#pragma unroll
    for (int s = 0; s < KPL; ++s) {
      const int jj = s * 32 + lane;
      if (jj < k) {
        const uint64_t key = m.v[s];
        if (a.out_keys) a.out_keys[ob + jj] = valid ? key : 0ull;
        if (a.out_score) a.out_score[ob + jj] = valid ? key_score(key) : __int_as_float(0x7fc00000);
        if (a.out_id) a.out_id[ob + jj] = valid ? key_id(key) : -1;
      }
    }
  }
  if (tid == 0) *a.counter = 0u;
  trace_mark(a.trace, 6);
  }  // KPL > 0
}

}  // namespace fmoe
