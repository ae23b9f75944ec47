// rerank.cu -- exact re-rank of the tensor-core semantic scan's candidates.
//
// The tcgen05 semantic scan (approx mode, scan_umma.cu) accumulates each dot
// over D/16 MMAs in ONE TMEM accumulator; tcgen05 fp32 accumulation truncates
// per MMA, so its scores carry an error of up to ~n_mma * 2^-23 (measured
// 1.4e-5 at D = 4096, P:461-466 scores are cosines in [-1, 1]).  Instead of
// splitting K over two accumulators (which takes the TMEM double buffer), the
// scan keeps k_ext > k candidates per query by approximate score and this
// kernel recomputes Eq. 1 for them exactly:
//   score = (sum_i q~_i e~_i in float64) / ||q~|| * r_e[y]
// (q~ the bf16 query, e~ the stored bf16 row: every product is exact), sorts
// them by (score desc, id asc) and writes the top k.
//
// Verification: every row outside the candidate list has approximate score
// <= a_last (the k_ext-th candidate's), so its exact score is <= a_last + eps,
// eps = the approximation bound.  If a_last + eps < s_k (the k-th exact
// score) the exact top-k is complete; otherwise (near-ties across the list
// boundary, e.g. more than k_ext duplicates of one row) the query is queued
// for the exact GEMV scan (fallback), whose results replace the re-rank's.
#include "common.cuh"
#include "kernels.cuh"

namespace fmoe {

constexpr int kRerankThreads = 256;
constexpr int kRerankWarps = kRerankThreads / 32;

__global__ void __launch_bounds__(kRerankThreads) rerank_kernel(const RerankArgs r) {
  extern __shared__ __align__(16) float qv[];          // [Dp] the bf16 query as fp32
  __shared__ uint64_t ck[kMaxK], ek[kMaxK], sorted[kMaxK];
  __shared__ double red[kRerankWarps];
  __shared__ double s_qn;
  __shared__ int s_slot;
  pdl_wait();
  const int x = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int D = r.D, Dp = r.Dp, ke = r.ke, k = r.k;
  double part = 0.0;
  for (int e = tid; e < Dp; e += kRerankThreads) {
    const float v = e < D ? __bfloat162float(__float2bfloat16_rn(r.q_emb[int64_t(x) * D + e])) : 0.f;
    qv[e] = v;
    part += double(v) * double(v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[warp] = part;
  if (tid < kMaxK) {
    ck[tid] = tid < ke ? r.keys[int64_t(x) * ke + tid] : 0ull;
    sorted[tid] = 0ull;
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kRerankWarps; ++w) t += red[w];
    s_qn = t;
    s_slot = -1;
  }
  __syncthreads();
  const double rq = s_qn > 0.0 ? 1.0 / sqrt(s_qn) : 0.0;
  const __nv_bfloat16* emb = static_cast<const __nv_bfloat16*>(r.emb);
  for (int j = warp; j < ke; j += kRerankWarps) {
    const uint64_t key = ck[j];
    if (key == 0ull) {
      if (lane == 0) ek[j] = 0ull;
      continue;
    }
    const int64_t gid = key_id(key);
    const int64_t y = gid - int64_t(r.id_offset);
    const uint4* row = reinterpret_cast<const uint4*>(emb + y * Dp);
    double dot = 0.0;
    for (int c = lane; c < Dp / 8; c += 32) {
      float f[8];
      unpack8(__ldg(row + c), f, Bf16Tag());
#pragma unroll
      for (int i = 0; i < 8; ++i) dot = fma(double(f[i]), double(qv[c * 8 + i]), dot);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) ek[j] = pack_key(float(dot * rq * double(__ldg(r.r_e + y))), uint32_t(gid));
  }
  __syncthreads();
  if (tid < ke && ek[tid] != 0ull) {             // keys are distinct (distinct ids): rank sort
    const uint64_t v = ek[tid];
    int rank = 0;
    for (int i = 0; i < ke; ++i) rank += ek[i] > v ? 1 : 0;
    sorted[rank] = v;
  }
  __syncthreads();
  const bool valid = r.valid == nullptr || r.valid[x] != 0.f;
  if (tid < k) {
    const uint64_t key = valid ? sorted[tid] : 0ull;
    const int64_t o = int64_t(x) * k + tid;
    if (r.out_keys) r.out_keys[o] = key;
    if (r.out_score) r.out_score[o] = valid ? key_score(key) : __int_as_float(0x7fc00000);
    if (r.out_id) r.out_id[o] = valid ? key_id(key) : -1;
  }
  if (tid == 0 && valid) {
    int nv = 0;
    for (int i = 0; i < ke; ++i) nv += ck[i] != 0ull ? 1 : 0;
    // list not full: every stored row is a candidate
    const bool complete = nv < ke || (sorted[k - 1] != 0ull &&
                                      key_score(ck[ke - 1]) + r.eps < key_score(sorted[k - 1]));
    if (!complete) {
      const int slot = atomicAdd(r.nfail, 1);
      r.qmap[slot] = x;
      s_slot = slot;
    }
  }
  __syncthreads();
  if (s_slot >= 0)
    for (int e = tid; e < D; e += kRerankThreads) r.qc[int64_t(s_slot) * D + e] = r.q_emb[int64_t(x) * D + e];
  pdl_trigger();
}

// Results of the fallback scan (compacted slots) -> the queries' output rows;
// resets the failure count for the next call.
__global__ void __launch_bounds__(256) rerank_scatter_kernel(const int* nfail_p, const int* qmap, int k,
                                                             const float* fb_s, const int64_t* fb_i,
                                                             const uint64_t* fb_keys, float* out_score,
                                                             int64_t* out_id, uint64_t* out_keys, int* nfail_w) {
  pdl_wait();
  const int nfail = *nfail_p;
  for (int t = threadIdx.x; t < nfail * k; t += blockDim.x) {
    const int slot = t / k, j = t - slot * k;
    const int64_t o = int64_t(qmap[slot]) * k + j, f = int64_t(slot) * k + j;
    if (out_keys) out_keys[o] = fb_keys[f];
    if (out_score) out_score[o] = fb_s[f];
    if (out_id) out_id[o] = fb_i[f];
  }
  __syncthreads();
  if (threadIdx.x == 0) *nfail_w = 0;
  pdl_trigger();
}

cudaError_t launch_rerank(const RerankArgs& r, cudaStream_t s) {
  const size_t smem = size_t(r.Dp) * 4;
  static size_t set = 0;
  if (smem > 48 * 1024 && smem > set) {
    cudaError_t e = cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    set = smem;
  }
  count_launch();
  return launch_pdl(rerank_kernel, dim3(r.B), dim3(kRerankThreads), smem, s, r);
}

cudaError_t launch_rerank_scatter(const int* nfail, const int* qmap, int k, const float* fb_s, const int64_t* fb_i,
                                  const uint64_t* fb_keys, float* out_score, int64_t* out_id, uint64_t* out_keys,
                                  int* nfail_w, cudaStream_t s) {
  count_launch();
  return launch_pdl(rerank_scatter_kernel, dim3(1), dim3(256), 0, s, nfail, qmap, k, fb_s, fb_i, fb_keys, out_score,
                    out_id, out_keys, nfail_w);
}

}  // namespace fmoe
