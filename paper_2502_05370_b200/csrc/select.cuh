// select.cuh -- the Eq. 4-6 selection of one (query, layer) by one warp,
// shared by the select kernel (select_insert.cu) and the fused selection at
// the end of a trajectory-session step (traj_session.cu).
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace fmoe {

// ------------------------------------------------------------------ K5 select (Eq. 4-6)
// One warp per (query, target layer).  The E <= 64 probabilities of the
// matched row are ranked by (p desc, index asc) in registers (each lane owns
// entries lane and lane+32), scattered into shared memory in rank order, and
// one lane accumulates them in float64 in that order -- the exact order and
// precision of the oracle, so sets are bit-identical given the same score.
constexpr int kSelWarps = 8;

template <class Tag>
__device__ __forceinline__ float load_p(const StoreView& st, int t, int64_t row, int j) {
  using T = typename StoreT<Tag>::T;
  const T* m = static_cast<const T*>(st.maps);
  if constexpr (sizeof(T) == 2)
    return __bfloat162float(m[(int64_t(t) * st.cap + row) * st.Ep + j]);
  else
    return m[(int64_t(t) * st.cap + row) * st.Ep + j];
}

// delta = Clip(1 - score, 0, 1) in float64 (score clamped to [-1, 1], NaN -> 1), or the fixed delta
__device__ __forceinline__ double selection_delta(float delta, float s) {
  if (delta >= 0.f) return double(delta);
  if (s != s) return 1.0;
  double sd = double(s);
  sd = sd < -1.0 ? -1.0 : (sd > 1.0 ? 1.0 : sd);
  const double v = 1.0 - sd;
  return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
}

// Eq. 4-6 for row `loc`, layer t, by one warp: rank the E <= 64 probabilities
// by (p desc, index asc) in registers, scatter them in rank order to the warp's
// scratch sp/si, and accumulate in float64 in that order on lane 0 (the order
// and precision of the oracle).  Returns (on every lane) the mask and count;
// sp/si[0..count) then hold the picked experts in selection order.
template <class Tag>
__device__ __forceinline__ void warp_select(const StoreView& st, int t, int64_t loc, double dl, int K, float* sp,
                                            int* si, uint64_t* mask_out, int* count_out) {
  const int lane = threadIdx.x & 31;
  const int E = st.E;
  const float NEG = -__int_as_float(0x7f800000);
  const float p0 = lane < E ? load_p<Tag>(st, t, loc, lane) : NEG;
  const float p1 = lane + 32 < E ? load_p<Tag>(st, t, loc, lane + 32) : NEG;
  int r0 = 0, r1 = 0;
  for (int j = 0; j < E; ++j) {
    const float a = __shfl_sync(0xffffffffu, p0, j & 31);
    const float b = __shfl_sync(0xffffffffu, p1, j & 31);
    const float pj = j < 32 ? a : b;
    r0 += (pj > p0) || (pj == p0 && j < lane);
    r1 += (pj > p1) || (pj == p1 && j < lane + 32);
  }
  if (lane < E) { sp[r0] = p0; si[r0] = lane; }
  if (lane + 32 < E) { sp[r1] = p1; si[r1] = lane + 32; }
  __syncwarp();
  uint64_t mask = 0ull;
  int m = E;
  if (lane == 0) {
    double cum = 0.0;
    for (int r = 0; r < E; ++r) {
      cum = cum + double(sp[r]);
      if (cum >= dl && r + 1 >= K) { m = r + 1; break; }
    }
    for (int r = 0; r < m; ++r) mask |= 1ull << si[r];
  }
  *mask_out = shfl_u64(mask, 0);
  *count_out = __shfl_sync(0xffffffffu, m, 0);
}

}  // namespace fmoe
