// traj_session.cu -- incremental trajectory search.
//
// A request observes its gate distributions layer by layer; after layer ell
// the trajectory search (Eq. 2) scores the prefix 1..ell.  The
// stateless call re-reads ell slabs per row; a session keeps, per query and
// per stored row, the running dot product  acc[q][y] = sum_{l<ell} q_l . M_y,l
// (fp32, the same sequential accumulation order as the stateless GEMV), so
// step ell reads one 16..256-byte slab row + 4 bytes of accumulator per query
// and writes the accumulator back:
//   score = acc * r_q(ell) / sqrt(psq[ell-1][y])
// with r_q(ell) from a running float64 sum of the query's squared entries and
// psq the store's prefix squared-norm table.  The result is Eq. 2 at prefix ell
// (summation order differs only in the prefix norm, taken from the table).
//
// Mapping: GT lanes per row (GT = 16-byte chunks per slab row, power of two),
// 32/GT rows per pass, PASSES passes per warp iteration so a lane keeps 8
// slab loads in flight; fused top-k via merge.cuh.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"
#include "merge.cuh"
#include "select.cuh"

namespace fmoe {

constexpr int kSessThreads = 256;
constexpr int kSessWarps = kSessThreads / 32;
constexpr int kPasses = 8;

template <class Tag>
__device__ __forceinline__ void unpack_sess(const uint4& u, float (&x)[8]) {
  if constexpr (StoreT<Tag>::kBytes == 2) {
    unpack8(u, x, Bf16Tag());
  } else {
    x[0] = __uint_as_float(u.x); x[1] = __uint_as_float(u.y);
    x[2] = __uint_as_float(u.z); x[3] = __uint_as_float(u.w);
    x[4] = x[5] = x[6] = x[7] = 0.f;
  }
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int pow2_at_least(int c) {
  int g = 1;
  while (g < c) g <<= 1;
  return g;
}

template <class Tag, int NQ, int KPL>
__global__ void __launch_bounds__(kSessThreads, NQ == 1 ? 4 : 2) traj_session_kernel(const ScanArgs a, SessionArgs s) {
  using ST = StoreT<Tag>;
  constexpr int EP = ST::kElemsPer16B;
  constexpr int SB = ST::kBytes;
  __shared__ __align__(16) float qs[NQ][kMaxE];   // layer ell-1 of the queries (store dtype values)
  __shared__ double red[kSessWarps][NQ];
  __shared__ float rq[NQ];
  __shared__ int s_valid[NQ];
  __shared__ int s_last;
  __shared__ __align__(16) uint64_t sk[kSessWarps * NQ * kMaxK];

  const StoreView& st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Ep = st.Ep, E = st.E, layer = s.layer;   // 0-based layer consumed by this step
  trace_mark(a.trace, 0);
  pdl_wait();
  trace_mark(a.trace, 1);

  // ---- the new layer of each query, and the running query norm
  double part[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    part[q] = 0.0;
    for (int j = tid; j < kMaxE; j += kSessThreads) {
      float v = 0.f;
      if (q < a.nq && j < E) v = to_store_value(s.q_layer[int64_t(a.q0 + q) * E + j], Tag());
      qs[q][j] = v;
      part[q] += double(v) * double(v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
    if (lane == 0) red[warp][q] = part[q];
  }
  __syncthreads();
  if (tid < NQ) {
    double t = layer > 0 ? s.qn_prev[a.q0 + tid] : 0.0;
    for (int w = 0; w < kSessWarps; ++w) t += red[w][tid];
    rq[tid] = t > 0.0 ? float(1.0 / sqrt(t)) : 0.f;
    // an abandoned sweep left the accumulators half-updated: no valid result
    // until the session is reset
    s_valid[tid] = t > 0.0 && !(s.abort && ld_acquire_u32(s.abort) != 0u);
    if (blockIdx.x == 0 && tid < a.nq) s.qn_next[a.q0 + tid] = t;   // double-buffered: others read qn_prev
  }
  __syncthreads();
  trace_mark(a.trace, 2);
  float rq_r[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) rq_r[q] = rq[q];

  WarpTopK<KPL> lists[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) lists[q].init();

  const int CPY = Ep / EP;                      // 16-byte chunks per slab row
  const int GT = pow2_at_least(CPY);
  const int rpp = 32 / GT, g = lane / GT, cl = lane % GT;
  const bool lead = cl == 0;
  const int64_t n = a.n_rows, cap = st.cap;
  const char* slab = static_cast<const char*>(st.maps) + int64_t(layer) * cap * Ep * SB;
  const float* psq = st.psq + int64_t(layer) * cap;
  const int64_t rows_per_iter = int64_t(rpp) * kPasses;
  const int64_t wg = int64_t(blockIdx.x) * kSessWarps + warp;
  // this warp's rows: one contiguous range, equal for every warp of the grid
  const int64_t r0 = wg * s.rpw;
  const int64_t r1 = r0 + s.rpw < n ? r0 + s.rpw : n;

  for (int64_t base = r0; base < r1; base += rows_per_iter) {
    uint4 buf[kPasses];
#pragma unroll
    for (int p = 0; p < kPasses; ++p) {
      const int64_t row = base + p * rpp + g;
      buf[p] = (row < r1 && cl < CPY) ? ld_stream(slab + row * Ep * SB + cl * 16) : make_uint4(0u, 0u, 0u, 0u);
    }
    float accv[kPasses][NQ], ps[kPasses];
#pragma unroll
    for (int p = 0; p < kPasses; ++p) {
      const int64_t row = base + p * rpp + g;
      const bool ok = lead && row < r1;
      ps[p] = ok ? __ldcs(psq + row) : 0.f;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        accv[p][q] = (ok && layer > 0 && q < a.nq) ? __ldcs(s.acc + int64_t(a.q0 + q) * cap + row) : 0.f;
    }
#pragma unroll
    for (int p = 0; p < kPasses; ++p) {
      float x[8];
      unpack_sess<Tag>(buf[p], x);
      float d[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        d[q] = 0.f;
        if (cl < CPY) {
#pragma unroll
          for (int e = 0; e < EP; ++e) d[q] = fmaf(x[e], qs[q][cl * EP + e], d[q]);
        }
        for (int o = GT >> 1; o > 0; o >>= 1) d[q] += __shfl_xor_sync(0xffffffffu, d[q], o);
      }
      const int64_t row = base + p * rpp + g;
      const bool ok = lead && row < r1;
      const float rm = ps[p] > 0.f ? rsqrtf(ps[p]) : 0.f;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float acc = accv[p][q] + d[q];
        if (ok && q < a.nq) __stcs(s.acc + int64_t(a.q0 + q) * cap + row, acc);
        const float sc = acc * rq_r[q] * rm;
        lists[q].offer(ok ? pack_key(sc, a.id_offset + uint32_t(row)) : 0ull, a.k);
      }
    }
  }
  trace_mark(a.trace, 3);
  pdl_trigger();
  finish_topk<NQ, KPL, kSessWarps>(lists, sk, a, s_valid, &s_last);
  if (s.sel_T <= 0) return;
  // ---- fused selection (Eq. 4-6) on the final top-1 of each query,
  // by the block that wrote it (its writes are visible after the barrier): one
  // warp per (query, target layer), the same warp_select as the select kernel
  __syncthreads();
  if (!s_last) return;
  __shared__ float sel_p[kSessWarps][kMaxE];
  __shared__ int sel_i[kSessWarps][kMaxE];
  for (int w = warp; w < a.nq * s.sel_T; w += kSessWarps) {
    const int q = w / s.sel_T, tt = w - q * s.sel_T;
    const int64_t ob = int64_t(a.q0 + q);
    const int64_t id = a.out_id[ob * a.k];
    const int64_t loc = id - int64_t(a.id_offset);
    const int64_t o = ob * s.sel_T + tt;
    if (id < 0 || loc < 0 || loc >= a.n_rows) {
      if (lane == 0) { s.sel_mask[o] = 0ull; s.sel_count[o] = 0; }
      continue;
    }
    const double dl = selection_delta(s.sel_delta, a.out_score[ob * a.k]);
    uint64_t mask;
    int m;
    warp_select<Tag>(st, s.sel_lb + tt, loc, dl, s.sel_K, sel_p[warp], sel_i[warp], &mask, &m);
    if (lane == 0) { s.sel_mask[o] = mask; s.sel_count[o] = m; }
    __syncwarp();
  }
}

cudaError_t launch_traj_session(const ScanArgs& a, const SessionArgs& s, cudaStream_t stream) {
  using Fn = void (*)(const ScanArgs, SessionArgs);
  Fn fn;
  const int NQ = a.nq <= 1 ? 1 : (a.nq <= 2 ? 2 : 4);
  const int kp = a.k == 1 ? 0 : (a.k <= 32 ? 1 : 2);
#define FMOE_SESS_PICK(TAG)                                                                          \
  if (NQ == 1) fn = kp == 0 ? traj_session_kernel<TAG, 1, 0> : kp == 1 ? traj_session_kernel<TAG, 1, 1> \
                                                                        : traj_session_kernel<TAG, 1, 2>; \
  else if (NQ == 2) fn = kp == 0 ? traj_session_kernel<TAG, 2, 0> : kp == 1 ? traj_session_kernel<TAG, 2, 1> \
                                                                             : traj_session_kernel<TAG, 2, 2>; \
  else fn = kp == 0 ? traj_session_kernel<TAG, 4, 0> : kp == 1 ? traj_session_kernel<TAG, 4, 1>           \
                                                              : traj_session_kernel<TAG, 4, 2>;
  if (a.st.bf16) { FMOE_SESS_PICK(Bf16Tag) } else { FMOE_SESS_PICK(F32Tag) }
#undef FMOE_SESS_PICK
  // equal contiguous row ranges per warp, in whole 32/GT-row passes
  const int esz = a.st.bf16 ? 2 : 4;
  int cpy = a.st.Ep * esz / 16, gt = 1;
  while (gt < cpy) gt <<= 1;
  const int64_t rpp = 32 / gt, nw = int64_t(a.grid) * kSessWarps;
  SessionArgs s2 = s;
  s2.rpw = ((a.n_rows + nw - 1) / nw + rpp - 1) / rpp * rpp;
  if (s2.rpw < rpp) s2.rpw = rpp;
  count_launch();
  return launch_pdl(fn, dim3(a.grid), dim3(kSessThreads), 0, stream, a, s2);
}

int traj_session_grid(const ScanArgs& a) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int esz = a.st.bf16 ? 2 : 4;
  int cpy = a.st.Ep * esz / 16, gt = 1;
  while (gt < cpy) gt <<= 1;
  const int64_t rows_per_iter = int64_t(32 / gt) * kPasses;
  const int64_t want = (a.n_rows + rows_per_iter * kSessWarps - 1) / (rows_per_iter * kSessWarps);
  // one full wave (every SM the same number of CTAs, rows spread evenly by
  // launch_traj_session), and (N = 1M, B = 1) at most one iteration per warp
  const int64_t full = int64_t(a.nq <= 1 ? 4 : 2) * sms;
  if (getenv("FMOE_SESS_BALANCE") == nullptr || atoi(getenv("FMOE_SESS_BALANCE")) != 0)
    if (want > full / 2) return int(full);
  const int64_t gsz = want < full ? want : full;
  return int(gsz < 1 ? 1 : gsz);
}

// ------------------------------------------------------------------ sweep: n session steps, one launch
// The steps of one request (B = 1, k = 1) over layers layer0 .. layer0+n-1 in
// ONE launch (fmoe_traj_session_sweep).  Each thread owns up to kSweepRows
// fixed rows (row = gtid + i * threads) and keeps their running dot products
// in REGISTERS across the steps, so step ell reads only the 16-byte slab row
// and the prefix-norm entry (20 B/row instead of the step kernel's 28 B) and
// the accumulators are written back once at the end.  Blocks never wait for
// each other: per step, one atomicMax per block into best[s] and a ticket;
// the last block of step s writes its top-1 and runs the Eq. 4-6 selection
// of target layer + sel_d (warp_select, as the step kernel), then publishes
// guidance_ready[s].  Optional layer_ready[s] flags (set by the producer of
// the gates, e.g. the MoE forward) gate step s: the device-side
// publisher/subscriber of P:528-533.  Arithmetic (query quantisation, fp64
// running query norm in the same reduction order, fmaf order over the row,
// acc + d, acc * r_q * rsqrt(psq)) is the step kernel's, so every output is
// bit-identical to n calls of fmoe_traj_session_step_select.
constexpr int kSweepThreads = 256;
constexpr int kSweepWarps = kSweepThreads / 32;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int kSweepMaxSteps = 64;

// A sweep that cannot run its steps (a poisoned session, or a layer that never
// became ready) marks them abandoned: guidance_ready = 2 for steps [s0, n), so
// a subscriber waiting on the flag wakes up, and the session's status word is
// set (fmoe_traj_session_abandoned; steps of the session report (NaN, -1)
// until it is reset).  Outputs of a poisoned session's steps are (NaN, -1).
__device__ __forceinline__ void sweep_abandon(const SweepArgs& a, int s0, bool write_outputs) {
  if (threadIdx.x != 0) return;
  if (write_outputs && blockIdx.x == 0)
    for (int f = s0; f < a.n_steps; ++f) {
      a.out_score[f] = __int_as_float(0x7fc00000);
      a.out_id[f] = -1;
      if (a.sel_mask) { a.sel_mask[f] = 0ull; a.sel_count[f] = 0; }
    }
  if (a.abort) atomicExch(a.abort, 1u);
  __threadfence();
  if (a.guidance_ready)
    for (int f = s0; f < a.n_steps; ++f) atomicCAS(a.guidance_ready + f, 0u, 2u);
}


// running query norm of step s from the per-warp partial sums, in the step
// kernel's order: t = (layer > 0 ? t_prev : 0) + red[0] + ... + red[7]
__device__ __forceinline__ double sweep_norm(double t_prev, int layer, const double* red) {
  double t = layer > 0 ? t_prev : 0.0;
  for (int w = 0; w < kSweepWarps; ++w) t += red[w];
  return t;
}

template <class Tag, int R>
__device__ __forceinline__ void sweep_issue(const StoreView& st, int layer, int gt, int nthr, int n,
                                            uint4 (&buf)[R], float (&ps)[R]) {
  const char* slab = static_cast<const char*>(st.maps) + int64_t(layer) * st.cap * 16;
  const float* psq = st.psq + int64_t(layer) * st.cap;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int row = gt + i * nthr;
    buf[i] = row < n ? ld_stream(slab + int64_t(row) * 16) : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int row = gt + i * nthr;
    ps[i] = row < n ? __ldcs(psq + row) : 0.f;
  }
}

template <class Tag, int R>
__global__ void __launch_bounds__(kSweepThreads, 4) traj_sweep_kernel(const SweepArgs a) {
  using ST = StoreT<Tag>;
  constexpr int EP = ST::kElemsPer16B;
  __shared__ __align__(16) float qs[kSweepMaxSteps][8];   // query layers (store-dtype values; 16-B rows: E <= 8)
  __shared__ float rqs[kSweepMaxSteps];
  __shared__ int valids[kSweepMaxSteps];
  __shared__ double red[kSweepWarps];
  __shared__ uint64_t sk[kSweepWarps];
  __shared__ int s_last, s_abort, s_fin;
  __shared__ float sel_p[kMaxE];
  __shared__ int sel_i[kMaxE];

  const StoreView& st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = st.E;
  const int n = int(a.n_rows);                      // < 2^31 (the register sweep holds <= 8 rows per thread)
  const int nthr = int(gridDim.x) * kSweepThreads;
  const int gt = int(blockIdx.x) * kSweepThreads + tid;
  const bool flags = a.layer_ready != nullptr;
  pdl_wait();
  if (a.abort && ld_acquire_u32(a.abort) != 0u) {   // poisoned by an earlier abandoned sweep
    sweep_abandon(a, 0, true);
    return;
  }

  // the first step's store rows are in flight while the queries are staged
  uint4 buf[R];
  float ps[R];
  sweep_issue<Tag, R>(st, a.layer0, gt, nthr, n, buf, ps);
  float acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int row = gt + i * nthr;
    acc[i] = (a.layer0 > 0 && row < n) ? __ldcs(a.acc + row) : 0.f;
  }
  double qn = a.layer0 > 0 ? a.qn_in[0] : 0.0;
  if (tid == 0) s_abort = 0;

  // Stage one query layer (thread j < 8 holds entry j: the step kernel's
  // partial-sum layout, warps 1..7 contribute 0) and its running norm.
  auto stage = [&](int s) {
    double part = 0.0;
    if (tid < 8) {
      const float v = tid < E ? to_store_value(a.q_layers[int64_t(s) * E + tid], Tag()) : 0.f;
      qs[s][tid] = v;
      part = double(v) * double(v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      qn = sweep_norm(qn, a.layer0 + s, red);
      rqs[s] = qn > 0.0 ? float(1.0 / sqrt(qn)) : 0.f;
      valids[s] = qn > 0.0;
    }
    __syncthreads();
  };
  if (!flags)   // every layer is already observed: stage them all up front
    for (int s = 0; s < a.n_steps; ++s) stage(s);

  // top-1 of step f (complete: this block took its last ticket), its Eq. 4-6
  // selection by warp 0, scratch reset, then guidance_ready[f]
  auto finalize = [&](int f) {
    if (warp != 0) return;
    __threadfence();
    const uint64_t key = __ldcg(a.best + f);
    const bool valid = valids[f] != 0;
    const int64_t id = valid ? key_id(key) : -1;
    const float score = valid ? key_score(key) : __int_as_float(0x7fc00000);
    if (lane == 0) {
      a.out_score[f] = score;
      a.out_id[f] = id;
    }
    const int tgt = a.layer0 + f + a.sel_d;
    if (a.sel_mask) {
      const int64_t loc = id - int64_t(a.id_offset);
      if (tgt >= st.L || id < 0 || loc < 0 || loc >= n) {
        if (lane == 0) { a.sel_mask[f] = 0ull; a.sel_count[f] = 0; }
      } else {
        uint64_t mask;
        int m;
        warp_select<Tag>(st, tgt, loc, selection_delta(a.sel_delta, score), a.sel_K, sel_p, sel_i, &mask, &m);
        if (lane == 0) { a.sel_mask[f] = mask; a.sel_count[f] = m; }
      }
    }
    __syncwarp();
    if (lane == 0) {
      a.best[f] = 0ull;
      a.tickets[f] = 0u;
      __threadfence();
      if (a.guidance_ready) st_release_u32(a.guidance_ready + f, 1u);
    }
  };
  unsigned pend_ticket = 0u;   // tid 0: ticket of step pend_s
  int pend_s = -1;

  for (int s = 0; s < a.n_steps; ++s) {
    const int layer = a.layer0 + s;
    if (flags) {
      if (tid == 0) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_u32(a.layer_ready + s) == 0u) {
          __nanosleep(200);
          if (globaltimer_ns() - t0 > a.timeout_ns) { s_abort = 1; break; }
        }
      }
      __syncthreads();
      if (s_abort) {
        // finish the step this block may hold the last ticket of, then abandon the rest
        if (tid == 0) {
          s_last = pend_s >= 0 && pend_ticket == gridDim.x - 1;
          s_fin = pend_s;
        }
        __syncthreads();
        if (s_last) finalize(s_fin);
        sweep_abandon(a, s, false);
        return;
      }
      stage(s);
    }
    const float rq = rqs[s];
    const float* qv = qs[s];
    uint64_t best = 0ull;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int row = gt + i * nthr;
      float x[8];
      unpack_sess<Tag>(buf[i], x);
      float d = 0.f;
#pragma unroll
      for (int e = 0; e < EP; ++e) d = fmaf(x[e], qv[e], d);
      acc[i] = acc[i] + d;
      const float rm = ps[i] > 0.f ? rsqrtf(ps[i]) : 0.f;
      const float sc = acc[i] * rq * rm;
      const uint64_t key = row < n ? pack_key(sc, a.id_offset + uint32_t(row)) : 0ull;
      best = key > best ? key : best;
    }
    // the next step's rows load while this step reduces and publishes
    if (s + 1 < a.n_steps) sweep_issue<Tag, R>(st, layer + 1, gt, nthr, n, buf, ps);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t x2 = shfl_u64(best, lane ^ o);
      best = x2 > best ? x2 : best;
    }
    if (lane == 0) sk[warp] = best;
    __syncthreads();
    // Ticket of step s is taken here but consumed one step later (tid 0 keeps
    // it in a register), so the block does not wait for the atomics' round
    // trip: the last block of step s - 1 finalises it now.
    uint64_t b = 0ull;
    if (tid == 0) {
      for (int w = 0; w < kSweepWarps; ++w) b = b > sk[w] ? b : sk[w];
      s_last = pend_s >= 0 && pend_ticket == gridDim.x - 1;
      s_fin = pend_s;
    }
    __syncthreads();
    if (tid == 0) {
      if (b) atomicMax(a.best + s, static_cast<unsigned long long>(b));
      __threadfence();
      pend_ticket = atomicAdd(a.tickets + s, 1u);
      pend_s = s;
    }
    if (s_last) finalize(s_fin);
  }
  if (tid == 0) {
    s_last = pend_s >= 0 && pend_ticket == gridDim.x - 1;
    s_fin = pend_s;
  }
  __syncthreads();
  if (s_last) finalize(s_fin);
  pdl_trigger();
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int row = gt + i * nthr;
    if (row < n) __stcs(a.acc + row, acc[i]);
  }
  if (blockIdx.x == 0 && tid == 0) a.qn_out[0] = qn;
}

// ------------------------------------------------------------------ sweep, shared-memory staged
// Same computation and outputs as traj_sweep_kernel (bit for bit), with the
// slab rows moved by the TMA engine: block b owns the contiguous rows
// [b*R*T, (b+1)*R*T) (thread t: rows b*R*T + i*T + t), so a step's slab chunk
// is one contiguous range, copied by one cp.async.bulk into a 2-stage shared
// ring issued two steps ahead (the copy of step s+2 starts when step s's
// stage is free).  The prefix-norm entries are prefetched two steps ahead in
// registers.  A step then costs max(transfer, compute) instead of
// load latency + transfer + compute.
constexpr int kSweepTmaThreads = 512;
constexpr int kSweepTmaR = 7;
constexpr int kSweepTmaWarps = kSweepTmaThreads / 32;
constexpr size_t kSweepTmaStage = size_t(kSweepTmaR) * kSweepTmaThreads * 16;

template <class Tag>
__global__ void __launch_bounds__(kSweepTmaThreads, 2) traj_sweep_tma_kernel(const SweepArgs a) {
  using ST = StoreT<Tag>;
  constexpr int EP = ST::kElemsPer16B;
  constexpr int R = kSweepTmaR, T = kSweepTmaThreads;
  extern __shared__ __align__(128) unsigned char ring[];            // [2][R*T][16 B]
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ __align__(16) float qs[kSweepMaxSteps][8];
  __shared__ float rqs[kSweepMaxSteps];
  __shared__ int valids[kSweepMaxSteps];
  __shared__ double red[kSweepTmaWarps];
  __shared__ uint64_t sk[kSweepTmaWarps];
  __shared__ int s_last, s_abort, s_fin;
  __shared__ float sel_p[kMaxE];
  __shared__ int sel_i[kMaxE];

  const StoreView& st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = st.E;
  const int n = int(a.n_rows);
  const int base = int(blockIdx.x) * R * T;
  const int cnt = n - base < R * T ? n - base : R * T;               // rows of this block (> 0)
  const bool flags = a.layer_ready != nullptr;
  const uint64_t pol = policy_evict_first();
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
    s_abort = 0;
  }
  __syncthreads();
  pdl_wait();
  if (a.abort && ld_acquire_u32(a.abort) != 0u) {
    sweep_abandon(a, 0, true);
    return;
  }
  auto issue = [&](int s) {   // tid 0: slab chunk of step s into stage s & 1
    const char* src = static_cast<const char*>(st.maps) + (int64_t(a.layer0 + s) * st.cap + base) * 16;
    mbar_arrive_expect_tx(&bar[s & 1], unsigned(cnt) * 16u);
    bulk_g2s(ring + (s & 1) * kSweepTmaStage, src, unsigned(cnt) * 16u, &bar[s & 1], pol);
  };
  if (tid == 0) {
    issue(0);
    if (a.n_steps > 1) issue(1);
  }
  float ps0[R], ps1[R];      // prefix-norm entries of steps s and s + 1
  auto load_ps = [&](int s, float (&ps)[R]) {
    const float* psq = st.psq + int64_t(a.layer0 + s) * st.cap + base;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = i * T + tid;
      ps[i] = r < cnt ? __ldcs(psq + r) : 0.f;
    }
  };
  load_ps(0, ps0);
  if (a.n_steps > 1) load_ps(1, ps1);
  float acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int r = i * T + tid;
    acc[i] = (a.layer0 > 0 && r < cnt) ? __ldcs(a.acc + base + r) : 0.f;
  }
  double qn = a.layer0 > 0 ? a.qn_in[0] : 0.0;

  auto stage = [&](int s) {
    double part = 0.0;
    if (tid < 8) {
      const float v = tid < E ? to_store_value(a.q_layers[int64_t(s) * E + tid], Tag()) : 0.f;
      qs[s][tid] = v;
      part = double(v) * double(v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0 && warp < kSweepWarps) red[warp] = part;   // the step kernel's 8-warp partial sums
    __syncthreads();
    if (tid == 0) {
      qn = sweep_norm(qn, a.layer0 + s, red);
      rqs[s] = qn > 0.0 ? float(1.0 / sqrt(qn)) : 0.f;
      valids[s] = qn > 0.0;
    }
    __syncthreads();
  };
  if (!flags)
    for (int s = 0; s < a.n_steps; ++s) stage(s);

  auto finalize = [&](int f) {
    if (warp != 0) return;
    __threadfence();
    const uint64_t key = __ldcg(a.best + f);
    const bool valid = valids[f] != 0;
    const int64_t id = valid ? key_id(key) : -1;
    const float score = valid ? key_score(key) : __int_as_float(0x7fc00000);
    if (lane == 0) {
      a.out_score[f] = score;
      a.out_id[f] = id;
    }
    const int tgt = a.layer0 + f + a.sel_d;
    if (a.sel_mask) {
      const int64_t loc = id - int64_t(a.id_offset);
      if (tgt >= st.L || id < 0 || loc < 0 || loc >= n) {
        if (lane == 0) { a.sel_mask[f] = 0ull; a.sel_count[f] = 0; }
      } else {
        uint64_t mask;
        int m;
        warp_select<Tag>(st, tgt, loc, selection_delta(a.sel_delta, score), a.sel_K, sel_p, sel_i, &mask, &m);
        if (lane == 0) { a.sel_mask[f] = mask; a.sel_count[f] = m; }
      }
    }
    __syncwarp();
    if (lane == 0) {
      a.best[f] = 0ull;
      a.tickets[f] = 0u;
      __threadfence();
      if (a.guidance_ready) st_release_u32(a.guidance_ready + f, 1u);
    }
  };
  unsigned pend_ticket = 0u;
  int pend_s = -1;

  for (int s = 0; s < a.n_steps; ++s) {
    if (flags) {
      if (tid == 0) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_u32(a.layer_ready + s) == 0u) {
          __nanosleep(200);
          if (globaltimer_ns() - t0 > a.timeout_ns) { s_abort = 1; break; }
        }
      }
      __syncthreads();
      if (s_abort) {
        // drain the bulk copies still landing in this block's shared memory
        mbar_wait(&bar[s & 1], unsigned((s >> 1) & 1));
        if (s + 1 < a.n_steps) mbar_wait(&bar[(s + 1) & 1], unsigned(((s + 1) >> 1) & 1));
        if (tid == 0) {
          s_last = pend_s >= 0 && pend_ticket == gridDim.x - 1;
          s_fin = pend_s;
        }
        __syncthreads();
        if (s_last) finalize(s_fin);
        sweep_abandon(a, s, false);
        return;
      }
      stage(s);
    }
    const float rq = rqs[s];
    const float* qv = qs[s];
    mbar_wait(&bar[s & 1], unsigned((s >> 1) & 1));
    const uint4* chunk = reinterpret_cast<const uint4*>(ring + (s & 1) * kSweepTmaStage);
    uint64_t best = 0ull;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = i * T + tid;
      float x[8];
      unpack_sess<Tag>(r < cnt ? chunk[r] : make_uint4(0u, 0u, 0u, 0u), x);
      float d = 0.f;
#pragma unroll
      for (int e = 0; e < EP; ++e) d = fmaf(x[e], qv[e], d);
      acc[i] = acc[i] + d;
      const float rm = ps0[i] > 0.f ? rsqrtf(ps0[i]) : 0.f;
      const float sc = acc[i] * rq * rm;
      const uint64_t key = r < cnt ? pack_key(sc, a.id_offset + uint32_t(base + r)) : 0ull;
      best = key > best ? key : best;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) ps0[i] = ps1[i];
    if (s + 2 < a.n_steps) load_ps(s + 2, ps1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t x2 = shfl_u64(best, lane ^ o);
      best = x2 > best ? x2 : best;
    }
    if (lane == 0) sk[warp] = best;
    __syncthreads();                      // also: every thread is done with stage s & 1
    uint64_t b = 0ull;
    if (tid == 0) {
      if (s + 2 < a.n_steps) issue(s + 2);
      for (int w = 0; w < kSweepTmaWarps; ++w) b = b > sk[w] ? b : sk[w];
      s_last = pend_s >= 0 && pend_ticket == gridDim.x - 1;
      s_fin = pend_s;
    }
    __syncthreads();
    if (tid == 0) {
      if (b) atomicMax(a.best + s, static_cast<unsigned long long>(b));
      __threadfence();
      pend_ticket = atomicAdd(a.tickets + s, 1u);
      pend_s = s;
    }
    if (s_last) finalize(s_fin);
  }
  if (tid == 0) {
    s_last = pend_s >= 0 && pend_ticket == gridDim.x - 1;
    s_fin = pend_s;
  }
  __syncthreads();
  if (s_last) finalize(s_fin);
  pdl_trigger();
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int r = i * T + tid;
    if (r < cnt) __stcs(a.acc + base + r, acc[i]);
  }
  if (blockIdx.x == 0 && tid == 0) a.qn_out[0] = qn;
}

// ------------------------------------------------------------------ sweep, row-major (every layer observed)
// When every layer of the sweep is already observed (no layer_ready /
// guidance_ready flags: trace replay, a request whose gates are all known),
// the steps need no order between them except through each row's running dot,
// which is private to the row.  So the sweep walks ROWS in the outer loop and
// the steps in the inner loop: a thread takes a row, streams its n_steps slab
// entries (16 B) and prefix-norm entries (4 B) in chunks of CH (8 or 16) loads,
// carries acc in one register from step to step, and folds each step's key
// into its own per-step best in shared memory.  Nothing synchronises between
// steps, so the loads of the next chunk / row are never held back by a step
// barrier (the step-major kernel pays load latency + transfer + reduction per
// step).  One reduction per block at the end (per-step atomicMax); a second,
// PDL-launched kernel (one warp per step) writes every step's top-1 and runs
// the Eq. 4-6 selections, all steps in parallel.  Arithmetic per (row, step)
// is the step kernel's (same fmaf order, acc + d, acc * r_q * rsqrt(psq)) and
// the max of packed keys is order-free, so outputs are bit-identical to the
// step-major kernel.  Any number of rows (no register-residency limit).


// Query layers of steps [0, ns) (store-dtype values, qs[s][0..8)) and their
// running norms, all steps at once (warp w: steps w, w+8, ...), in the step
// kernel's order: part_s = butterfly sum of v^2 over lanes 0..7 of one warp,
// t_s = (layer > 0 ? t_{s-1} : 0) + part_s (the step kernel adds the other
// seven warps' zero partials, which leaves the double unchanged).  Returns the
// norm after the last step on tid 0.
template <class Tag>
__device__ __forceinline__ double sweep_stage_all(const SweepArgs& a, float (*qs)[8], float* rqs, int* valids,
                                                  double* parts) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = a.st.E, ns = a.n_steps;
  for (int s = warp; s < ns; s += kSweepWarps) {
    double part = 0.0;
    if (lane < 8) {
      const float v = lane < E ? to_store_value(a.q_layers[int64_t(s) * E + lane], Tag()) : 0.f;
      qs[s][lane] = v;
      part = double(v) * double(v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) parts[s] = part;
  }
  __syncthreads();
  double qn = a.layer0 > 0 ? a.qn_in[0] : 0.0;
  if (tid == 0)
    for (int s = 0; s < ns; ++s) {
      double red[kSweepWarps] = {parts[s]};      // warps 1..7 contribute 0, as in the step kernel
      qn = sweep_norm(qn, a.layer0 + s, red);
      rqs[s] = qn > 0.0 ? float(1.0 / sqrt(qn)) : 0.f;
      valids[s] = qn > 0.0;
    }
  __syncthreads();
  return qn;
}

template <class Tag, int CH>
__global__ void __launch_bounds__(kSweepThreads, CH > 8 ? 2 : 3) traj_sweep_rowmajor_kernel(const SweepArgs a) {
  using ST = StoreT<Tag>;
  constexpr int EP = ST::kElemsPer16B;
  extern __shared__ __align__(16) unsigned long long bk[];   // [n_steps][kSweepThreads] per-thread best keys
  __shared__ __align__(16) float qs[kSweepMaxSteps][8];
  __shared__ float rqs[kSweepMaxSteps];
  __shared__ int valids[kSweepMaxSteps];
  __shared__ double parts[kSweepMaxSteps];

  const StoreView& st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n_rows;
  const int ns = a.n_steps;
  const int64_t nthr = int64_t(gridDim.x) * kSweepThreads;
  const char* maps = static_cast<const char*>(st.maps);
  pdl_wait();
  pdl_trigger();                 // the finalize kernel may be scheduled; it waits for this grid
  if (a.abort && ld_acquire_u32(a.abort) != 0u) return;   // poisoned: the finalize kernel reports it
  // the first chunk of this thread's first row is in flight while the queries are staged
  const int64_t row0 = int64_t(blockIdx.x) * kSweepThreads + tid;
  uint4 buf[CH];
  float ps[CH];
  auto issue = [&](int64_t row, int s0) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int64_t layer = a.layer0 + s0 + j;
      buf[j] = (row < n && s0 + j < ns) ? ld_stream(maps + (layer * st.cap + row) * 16) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int64_t layer = a.layer0 + s0 + j;
      ps[j] = (row < n && s0 + j < ns) ? __ldcs(st.psq + layer * st.cap + row) : 0.f;
    }
  };
  issue(row0, 0);
  sweep_stage_all<Tag>(a, qs, rqs, valids, parts);
  for (int s = 0; s < ns; ++s) bk[s * kSweepThreads + tid] = 0ull;

  for (int64_t row = row0; row < n; row += nthr) {
    float acc = a.layer0 > 0 ? __ldcs(a.acc + row) : 0.f;
    const uint32_t gid = a.id_offset + uint32_t(row);
    for (int s0 = 0; s0 < ns; s0 += CH) {
      if (row != row0 || s0 != 0) issue(row, s0);
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int s = s0 + j;
        if (s < ns) {
          float x[8];
          unpack_sess<Tag>(buf[j], x);
          const float* qv = qs[s];
          float d = 0.f;
#pragma unroll
          for (int e = 0; e < EP; ++e) d = fmaf(x[e], qv[e], d);
          acc = acc + d;
          const float rm = ps[j] > 0.f ? rsqrtf(ps[j]) : 0.f;
          const float sc = acc * rqs[s] * rm;
          const unsigned long long key = pack_key(sc, gid);
          unsigned long long& b = bk[s * kSweepThreads + tid];
          b = key > b ? key : b;
        }
      }
    }
    __stcs(a.acc + row, acc);
  }
  __syncthreads();
  for (int s = warp; s < ns; s += kSweepWarps) {
    unsigned long long b = 0ull;
#pragma unroll
    for (int j = 0; j < kSweepThreads / 32; ++j) {
      const unsigned long long v = bk[s * kSweepThreads + j * 32 + lane];
      b = v > b ? v : b;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x2 = shfl_u64(b, lane ^ o);
      b = x2 > b ? x2 : b;
    }
    if (lane == 0 && b) atomicMax(a.best + s, b);
  }
}

// Outputs of a row-major sweep: one warp per step (after the sweep grid
// completed): top-1 from the packed best key, the Eq. 4-6 selection of target
// layer layer0 + s + sel_d (warp_select, as the step kernel), best reset; the
// running query norm goes to qn_out.  A poisoned session reports (NaN, -1).
template <class Tag>
__global__ void __launch_bounds__(kSweepThreads) traj_sweep_finalize_kernel(const SweepArgs a) {
  __shared__ __align__(16) float qs[kSweepMaxSteps][8];
  __shared__ float rqs[kSweepMaxSteps];
  __shared__ int valids[kSweepMaxSteps];
  __shared__ double parts[kSweepMaxSteps];
  __shared__ float sel_p[kSweepWarps][kMaxE];
  __shared__ int sel_i[kSweepWarps][kMaxE];
  const StoreView& st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();
  const bool poisoned = a.abort && ld_acquire_u32(a.abort) != 0u;
  const double qn = sweep_stage_all<Tag>(a, qs, rqs, valids, parts);
  for (int f = int(blockIdx.x) * kSweepWarps + warp; f < a.n_steps; f += int(gridDim.x) * kSweepWarps) {
    const uint64_t key = __ldcg(a.best + f);
    const bool valid = valids[f] != 0 && !poisoned;
    const int64_t id = valid ? key_id(key) : -1;
    const float score = valid ? key_score(key) : __int_as_float(0x7fc00000);
    if (lane == 0) {
      a.out_score[f] = score;
      a.out_id[f] = id;
    }
    const int tgt = a.layer0 + f + a.sel_d;
    if (a.sel_mask) {
      const int64_t loc = id - int64_t(a.id_offset);
      if (tgt >= st.L || id < 0 || loc < 0 || loc >= a.n_rows) {
        if (lane == 0) { a.sel_mask[f] = 0ull; a.sel_count[f] = 0; }
      } else {
        uint64_t mask;
        int m;
        warp_select<Tag>(st, tgt, loc, selection_delta(a.sel_delta, score), a.sel_K, sel_p[warp], sel_i[warp],
                         &mask, &m);
        if (lane == 0) { a.sel_mask[f] = mask; a.sel_count[f] = m; }
      }
    }
    __syncwarp();
    if (lane == 0) a.best[f] = 0ull;
  }
  if (blockIdx.x == 0 && tid == 0 && !poisoned) a.qn_out[0] = qn;
  pdl_trigger();
}

int traj_sweep_rows(int64_t n_rows, int* grid_out) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t grid = int64_t(4) * sms;
  const int64_t need = (n_rows + kSweepThreads - 1) / kSweepThreads;
  if (need < grid) grid = need < 1 ? 1 : need;
  const int64_t rpt = (n_rows + grid * kSweepThreads - 1) / (grid * kSweepThreads);
  *grid_out = int(grid);
  return rpt <= 4 ? 4 : (rpt <= 7 ? 7 : (rpt <= 8 ? 8 : 0));   // 0: too many rows for registers
}

cudaError_t launch_traj_sweep(const SweepArgs& a, cudaStream_t stream) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // Kernel choice (FMOE_SWEEP_KERNEL, read per call: a measurement/test knob):
  //  "row" (default) -- row-major sweep when no ready flags are given;
  //  "reg" -- the step-major register kernel; "tma" -- the step-major
  //  shared-memory staged kernel (measured slower at C2: 0.262 vs 0.217 ms,
  //  profiles/r01f_c2_sweep.md).  Ready flags always take a step-major kernel.
  const char* env = getenv("FMOE_SWEEP_KERNEL");
  const bool want_tma = env != nullptr && strcmp(env, "tma") == 0;
  const bool want_reg = env != nullptr && strcmp(env, "reg") == 0;
  int unused_grid = 0;
  const bool flagless = !a.layer_ready && !a.guidance_ready;
  if (flagless && ((!want_tma && !want_reg) || traj_sweep_rows(a.n_rows, &unused_grid) == 0)) {
    using Fn = void (*)(const SweepArgs);
    // loads in flight per thread (FMOE_SWEEP_CHUNK = 8 or 16; measurement knob)
    const char* ce = getenv("FMOE_SWEEP_CHUNK");
    const int ch = ce && atoi(ce) == 8 ? 8 : 16;
    Fn fn = a.st.bf16 ? (ch == 8 ? traj_sweep_rowmajor_kernel<Bf16Tag, 8> : traj_sweep_rowmajor_kernel<Bf16Tag, 16>)
                      : (ch == 8 ? traj_sweep_rowmajor_kernel<F32Tag, 8> : traj_sweep_rowmajor_kernel<F32Tag, 16>);
    const int smem = a.n_steps * kSweepThreads * 8;
    // the attribute allows the largest sweep (64 steps), set once per kernel;
    // resident blocks per SM cached by (dtype, n_steps)
    static int occ[4][kSweepMaxSteps + 1];
    static bool attr_set[4];
    const int di = (a.st.bf16 ? 1 : 0) + (ch == 8 ? 0 : 2);
    int& per_sm = occ[di][a.n_steps];
    if (per_sm == 0) {
      cudaError_t e = cudaSuccess;
      if (!attr_set[di]) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepMaxSteps * kSweepThreads * 8);
        if (e == cudaSuccess) attr_set[di] = true;
      }
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSweepThreads, size_t(smem));
      if (e != cudaSuccess) return e;
      if (per_sm < 1) return cudaErrorInvalidConfiguration;
    }
    int64_t grid = int64_t(per_sm) * sms;
    const int64_t need = (a.n_rows + kSweepThreads - 1) / kSweepThreads;
    if (need < grid) grid = need < 1 ? 1 : need;
    count_launch(2);
    cudaError_t e = launch_pdl(fn, dim3(unsigned(grid)), dim3(kSweepThreads), size_t(smem), stream, a);
    if (e != cudaSuccess) return e;
    Fn fin = a.st.bf16 ? traj_sweep_finalize_kernel<Bf16Tag> : traj_sweep_finalize_kernel<F32Tag>;
    return launch_pdl(fin, dim3(unsigned((a.n_steps + kSweepWarps - 1) / kSweepWarps)), dim3(kSweepThreads), 0,
                      stream, a);
  }
  const bool tma_ok = want_tma;
  const int64_t per_block = int64_t(kSweepTmaR) * kSweepTmaThreads;
  const int64_t tgrid = (a.n_rows + per_block - 1) / per_block;
  if (tma_ok && tgrid <= int64_t(2) * sms) {
    using Fn = void (*)(const SweepArgs);
    Fn fn = a.st.bf16 ? traj_sweep_tma_kernel<Bf16Tag> : traj_sweep_tma_kernel<F32Tag>;
    const int smem = int(2 * kSweepTmaStage);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    count_launch();
    return launch_pdl(fn, dim3(unsigned(tgrid)), dim3(kSweepTmaThreads), size_t(smem), stream, a);
  }
  int grid = 1;
  const int R = traj_sweep_rows(a.n_rows, &grid);
  using Fn = void (*)(const SweepArgs);
  Fn fn = nullptr;
  if (R == 0) return cudaErrorInvalidValue;
  if (a.st.bf16) fn = R == 4 ? traj_sweep_kernel<Bf16Tag, 4> : R == 7 ? traj_sweep_kernel<Bf16Tag, 7>
                                                              : traj_sweep_kernel<Bf16Tag, 8>;
  else fn = R == 4 ? traj_sweep_kernel<F32Tag, 4> : R == 7 ? traj_sweep_kernel<F32Tag, 7>
                                                           : traj_sweep_kernel<F32Tag, 8>;
  count_launch();
  return launch_pdl(fn, dim3(grid), dim3(kSweepThreads), 0, stream, a);
}

}  // namespace fmoe
