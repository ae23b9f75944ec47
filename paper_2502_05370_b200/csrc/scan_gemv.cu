// scan_gemv.cu -- K2: bandwidth-bound scoring of B <= 4 queries against the
// whole store, fused with a per-warp top-k.
//
// What it computes, per query x and stored row y:
//   sem  = (q~_x . e~_y) * r_q * r_e[y]                      cosine, Eq. 1
//   traj = (q~_x[0:ell] . M~_y[0:ell]) * r_q(ell) / ||M~_y[0:ell]||   Eq. 2
//   score = w*sem + (1-w)*traj                               RDY / blend
// where ~ is the store dtype (bf16 RNE or fp32) and all dots accumulate in
// fp32.  The prefix norm of the stored map is accumulated on the fly from the
// same bytes (no norm-table read: at ell = 1 a table would add 25% traffic).
//
// Mapping: a warp owns a tile of 32 consecutive rows.  The
// semantic dot of one row is spread over GS lanes (GS = 32 for D >= 256 bf16),
// each lane streaming 16-byte chunks with ld.global.nc.L1::no_allocate, 8
// chunks in flight per lane; the trajectory dot of one row is spread over GT
// lanes (GT = 1 for Mixtral bf16: each lane reads its row's 16-byte slab
// entry, so a warp instruction reads 512 contiguous bytes of a layer slab).
// Results are shuffled so that lane r holds row y0+r, then offered to the
// warp's register-resident top-k lists (WarpTopK).  Queries are staged once
// per block in shared memory as fp32 values of the store dtype.
#include <cstdio>
#include <mutex>
#include <map>
#include "common.cuh"
#include "kernels.cuh"
#include "merge.cuh"

namespace fmoe {

constexpr int kScanThreads = 256;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kU = 8;  // 16-byte loads in flight per lane per batch

template <class Tag>
__device__ __forceinline__ void unpack_chunk(const uint4& u, float (&x)[8]);
template <>
__device__ __forceinline__ void unpack_chunk<Bf16Tag>(const uint4& u, float (&x)[8]) {
  unpack8(u, x, Bf16Tag());
}
template <>
__device__ __forceinline__ void unpack_chunk<F32Tag>(const uint4& u, float (&x)[8]) {
  x[0] = __uint_as_float(u.x); x[1] = __uint_as_float(u.y);
  x[2] = __uint_as_float(u.z); x[3] = __uint_as_float(u.w);
  x[4] = x[5] = x[6] = x[7] = 0.f;
}

__device__ __forceinline__ int group_size(int chunks) {
  int g = 1;
  while (g < chunks && g < 32) g <<= 1;
  return g;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// TPI >= 1 (trajectory-only, 16-byte map rows): a warp streams TPI
// consecutive 32-row tiles per iteration, LB = 16/TPI layers per load batch,
// so each lane keeps 16 16-byte loads in flight at every prefix length (the
// 8-deep generic path was latency-bound below ell ~ 16).  TPI = 0: generic.
// Occupancy: the generic path needs >= 3 CTAs (24 warps) per SM to cover HBM
// latency with 8 loads per lane; the multi-tile path keeps 16 loads per lane
// and runs at 2 CTAs per SM.
template <class Tag, int NQ, int KPL, bool SEM, bool TRAJ, int TPI>
__global__ void __launch_bounds__(kScanThreads, TPI >= 1 ? 2 : 3) scan_gemv_kernel(const ScanArgs a) {
  using ST = StoreT<Tag>;
  constexpr int EP = ST::kElemsPer16B;
  constexpr int SB = ST::kBytes;
  extern __shared__ __align__(16) float smem[];
  __shared__ double red[kScanWarps][2 * NQ];
  __shared__ float rq[2][NQ];
  __shared__ int s_valid[NQ];
  __shared__ int s_last;

  const StoreView& st = a.st;
  const int Dp = st.Dp, Ep = st.Ep, E = st.E, D = st.D, ell = a.ell;
  const int tl = ell * Ep;
  float* qsem = smem;                              // [NQ][Dp]
  float* qtraj = smem + (SEM ? NQ * Dp : 0);       // [NQ][ell][Ep]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  trace_mark(a.trace, 0);
  pdl_wait();
  trace_mark(a.trace, 1);
  if (a.run_if_gt && *a.run_if_gt <= a.q0) return;   // a fallback pass with no queries

  // ---- 1. stage the queries (quantised to the store dtype) + their norms
  double part[2 * NQ];
#pragma unroll
  for (int i = 0; i < 2 * NQ; ++i) part[i] = 0.0;
  if (SEM) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      for (int e = tid; e < Dp; e += kScanThreads) {
        float v = 0.f;
        if (q < a.nq && e < D) v = to_store_value(a.q_emb[int64_t(a.q0 + q) * D + e], Tag());
        qsem[q * Dp + e] = v;
        part[q] += double(v) * double(v);
      }
  }
  if (TRAJ) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      for (int i = tid; i < tl; i += kScanThreads) {
        const int l = i / Ep, j = i - l * Ep;
        float v = 0.f;
        if (q < a.nq && j < E) v = to_store_value(a.q_prefix[int64_t(a.q0 + q) * a.q_stride + l * E + j], Tag());
        qtraj[q * tl + i] = v;
        part[NQ + q] += double(v) * double(v);
      }
  }
#pragma unroll
  for (int i = 0; i < 2 * NQ; ++i) {
    const double s = warp_sum_d(part[i]);
    if (lane == 0) red[warp][i] = s;
  }
  __syncthreads();
  if (tid < NQ) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < kScanWarps; ++w) { s0 += red[w][tid]; s1 += red[w][NQ + tid]; }
    rq[0][tid] = s0 > 0.0 ? float(1.0 / sqrt(s0)) : 0.f;
    rq[1][tid] = s1 > 0.0 ? float(1.0 / sqrt(s1)) : 0.f;
    s_valid[tid] = (!SEM || s0 > 0.0) && (!TRAJ || s1 > 0.0);
  }
  __syncthreads();

  trace_mark(a.trace, 2);
  float rq0[NQ], rq1[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) { rq0[q] = rq[0][q]; rq1[q] = rq[1][q]; }

  // ---- 2. stream 32-row tiles
  WarpTopK<KPL> lists[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) lists[q].init();

  // Work partition: tiles of TS rows dealt round-robin over the nw warps
  // (neighbouring warps stream neighbouring rows: DRAM-page friendly), and the
  // rows left after the last full round split evenly into one partial tile per
  // warp, so per-warp work differs by at most one row (plain round-robin left a
  // 5-13% tail whenever the tile count was not a multiple of nw).
  const int64_t nw = int64_t(gridDim.x) * kScanWarps;
  const int64_t wg = int64_t(blockIdx.x) * kScanWarps + warp;
  const int64_t TS = TPI >= 1 ? 32 * TPI : 32;
  const int64_t full_rounds = a.n_rows / (nw * TS);
  const int64_t rem_base = full_rounds * nw * TS, rem = a.n_rows - rem_base;
  auto tile_of = [&](int64_t r, int64_t& y0, int64_t& y1) -> bool {
    if (r < full_rounds) { y0 = (r * nw + wg) * TS; y1 = y0 + TS; return true; }
    y0 = rem_base + rem * wg / nw;
    y1 = rem_base + rem * (wg + 1) / nw;
    return r == full_rounds && y0 < y1;
  };
  const int CPR = Dp / EP;          // 16-byte chunks per embedding row
  const int GS = group_size(CPR);
  const int rpp = 32 / GS, sg = lane / GS, sgl = lane % GS;
  const int cpl = (CPR + GS - 1) / GS;
  const int CPY = Ep / EP;          // 16-byte chunks per map-layer row
  const int GT = group_size(CPY);
  const int rppt = 32 / GT, tg = lane / GT, tcl = lane % GT;
  const char* embp = static_cast<const char*>(st.emb);
  const char* mapp = static_cast<const char*>(st.maps);
  const int64_t slab = st.cap * int64_t(Ep) * SB;
  const float w = a.w_sem, w1 = 1.f - a.w_sem;

  if constexpr (TPI >= 1) {
    // ---- 2a. trajectory-only, one 16-byte chunk per row-layer (GT == 1)
    constexpr int LB = 16 / TPI;
    int64_t y0, n_rows;
    for (int64_t rr = 0; tile_of(rr, y0, n_rows); ++rr) {
      float acc[TPI][NQ], sq[TPI];
#pragma unroll
      for (int i = 0; i < TPI; ++i) {
        sq[i] = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[i][q] = 0.f;
      }
      for (int l0 = 0; l0 < ell; l0 += LB) {
        uint4 buf[TPI][LB];
#pragma unroll
        for (int i = 0; i < TPI; ++i)
#pragma unroll
          for (int u = 0; u < LB; ++u) {
            const int64_t row = y0 + i * 32 + lane;
            buf[i][u] = (row < n_rows && l0 + u < ell) ? ld_stream(mapp + row * 16 + int64_t(l0 + u) * slab)
                                                       : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          if (l0 + u < ell) {
#pragma unroll
            for (int i = 0; i < TPI; ++i) {
              float x[8];
              unpack_chunk<Tag>(buf[i][u], x);
#pragma unroll
              for (int e = 0; e < EP; ++e) sq[i] = fmaf(x[e], x[e], sq[i]);
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                const float4* qp = reinterpret_cast<const float4*>(qtraj + q * tl + (l0 + u) * Ep);
#pragma unroll
                for (int e4 = 0; e4 < EP / 4; ++e4) {
                  const float4 qv = qp[e4];
                  acc[i][q] = fmaf(x[4 * e4 + 0], qv.x, acc[i][q]);
                  acc[i][q] = fmaf(x[4 * e4 + 1], qv.y, acc[i][q]);
                  acc[i][q] = fmaf(x[4 * e4 + 2], qv.z, acc[i][q]);
                  acc[i][q] = fmaf(x[4 * e4 + 3], qv.w, acc[i][q]);
                }
              }
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < TPI; ++i) {
        const int64_t y = y0 + i * 32 + lane;
        const bool ok = y < n_rows;
        const float rm = sq[i] > 0.f ? rsqrtf(sq[i]) : 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float sc = fmaf(w1, acc[i][q] * rq1[q] * rm, 0.f);
          lists[q].offer(ok ? pack_key(sc, a.id_offset + uint32_t(y)) : 0ull, a.k);
        }
      }
    }
  } else {
  int64_t y0, n_rows;
  for (int64_t rr = 0; tile_of(rr, y0, n_rows); ++rr) {
    float sem[NQ], trj[NQ], msq = 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) { sem[q] = 0.f; trj[q] = 0.f; }

    if (SEM) {
      for (int p = 0; p < GS; ++p) {
        const int64_t row = y0 + p * rpp + sg;
        const bool rok = row < n_rows;
        const char* rp = embp + row * int64_t(Dp) * SB;
        float acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.f;
        for (int j0 = 0; j0 < cpl; j0 += kU) {
          uint4 buf[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int c = sgl + (j0 + u) * GS;
            buf[u] = (rok && j0 + u < cpl && c < CPR) ? ld_stream(rp + int64_t(c) * 16) : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int c = sgl + (j0 + u) * GS;
            if (j0 + u < cpl && c < CPR) {
              float x[8];
              unpack_chunk<Tag>(buf[u], x);
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                const float4* qp = reinterpret_cast<const float4*>(qsem + q * Dp + c * EP);
#pragma unroll
                for (int e4 = 0; e4 < EP / 4; ++e4) {
                  const float4 qv = qp[e4];
                  acc[q] = fmaf(x[4 * e4 + 0], qv.x, acc[q]);
                  acc[q] = fmaf(x[4 * e4 + 1], qv.y, acc[q]);
                  acc[q] = fmaf(x[4 * e4 + 2], qv.z, acc[q]);
                  acc[q] = fmaf(x[4 * e4 + 3], qv.w, acc[q]);
                }
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          for (int o = GS >> 1; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
          const float v = __shfl_sync(0xffffffffu, acc[q], (lane % rpp) * GS);
          if (lane / rpp == p) sem[q] = v;
        }
      }
    }

    if (TRAJ) {
      for (int p = 0; p < GT; ++p) {
        const int64_t row = y0 + p * rppt + tg;
        const bool active = tcl < CPY;
        const bool rok = row < n_rows && active;
        const char* rp = mapp + row * int64_t(Ep) * SB + tcl * 16;
        float acc[NQ], sq = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.f;
        for (int l0 = 0; l0 < ell; l0 += kU) {
          uint4 buf[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u)
            buf[u] = (rok && l0 + u < ell) ? ld_stream(rp + int64_t(l0 + u) * slab) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            if (active && l0 + u < ell) {
              float x[8];
              unpack_chunk<Tag>(buf[u], x);
#pragma unroll
              for (int e = 0; e < EP; ++e) sq = fmaf(x[e], x[e], sq);
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                const float4* qp = reinterpret_cast<const float4*>(qtraj + q * tl + (l0 + u) * Ep + tcl * EP);
#pragma unroll
                for (int e4 = 0; e4 < EP / 4; ++e4) {
                  const float4 qv = qp[e4];
                  acc[q] = fmaf(x[4 * e4 + 0], qv.x, acc[q]);
                  acc[q] = fmaf(x[4 * e4 + 1], qv.y, acc[q]);
                  acc[q] = fmaf(x[4 * e4 + 2], qv.z, acc[q]);
                  acc[q] = fmaf(x[4 * e4 + 3], qv.w, acc[q]);
                }
              }
            }
          }
        }
        for (int o = GT >> 1; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        const int src = (lane % rppt) * GT;
        const bool mine = lane / rppt == p;
        {
          const float v = __shfl_sync(0xffffffffu, sq, src);
          if (mine) msq = v;
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          for (int o = GT >> 1; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
          const float v = __shfl_sync(0xffffffffu, acc[q], src);
          if (mine) trj[q] = v;
        }
      }
    }

    // ---- epilogue: lane r scores row y0 + r and offers it to the lists
    const int64_t y = y0 + lane;
    // rows claimed by an earlier sub-batch of the same insert (R8) are no candidates
    const bool ok = y < n_rows && !(a.excl && ((__ldg(a.excl + (y >> 5)) >> (y & 31)) & 1u));
    const float re = (SEM && ok) ? st.r_e[y] : 0.f;
    const float rm = (TRAJ && msq > 0.f) ? rsqrtf(msq) : 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float s = 0.f;
      if (SEM) {
        const float c = sem[q] * rq0[q] * re;          // the semantic cosine (Eq. 1)
        if (a.out_cos && ok && q < a.nq) a.out_cos[int64_t(a.q0 + q) * a.cos_stride + y] = c;
        s = w * c;
      } else if (a.sem_cos) {                          // cached cosine of this (query, row)
        s = (ok && q < a.nq) ? w * __ldcs(a.sem_cos + int64_t(a.q0 + q) * a.cos_stride + y) : 0.f;
      }
      if (TRAJ) s = fmaf(w1, trj[q] * rq1[q] * rm, s);
      const uint64_t key = ok ? pack_key(s, a.id_offset + uint32_t(y)) : 0ull;
      lists[q].offer(key, a.k);
    }
  }
  }  // generic path

  // ---- 3. block merge + grid merge (last block)
  trace_mark(a.trace, 3);
  pdl_trigger();
  finish_topk<NQ, KPL, kScanWarps>(lists, reinterpret_cast<uint64_t*>(smem), a, s_valid, &s_last);
}

// ------------------------------------------------------------------ host side
using KernelFn = void (*)(const ScanArgs);

// multi-tile trajectory path: trajectory-only, one 16-byte chunk per
// row-layer; TPI*LB = 16 loads in flight per lane, TPI capped by registers.
static bool sem_in(const ScanArgs& a) { return a.w_sem != 0.f && !a.sem_cos; }

static int traj_tpi(const ScanArgs& a) {
  const int esz = a.st.bf16 ? 2 : 4;
  if (sem_in(a) || a.sem_cos || a.st.Ep * esz != 16) return 0;
  const int cap = a.nq <= 1 ? 16 : (a.nq <= 2 ? 8 : 4);
  int tpi = 1;
  while (tpi * 2 <= cap && tpi * 2 * a.ell <= 16) tpi *= 2;
  return tpi;
}

template <class Tag, int NQ, int KPL>
static KernelFn pick_mode(const ScanArgs& a) {
  if (a.w_sem == 1.f) return scan_gemv_kernel<Tag, NQ, KPL, true, false, 0>;
  if (!sem_in(a)) {
    switch (traj_tpi(a)) {
      case 16: if constexpr (NQ == 1) return scan_gemv_kernel<Tag, NQ, KPL, false, true, 16>; break;
      case 8: if constexpr (NQ <= 2) return scan_gemv_kernel<Tag, NQ, KPL, false, true, 8>; break;
      case 4: return scan_gemv_kernel<Tag, NQ, KPL, false, true, 4>;
      case 2: return scan_gemv_kernel<Tag, NQ, KPL, false, true, 2>;
      case 1: return scan_gemv_kernel<Tag, NQ, KPL, false, true, 1>;
      default: break;
    }
    return scan_gemv_kernel<Tag, NQ, KPL, false, true, 0>;
  }
  return scan_gemv_kernel<Tag, NQ, KPL, true, true, 0>;
}
template <class Tag, int NQ>
static KernelFn pick_kpl(const ScanArgs& a) {
  if (a.k == 1) return pick_mode<Tag, NQ, 0>(a);
  return a.k <= 32 ? pick_mode<Tag, NQ, 1>(a) : pick_mode<Tag, NQ, 2>(a);
}
template <class Tag>
static KernelFn pick_nq(const ScanArgs& a, int* NQ) {
  if (a.nq <= 1) { *NQ = 1; return pick_kpl<Tag, 1>(a); }
  if (a.nq <= 2) { *NQ = 2; return pick_kpl<Tag, 2>(a); }
  *NQ = 4;
  return pick_kpl<Tag, 4>(a);
}
static KernelFn pick(const ScanArgs& a, int* NQ) {
  return a.st.bf16 ? pick_nq<Bf16Tag>(a, NQ) : pick_nq<F32Tag>(a, NQ);
}

static size_t scan_smem(const ScanArgs& a, int NQ) {
  size_t f = 0;
  if (sem_in(a)) f += size_t(NQ) * a.st.Dp;
  if (a.w_sem != 1.f) f += size_t(NQ) * a.ell * a.st.Ep;
  size_t bytes = f * 4;
  const size_t merge = size_t(kScanWarps) * NQ * a.k * 8;
  return bytes > merge ? bytes : merge;
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// Per-kernel launch facts, computed once: the max dynamic smem attribute per
// kernel and blocks/SM per (kernel, smem) (host-side cache; the ABI may be
// called from several threads).
static std::mutex g_info_mu;
static std::map<const void*, size_t> g_smem_set;
static std::map<std::pair<const void*, size_t>, int> g_occ;

static int prepare(KernelFn fn, size_t smem) {
  const void* f = reinterpret_cast<const void*>(fn);
  std::lock_guard<std::mutex> lk(g_info_mu);
  size_t& set = g_smem_set[f];
  if (set < smem) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    set = smem;
  }
  int& per_sm = g_occ[{f, smem}];
  if (per_sm == 0) {
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, f, kScanThreads, smem);
    per_sm = v < 1 ? 1 : v;
  }
  return per_sm;
}

int scan_gemv_grid(const ScanArgs& a) {
  int NQ = 1;
  KernelFn fn = pick(a, &NQ);
  const size_t smem = scan_smem(a, NQ);
  const int per_sm = prepare(fn, smem);
  const int tpi = traj_tpi(a) > 0 ? traj_tpi(a) : 1;
  const int64_t ntiles = (a.n_rows + 32 * tpi - 1) / (32 * tpi);
  int64_t want = (ntiles + kScanWarps - 1) / kScanWarps;   // >= one tile per warp
  int64_t full = int64_t(per_sm) * sm_count();
  int64_t g = want < full ? want : full;
  return int(g < 1 ? 1 : g);
}

cudaError_t launch_scan_gemv(const ScanArgs& a, cudaStream_t s) {
  int NQ = 1;
  KernelFn fn = pick(a, &NQ);
  const size_t smem = scan_smem(a, NQ);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  prepare(fn, smem);
  count_launch();
  return launch_pdl(fn, dim3(a.grid), dim3(kScanThreads), smem, s, a);
}

}  // namespace fmoe
