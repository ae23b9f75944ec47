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
#include "common.cuh"
#include "kernels.cuh"

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

template <class Tag, int NQ, int KPL, bool SEM, bool TRAJ>
__global__ void __launch_bounds__(kScanThreads) scan_gemv_kernel(const ScanArgs a) {
  using ST = StoreT<Tag>;
  constexpr int EP = ST::kElemsPer16B;
  constexpr int SB = ST::kBytes;
  extern __shared__ __align__(16) float smem[];
  __shared__ double red[kScanWarps][2 * NQ];
  __shared__ float rq[2][NQ];

  const StoreView& st = a.st;
  const int Dp = st.Dp, Ep = st.Ep, E = st.E, D = st.D, ell = a.ell;
  const int tl = ell * Ep;
  float* qsem = smem;                              // [NQ][Dp]
  float* qtraj = smem + (SEM ? NQ * Dp : 0);       // [NQ][ell][Ep]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

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
    if (blockIdx.x == 0 && tid < a.nq && a.qinfo)
      a.qinfo[a.q0 + tid] = ((!SEM || s0 > 0.0) && (!TRAJ || s1 > 0.0)) ? 1.f : 0.f;
  }
  __syncthreads();

  float rq0[NQ], rq1[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) { rq0[q] = rq[0][q]; rq1[q] = rq[1][q]; }

  // ---- 2. stream 32-row tiles
  WarpTopK<KPL> lists[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) lists[q].init();

  const int64_t n_rows = a.n_rows;
  const int64_t ntiles = (n_rows + 31) / 32;
  const int64_t wstride = int64_t(gridDim.x) * kScanWarps;
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

  for (int64_t t = int64_t(blockIdx.x) * kScanWarps + warp; t < ntiles; t += wstride) {
    const int64_t y0 = t * 32;
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
    const bool ok = y < n_rows;
    const float re = (SEM && ok) ? st.r_e[y] : 0.f;
    const float rm = (TRAJ && msq > 0.f) ? 1.f / sqrtf(msq) : 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float s = 0.f;
      if (SEM) s = w * (sem[q] * rq0[q] * re);
      if (TRAJ) s = fmaf(w1, trj[q] * rq1[q] * rm, s);
      const uint64_t key = ok ? pack_key(s, a.id_offset + uint32_t(y)) : 0ull;
      lists[q].offer(key, a.k);
    }
  }

  // ---- 3. block merge of the warps' lists, one warp per query
  __syncthreads();
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem);  // [kScanWarps][NQ][k]
  const int k = a.k;
#pragma unroll
  for (int q = 0; q < NQ; ++q) lists[q].store(sk + (warp * NQ + q) * k, k);
  __syncthreads();
  if (warp < a.nq) {
    const int q = warp;
    WarpTopK<KPL> m;
#pragma unroll
    for (int s = 0; s < KPL; ++s) {
      const int j = s * 32 + lane;
      m.v[s] = j < k ? sk[q * k + j] : 0ull;
    }
    for (int w2 = 1; w2 < kScanWarps; ++w2)
      for (int j0 = 0; j0 < k; j0 += 32) {
        const uint64_t key = (j0 + lane < k) ? sk[(w2 * NQ + q) * k + j0 + lane] : 0ull;
        m.offer(key, k);
      }
    m.store(a.cand + (int64_t(a.q0 + q) * a.grid + blockIdx.x) * k, k);
  }
}

// ------------------------------------------------------------------ host side
using KernelFn = void (*)(const ScanArgs);

template <class Tag, int NQ, int KPL>
static KernelFn pick_mode(float w) {
  if (w == 1.f) return scan_gemv_kernel<Tag, NQ, KPL, true, false>;
  if (w == 0.f) return scan_gemv_kernel<Tag, NQ, KPL, false, true>;
  return scan_gemv_kernel<Tag, NQ, KPL, true, true>;
}
template <class Tag, int NQ>
static KernelFn pick_kpl(const ScanArgs& a) {
  return a.k <= 32 ? pick_mode<Tag, NQ, 1>(a.w_sem) : pick_mode<Tag, NQ, 2>(a.w_sem);
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
  if (a.w_sem != 0.f) f += size_t(NQ) * a.st.Dp;
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

int scan_gemv_grid(const ScanArgs& a) {
  int NQ = 1;
  KernelFn fn = pick(a, &NQ);
  const size_t smem = scan_smem(a, NQ);
  cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(fn), kScanThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t ntiles = (a.n_rows + 31) / 32;
  int64_t want = (ntiles + kScanWarps - 1) / kScanWarps;
  int64_t full = int64_t(per_sm) * sm_count();
  int64_t g = want < full ? want : full;
  return int(g < 1 ? 1 : g);
}

cudaError_t launch_scan_gemv(const ScanArgs& a, cudaStream_t s, int* grid_out) {
  int NQ = 1;
  KernelFn fn = pick(a, &NQ);
  const size_t smem = scan_smem(a, NQ);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  if (grid_out) *grid_out = a.grid;
  fn<<<a.grid, kScanThreads, smem, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace fmoe
