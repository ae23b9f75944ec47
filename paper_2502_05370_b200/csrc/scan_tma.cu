// scan_tma.cu -- K2t: trajectory scan fed by a TMA bulk-copy ring.
//
// Computes, per query x and stored row y (Eq. 2; Reading R1):
//   traj = (q~_x[0:ell] . M~_y[0:ell]) * r_q(ell) / ||M~_y[0:ell]||
// with the map tiles held layer-major ([L][cap][Ep]),
// so the prefix of R consecutive rows is ell contiguous slab segments of R*RB
// bytes (RB = Ep * sizeof(dtype)).
//
// Why a TMA ring: a register-streaming GEMV keeps at most ~8 16-byte loads per
// lane in flight, which at prefix length 1..8 (16..128 bytes of map per row)
// cannot cover HBM latency.  Here one producer lane per CTA issues
// cp.async.bulk copies of whole slab segments (up to 64 KB per stage, 2-3
// stages, mbarrier complete_tx) while 8 consumer warps score rows out of shared
// memory; the bytes in flight per SM no longer depend on the prefix length.
// One CTA per SM (persistent, ~200 KB smem); tiles of R rows are dealt
// round-robin; every stage carries LC layers of one tile.
//
// Shared-memory reads are bank-conflict free: lanes read consecutive rows, and
// when a row-layer spans CPY > 1 16-byte chunks the chunk order is rotated by
// lane so that the 8 lanes of an LDS.128 phase hit 8 distinct 16-byte bank
// groups.  The query is staged in the same dtype/layout as the data.
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "merge.cuh"

namespace fmoe {

constexpr int kTmaConsumerWarps = 8;
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;   // + 1 producer warp
constexpr int kStageBytes = 64 * 1024;
constexpr int kMaxStages = 3;

template <class Tag>
__device__ __forceinline__ void unpack_any(const uint4& u, float (&x)[8]);
template <>
__device__ __forceinline__ void unpack_any<Bf16Tag>(const uint4& u, float (&x)[8]) {
  unpack8(u, x, Bf16Tag());
}
template <>
__device__ __forceinline__ void unpack_any<F32Tag>(const uint4& u, float (&x)[8]) {
  x[0] = __uint_as_float(u.x); x[1] = __uint_as_float(u.y);
  x[2] = __uint_as_float(u.z); x[3] = __uint_as_float(u.w);
  x[4] = x[5] = x[6] = x[7] = 0.f;
}

// chunk rotation making an LDS.128 phase (8 lanes, consecutive rows) conflict-free
__device__ __forceinline__ int chunk_rot(int lane, int cpy) {
  const int i = lane & 7;
  if (cpy == 1 || (cpy & (cpy - 1)) != 0) return 0;   // 1 chunk, or odd strides already spread
  return cpy >= 8 ? i : i / (8 / cpy);
}

template <class Tag, int NQ, int KPL, int RPT>
__global__ void __launch_bounds__(kTmaThreads, 1) scan_traj_tma_kernel(const ScanArgs a, int LC, int S) {
  using ST = StoreT<Tag>;
  using T = typename ST::T;
  constexpr int EP = ST::kElemsPer16B;
  constexpr int SB = ST::kBytes;
  constexpr int R = RPT * kTmaConsumerWarps * 32;       // rows per tile
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ double red[kTmaConsumerWarps + 1][NQ];
  __shared__ float rq[NQ];
  __shared__ int s_valid[NQ];
  __shared__ int s_last;

  const StoreView& st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Ep = st.Ep, E = st.E, ell = a.ell;
  const int RB = Ep * SB, CPY = RB / 16;
  const int tl = ell * Ep;                               // query elements per query
  unsigned char* stages = smem_raw;
  T* qs = reinterpret_cast<T*>(smem_raw + size_t(S) * kStageBytes);   // [NQ][ell][Ep] store dtype

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumerWarps);
    }
    mbar_fence_init();
  }
  trace_mark(a.trace, 0);
  pdl_wait();
  trace_mark(a.trace, 1);

  // ---- stage the trajectory queries (store dtype) and their norms
  double part[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    part[q] = 0.0;
    for (int i = tid; i < tl; i += kTmaThreads) {
      const int l = i / Ep, j = i - l * Ep;
      float v = 0.f;
      if (q < a.nq && j < E) v = to_store_value(a.q_prefix[int64_t(a.q0 + q) * a.q_stride + l * E + j], Tag());
      if constexpr (SB == 2) qs[q * tl + i] = __float2bfloat16_rn(v);
      else qs[q * tl + i] = v;
      part[q] += double(v) * double(v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
    if (lane == 0) red[warp][q] = part[q];
  }
  __syncthreads();
  if (tid < NQ) {
    double s1 = 0.0;
    for (int w = 0; w <= kTmaConsumerWarps; ++w) s1 += red[w][tid];
    rq[tid] = s1 > 0.0 ? float(1.0 / sqrt(s1)) : 0.f;
    s_valid[tid] = s1 > 0.0;
  }
  __syncthreads();
  trace_mark(a.trace, 2);

  WarpTopK<KPL> lists[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) lists[q].init();

  const int64_t n = a.n_rows;
  const int64_t ntiles = (n + R - 1) / R;
  const int nch = (ell + LC - 1) / LC;
  const unsigned char* maps = static_cast<const unsigned char*>(st.maps);

  if (warp == kTmaConsumerWarps) {
    // ---- producer: one lane streams slab segments into the ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      unsigned u = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t y0 = t * R;
        const int rows = int(n - y0 < R ? n - y0 : R);
        for (int c = 0; c < nch; ++c, ++u) {
          const int s = int(u % unsigned(S));
          mbar_wait(&empty[s], ((u / unsigned(S)) & 1u) ^ 1u);
          const int l0 = c * LC, lc = ell - l0 < LC ? ell - l0 : LC;
          mbar_arrive_expect_tx(&full[s], unsigned(lc * rows * RB));
          for (int l = 0; l < lc; ++l)
            bulk_g2s(stages + size_t(s) * kStageBytes + size_t(l) * R * RB,
                     maps + (int64_t(l0 + l) * st.cap + y0) * RB, unsigned(rows * RB), &full[s], pol);
        }
      }
    }
  } else {
    // ---- consumers: thread tid owns rows tid + 256*j of every tile
    const int rot = chunk_rot(lane, CPY);
    float rq1[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) rq1[q] = rq[q];
    unsigned u = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t y0 = t * R;
      const int rows = int(n - y0 < R ? n - y0 : R);
      float acc[RPT][NQ], sq[RPT];
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        sq[j] = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[j][q] = 0.f;
      }
      for (int c = 0; c < nch; ++c, ++u) {
        const int s = int(u % unsigned(S));
        mbar_wait(&full[s], (u / unsigned(S)) & 1u);
        const unsigned char* sb = stages + size_t(s) * kStageBytes;
        const int l0 = c * LC, lc = ell - l0 < LC ? ell - l0 : LC;
        for (int l = 0; l < lc; ++l) {
          for (int cc = 0; cc < CPY; ++cc) {
            int ch = cc + rot;
            if (ch >= CPY) ch -= CPY;
            float qv[NQ][8];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const uint4 qu = *reinterpret_cast<const uint4*>(qs + q * tl + (l0 + l) * Ep + ch * EP);
              unpack_any<Tag>(qu, qv[q]);
            }
            const unsigned char* base = sb + size_t(l) * R * RB + ch * 16;
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
              const int r = tid + j * (kTmaConsumerWarps * 32);
              if (r < rows) {
                const uint4 du = *reinterpret_cast<const uint4*>(base + size_t(r) * RB);
                float x[8];
                unpack_any<Tag>(du, x);
#pragma unroll
                for (int e = 0; e < EP; ++e) sq[j] = fmaf(x[e], x[e], sq[j]);
#pragma unroll
                for (int q = 0; q < NQ; ++q)
#pragma unroll
                  for (int e = 0; e < EP; ++e) acc[j][q] = fmaf(x[e], qv[q][e], acc[j][q]);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int r = tid + j * (kTmaConsumerWarps * 32);
        const bool ok = r < rows;
        const float rm = sq[j] > 0.f ? rsqrtf(sq[j]) : 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float sc = fmaf(1.f, acc[j][q] * rq1[q] * rm, 0.f);
          lists[q].offer(ok ? pack_key(sc, a.id_offset + uint32_t(y0 + r)) : 0ull, a.k);
        }
      }
    }
  }

  trace_mark(a.trace, 3);
  pdl_trigger();
  finish_topk<NQ, KPL, kTmaConsumerWarps + 1>(lists, reinterpret_cast<uint64_t*>(smem_raw), a, s_valid, &s_last);
}

// ------------------------------------------------------------------ host side
using TmaFn = void (*)(const ScanArgs, int, int);

template <class Tag, int NQ, int KPL>
static TmaFn pick_rpt(int rpt) {
  switch (rpt) {
    case 8: return scan_traj_tma_kernel<Tag, NQ, KPL, 8>;
    case 4: return scan_traj_tma_kernel<Tag, NQ, KPL, 4>;
    case 2: return scan_traj_tma_kernel<Tag, NQ, KPL, 2>;
    default: return scan_traj_tma_kernel<Tag, NQ, KPL, 1>;
  }
}
template <class Tag, int NQ>
static TmaFn pick_k(int k, int rpt) {
  if (k == 1) return pick_rpt<Tag, NQ, 0>(rpt);
  return k <= 32 ? pick_rpt<Tag, NQ, 1>(rpt) : pick_rpt<Tag, NQ, 2>(rpt);
}
template <class Tag>
static TmaFn pick_q(int nq, int k, int rpt, int* NQ) {
  if (nq <= 1) { *NQ = 1; return pick_k<Tag, 1>(k, rpt); }
  if (nq <= 2) { *NQ = 2; return pick_k<Tag, 2>(k, rpt); }
  *NQ = 4;
  return pick_k<Tag, 4>(k, rpt);
}

struct TmaPlan { TmaFn fn; int rpt, LC, S, NQ; size_t smem; };

static TmaPlan plan(const ScanArgs& a) {
  TmaPlan p{};
  const int esz = a.st.bf16 ? 2 : 4;
  const int RB = a.st.Ep * esz;
  int rows = kStageBytes / RB;                 // rows of one layer that fit a stage
  int rpt = 8;
  while (rpt > 1 && rpt * kTmaConsumerWarps * 32 > rows) rpt >>= 1;
  p.rpt = rpt;
  const int R = rpt * kTmaConsumerWarps * 32;
  p.LC = kStageBytes / (R * RB);
  if (p.LC < 1) p.LC = 1;
  int NQ = 1;
  p.fn = a.st.bf16 ? pick_q<Bf16Tag>(a.nq, a.k, rpt, &NQ) : pick_q<F32Tag>(a.nq, a.k, rpt, &NQ);
  p.NQ = NQ;
  const size_t qbytes = size_t(NQ) * a.ell * a.st.Ep * esz;
  const size_t budget = 220 * 1024;
  int S = int((budget - qbytes) / kStageBytes);
  p.S = S > kMaxStages ? kMaxStages : S;
  p.smem = size_t(p.S) * kStageBytes + ((qbytes + 15) & ~size_t(15));
  return p;
}

bool scan_tma_supported(const ScanArgs& a) {
  const int esz = a.st.bf16 ? 2 : 4;
  return a.w_sem == 0.f && a.st.Ep * esz <= kStageBytes / (kTmaConsumerWarps * 32) && plan(a).S >= 2;
}

static int sm_count_tma() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int scan_tma_grid(const ScanArgs& a) {
  const TmaPlan p = plan(a);
  const int64_t R = int64_t(p.rpt) * kTmaConsumerWarps * 32;
  const int64_t ntiles = (a.n_rows + R - 1) / R;
  const int64_t g = ntiles < sm_count_tma() ? ntiles : sm_count_tma();
  return int(g < 1 ? 1 : g);
}

cudaError_t launch_scan_tma(const ScanArgs& a, cudaStream_t s) {
  const TmaPlan p = plan(a);
  {
    static std::mutex mu;
    static std::map<const void*, size_t> set;
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = set[reinterpret_cast<const void*>(p.fn)];
    if (cur < p.smem) {
      cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(p.fn),
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(p.smem));
      if (e != cudaSuccess) return e;
      cur = p.smem;
    }
  }
  count_launch();
  return launch_pdl(p.fn, dim3(a.grid), dim3(kTmaThreads), p.smem, s, a, p.LC, p.S);
}

}  // namespace fmoe
