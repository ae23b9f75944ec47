// scan_f32mm.cu -- K2b: batched scoring of an fp32 store, 5 <= nq <= 64
// queries per pass, read from HBM ONCE per pass (the GEMV K2 streams the
// store once per 4 queries), fused with per-warp top-k lists.
//
// What it computes (Eq. 1, Eq. 2 and the RDY blend):
//   S_sem [x][y] = (q_x . e_y) * r_q(x) * r_e[y]
//   S_traj[x][y] = (q_x[0:ell] . M_y[0:ell]) * r_q(ell,x) / sqrt(psq[ell-1][y])
//   S = w*S_sem + (1-w)*S_traj      (S_sem optionally from cached cosines)
// and the k best (score desc, id asc) per x.  fp32 operands, fp32 FFMA
// accumulation (round-to-nearest at every step), so the scores carry the
// GEMV's precision -- no re-rank needed for the 1e-5 parity bar.
//
// Why FFMA and not the tensor cores: the store is fp32 and the paper's scores
// are fp32; kind::tf32 truncates both operands to 10 mantissa
// bits (|error| up to ~2^-9 on a cosine), so a tensor-core fp32 path needs a
// 3xTF32 split of the streamed tile in shared memory plus an exact re-rank.
// At B = 64 the pass does 32 FLOP per store byte, above the FFMA ridge
// (~72 TFLOP/s / 6.5 TB/s = 11), so it is ALU-bound (roofline "alu").
//
// Structure: 256 threads, 1 CTA per SM, persistent over tiles of RT store
// rows (round-robin).  K runs in chunks of 32 floats (128 B per row): the
// semantic chunks over D, then the trajectory chunks over the flattened
// prefix [ell][Ep] (a chunk gathers 16-byte pieces of several layer slabs).
// A 3-stage cp.async ring holds, per chunk, the RT store rows and the 64
// query rows (prepared operand, L2-resident), both 128-byte-XOR swizzled so
// a warp's row fragments are conflict-free and its query fragments are
// broadcasts.  Warp w owns query group wq = w % WQ (8 queries) and row block
// wr = w / WQ; a thread accumulates 8 queries x TR rows (rows lane + 32j of
// the block).  Epilogue per tile: scale, blend, exclusion bitmap, cosine side
// output / input, then each (warp, query) keeps its own sorted top-k list in
// shared memory (ballot the keys beating the list's k-th, insert warp-
// cooperatively); lists go to cand[q][CTA*(8/WQ) + wr][k] and the merge
// kernel finishes.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace fmoe {

#ifndef FMOE_F32MM_UNROLL
#define FMOE_F32MM_UNROLL 2
#endif
constexpr int kMmUnroll = FMOE_F32MM_UNROLL;   // k-steps of the FFMA loop unrolled (code size vs. scheduling)
constexpr int kMmThreads = 256;
constexpr int kMmWarps = kMmThreads / 32;
constexpr int kMmQ = 64;            // queries per pass (8 per warp query group)
constexpr int kMmStages = 3;
constexpr int kMmQStage = kMmQ * 128;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;     // src-size 0: zero-fill, nothing read
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Insert key into the warp's sorted (desc) list lb[0..cnt) of capacity k (all
// lanes, warp-uniform key > current k-th).  Entries j and j + 32 live in lane j.
__device__ __forceinline__ void list_insert(uint64_t* lb, int k, int& cnt, uint64_t key, int lane) {
  const uint64_t v0 = lane < cnt ? lb[lane] : 0ull;
  const uint64_t v1 = lane + 32 < cnt ? lb[lane + 32] : 0ull;
  const int pos = __popc(__ballot_sync(0xffffffffu, lane < cnt && v0 > key)) +
                  __popc(__ballot_sync(0xffffffffu, lane + 32 < cnt && v1 > key));
  const int nc = cnt + 1 < k ? cnt + 1 : k;
  const uint64_t p0 = shfl_up_u64(v0, 1);
  const uint64_t top = shfl_u64(v0, 31);
  const uint64_t u1 = shfl_up_u64(v1, 1);     // every lane shuffles (full-mask shfl.sync)
  const uint64_t p1 = lane == 0 ? top : u1;
  __syncwarp();
  if (lane < nc) {
    if (lane == pos) lb[lane] = key;
    else if (lane > pos) lb[lane] = p0;
  }
  if (lane + 32 < nc) {
    if (lane + 32 == pos) lb[lane + 32] = key;
    else if (lane + 32 > pos) lb[lane + 32] = p1;
  }
  __syncwarp();
  cnt = nc;
}

// (plain C++ shared loads, not asm: the compiler may hoist the next query
// fragment above the current FFMAs; the barrier intrinsics still order them)
template <int TR>
__device__ __forceinline__ void mm_chunk(const unsigned char* rows, const unsigned char* qs, int wq, int lane, int wr,
                                         float (&acc)[8][TR]) {
  const unsigned char* rb = rows + (wr * 32 * TR + lane) * 128;
  const unsigned char* qb = qs + wq * 8 * 128;
#pragma unroll kMmUnroll
  for (int kk = 0; kk < 8; ++kk) {
    const int sw = (kk ^ (lane & 7)) * 16;
    float4 x[TR];
#pragma unroll
    for (int j = 0; j < TR; ++j) x[j] = *reinterpret_cast<const float4*>(rb + j * 32 * 128 + sw);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 q = *reinterpret_cast<const float4*>(qb + i * 128 + ((kk ^ i) * 16));
#pragma unroll
      for (int j = 0; j < TR; ++j) {
        acc[i][j] = fmaf(x[j].x, q.x, acc[i][j]);
        acc[i][j] = fmaf(x[j].y, q.y, acc[i][j]);
        acc[i][j] = fmaf(x[j].z, q.z, acc[i][j]);
        acc[i][j] = fmaf(x[j].w, q.w, acc[i][j]);
      }
    }
  }
}

template <int TR, bool SEM, bool TRAJ, int MINB = 1>
__global__ void __launch_bounds__(kMmThreads, MINB) scan_f32mm_kernel(const F32mmArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const StoreView& st = a.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int WQ = a.wq, RB = kMmWarps / WQ;                 // query groups, row blocks
  const int RT = RB * 32 * TR;                               // rows per tile
  const int wq = warp % WQ, wr = warp / WQ;
  const int stage_bytes = RT * 128 + kMmQStage;
  uint64_t* lists = reinterpret_cast<uint64_t*>(smem + kMmStages * stage_bytes);   // [64][k]
  const uint32_t ring = smem_u32(smem);
  const int k = a.k;
  const int64_t n = a.n_rows;
  const int n_tiles = int((n + RT - 1) / RT);
  const int nch = a.n_sem_ch + a.n_traj_ch;
  const int my_tiles = int(blockIdx.x) < n_tiles ? (n_tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  const int total = my_tiles * nch;
  const char* embp = static_cast<const char*>(st.emb);
  const char* mapp = static_cast<const char*>(st.maps);
  const int Dp = st.Dp, Ep = st.Ep, tl = a.ell * Ep;

  pdl_wait();
  // chunk `it` of this CTA -> (tile, c): its store rows and query rows into stage it % S
  auto issue = [&](int it) {
    if (it < total) {
      const int t = int(blockIdx.x) + (it / nch) * int(gridDim.x);
      const int c = it % nch;
      const uint32_t sb = ring + uint32_t((it % kMmStages) * stage_bytes);
      const int pieces = RT * 8;
      for (int pc = tid; pc < pieces; pc += kMmThreads) {
        const int r = pc >> 3, p = pc & 7;
        const int64_t y = int64_t(t) * RT + r;
        const char* src = embp;
        bool ok = y < n;
        if (c < a.n_sem_ch) {
          const int f = c * 32 + p * 4;
          ok = ok && f < Dp;
          src = embp + (y * Dp + f) * 4;
        } else {
          const int f = (c - a.n_sem_ch) * 32 + p * 4;
          ok = ok && f < tl;
          const int layer = f / Ep, col = f - layer * Ep;
          src = mapp + ((int64_t(layer) * st.cap + y) * Ep + col) * 4;
        }
        cp_async16(sb + uint32_t(r * 128 + ((p ^ (r & 7)) * 16)), ok ? src : embp, ok);
      }
      const uint32_t qb = sb + uint32_t(RT * 128);
      for (int pc = tid; pc < kMmQ * 8; pc += kMmThreads) {
        const int x = pc >> 3, p = pc & 7;
        const bool ok = x < a.nq;
        const float* src = a.qop + int64_t(ok ? x : 0) * a.qpitch + c * 32 + p * 4;
        cp_async16(qb + uint32_t(x * 128 + ((p ^ (x & 7)) * 16)), src, ok);
      }
    }
    cp_async_commit();   // (an empty group past the end keeps the wait count uniform)
  };

  // per-warp lists: this warp's 8 queries in row block wr
  for (int i = tid; i < kMmQ * k; i += kMmThreads) lists[i] = 0ull;
  uint64_t thr[8];
  int cnt[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { thr[i] = 0ull; cnt[i] = 0; }
  const float w = a.w, w1 = 1.f - a.w;

  for (int s = 0; s < kMmStages - 1; ++s) issue(s);
  float accs[8][TR], acct[8][TR];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TR; ++j) { accs[i][j] = 0.f; acct[i][j] = 0.f; }
  __syncthreads();   // lists zeroed

  for (int it = 0; it < total; ++it) {
    cp_async_wait<kMmStages - 2>();
    __syncthreads();                      // chunk it landed for everyone; stage (it-1) % S is free
    issue(it + kMmStages - 1);
    const unsigned char* sb = smem + (it % kMmStages) * stage_bytes;
    const int c = it % nch;
    if (SEM && (!TRAJ || c < a.n_sem_ch)) mm_chunk<TR>(sb, sb + RT * 128, wq, lane, wr, accs);
    else mm_chunk<TR>(sb, sb + RT * 128, wq, lane, wr, acct);
    if (c != nch - 1) continue;

    // ---- epilogue of tile t
    const int t = int(blockIdx.x) + (it / nch) * int(gridDim.x);
#pragma unroll
    for (int j = 0; j < TR; ++j) {
      const int64_t y = int64_t(t) * RT + wr * 32 * TR + j * 32 + lane;
      const bool ok = y < n && !(a.excl && ((__ldg(a.excl + (y >> 5)) >> (y & 31)) & 1u));
      const float re = (SEM && ok) ? st.r_e[y] : 0.f;
      float rm = 0.f;
      if (TRAJ && ok) {
        const float ps = st.psq[int64_t(a.ell - 1) * st.cap + y];
        rm = ps > 0.f ? rsqrtf(ps) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int q = wq * 8 + i;
        float s = 0.f;
        if (q < a.nq) {
          if (SEM) {
            const float cs = accs[i][j] * a.rq_s[q] * re;     // the semantic cosine (Eq. 1)
            if (a.out_cos && ok) a.out_cos[int64_t(q) * a.cos_stride + y] = cs;
            s = w * cs;
          } else if (a.sem_cos) {
            s = ok ? w * __ldcs(a.sem_cos + int64_t(q) * a.cos_stride + y) : 0.f;
          }
          if (TRAJ) s = fmaf(w1, acct[i][j] * a.rq_t[q] * rm, s);
        }
        const uint64_t key = (ok && q < a.nq) ? pack_key(s, a.id_offset + uint32_t(y)) : 0ull;
        unsigned m = __ballot_sync(0xffffffffu, key > thr[i]);
        uint64_t* lb = lists + (wr * (8 * WQ) + q) * k;
        while (m) {
          const int src = __ffs(m) - 1;
          m &= m - 1;
          const uint64_t kv = shfl_u64(key, src);
          if (kv > thr[i]) {
            list_insert(lb, k, cnt[i], kv, lane);
            if (cnt[i] == k) thr[i] = lb[k - 1];
          }
        }
        accs[i][j] = 0.f;
        acct[i][j] = 0.f;
      }
    }
  }
  cp_async_wait<0>();
  pdl_trigger();
  // ---- lists -> cand[q][CTA * RB + wr][k]
  __syncwarp();
  const int n_lists = int(gridDim.x) * RB;
  for (int i = 0; i < 8; ++i) {
    const int q = wq * 8 + i;
    if (q >= a.nq) continue;
    const uint64_t* lb = lists + (wr * (8 * WQ) + q) * k;
    uint64_t* dst = a.cand + (int64_t(a.cand_q0 + q) * n_lists + int64_t(blockIdx.x) * RB + wr) * k;
    for (int e = lane; e < k; e += 32) dst[e] = e < cnt[i] ? lb[e] : 0ull;
  }
}

// Prepared query operand of one pass: row x = [sem: Dp floats zero-padded to
// n_sem_ch*32 | traj: the prefix as [ell][Ep] (pad columns 0) zero-padded to
// n_traj_ch*32]; fp64 norms -> rq_s, rq_t; valid = the query's used parts
// have non-zero norm (a zero-norm query reports (NaN, -1), Reading R3).
__global__ void __launch_bounds__(256) f32mm_prep_kernel(const F32mmPrep p) {
  __shared__ double red[2][8];
  const int x = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();
  float* row = p.qop + int64_t(x) * p.qpitch;
  double s0 = 0.0, s1 = 0.0;
  const int ns = p.n_sem_ch * 32, nt = p.n_traj_ch * 32, tl = p.ell * p.Ep;
  for (int f = tid; f < ns; f += 256) {
    const float v = (p.q_emb && f < p.D) ? p.q_emb[int64_t(x) * p.D + f] : 0.f;
    row[f] = v;
    s0 += double(v) * double(v);
  }
  for (int f = tid; f < nt; f += 256) {
    float v = 0.f;
    if (p.q_prefix && f < tl) {
      const int l = f / p.Ep, j = f - l * p.Ep;
      if (j < p.E) v = p.q_prefix[int64_t(x) * p.q_stride + l * p.E + j];
    }
    row[ns + f] = v;
    s1 += double(v) * double(v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if (lane == 0) { red[0][warp] = s0; red[1][warp] = s1; }
  __syncthreads();
  if (tid == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int w = 0; w < 8; ++w) { t0 += red[0][w]; t1 += red[1][w]; }
    p.rq_s[x] = t0 > 0.0 ? float(1.0 / sqrt(t0)) : 0.f;
    p.rq_t[x] = t1 > 0.0 ? float(1.0 / sqrt(t1)) : 0.f;
    p.valid[x] = ((!p.sem || t0 > 0.0) && (!p.traj || t1 > 0.0)) ? 1.f : 0.f;
  }
  pdl_trigger();
}

int f32mm_wq(int nq) { return nq <= 8 ? 1 : nq <= 16 ? 2 : nq <= 32 ? 4 : 8; }

// Two CTAs per SM for single-part passes of > 32 queries: thread tiles of
// 8 queries x 4 rows, <= 128 registers, 128-row tiles, twice the warps per SM
// to hide the shared-memory and FMA latencies.  Measured (Qwen shape, N = 1M,
// B = 64, profiles/r02p_f32mm_2cta.md): semantic 8.40 -> 8.12 ms, trajectory
// ell = 16 5.29 -> 4.37 ms; a blend (two accumulator sets -> 8 x 2 tiles) got
// slower (13.4 -> 15.3 ms) and keeps one CTA per SM.  FMOE_F32MM_2CTA=0: off.
static bool f32mm_2cta(int wq, bool blend) {
  static const bool off = getenv("FMOE_F32MM_2CTA") && atoi(getenv("FMOE_F32MM_2CTA")) == 0;
  return !off && wq == 8 && !blend;
}
// thread tile rows: TR = WQ (RT = 256 rows per tile); a blend keeps two
// accumulator sets, so TR <= 4 there (RT = 128 at WQ = 8)
static int f32mm_tr(int wq, bool blend) {
  if (f32mm_2cta(wq, blend)) return 4;
  return blend && wq > 4 ? 4 : wq;
}

static size_t f32mm_smem(int wq, int k, bool blend) {
  const int rt = (kMmWarps / wq) * 32 * f32mm_tr(wq, blend);
  return size_t(kMmStages) * (rt * 128 + kMmQStage) + size_t(kMmQ) * k * 8;
}

int f32mm_grid(int64_t n_rows, int nq, bool blend) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int wq = f32mm_wq(nq);
  const int rt = (kMmWarps / wq) * 32 * f32mm_tr(wq, blend);
  const int64_t tiles = (n_rows + rt - 1) / rt;
  const int units = f32mm_2cta(wq, blend) ? 2 * sms : sms;
  return int(tiles < units ? (tiles < 1 ? 1 : tiles) : units);
}

int f32mm_lists_per_cta(int nq) { return kMmWarps / f32mm_wq(nq); }

cudaError_t launch_f32mm_prep(const F32mmPrep& p, int nq, cudaStream_t s) {
  count_launch();
  return launch_pdl(f32mm_prep_kernel, dim3(unsigned(nq)), dim3(256), 0, s, p);
}

template <int TR, int MINB = 1>
static cudaError_t launch_tr(const F32mmArgs& a, bool sem, bool traj, size_t smem, int grid, cudaStream_t s) {
  using Fn = void (*)(const F32mmArgs);
  Fn fn = nullptr;
  if constexpr (MINB == 1)   // (two-CTA launches are single-part: no blend variant)
    fn = sem && traj ? scan_f32mm_kernel<(TR > 4 ? 4 : TR), true, true, 1>
                     : sem ? scan_f32mm_kernel<TR, true, false, 1> : scan_f32mm_kernel<TR, false, true, 1>;
  else
    fn = sem ? scan_f32mm_kernel<TR, true, false, MINB> : scan_f32mm_kernel<TR, false, true, MINB>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  count_launch();
  return launch_pdl(fn, dim3(unsigned(grid)), dim3(kMmThreads), smem, s, a);
}

cudaError_t launch_f32mm(const F32mmArgs& a, cudaStream_t s) {
  const bool sem = a.n_sem_ch > 0, traj = a.n_traj_ch > 0;
  const bool blend = sem && traj;
  if ((a.wq != 1 && a.wq != 2 && a.wq != 4 && a.wq != 8) || a.nq < 1 || a.nq > 8 * a.wq || a.k < 1 ||
      a.k > kMaxK)
    return cudaErrorInvalidValue;
  const size_t smem = f32mm_smem(a.wq, a.k, blend);
  const int grid = a.grid;
  if (f32mm_2cta(a.wq, blend)) return launch_tr<4, 2>(a, sem, traj, smem, grid, s);
  switch (f32mm_tr(a.wq, blend)) {
    case 1: return launch_tr<1>(a, sem, traj, smem, grid, s);
    case 2: return launch_tr<2>(a, sem, traj, smem, grid, s);
    case 4: return launch_tr<4>(a, sem, traj, smem, grid, s);
    default: return launch_tr<8>(a, sem, traj, smem, grid, s);
  }
}

}  // namespace fmoe
