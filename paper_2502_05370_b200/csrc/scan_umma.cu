// scan_umma.cu -- K3: batched scoring on the 5th-gen tensor cores (tcgen05),
// fused with a per-query top-k epilogue.  bf16 stores, 5 <= B <= 128 queries
// per pass on single CTAs, 129..256 on CTA pairs (cta_group::2, M = 256: each
// CTA of a pair holds 128 query rows and half of every 256-row store tile, the
// leader issues the MMAs for both, each CTA's TMEM receives its own queries'
// accumulators; the peer's loads are relayed to the leader's stage barrier and
// the MMA commits multicast to both CTAs).
//
// What it computes (Eq. 1, Eq. 2 and the RDY blend):
//   S_sem [x][y] = (q~_x . e~_y) * r_q(x) * r_e[y]
//   S_traj[x][y] = (q~_x[0:ell] . M~_y[0:ell]) * r_q(ell,x) / sqrt(psq[ell-1][y])
//   S = w*S_sem + (1-w)*S_traj,  then the k best (score desc, id asc) per x.
// The two dot products are real dense contractions once B >= 16: queries sit
// on the UMMA M dimension (128 lanes of TMEM, zero-padded), store rows on N
// (256 per tile), and K runs over D (64-element SW128 boxes) and over the
// observed layers of the layer-major map slabs.
//
// Structure (one CTA per SM, persistent over 256-row tiles, round-robin):
//   warp 0      TMA producer: cp.async.bulk.tensor boxes of the query and
//               store tiles into an S-stage smem ring (mbarrier complete_tx)
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma kind::f16
//               (bf16 x bf16 -> fp32 in TMEM), tcgen05.commit frees stages and
//               publishes finished accumulators
//   warp 2      TMEM allocator (512 columns)
//   warps 4..11 epilogue: tcgen05.ld 32x32b (thread = query lane, warp pair
//               = two column halves), scale, blend, threshold test against the
//               thread's k-th key; the rare winners go into a per-thread min-heap
//               in shared memory (out-of-line replace-root keeps the hot loop
//               small: a fully unrolled version thrashed the instruction cache)
// Accumulators: 1 (semantic or trajectory) or 2 (blend) x 256 fp32 columns,
// double-buffered in TMEM when they fit (512 columns).
// Per-CTA lists (one per column half) go to cand[q][2*cta+half][k]; a tiny
// merge kernel (PDL) finishes.
//
// Trajectory K layout by map row width RB = Ep*2 bytes (SURVEY §8(a) layout
// note): RB = 16 (Mixtral, E = 8): SWIZZLE_NONE core matrices, one K = 16 MMA
// spans two layers (LBO = the layer stride inside the stage); RB = 32 (Phi):
// SWIZZLE_32B, one MMA per layer; RB = 64: SWIZZLE_64B, 2 MMAs per layer;
// RB = 128 (Qwen, E = 60 padded to 64): SWIZZLE_128B, 4 MMAs per layer.
// RB = 16 operands are moved with 1-D bulk copies (a layer's rows of a tile are
// one contiguous run of the slab): 16-byte-wide tensor boxes cost one TMA
// request per row and held the Mixtral-shape trajectory scan at 1.6 TB/s.
#include <cuda.h>

#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace fmoe {

constexpr int UM_M = 128;
constexpr int UM_N = 256;
constexpr int kUmEpiWarps = 8;               // 2 per SM sub-partition: two column halves
constexpr int kUmThreads = (4 + kUmEpiWarps) * 32;
constexpr int kStageA = UM_M * 128;          // 16 KB of queries per stage (per CTA)
// Tile height TN: 256 store rows, or 128 when a tile needs two accumulators
// (blend, or the K-split semantic scan) so that two tiles' accumulators still
// fit TMEM's 512 columns double-buffered (2 x 2 x 128).  Store rows per CTA
// and tile: all TN (cta_group::1), or half (cta_group::2).
__host__ __device__ constexpr int um_rows(int cg, int tn = UM_N) { return tn / cg; }
__host__ __device__ constexpr int um_stage_bytes(int cg, int tn = UM_N) { return kStageA + um_rows(cg, tn) * 128; }
constexpr int kUmMaxStages = 8;

__device__ __forceinline__ int nvalid_rows(int64_t yc, int64_t n_rows, bool live) {
  if (!live) return 0;
  const int64_t left = n_rows - yc;
  return left >= 32 ? 32 : (left <= 0 ? 0 : int(left));
}

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// cta_group::2: the commit arrives on the barrier at the same offset in both
// CTAs of the pair (multicast mask 0b11)
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
template <int CG>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
// thread-block cluster helpers (CTA pairs)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// L2 prefetches (no smem, no barrier): the store operand of a k-block issued
// ahead of the smem ring, so its TMA load later hits L2
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// Non-critical waiter (the epilogue warps wait most of a tile for its
// accumulators): poll with test_wait and a real sleep in between.  The
// try_wait suspend loop wakes on every mbarrier event of the CTA -- each TMA
// complete_tx -- so eight warps waking every ~100 cycles competed with the
// producer/MMA barrier traffic.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, unsigned parity, unsigned ns) {
  while (!mbar_test(bar, parity)) __nanosleep(ns);
}
// global -> shared 1-D bulk copy without a cache hint (query operands: re-read by every tile)
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// per-tile role timeline of CTA 0 (debug tracer): flat slot 8192 + role*256 + tile
__device__ __forceinline__ void tile_mark(unsigned long long* trace, int role, unsigned ti) {
  if (trace && blockIdx.x == 0 && ti < 256) trace[8192 + role * 256 + ti] = globaltimer();
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// shared -> global tensor store (bulk group) and its completion waits
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
// shared -> global 1-D bulk copy (bulk group)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

// UMMA shared-memory matrix descriptor (K-major), sm_100 "version 1".
//  layout: 0 none (interleaved core matrices), 6 SW32, 4 SW64, 2 SW128
__device__ __forceinline__ uint64_t umma_desc(const void* smem, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((smem_u32(smem) >> 4) & 0x3fff);
  d |= uint64_t((lbo_bytes >> 4) & 0x3fff) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3fff) << 32;
  d |= uint64_t(1) << 46;                      // version (Blackwell)
  d |= uint64_t(layout & 7) << 61;
  return d;
}
// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major.
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

struct UmmaParams {
  int64_t n_rows;       // rows to scan
  int n_tiles;
  int k;                // list length
  int nq;               // queries of this pass (<= 128 * CG; CTA r of a pair owns rows r*128..)
  float w;              // blend weight
  int n_sem_kb;         // semantic k-blocks (64 elements), 0 if no semantic part
  int n_traj_kb;        // trajectory k-blocks (stages)
  int ell_pad;          // layers covered by trajectory k-blocks (ell, even for RB = 16)
  int tmode;            // 0: RB 16, 1: RB 32, 2: RB 64, 3: RB 128
  int lc;               // layers per trajectory stage
  int stages;
  int acc_stages;       // TMEM accumulator buffers (1 or 2)
  int fake_loads;       // debug knob (FMOE_FAKE_LOADS=1): skip the loads, results are garbage
  int epi_sleep;        // epilogue accumulator wait: ns between polls (0 = try_wait suspend loop)
  int l2pf;             // L2 prefetch distance of the store operand, in k-blocks (0 = off)
  int split_kb;         // semantic-only: k-blocks >= split_kb accumulate into a second TMEM
                        // accumulator, summed in fp32 by the epilogue (0 = no split)
  int64_t cap;          // slab stride (rows) of the map tensor
  int L;                // map layers (slabs)
  const unsigned char* maps;   // map slabs (bulk-copy path, RB = 16)
  const unsigned char* qt;     // trajectory query operand [CG][ell_pad][128][Ep] (bulk-copy path)
  const unsigned char* qs;     // semantic query operand, UMMA-tiled [CG][n_sem_kb][128][128 B] (SW128 image)
  const void* emb_raw;         // experiment knob FMOE_TILED_B_EXP
  size_t emb_bytes;
  int tiled_b_exp;
  uint32_t id_offset;
  const float* rq_s;    // [128] query inverse norms (0 for padding rows)
  const float* rq_t;
  const float* r_e;     // [cap]
  const float* psq;     // [cap] prefix squared norms at layer ell-1 (traj)
  uint64_t* cand;       // [B][grid][k]
  int cand_q0;          // query offset of this pass in cand
  int grid;             // lists per query = CTAs / CG
  const int* gate;      // nullable device flag: 0 -> return at once
  int rep;              // query replication R (1, 2, 4): A rows r and r + 128/R hold the same
                        // query, so all four TMEM lane quadrants (= SM sub-partitions) carry
                        // live queries when nq <= 64; each replica scores 1/R of the columns
  unsigned long long* trace;
  float* out_cos;               // semantic kernels: cosines [B][cos_stride] (optional; this pass's first row)
  const float* sem_cos;         // trajectory kernels: cached semantic cosines to blend (optional)
  int64_t cos_stride;
  unsigned long long* gthr;     // [nq] shared admission threshold per query (zeroed by prep)
  const uint32_t* excl;         // nullable bitmap over rows: no candidates (insert sub-batches)
  int cos_ring;                 // cached-cosine ring depth (trajectory scans with cos_tma)
  int cos_bound;                // trajectory scans with sem_cos: read only the cosines whose blend bound
                                // reaches the admission threshold (direct loads, no TMA ring)
  int cos_tiled_exp;            // experiment knob FMOE_COS_TILED_EXP: cosine boxes as contiguous 4 KB blocks
  size_t cos_bytes;
  int cos_tma;                  // semantic scans: out_cos written through a swizzled smem stage + TMA
                                // tensor stores; trajectory scans: sem_cos read by per-warp TMA loads
                                // (a 3-buffer ring, 2 chunks ahead) instead of lane-per-query loads
  int no_epi;                   // debug knob (FMOE_NO_EPI=1): the epilogue only hands the accumulators
                                // back (measures the MMA + feed pipeline alone; results garbage)
  int no_a_reload;              // debug knob (FMOE_NO_A_RELOAD=1): query operand loaded only into the
                                // first ring pass, reused stale afterwards (results garbage; measures
                                // the L2 traffic of re-reading it per tile)
};
constexpr float kCosMax = 1.001f;               // bound on a cached cosine (|cos| <= 1 plus rounding)
constexpr int kCosStage = 32 * 128;             // per epilogue warp: 32 queries x 32 columns fp32 (SW128)
constexpr int kCosRingMax = 6;                  // cached-cosine loads: buffers per epilogue warp (ring - 1 chunks ahead)
// ring depth of the cached-cosine loads (FMOE_COS_RING, 2..6; measurement knob)
static int cos_ring() {
  static const int r = getenv("FMOE_COS_RING") ? atoi(getenv("FMOE_COS_RING")) : 3;
  return r < 2 ? 2 : (r > kCosRingMax ? kCosRingMax : r);
}
// bounded cached-cosine reads for blends / RDY scans with sem_cos (opt-in,
// FMOE_COS_BOUND=1).  Measured slower on the synthetic C5 workload (2M shard,
// B = 256, ell = 31: 1070 vs 955 us, profiles/r02i_cos_bound.md): the
// softmax gate maps give many rows trajectory cosines close to the admission
// threshold, so most chunks still need their cosines, now through per-lane
// loads instead of the TMA ring.  Kept for stores whose trajectories separate.
bool umma_cos_bound() {
  static const bool on = getenv("FMOE_COS_BOUND") && atoi(getenv("FMOE_COS_BOUND")) == 1;
  return on;
}
static int cos_stage_bytes(bool sem) { return kUmEpiWarps * kCosStage * (sem ? 1 : cos_ring()); }

// Sorted insert into a per-thread list in shared memory (entry i at
// l[i*stride]); called rarely (only for keys beating the k-th), kept out of
// line so the hot epilogue loop stays small enough for the instruction cache.
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
// Per-thread top-k list in shared memory kept as a binary MIN-heap of k keys
// (entry i at l + i*stride; empty entries are key 0): the root is the current
// k-th best key, a better key replaces it and sifts down (log2 k levels, no
// shifting -- the sorted-array insert cost O(k) smem moves and dominated the
// k = 64 RDY scan).  The merge kernel takes the lists unsorted.  Called only
// for keys beating the root, out of line.  Returns the new root.
__device__ __noinline__ uint64_t heap_sift(uint32_t l, uint32_t stride, int k, int i, uint64_t key) {
  while (true) {
    const int c1 = 2 * i + 1;
    if (c1 >= k) break;
    int c = c1;
    uint64_t vc = lds64(l + uint32_t(c1) * stride);
    if (c1 + 1 < k) {
      const uint64_t v2 = lds64(l + uint32_t(c1 + 1) * stride);
      if (v2 < vc) { vc = v2; c = c1 + 1; }
    }
    if (vc >= key) break;
    sts64(l + uint32_t(i) * stride, vc);
    i = c;
  }
  sts64(l + uint32_t(i) * stride, key);
  return lds64(l);
}
__device__ __forceinline__ uint64_t heap_replace_root(uint32_t l, uint32_t stride, int k, uint64_t key) {
  return heap_sift(l, stride, k, 0, key);
}
// Bottom-up heap construction over an unordered list of k keys; returns the root.
__device__ __noinline__ uint64_t heapify(uint32_t l, uint32_t stride, int k) {
  for (int i = k / 2 - 1; i >= 0; --i) heap_sift(l, stride, k, i, lds64(l + uint32_t(i) * stride));
  return lds64(l);
}
// Admit key into a thread's list holding cnt keys: append while filling
// (cnt < k; the k-th append builds the heap), else replace the root.  Returns
// the list's k-th key once full, else 0.
__device__ __noinline__ uint64_t list_admit(uint32_t l, uint32_t stride, int k, int cnt, uint64_t key) {
  if (cnt < k) {
    sts64(l + uint32_t(cnt) * stride, key);
    return cnt + 1 == k ? heapify(l, stride, k) : 0ull;
  }
  return heap_sift(l, stride, k, 0, key);
}
// Relaxed 64-bit read / max of the shared per-query admission threshold
__device__ __forceinline__ uint64_t ld_relaxed_u64(const unsigned long long* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_max_u64(unsigned long long* p, uint64_t v) {
  asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Epilogue cycle accounting for tools/trace.py (build with -DFMOE_EPI_PROFILE):
// per epilogue thread of CTA 0, clock64 cycles in [tile 0, tile 1, rest] x
// [tfull wait, named barrier, TMEM load, fast path, rare path, other].
#ifdef FMOE_EPI_PROFILE
#define EPI_T(slot) do { const long long c_ = clock64(); cyc[ti < 2 ? ti : 2][slot] += c_ - c_last; c_last = c_; } while (0)
#else
#define EPI_T(slot) do { } while (0)
#endif

template <bool SEM, bool TRAJ, int CG, int TN>
__global__ void __launch_bounds__(kUmThreads, 1)
    scan_umma_kernel(const __grid_constant__ CUtensorMap tm_qs, const __grid_constant__ CUtensorMap tm_es,
                     const __grid_constant__ CUtensorMap tm_qt, const __grid_constant__ CUtensorMap tm_mt,
                     const __grid_constant__ CUtensorMap tm_cos, const UmmaParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kUmMaxStages], empty[kUmMaxStages], tfull[2], tempty[2];
  __shared__ __align__(8) uint64_t cbar_all[kUmEpiWarps * kCosRingMax];   // cached-cosine ring (TRAJ + sem_cos)
  if (p.gate) {                                  // a conditional (fallback) scan
    pdl_wait();
    if (*p.gate == 0) {                          // (both CTAs of a pair read the same flag)
      pdl_trigger();
      return;
    }
  }
  __shared__ uint32_t tmem_base_sh;
  // row scales (re, rm) of each half tile, one buffer per TMEM accumulator stage
  __shared__ __align__(16) float escale[2][2][2][TN / 2];

  // 1024-byte alignment for the SW128 atoms (the same offsets in both CTAs of a pair)
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int NB = um_rows(CG, TN);            // store rows of a tile held by this CTA
  constexpr int SBY = um_stage_bytes(CG, TN);
  // [8 warps][kCosStage] cosine staging (cos_tma), then the lists [2R][k][LQ]
  unsigned char* cstage_all = smem + size_t(p.stages) * SBY;
  uint64_t* lists = reinterpret_cast<uint64_t*>(cstage_all + (p.cos_tma ? kUmEpiWarps * kCosStage * (SEM ? 1 : p.cos_ring) : 0));
  // CTA pair (cta_group::2): rank r owns query rows r*128.. of the M = 256
  // operand and store rows r*128.. of each 256-row tile; the leader (rank 0)
  // issues the MMAs for both, the accumulators of its queries land in each
  // CTA's own TMEM
  const int rank = CG == 2 ? int(cluster_rank()) : 0;
  const bool leader = rank == 0;
  const int cid = int(blockIdx.x) / CG, ncl = int(gridDim.x) / CG;
  const int nq_c = p.nq - rank * UM_M < 0 ? 0 : (p.nq - rank * UM_M > UM_M ? UM_M : p.nq - rank * UM_M);
  const int LQ = (nq_c + 31) / 32 * 32;          // list stride: queries rounded up to a warp

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // accumulators per tile: semantic + trajectory, or semantic K-halves when
  // split_kb > 0 (second slot), else one
  const int NACC = ((SEM && TRAJ) || p.split_kb > 0) ? 2 : 1;
  const int S = p.stages, AS = p.acc_stages;

  if (tid == 0) {
    // the leader's stage barrier also waits for the peer's relay arrival
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], (CG == 2 && leader) ? 2 : 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < AS; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], CG * kUmEpiWarps); }
    if (!SEM && p.cos_tma)
      for (int i = 0; i < kUmEpiWarps * p.cos_ring; ++i) mbar_init(&cbar_all[i], 1);
    mbar_fence_init();
  }
  if (warp == 0 && lane == 0) {
    if (SEM) tma_prefetch(&tm_es);
    if (TRAJ) { tma_prefetch(&tm_qt); tma_prefetch(&tm_mt); }
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  // empty top-k lists
  for (int i = tid; i < 2 * p.rep * p.k * LQ; i += kUmThreads) lists[i] = 0ull;
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all();      // peer barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  trace_mark(p.trace, 0);
  pdl_wait();

  const int n_kb = p.n_sem_kb + p.n_traj_kb;
  const int RB = 16 << p.tmode;                        // trajectory row bytes

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      // store operand of k-block kb of tile t -> L2
      auto prefetch = [&](int t, int kb) {
        const int y0 = t * TN + rank * NB;
        if (SEM && kb < p.n_sem_kb) {
          if constexpr (TN == 512) {                    // the two 128-row boxes this CTA loads
            tma_prefetch_l2(&tm_es, kb * 64, t * TN + rank * UM_M);
            tma_prefetch_l2(&tm_es, kb * 64, t * TN + 256 + rank * UM_M);
          } else {
            tma_prefetch_l2(&tm_es, kb * 64, y0);
          }
          return;
        }
        const int l0 = (kb - p.n_sem_kb) * p.lc;
        const int nl = p.ell_pad - l0 < p.lc ? p.ell_pad - l0 : p.lc;
        if (p.tmode == 0) {
          const int64_t left = p.cap - y0;
          const int rows = left >= NB ? NB : (left <= 0 ? 0 : int(left));
          if (rows > 0)
            for (int l = 0; l < nl && l0 + l < p.L; ++l)
              bulk_prefetch_l2(p.maps + (int64_t(l0 + l) * p.cap + y0) * 16, unsigned(rows * 16));
        } else {
          for (int l = 0; l < nl; ++l) tma_prefetch_l2(&tm_mt, 0, int((l0 + l) * p.cap + y0));
        }
      };
      int pt = cid, pkb = 0;                     // prefetch cursor, l2pf k-blocks ahead
      for (int i = 0; i < p.l2pf && pt < p.n_tiles; ++i)
        if (++pkb == n_kb) { pkb = 0; pt += ncl; }
      unsigned u = 0;
      for (int t = cid; t < p.n_tiles; t += ncl) {
        const int y0 = t * TN + rank * NB;             // this CTA's store rows of the tile
        for (int kb = 0; kb < n_kb; ++kb, ++u) {
          const int s = int(u % unsigned(S));
          if (p.l2pf > 0 && pt < p.n_tiles) {
            prefetch(pt, pkb);
            if (++pkb == n_kb) { pkb = 0; pt += ncl; }
          }
          mbar_wait(&empty[s], ((u / unsigned(S)) & 1u) ^ 1u);
          if (p.trace && blockIdx.x == 0 && u < 1024u) p.trace[16384 + u] = globaltimer();
          unsigned char* sa = smem + size_t(s) * SBY;
          unsigned char* sb = sa + kStageA;
          if (p.fake_loads) {                    // debug: MMAs on stale smem (feed excluded)
            mbar_arrive(&full[s]);
            continue;
          }
          if (SEM && kb < p.n_sem_kb) {
            const bool load_a = !p.no_a_reload || u < unsigned(S);
            mbar_arrive_expect_tx(&full[s], unsigned(load_a ? SBY : SBY - kStageA));
            if (load_a) bulk_g2s_plain(sa, p.qs + (size_t(rank) * p.n_sem_kb + kb) * kStageA, kStageA, &full[s]);
            if (p.tiled_b_exp) {
              // experiment: the same bytes as contiguous 16 KB blocks (results garbage);
              // 1: [row block][kb] order, 2: [kb][row block] order (a K-slab-major layout)
              const unsigned char* eb = static_cast<const unsigned char*>(p.emb_raw);
              const size_t nblk = size_t(p.cap / 128);
              for (int h = 0; h < NB / 128; ++h) {
                const size_t blk = TN == 512 ? size_t(t) * 4 + size_t(h) * 2 + rank : size_t(y0 / 128 + h);
                const size_t off = p.tiled_b_exp == 2 ? (size_t(kb) * nblk + blk) : (blk * p.n_sem_kb + kb);
                bulk_g2s(sb + h * 16384, eb + (off * 16384) % p.emb_bytes, 16384u, &full[s], pol);
              }
            } else if constexpr (TN == 512) {
              // two 128-row boxes: the halves this CTA feeds to the two N = 256 MMAs
              // (rows t*512 + g*256 + rank*128: TMEM column g*256 + j is row t*512 + g*256 + j)
              tma_load_2d(sb, &tm_es, kb * 64, t * TN + rank * UM_M, &full[s]);
              tma_load_2d(sb + UM_M * 128, &tm_es, kb * 64, t * TN + 256 + rank * UM_M, &full[s]);
            } else
            tma_load_2d(sb, &tm_es, kb * 64, y0, &full[s]);
          } else {
            const int j = kb - p.n_sem_kb;
            const int l0 = j * p.lc;
            const int nl = p.ell_pad - l0 < p.lc ? p.ell_pad - l0 : p.lc;
            if (p.tmode == 0) {
              // 16-byte rows: a layer's NB rows are one contiguous run of the
              // slab and already the no-swizzle K-major core-matrix layout, so
              // 1-D bulk copies replace 16-byte-wide tensor boxes (which cost
              // one TMA request per row)
              const int64_t left = p.cap - y0;
              const int rows = left >= NB ? NB : (left <= 0 ? 0 : int(left));
              const unsigned ba = unsigned(nl * UM_M * 16), bb = unsigned(rows * 16);
              mbar_arrive_expect_tx(&full[s], ba + unsigned(nl) * bb);
              bulk_g2s_plain(sa, p.qt + (size_t(rank) * p.ell_pad + l0) * UM_M * 16, ba, &full[s]);
              if (rows > 0)
                for (int l = 0; l < nl; ++l) {
                  // a padding layer past the last slab re-reads a real one: finite
                  // values against the zero query columns
                  const int ls = l0 + l < p.L ? l0 + l : p.L - 1;
                  bulk_g2s(sb + l * NB * 16, p.maps + (int64_t(ls) * p.cap + y0) * 16, bb, &full[s], pol);
                }
            } else {
              mbar_arrive_expect_tx(&full[s], unsigned(nl * (UM_M + NB) * RB));
              for (int l = 0; l < nl; ++l) {
                tma_load_2d(sa + l * UM_M * RB, &tm_qt, 0, (rank * p.ell_pad + l0 + l) * UM_M, &full[s]);
                tma_load_2d(sb + l * NB * RB, &tm_mt, 0, int((l0 + l) * p.cap + y0), &full[s]);
              }
            }
          }
        }
        tile_mark(p.trace, 0, unsigned((t - cid) / ncl));
      }
      trace_mark_here(p.trace, 5);
    }
  } else if (warp == 1 && CG == 2 && !leader) {
    // ---------------------------------------------------------------- peer relay
    // the leader's MMAs read this CTA's stage too: forward each completed
    // stage to the leader's barrier
    if (lane == 0) {
      const uint32_t rfull = mapa_rank(&full[0], 0);
      unsigned u = 0;
      for (int t = cid; t < p.n_tiles; t += ncl)
        for (int kb = 0; kb < n_kb; ++kb, ++u) {
          const int s = int(u % unsigned(S));
          mbar_wait(&full[s], (u / unsigned(S)) & 1u);
          mbar_arrive_remote(rfull + uint32_t(s) * 8u);
        }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc(UM_M * CG, TN > 256 ? 256 : TN);
      unsigned u = 0, ti = 0;
      for (int t = cid; t < p.n_tiles; t += ncl, ++ti) {
        const int as = int(ti % unsigned(AS));
        mbar_wait(&tempty[as], ((ti / unsigned(AS)) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d_sem = tmem_base + uint32_t(as * NACC * TN);
        const uint32_t d_trj = d_sem + (NACC == 2 ? TN : 0);
        for (int kb = 0; kb < n_kb; ++kb, ++u) {
          const int s = int(u % unsigned(S));
          mbar_wait(&full[s], (u / unsigned(S)) & 1u);
          if (p.trace && blockIdx.x == 0 && u < 1024u) p.trace[17408 + u] = globaltimer();
          tc_fence_after();
          const unsigned char* sa = smem + size_t(s) * SBY;
          const unsigned char* sb = sa + kStageA;
          if (SEM && kb < p.n_sem_kb) {
            const bool hi = !TRAJ && p.split_kb > 0 && kb >= p.split_kb;
            const uint32_t d = hi ? d_trj : d_sem;
            const int kb0 = hi ? p.split_kb : 0;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              tc_mma<CG>(d, umma_desc(sa + kk * 32, 16, 1024, 2), umma_desc(sb + kk * 32, 16, 1024, 2), idesc,
                         (kb != kb0 || kk) ? 1u : 0u);
              if constexpr (TN == 512)      // second N = 256 column group, same A
                tc_mma<CG>(d + 256, umma_desc(sa + kk * 32, 16, 1024, 2),
                           umma_desc(sb + UM_M * 128 + kk * 32, 16, 1024, 2), idesc, (kb != kb0 || kk) ? 1u : 0u);
            }
          } else {
            const int j = kb - p.n_sem_kb;
            const int l0 = j * p.lc;
            const int nl = p.ell_pad - l0 < p.lc ? p.ell_pad - l0 : p.lc;
            const bool first = (j == 0);
            if (p.tmode == 0) {
              // two 16-byte layers per K=16 MMA: LBO = the layer stride
              for (int l = 0; l < nl; l += 2)
                tc_mma<CG>(d_trj, umma_desc(sa + l * UM_M * 16, UM_M * 16, 128, 0),
                           umma_desc(sb + l * NB * 16, NB * 16, 128, 0), idesc, (first && l == 0) ? 0u : 1u);
            } else {
              const uint32_t layout = p.tmode == 1 ? 6u : (p.tmode == 2 ? 4u : 2u);
              const int ksteps = RB / 32;
              for (int l = 0; l < nl; ++l)
                for (int kk = 0; kk < ksteps; ++kk)
                  tc_mma<CG>(d_trj, umma_desc(sa + l * UM_M * RB + kk * 32, 16, 8 * RB, layout),
                             umma_desc(sb + l * NB * RB + kk * 32, 16, 8 * RB, layout), idesc,
                             (first && l == 0 && kk == 0) ? 0u : 1u);
            }
          }
          // stage s may be refilled (in both CTAs of a pair) once these MMAs retire
          if constexpr (CG == 2) tc_commit_pair(&empty[s]); else tc_commit(&empty[s]);
        }
        // accumulators of tile t complete
        if constexpr (CG == 2) tc_commit_pair(&tfull[as]); else tc_commit(&tfull[as]);
        tile_mark(p.trace, 1, ti);
      }
      trace_mark_here(p.trace, 7);
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    // warp 4+e: TMEM lane quadrant e%4 (a warp may only read its own
    // quadrant), column half e/4.  With replication R the quadrants hold R
    // copies of 4/R query quadrants; copy `sub` scores the sub-th 1/R of the
    // half's columns.  Thread = (query, column group): its own top-k list.
    const int e = warp - 4, qd = e & 3, half = e >> 2;
    const int R = p.rep, QA = 4 / R;              // query quadrants per replica
    const int sub = qd / QA;                      // replica index
    const int NC = (TN / 2) / 32 / R;             // 32-column chunks per tile and warp
    const int q = (qd % QA) * 32 + lane;          // query of this thread (this CTA's TMEM lane)
    const int qg = rank * UM_M + q;               // ... and its row in the pass
    const bool live = q < nq_c;
    const int gi = half * R + sub;                // list (column group) index
    const float rqs = (SEM && live) ? p.rq_s[qg] : 0.f;
    const float rqt = (TRAJ && live) ? p.rq_t[qg] : 0.f;
    const float w = p.w, w1 = 1.f - p.w;
    const int k = p.k;
    const bool split = p.split_kb > 0;
    const bool vec4 = (p.cos_stride & 3) == 0;      // 16-byte aligned cosine rows
    constexpr int HC = TN / 2;                    // columns per half
    uint64_t* ml = lists + size_t(gi) * k * LQ + q;     // this thread's list: entry i at ml[i*LQ]
    const uint32_t ml_s = smem_u32(ml);
    // Admission: a key enters this thread's list if it beats the list's k-th
    // key (thr) and the query's shared threshold g: the largest k-th key any
    // list of this query (any CTA, any column group) has reached -- k better
    // keys already exist, so nothing below it can be in the final top-k.
    // The list fills unordered (cnt < k, no sifting) and becomes a min-heap
    // when full.
    uint64_t g = 0ull, published = 0ull;
    int cnt = 0;
    // filter score (fast path: score >= thr_s); +inf keeps idle lanes out
    float thr_s = live ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000);
    unsigned long long* gq = p.gthr + (live ? qg : 0);
    if (live) {                                    // a seeded scan starts at the seed bound
      g = ld_relaxed_u64(gq);
      if (g) thr_s = key_score(g);
    }
#ifdef FMOE_EPI_PROFILE
    const uint64_t g_init = g;
#endif
    // single-part scans: fold the (exactly 1) weight and the query norm
    const float cs = SEM && !TRAJ ? rqs : w * rqs, ct = TRAJ && !SEM ? rqt : w1 * rqt;
    unsigned ti = 0;
#ifdef FMOE_EPI_PROFILE
    long long cyc[3][6] = {}, c_last = clock64();
    unsigned n_cand_rest = 0;
#endif
    // per-row scales of the next half tile, loaded one tile ahead by the
    // warp that publishes them
    float re_n[HC / 32], rm_n[HC / 32];
    auto fetch = [&](int t) {
#pragma unroll
      for (int c = 0; c < HC / 32; ++c) {
        const int64_t yl = int64_t(t) * TN + half * HC + c * 32 + lane;
        const bool yok = qd == 0 && t < p.n_tiles && yl < p.n_rows;
        re_n[c] = (SEM && yok) ? __ldg(p.r_e + yl) : 0.f;
        rm_n[c] = (TRAJ && yok) ? __ldg(p.psq + yl) : 0.f;
      }
    };
    fetch(cid);
    // cached cosines (TRAJ + sem_cos, cos_tma): chunk i of this warp's sequence
    // (tile cid + (i / NC) * ncl, chunk i % NC) lands in ring buffer i % 3
    const bool cin = !SEM && p.sem_cos && p.cos_tma;
    const int CR = p.cos_ring;
    uint64_t* cbar = cbar_all + e * CR;
    unsigned char* cring = cstage_all + size_t(e) * CR * kCosStage;
    const int crow = rank * UM_M + (qd % QA) * 32;      // first query row of this warp's box
    auto cos_issue = [&](unsigned i) {                  // lane 0
      const int t2 = cid + int(i / unsigned(NC)) * ncl;
      if (t2 >= p.n_tiles) return;
      const int col = t2 * TN + half * HC + sub * NC * 32 + int(i % unsigned(NC)) * 32;
      uint64_t* b = &cbar[i % unsigned(CR)];
      mbar_arrive_expect_tx(b, unsigned(kCosStage));
      if (p.cos_tiled_exp) {   // experiment: the same bytes as contiguous 4 KB blocks (results garbage)
        const size_t blk = (size_t(col) / 32) * size_t((p.nq + 31) / 32) + size_t(crow) / 32;
        bulk_g2s_plain(cring + (i % unsigned(CR)) * kCosStage,
                       reinterpret_cast<const unsigned char*>(p.sem_cos) + (blk * kCosStage) % p.cos_bytes,
                       unsigned(kCosStage), b);
      } else
      tma_load_2d(cring + (i % unsigned(CR)) * kCosStage, &tm_cos, col, crow, b);
    };
    if (cin && lane == 0)
      for (int i = 0; i < CR - 1; ++i) cos_issue(unsigned(i));
    unsigned ci = 0;                                    // this warp's chunk sequence number
    uint64_t st0 = 0ull, st1 = 0ull, st2 = 0ull, st3 = 0ull;   // candidate stash (see the rare path)
    int ns = 0;
    auto admit = [&](uint64_t key) {
      if (key > g) {
        const uint64_t root = list_admit(ml_s, uint32_t(LQ) * 8, k, cnt, key);
        cnt += cnt < k ? 1 : 0;
        if (root > g) {                                 // a full list: its k-th key bounds the query
          g = root;
          thr_s = key_score(g);
        }
      }
    };
    auto flush = [&]() {
      if (ns > 0) admit(st0);
      if (ns > 1) admit(st1);
      if (ns > 2) admit(st2);
      if (ns > 3) admit(st3);
      ns = 0;
    };
    if (p.no_epi) {
      for (int t = cid; t < p.n_tiles; t += ncl, ++ti) {
        const int as = int(ti % unsigned(AS));
        mbar_wait(&tfull[as], (ti / unsigned(AS)) & 1u);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2 && !leader) mbar_arrive_remote(mapa_rank(&tempty[as], 0));
          else mbar_arrive(&tempty[as]);
        }
      }
    }
    for (int t = p.no_epi ? p.n_tiles : cid; t < p.n_tiles; t += ncl, ++ti) {
      const int as = int(ti % unsigned(AS));
      const int ybase = t * TN + half * HC + sub * NC * 32;     // first column of this warp
      // this warp's copy of the half tile's row scales, read back as broadcast
      // LDS.128 (4 columns per load) instead of one shuffle per column
      float re_c[HC / 32], rm_c[HC / 32];
#pragma unroll
      for (int c = 0; c < HC / 32; ++c) {
        re_c[c] = re_n[c];
        rm_c[c] = rm_n[c] > 0.f ? rsqrtf(rm_n[c]) : 0.f;
      }
      fetch(t + ncl);
      if (ti == 0 && tid == 128) trace_mark_here(p.trace, 2);
      EPI_T(5);
      if (p.epi_sleep > 0) mbar_wait_backoff(&tfull[as], (ti / unsigned(AS)) & 1u, unsigned(p.epi_sleep));
      else mbar_wait(&tfull[as], (ti / unsigned(AS)) & 1u);
      EPI_T(0);
      // one warp per half publishes the scales, after this tile's accumulators
      // are full (so every warp has released the previous tile of this stage);
      // a named barrier per half orders the reads
      if (qd == 0) {
#pragma unroll
        for (int c = 0; c < HC / 32; ++c) {
          escale[as][half][0][c * 32 + lane] = re_c[c];
          escale[as][half][1][c * 32 + lane] = rm_c[c];
        }
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + half) : "memory");
      EPI_T(1);
      if (ti == 0 && tid == 128) trace_mark_here(p.trace, 4);
      if (tid == 128) tile_mark(p.trace, 2, ti);
      tc_fence_after();
      // the shared threshold, read now and applied after this tile's chunks
      const uint64_t g_new = live ? ld_relaxed_u64(gq) : 0ull;
      const uint32_t lane_addr = uint32_t(qd * 32) << 16;
      const uint32_t c_sem = tmem_base + lane_addr + uint32_t(as * NACC * TN + half * HC + sub * NC * 32);
      const uint32_t c_trj = c_sem + (NACC == 2 ? TN : 0);
#pragma unroll 1
      for (int c = 0; c < NC; ++c) {
        uint32_t vs[32], vt[32];
        if (SEM) tc_ld32(c_sem + c * 32, vs);
        if (TRAJ || p.split_kb > 0) tc_ld32(c_trj + c * 32, vt);
        const int64_t yc = int64_t(ybase) + c * 32;
        const int64_t left = p.n_rows - yc;
        const unsigned vmask = !live ? 0u : (left >= 32 ? 0xffffffffu : (left <= 0 ? 0u : ((1u << left) - 1u)));
        float cached[32];
        if (cin) {
          // buffer (ci + CR - 1) % CR held chunk ci - 1, which every lane has read
          __syncwarp();
          if (lane == 0) {
            fence_proxy_async_smem();
            cos_issue(ci + unsigned(CR) - 1);
          }
          mbar_wait(&cbar[ci % unsigned(CR)], (ci / unsigned(CR)) & 1u);
          const uint32_t row = smem_u32(cring + (ci % unsigned(CR)) * kCosStage) + uint32_t(lane) * 128u;
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            float4 f;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(f.x), "=f"(f.y), "=f"(f.z), "=f"(f.w)
                         : "r"(row + (uint32_t(j4 ^ (lane & 7)) << 4)));
            cached[4 * j4] = f.x; cached[4 * j4 + 1] = f.y; cached[4 * j4 + 2] = f.z; cached[4 * j4 + 3] = f.w;
          }
          ++ci;
        } else if (!SEM && p.sem_cos && !p.cos_bound) {
          const float* cp = p.sem_cos + int64_t(qg) * p.cos_stride + yc;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            if (vec4 && j + 4 <= nvalid_rows(yc, p.n_rows, live)) {
              const float4 f = __ldcs(reinterpret_cast<const float4*>(cp + j));
              cached[j] = f.x; cached[j + 1] = f.y; cached[j + 2] = f.z; cached[j + 3] = f.w;
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u) cached[j + u] = (j + u < nvalid_rows(yc, p.n_rows, live)) ? cp[j + u] : 0.f;
            }
          }
        }
        const float4* res = reinterpret_cast<const float4*>(&escale[as][half][0][(sub * NC + c) * 32]);
        const float4* rms = reinterpret_cast<const float4*>(&escale[as][half][1][(sub * NC + c) * 32]);
        tc_wait_ld();
        // Bounded cached-cosine reads (cos_bound): cos <= 1, so a row's blend
        // is at most fmaf(w1, traj, w * kCosMax) (fmaf is monotone in its
        // addend; kCosMax covers the semantic scan's rounding).  Only the
        // columns whose bound reaches the thread's admission threshold can
        // enter the top-k, and only their cosines are read: after the first
        // tiles almost none, so the scan streams the map prefix instead of
        // B x 4 bytes of cosines per row.  Scores of the read columns are
        // computed exactly as on the unbounded path.
        unsigned need = 0u;
        if (!SEM && p.sem_cos && p.cos_bound) {
          const int nv = nvalid_rows(yc, p.n_rows, live);
          const float wc = w * kCosMax;
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 rm4 = rms[j4];
            const float rma[4] = {rm4.x, rm4.y, rm4.z, rm4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = 4 * j4 + u;
              const float b = fmaf(w1, __uint_as_float(vt[j]) * rqt * rma[u], wc);
              need |= (b >= thr_s ? 1u : 0u) << j;
            }
          }
          need &= nv >= 32 ? 0xffffffffu : ((1u << nv) - 1u);
          // no column of this chunk can reach any lane's list: nothing to read or score
          if (!__any_sync(0xffffffffu, need != 0u)) continue;
          const float* cp = p.sem_cos + int64_t(qg) * p.cos_stride + yc;
          if (need == 0xffffffffu && vec4) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 f = __ldcs(reinterpret_cast<const float4*>(cp + j));
              cached[j] = f.x; cached[j + 1] = f.y; cached[j + 2] = f.z; cached[j + 3] = f.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) cached[j] = ((need >> j) & 1u) ? __ldcs(cp + j) : 0.f;
          }
        }
        EPI_T(2);
        // fast path: 32 scores and their maximum, one compare against the k-th score
        float sc[32];
        float vmax = -__int_as_float(0x7f800000);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 re4 = SEM ? res[j4] : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 rm4 = TRAJ ? rms[j4] : make_float4(0.f, 0.f, 0.f, 0.f);
          const float rea[4] = {re4.x, re4.y, re4.z, re4.w};
          const float rma[4] = {rm4.x, rm4.y, rm4.z, rm4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 4 * j4 + u;
            float v = (!SEM && p.sem_cos) ? w * cached[j] : 0.f;
            if (SEM) {
              const float dot = (!TRAJ && split) ? __uint_as_float(vs[j]) + __uint_as_float(vt[j]) : __uint_as_float(vs[j]);
              v = TRAJ ? w * (dot * rqs * rea[u]) : dot * cs * rea[u];
            }
            if (TRAJ) v = SEM || p.sem_cos ? fmaf(w1, __uint_as_float(vt[j]) * rqt * rma[u], v)
                                           : __uint_as_float(vt[j]) * ct * rma[u];
            if (!SEM && p.sem_cos && p.cos_bound && !((need >> j) & 1u)) v = -__int_as_float(0x7f800000);
            sc[j] = v;
            vmax = fmaxf(vmax, v);
          }
        }
        unsigned m = 0;
        if (vmax >= thr_s) {
#pragma unroll
          for (int j = 0; j < 32; ++j) m |= (sc[j] >= thr_s ? 1u : 0u) << j;
        }
        m &= vmask;
        if (m && p.excl) m &= ~__ldg(p.excl + (yc >> 5));   // rows claimed by an earlier insert sub-batch
        EPI_T(3);
        if (SEM && !TRAJ && p.out_cos && p.cos_tma) {
          // warp-cooperative: the 32 x 32 block (queries of this warp x this
          // chunk's columns) is staged in shared memory with the 128-byte
          // swizzle (16-byte group j of row r at j ^ (r & 7): conflict-free
          // v4 stores) and written by one TMA tensor store, which also clips
          // rows >= nq and columns >= n_rows.  (Lane-per-query global stores
          // touched 32 rows per instruction.)
          if (__any_sync(0xffffffffu, live)) {
            unsigned char* cst = cstage_all + size_t(e) * kCosStage;
            if (lane == 0) bulk_wait_read0();            // the previous chunk's store has read the stage
            __syncwarp();
            const uint32_t row = smem_u32(cst) + uint32_t(lane) * 128u;
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4)
              sts128(row + (uint32_t(j4 ^ (lane & 7)) << 4), sc[4 * j4], sc[4 * j4 + 1], sc[4 * j4 + 2],
                     sc[4 * j4 + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (p.cos_tiled_exp) {   // experiment: contiguous 4 KB blocks (results garbage)
                const size_t blk = size_t(yc / 32) * size_t((p.nq + 31) / 32) + size_t(rank * UM_M + (qd % QA) * 32) / 32;
                bulk_s2g(reinterpret_cast<unsigned char*>(p.out_cos) + (blk * kCosStage) % p.cos_bytes, cst,
                         unsigned(kCosStage));
              } else
              tma_store_2d(&tm_cos, cst, int(yc), rank * UM_M + (qd % QA) * 32);
              bulk_commit();
            }
          }
        } else if (SEM && !TRAJ && p.out_cos && live) {
          float* op = p.out_cos + int64_t(qg) * p.cos_stride + yc;
          const int nv = nvalid_rows(yc, p.n_rows, live);
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            if (vec4 && j + 4 <= nv) __stcs(reinterpret_cast<float4*>(op + j), make_float4(sc[j], sc[j + 1], sc[j + 2], sc[j + 3]));
            else
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (j + u < nv) op[j + u] = sc[j + u];
          }
        }
        // rare path: exact key order (score desc, id asc) for the candidates
#ifdef FMOE_EPI_PROFILE
        if (ti >= 2) n_cand_rest += __popc(m);
#endif
#ifdef FMOE_NO_RARE
        m = 0;
#endif
        // (the scores go through a local copy: one indexed load per candidate
        // instead of a 31-deep select chain).  Candidates go to a 4-key
        // register stash admitted once per tile (or when it is full): a warp
        // then pays one divergent heap insert per stashed key of its busiest
        // lane, instead of one per chunk in which any lane had a candidate.
        if (m) {
          const uint32_t idb = p.id_offset + uint32_t(yc);
          float scl[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) scl[j] = sc[j];
          do {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const uint64_t key = pack_key(scl[j], idb + uint32_t(j));
            if (key > g) {
              if (ns == 4) flush();
              if (ns == 0) st0 = key;
              else if (ns == 1) st1 = key;
              else if (ns == 2) st2 = key;
              else st3 = key;
              ++ns;
            }
          } while (m);
        }
        EPI_T(4);
      }
      // hand the accumulator stage back first: the arrive is a release, and
      // placed after the threshold's global red it would wait for that red's
      // round trip (the MMA warp, not this warp, is what waits on it).  The
      // stashed candidates are admitted after it: the heap inserts touch only
      // this thread's list, and with a single-buffered accumulator (TN = 512)
      // the next tile's MMAs wait for the arrive.
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {                            // the leader's MMA waits for both CTAs' epilogues
        if (CG == 2 && !leader) mbar_arrive_remote(mapa_rank(&tempty[as], 0));
        else mbar_arrive(&tempty[as]);
      }
      flush();
      // publish this list's bound once per tile (atomics per insert contended
      // at k = 64), then take the shared one read at the start of this tile
      if (g > published) {
        red_max_u64(gq, g);
        published = g;
      }
      if (g_new > g) {
        g = g_new;
        thr_s = key_score(g);
      }
      if (ti == 0 && tid == 128) trace_mark_here(p.trace, 1);
      if (tid == 128) tile_mark(p.trace, 3, ti);
    }
    trace_mark(p.trace, 3);
#ifdef FMOE_EPI_PROFILE
    if (p.trace && blockIdx.x == 0)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 6; ++b)
          p.trace[12288 + (tid - 128) * 18 + a * 6 + b] =
              a == 2 && b == 5 ? n_cand_rest : a == 0 && b == 5 ? g_init : a == 1 && b == 5 ? g : cyc[a][b];
#endif
    if (SEM && !TRAJ && p.out_cos && p.cos_tma && lane == 0) bulk_wait_all0();   // cosines written
    // fold the 2R column-group lists of each query into group 0's heap, then
    // one list per (query, CTA) goes out
    if (live && cnt < k) heapify(ml_s, uint32_t(LQ) * 8, k);   // empty slots are key 0
    asm volatile("bar.sync 3, %0;" ::"r"(kUmEpiWarps * 32) : "memory");
    const int te = tid - 128;
    if (te < nq_c) {
      const uint32_t l0 = smem_u32(lists + te);
      uint64_t root = lists[te];
      for (int g = 1; g < 2 * R; ++g)
        for (int i = 0; i < k; ++i) {
          const uint64_t key = lists[(size_t(g) * k + i) * LQ + te];
          if (key > root) root = heap_replace_root(l0, uint32_t(LQ) * 8, k, key);
        }
      uint64_t* dst = p.cand + (int64_t(p.cand_q0 + rank * UM_M + te) * p.grid + cid) * k;
      for (int i = 0; i < k; ++i) dst[i] = lists[size_t(i) * LQ + te];
    }
  }
  pdl_trigger();
  tc_fence_before();
  __syncwarp();
  if constexpr (CG == 2) cluster_sync_all();      // no CTA leaves while its peer may still signal it
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
  trace_mark(p.trace, 6);
}

// ------------------------------------------------------------------ query preparation
// Quantises the batch to bf16 in the UMMA operand layouts (zero padding to
// 128 rows, to Dp columns and to ell_pad layers) and computes the inverse norms
// of the quantised rows (float64 sums) and the validity flags.
// Seeded trajectory scans (a session step seeded with the previous step's
// top-k ids): k distinct stored rows whose scores are known bound the k-th
// best key from below, so the scan may start its admission threshold there.
struct SeedArgs {
  const int64_t* ids = nullptr;   // [nq][stride] global ids (this pass); null = no seeds
  int stride = 0, n = 0, k = 0;   // n seeds per query (k <= n <= 64), bound = k-th best of them
  uint32_t id_offset = 0;
  int64_t n_rows = 0, cap = 0;
  const __nv_bfloat16* maps = nullptr;
  const float* psq = nullptr;     // prefix squared norms at layer ell-1
};
// Margin between a seed score computed here (fp32 FMA over ell*E) and the
// scan's score of the same row (tcgen05 fp32 accumulation, same bf16 operands):
// both are within ~1e-6 of the exact cosine; 1e-4 keeps the bound safe.
constexpr float kSeedMargin = 1e-4f;

__global__ void __launch_bounds__(256) umma_prep_kernel(const float* __restrict__ q_emb, const float* __restrict__ q_prefix,
                                                        int64_t q_stride, int nq, int D, int Dp, int E, int Ep, int ell,
                                                        int ell_pad, __nv_bfloat16* qs, __nv_bfloat16* qt, float* rq_s,
                                                        float* rq_t, float* valid, int sem, int traj, int qper,
                                                        unsigned long long* gthr, const SeedArgs sd,
                                                        const int* gate, int keep_gthr) {
  pdl_wait();
  if (gate && *gate == 0) return;
  __shared__ double red[2][8];
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x = q % qper;                        // source query of A row q (replication)
  const bool live = x < nq;
  double a = 0.0, b = 0.0;
  if (sem) {
    // UMMA-tiled: [q / 128][k-block][128 rows][128 B], 16-byte groups swizzled
    // within each 8-row atom (group c of row r at c ^ (r & 7), the SWIZZLE_128B
    // K-major image), so a k-block of 128 query rows is one contiguous 16 KB
    // block that one 1-D bulk copy moves (a 2-D tensor box costs one TMA
    // request per 128-byte row)
    const int nkb = (Dp + 63) / 64, half = q / UM_M, r = q % UM_M;
    for (int e = tid; e < nkb * 64; e += 256) {
      const float v = (live && e < D) ? __bfloat162float(__float2bfloat16_rn(q_emb[int64_t(x) * D + e])) : 0.f;
      const int kb = e >> 6, c = (e & 63) >> 3;
      qs[((int64_t(half) * nkb + kb) * UM_M + r) * 64 + ((c ^ (r & 7)) << 3) + (e & 7)] = __float2bfloat16_rn(v);
      a += double(v) * double(v);
    }
  }
  if (traj) {
    for (int i = tid; i < ell_pad * Ep; i += 256) {
      const int l = i / Ep, j = i - l * Ep;
      const float v = (live && l < ell && j < E)
                          ? __bfloat162float(__float2bfloat16_rn(q_prefix[int64_t(x) * q_stride + l * E + j]))
                          : 0.f;
      // [CG][ell_pad][128][Ep]: each CTA of a pair reads its own contiguous block
      qt[((int64_t(q / UM_M) * ell_pad + l) * UM_M + q % UM_M) * Ep + j] = __float2bfloat16_rn(v);
      b += double(v) * double(v);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (lane == 0) { red[0][warp] = a; red[1][warp] = b; }
  __syncthreads();
  if (tid == 0) {
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < 8; ++w) { sa += red[0][w]; sb += red[1][w]; }
    rq_s[q] = sa > 0.0 ? float(1.0 / sqrt(sa)) : 0.f;
    rq_t[q] = sb > 0.0 ? float(1.0 / sqrt(sb)) : 0.f;
    if (live && q == x) valid[q] = ((!sem || sa > 0.0) && (!traj || sb > 0.0)) ? 1.f : 0.f;
    if (live && q == x && !keep_gthr) gthr[q] = 0ull;   // keep: seeded by a sample pass
    red[0][0] = sb > 0.0 ? 1.0 / sqrt(sb) : 0.0;
  }
  // (no seed bound -- an unseeded scan -- when the prefix does not fit the staging below)
  if (!(sd.ids && traj && !sem && live && q == x && sd.k > 0 && sd.n >= sd.k && sd.n <= 64 && ell * Ep <= kMaxE * 64))
    return;
  // ---- seed bound: the k-th best trajectory score of the valid seed rows
  // (ids -1, e.g. from a short candidate union, are skipped), less a margin.
  // The query prefix (store-dtype values, pad columns 0) is staged in shared
  // memory; a seed's dot is spread over the warp as 16-byte chunks of its
  // layer rows (Ep*2 bytes each, 16-byte multiples), all loads independent.
  __shared__ unsigned s_sc[64];
  __shared__ __align__(16) float s_q[kMaxE * 64];      // [ell][Ep], ell * Ep <= 64 * 64
  for (int i = tid; i < ell * Ep; i += 256) {
    const int l = i / Ep, j = i - l * Ep;
    s_q[i] = j < E ? __bfloat162float(__float2bfloat16_rn(q_prefix[int64_t(x) * q_stride + l * E + j])) : 0.f;
  }
  __syncthreads();
  const float rq = float(red[0][0]);
  const int cpr = Ep / 8;                                // 16-byte chunks per layer row
  const int nch = ell * cpr;
  for (int i = warp; i < sd.n; i += 8) {
    const int64_t gid = sd.ids[int64_t(x) * sd.stride + i];
    const int64_t y = gid - int64_t(sd.id_offset);
    const bool ok = gid >= 0 && y >= 0 && y < sd.n_rows;
    float dot = 0.f;
    if (ok)
      for (int c = lane; c < nch; c += 32) {
        const int l = c / cpr, j0 = (c - l * cpr) * 8;
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(sd.maps + (int64_t(l) * sd.cap + y) * Ep + j0));
        float m8[8];
        unpack8(u, m8, Bf16Tag());
        const float* qv = s_q + l * Ep + j0;
#pragma unroll
        for (int e = 0; e < 8; ++e) dot = fmaf(qv[e], m8[e], dot);
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) {
      const float ps = ok ? sd.psq[y] : 0.f;
      const float sc = ps > 0.f ? dot * rq * rsqrtf(ps) : 0.f;
      s_sc[i] = (ok && sc == sc) ? orderable(sc) : 0u;    // 0: no seed (below every score)
    }
  }
  __syncthreads();
  if (tid < sd.n && s_sc[tid] != 0u) {
    // rank of seed tid among the valid seeds (ties by index): rank k-1 is the k-th best
    const unsigned v = s_sc[tid];
    int rank = 0;
    for (int i = 0; i < sd.n; ++i) rank += (s_sc[i] > v || (s_sc[i] == v && i < tid)) ? 1 : 0;
    if (rank == sd.k - 1) {
      const float lo = from_orderable(v) - kSeedMargin;
      gthr[q] = uint64_t(orderable(lo)) << 32;    // below every key of score >= lo
    }
  }
}

// Admission bound from a sample pass (approx semantic scans): the ke-th best
// approximate key of rows [0, S) -- those rows get bit-identical keys in the
// full scan, so the full scan's ke-th best key is >= this one.
__global__ void seed_from_sample_kernel(int B, int ke, const uint64_t* __restrict__ keys,
                                        unsigned long long* gthr) {
  pdl_wait();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < B) gthr[x] = keys[int64_t(x) * ke + ke - 1];
}
cudaError_t launch_seed_from_sample(int B, int ke, const uint64_t* keys, unsigned long long* gthr, cudaStream_t s) {
  count_launch();
  return launch_pdl(seed_from_sample_kernel, dim3((B + 127) / 128), dim3(128), 0, s, B, ke, keys, gthr);
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D bf16 tensor map: inner dim `cols` (contiguous), outer `rows`, box {bc, br}
static bool make_map(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t bc, uint32_t br,
                     CUtensorMapSwizzle sw) {
  EncodeFn enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {bc, br};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int tmode_of(int rb) { return rb == 16 ? 0 : rb == 32 ? 1 : rb == 64 ? 2 : rb == 128 ? 3 : -1; }

// CTA pairs (cta_group::2, M = 256) for passes of more than 128 queries
static int cg_of(const UmmaPlanIn& in) { return in.cg > 0 ? in.cg : (in.nq > UM_M ? 2 : 1); }
// smem: 1 KB alignment + S stages (48 KB; 32 KB per CTA of a pair) + 2R lists
// of k keys per query of the CTA, within 216 KB (+ ~10 KB static <= 227 KB)
static size_t lists_bytes(const UmmaPlanIn& in, int R) {
  const int nq = in.nq < UM_M ? in.nq : UM_M;
  return size_t(2 * R) * in.k * ((nq + 31) / 32 * 32) * 8 + (in.cos_out ? size_t(cos_stage_bytes(true)) : 0) +
         (in.cos_in ? size_t(cos_stage_bytes(false)) : 0);
}
// (planning uses TN = 256, the larger stage: a launch at TN = 128 fits as many)
// Semantic-only approximate scans on CTA pairs use 512-row tiles: two N = 256
// MMAs per K step share the query operand A, so a stage carries 16 KB of A for
// 32 KB of store rows (per CTA) instead of 16 + 16 -- the scan is paced by the
// bytes the L2 delivers per SM, and A is re-read for every tile.  The 512 TMEM
// columns then hold one tile (single-buffered accumulator).
static int umma_tn(const UmmaPlanIn& in, int cg) {
  static const int tn_env = getenv("FMOE_UMMA_TN") ? atoi(getenv("FMOE_UMMA_TN")) : 0;
  if (tn_env == 128) return 128;
  if (tn_env != 256 && cg == 2 && in.approx && in.w_sem == 1.f) return 512;
  return UM_N;
}
static int stages_for(const UmmaPlanIn& in, int R, int tn = UM_N) {
  const size_t l = lists_bytes(in, R);
  // dynamic smem budget (FMOE_UMMA_SMEM_KB, measurement knob; the static
  // shared memory is <= 9 KB, the per-block limit 227 KB)
  static const int kb_env = getenv("FMOE_UMMA_SMEM_KB") ? atoi(getenv("FMOE_UMMA_SMEM_KB")) : 216;
  const size_t budget = size_t(kb_env < 64 ? 64 : (kb_env > 218 ? 218 : kb_env)) * 1024;
  if (l + 1024 > budget) return 0;
  const int cg = cg_of(in);
  const int S = int((budget - 1024 - l) / size_t(um_stage_bytes(cg, tn)));
  static const int env = getenv("FMOE_UMMA_STAGES") ? atoi(getenv("FMOE_UMMA_STAGES")) : 0;
  const int cap = env > 0 ? env : (tn == 512 ? 4 : tn == UM_N ? (cg == 2 ? 6 : 4) : kUmMaxStages);
  return S > cap ? cap : S;
}
// Query replication: nq <= 32 uses one TMEM lane quadrant, nq <= 64 two; the
// other quadrants' epilogue warps (the other SM sub-partitions) would idle, so
// the query rows are repeated R = 4 / quadrants times and the replicas split
// the columns.  Backed off while the larger lists would cost pipeline stages.
int umma_rep(const UmmaPlanIn& in) {
  int R = in.nq <= 32 ? 4 : (in.nq <= 64 ? 2 : 1);   // (1 for CTA pairs: nq > 128)
  const int s1 = stages_for(in, 1), want = s1 < 3 ? s1 : 3;
  while (R > 1 && stages_for(in, R) < want) R /= 2;
  return R;
}

bool umma_supported(const UmmaPlanIn& in) {
  if (!in.bf16 || in.nq < 1 || in.nq > 2 * UM_M || in.k < 1 || in.k > kMaxK) return false;
  if (stages_for(in, 1) < 2) return false;   // keep >= 2 pipeline stages
  if (in.w_sem != 1.f && tmode_of(in.Ep * 2) < 0) return false;
  if (!encoder()) return false;
  return true;
}

// scratch layout (MQ = 256 rows, enough for either CTA mode):
//   qs [MQ][Dp] bf16 | qt [CG][ell+2][128][Ep] bf16 | rq_s, rq_t [MQ] f32
constexpr int kMQ = 2 * UM_M;
static size_t qt_offset(const UmmaPlanIn& in) { return size_t(kMQ) * ((in.Dp + 63) / 64 * 64) * 2; }
static size_t rq_offset(const UmmaPlanIn& in) { return qt_offset(in) + size_t(in.ell + 2) * kMQ * in.Ep * 2; }
size_t umma_scratch_bytes(const UmmaPlanIn& in) { return rq_offset(in) + 2 * kMQ * 4 + 256; }

int umma_grid(const UmmaPlanIn& in) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // one CTA (or CTA pair) per SM (pair of SMs), persistent over the tiles
  const int cg = cg_of(in);
  const int tn = umma_tn(in, cg);
  const int64_t tiles = (in.n_rows + tn - 1) / tn;
  const int64_t units = sms / cg;
  return cg * int(tiles < units ? (tiles < 1 ? 1 : tiles) : units);
}
int umma_cg(const UmmaPlanIn& in) { return cg_of(in); }

cudaError_t launch_umma(const UmmaLaunch& L, cudaStream_t s) {
  const UmmaPlanIn& in = L.in;
  const bool sem = in.w_sem != 0.f && !L.sem_cos, traj = in.w_sem != 1.f;
  const int ell_pad = traj ? in.ell + ((in.Ep * 2 == 16) ? (in.ell & 1) : 0) : 0;
  const int CG = cg_of(in);
  // tcgen05 fp32 accumulation is not round-to-nearest per step: over D/16 = 256
  // MMAs (D = 4096) the semantic dot drifted by ~1.4e-5 relative (measured,
  // C5).  Two ways to keep the 1e-5 contract:
  //  * approx (semantic searches, k <= kApproxMaxK): ONE accumulator (TMEM
  //    double-buffered, the epilogue overlaps the next tile's MMAs), lists of
  //    k_ext > k approximate candidates, then an exact fp64 re-rank of the
  //    candidates with a verified margin (rerank_kernel) and an exact GEMV
  //    fallback for any query whose margin does not hold;
  //  * otherwise split K over two accumulators (the epilogue adds them in IEEE
  //    fp32; D >= 3072; measured: D = 2048 stays within 7e-6).
  // Blends weight the semantic part by d/L and their trajectory K is short,
  // so they keep one accumulator per part.
  const int n_sem_kb = sem ? (in.Dp + 63) / 64 : 0;
  const int split_kb = (sem && !traj && !in.approx && n_sem_kb >= 48) ? n_sem_kb / 2 : 0;
  // Two accumulators per tile (blend or split) single-buffer the 256-row tile's
  // TMEM.  128-row tiles keep the double buffer (2 x 2 x 128 columns) but
  // measured slower: the epilogue, not the serialisation, paces these scans.
  // With the loads removed, a split D = 3072 scan ran 0.72 PFLOP/s at 256 rows
  // and 0.68 at 128 rows; B = 256 on CTA pairs went 5.5 -> 13.1 ms.  Kept as an
  // experiment knob (FMOE_UMMA_TN=128).
  const bool nacc2 = (sem && traj) || split_kb > 0;
  const int TN = umma_tn(in, CG);
  int R = CG == 2 || in.rep < 1 ? 1 : in.rep;
  if (TN == 128 && R > 2) R = 2;                  // >= one 32-column chunk per replica
  const int MQ = UM_M * CG;
  char* scr = static_cast<char*>(L.scratch);
  __nv_bfloat16* qs = reinterpret_cast<__nv_bfloat16*>(scr);
  __nv_bfloat16* qt = reinterpret_cast<__nv_bfloat16*>(scr + qt_offset(in));
  float* rq_s = reinterpret_cast<float*>(scr + rq_offset(in));
  float* rq_t = rq_s + kMQ;
  // 1. query preparation (+ the seed bound)
  SeedArgs sd;
  if (L.seed_ids && traj && !sem) {
    sd.ids = L.seed_ids;
    sd.stride = L.seed_stride;
    sd.n = L.seed_n;
    sd.k = in.k;
    sd.id_offset = in.id_offset;
    sd.n_rows = in.n_rows;
    sd.cap = in.cap;
    sd.maps = static_cast<const __nv_bfloat16*>(in.maps);
    sd.psq = in.psq + int64_t(in.ell - 1) * in.cap;
  }
  count_launch();
  cudaError_t e = launch_pdl(umma_prep_kernel, dim3(MQ), dim3(256), 0, s, L.q_emb, L.q_prefix, L.q_stride, in.nq,
                             in.D, in.Dp, in.E, in.Ep, in.ell, ell_pad, qs, qt, rq_s, rq_t, L.valid, sem ? 1 : 0,
                             traj ? 1 : 0, MQ / R, L.gthr, sd, L.gate, L.keep_gthr);
  if (e != cudaSuccess) return e;
  // 2. tensor maps
  CUtensorMap tq_s{}, te_s{}, tq_t{}, tm_t{}, tc_o{};
  // cosine side output: fp32 [nq][cos_stride] rows of this pass, box 32 x 32 with
  // the 128-byte swizzle; TMA clips rows >= nq and columns >= n_rows
  const bool cos_tma = (in.cos_out && L.out_cos && sem && !traj && (L.cos_stride % 4) == 0 &&
                        (reinterpret_cast<uintptr_t>(L.out_cos) & 15) == 0) ||
                       (in.cos_in && L.sem_cos && !sem && traj && (L.cos_stride % 4) == 0 &&
                        (reinterpret_cast<uintptr_t>(L.sem_cos) & 15) == 0);
  if (cos_tma) {
    EncodeFn enc = encoder();
    cuuint64_t dims[2] = {cuuint64_t(in.n_rows), cuuint64_t(in.nq)};
    cuuint64_t strides[1] = {cuuint64_t(L.cos_stride) * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    void* base = sem ? static_cast<void*>(L.out_cos) : const_cast<float*>(L.sem_cos);
    if (!enc || enc(&tc_o, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if (sem) {
    if (!make_map(&te_s, in.emb, in.Dp, in.cap, 64, TN == 512 ? UM_M : um_rows(CG, TN), CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  int tmode = 0, lc = 0, n_traj_kb = 0;
  if (traj) {
    const int rb = in.Ep * 2;
    tmode = tmode_of(rb);
    const CUtensorMapSwizzle sw = tmode == 0   ? CU_TENSOR_MAP_SWIZZLE_NONE
                                  : tmode == 1 ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : tmode == 2 ? CU_TENSOR_MAP_SWIZZLE_64B
                                               : CU_TENSOR_MAP_SWIZZLE_128B;
    if (!make_map(&tq_t, qt, in.Ep, uint64_t(CG) * ell_pad * UM_M, in.Ep, UM_M, sw) ||
        !make_map(&tm_t, in.maps, in.Ep, uint64_t(in.L) * in.cap, in.Ep, um_rows(CG, TN), sw))
      return cudaErrorInvalidValue;
    lc = kStageA / (UM_M * rb);
    n_traj_kb = (ell_pad + lc - 1) / lc;
  }
  UmmaParams p{};
  p.n_rows = in.n_rows;
  p.n_tiles = int((in.n_rows + TN - 1) / TN);
  p.k = in.k;
  p.nq = in.nq;
  p.w = in.w_sem;
  p.n_sem_kb = n_sem_kb;
  p.n_traj_kb = n_traj_kb;
  p.ell_pad = ell_pad;
  p.tmode = tmode;
  p.lc = lc;
  const size_t lists = lists_bytes(in, R);
  p.stages = stages_for(in, R, TN);
  if (p.stages < 2) return cudaErrorInvalidValue;
  p.rep = R;
  p.split_kb = split_kb;
  p.acc_stages = (nacc2 && TN == UM_N) || TN == 512 ? 1 : 2;
  {
    static const int pf_env = getenv("FMOE_L2PF") ? atoi(getenv("FMOE_L2PF")) : -1;
    // L2 prefetch of the store operand: measured +2..5 % for the 512-row semantic
    // tiles at 2 k-blocks ahead (3 smem stages; deeper hurts: 8 -> -6 %,
    // profiles/r02d_semantic_experiments.md), no gain elsewhere
    p.l2pf = pf_env >= 0 ? pf_env : (TN == 512 ? 2 : 0);
    static const int es_env = getenv("FMOE_EPI_SLEEP") ? atoi(getenv("FMOE_EPI_SLEEP")) : -1;
    p.epi_sleep = es_env >= 0 ? es_env : 0;
    static const int fk_env = getenv("FMOE_FAKE_LOADS") ? atoi(getenv("FMOE_FAKE_LOADS")) : 0;
    p.fake_loads = fk_env;   // measured neutral (64..1000 ns); kept as a knob
    static const int na_env = getenv("FMOE_NO_A_RELOAD") ? atoi(getenv("FMOE_NO_A_RELOAD")) : 0;
    p.no_a_reload = na_env;
    static const int ne_env = getenv("FMOE_NO_EPI") ? atoi(getenv("FMOE_NO_EPI")) : 0;
    p.no_epi = ne_env;
  }
  p.cos_tma = cos_tma ? 1 : 0;
  p.cos_ring = cos_ring();
  p.cos_bound = !sem && traj && L.sem_cos != nullptr && !cos_tma && umma_cos_bound();
  {
    static const int ct_env = getenv("FMOE_COS_TILED_EXP") ? atoi(getenv("FMOE_COS_TILED_EXP")) : 0;
    p.cos_tiled_exp = cos_tma ? ct_env : 0;
    p.cos_bytes = size_t(in.nq) * size_t(L.cos_stride) * 4 / kCosStage * kCosStage;
  }
  p.cap = in.cap;
  p.L = in.L;
  p.maps = static_cast<const unsigned char*>(in.maps);
  p.qt = reinterpret_cast<const unsigned char*>(qt);
  p.qs = reinterpret_cast<const unsigned char*>(qs);
  p.emb_raw = in.emb;
  p.emb_bytes = size_t(in.cap) * in.Dp * 2 / 16384 * 16384;
  {
    static const int tb_env = getenv("FMOE_TILED_B_EXP") ? atoi(getenv("FMOE_TILED_B_EXP")) : 0;
    p.tiled_b_exp = tb_env;
  }
  p.id_offset = in.id_offset;
  p.rq_s = rq_s;
  p.rq_t = rq_t;
  p.r_e = in.r_e;
  p.psq = traj ? in.psq + int64_t(in.ell - 1) * in.cap : in.psq;
  p.cand = L.cand;
  p.cand_q0 = L.cand_q0;
  p.grid = L.grid / CG;
  p.trace = L.trace;
  p.out_cos = L.out_cos;
  p.sem_cos = L.sem_cos;
  p.cos_stride = L.cos_stride;
  p.gthr = L.gthr;
  p.excl = L.excl;
  p.gate = L.gate;
  const size_t smem = 1024 + size_t(p.stages) * um_stage_bytes(CG, TN) + lists;
  using Fn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                     const UmmaParams);
#define FMOE_UMMA_PICK(CGV, TNV)                                                      \
  (sem && traj ? scan_umma_kernel<true, true, CGV, TNV>                               \
   : sem       ? scan_umma_kernel<true, false, CGV, TNV>                              \
               : scan_umma_kernel<false, true, CGV, TNV>)
  const Fn fn = CG == 2 ? (TN == 512 ? scan_umma_kernel<true, false, 2, 512>
                         : TN == 128 ? FMOE_UMMA_PICK(2, 128) : FMOE_UMMA_PICK(2, 256))
                        : (TN == 128 ? FMOE_UMMA_PICK(1, 128) : FMOE_UMMA_PICK(1, 256));
#undef FMOE_UMMA_PICK
  {
    static std::mutex mu;
    static std::map<const void*, size_t> set;
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = set[reinterpret_cast<const void*>(fn)];
    if (cur < smem) {
      e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(smem));
      if (e != cudaSuccess) return e;
      cur = smem;
    }
  }
  count_launch();
  if (CG == 1) return launch_pdl(fn, dim3(L.grid), dim3(kUmThreads), smem, s, tq_s, te_s, tq_t, tm_t, tc_o, p);
  // CTA pairs: clusters of 2 (one TPC), with programmatic dependent launch
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.grid);
  cfg.blockDim = dim3(kUmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 2;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fn, tq_s, te_s, tq_t, tm_t, tc_o, p);
}

}  // namespace fmoe
