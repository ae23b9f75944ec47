// store.cu -- the C ABI of include/fmoe.h: store object, argument checks,
// host/device staging, and dispatch of the sm_100a kernels.
#include <atomic>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda.h>

#include "../../include/fmoe.h"
#include "common.cuh"
#include "kernels.cuh"

namespace fmoe {
int64_t launch_count();
}

using namespace fmoe;

// Scratch reused by consecutive calls on one stream (stream-ordered, so no
// hazard between them): per-block candidate lists and the scan's ticket
// counters, which the last block of every scan resets to zero.
struct StreamScratch {
  char* buf = nullptr;
  size_t bytes = 0;
  unsigned* counters = nullptr;      // zero between calls
  int ncounters = 0;
  unsigned long long* best = nullptr;  // zero between calls (k == 1 merge)
  int nbest = 0;
};

struct fmoe_store {
  fmoe_store_config cfg;
  mutable std::mutex mu;
  mutable std::unordered_map<cudaStream_t, StreamScratch> scratch;
  int device;
  int bf16, esz, Dp, Ep;
  void* emb = nullptr;
  float* r_e = nullptr;
  void* maps = nullptr;
  float* psq = nullptr;
  int64_t n = 0;
  uint64_t gen = 0;       // bumped by every insert/write (invalidates trajectory sessions)
  struct Dist {           // sharded store (fmoe_store_create_sharded)
    fmoe::Comm comm;
    int64_t cap_total = 0, per = 0, n_total = 0;
  };
  Dist* dist = nullptr;
  uint32_t* excl = nullptr;   // [cap / 32] claimed-slot bitmap of an insert's sub-batches (zero between calls)

  StoreView view() const {
    StoreView v;
    v.emb = emb; v.r_e = r_e; v.maps = maps; v.psq = psq;
    v.cap = cfg.capacity; v.L = cfg.L; v.E = cfg.E; v.D = cfg.D; v.Dp = Dp; v.Ep = Ep; v.bf16 = bf16;
    return v;
  }
};

namespace {

thread_local std::string g_err;

fmoe_status fail(fmoe_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
fmoe_status cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? FMOE_ERR_OOM : FMOE_ERR_CUDA;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// 0 = host (pageable or pinned), 1 = device memory of `dev`, -1 = other device,
// -2 = a pointer the runtime rejects (CUDA >= 11 classifies plain host memory
// as cudaMemoryTypeUnregistered, so a failure is not "host")
int ptr_kind(const void* p, int dev) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return -2;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return at.device == dev ? 1 : -1;
  return 0;
}

// Stream-ordered scratch comes from a private memory pool per device (release
// threshold: keep everything), so the library never changes the process's
// default pool.
cudaMemPool_t scratch_pool(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    pool = nullptr;
  } else {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  pools[dev] = pool;
  return pool;
}
cudaError_t pool_malloc(void** p, size_t bytes, int dev, cudaStream_t s) {
  cudaMemPool_t pool = scratch_pool(dev);
  return pool ? cudaMallocFromPoolAsync(p, bytes, pool, s) : cudaMallocAsync(p, bytes, s);
}

// fmoe_set_host_sync: whether a call with host outputs synchronises its stream
std::atomic<int> g_host_sync{1};

// Staging arena of a (device, stream) for the calling thread: host arguments
// of a call are carved from one device buffer instead of one cudaMallocAsync /
// cudaFreeAsync pair each.  A later call on the same stream may reuse the
// bytes at once: its copies and kernels are ordered after the earlier call's.
// Grows (stream-ordered free + malloc) when a call needed more.
// The arena is capped at kArenaMax (a C5 host cosine matrix would otherwise
// pin 16 GB for the life of the thread); bigger staging is allocated and freed
// per call, stream-ordered.
constexpr size_t kArenaMax = size_t(64) << 20;
struct Arena {
  char* base = nullptr;
  size_t cap = 0, want = 0;
};
Arena& staging_arena(int dev, cudaStream_t s) {
  thread_local std::map<std::pair<int, cudaStream_t>, Arena> arenas;
  return arenas[{dev, s}];
}

// Stream-ordered staging of host arguments through device buffers.
struct Staging {
  cudaStream_t s;
  int dev;
  Arena* arena = nullptr;
  size_t used = 0;
  std::vector<void*> allocs;
  struct Back { void* host; void* dev; size_t bytes; };
  std::vector<Back> backs;
  cudaError_t err = cudaSuccess;
  const char* what = "";
  bool bad_device = false;
  bool bad_ptr = false;

  bool own_only = false;   // every buffer is a per-call allocation (a sharded call nests a local call,
                           // whose own Staging carves the thread's arena from offset 0)

  Staging(cudaStream_t s_, int dev_, bool own = false) : s(s_), dev(dev_), own_only(own) {}

  void* scratch(size_t bytes) {
    if (err != cudaSuccess) return nullptr;
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~size_t(255);
    if (own_only) {
      cudaError_t e = pool_malloc(&p, bytes, dev, s);
      if (e != cudaSuccess) { err = e; what = "cudaMallocAsync"; return nullptr; }
      allocs.push_back(p);
      return p;
    }
    if (!arena) arena = &staging_arena(dev, s);
    if (used + bytes <= arena->cap) {
      p = arena->base + used;
      used += bytes;
      return p;
    }
    // grow for the next call, up to kArenaMax; larger requests stay per-call
    if (used + bytes > arena->want && used + bytes <= kArenaMax) arena->want = used + bytes;
    cudaError_t e = pool_malloc(&p, bytes, dev, s);
    if (e != cudaSuccess) { err = e; what = "cudaMallocAsync"; return nullptr; }
    allocs.push_back(p);
    return p;
  }
  template <class T>
  const T* in(const T* p, size_t count) {
    if (!p) return nullptr;
    const int k = ptr_kind(p, dev);
    if (k == 1) return p;
    if (k < 0) { bad_device = true; bad_ptr = bad_ptr || k == -2; return nullptr; }
    T* d = static_cast<T*>(scratch(count * sizeof(T)));
    if (!d) return nullptr;
    if (count) {
      cudaError_t e = cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) { err = e; what = "H2D copy"; }
    }
    return d;
  }
  template <class T>
  T* out(T* p, size_t count) {
    if (!p) return nullptr;
    const int k = ptr_kind(p, dev);
    if (k == 1) return p;
    if (k < 0) { bad_device = true; bad_ptr = bad_ptr || k == -2; return nullptr; }
    T* d = static_cast<T*>(scratch(count * sizeof(T)));
    if (d) backs.push_back({p, d, count * sizeof(T)});
    return d;
  }
  fmoe_status check() const {
    if (bad_device) return fail(FMOE_ERR_INVALID_ARG, bad_ptr ? "pointer rejected by cudaPointerGetAttributes"
                                                              : "array on another device");
    if (err != cudaSuccess) return cuda_fail(err, what);
    return FMOE_OK;
  }
  // copies outputs back, frees scratch; synchronises if any output is host memory
  fmoe_status finish(fmoe_status st) {
    for (auto& b : backs) {
      if (st == FMOE_OK && b.bytes) {
        cudaError_t e = cudaMemcpyAsync(b.host, b.dev, b.bytes, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) st = cuda_fail(e, "D2H copy");
      }
    }
    for (void* p : allocs) cudaFreeAsync(p, s);
    if (arena && arena->want > arena->cap) {
      if (arena->base) cudaFreeAsync(arena->base, s);
      arena->base = nullptr;
      arena->cap = 0;
      const size_t nb = arena->want < (size_t(1) << 20) ? (size_t(1) << 20) : arena->want;
      if (pool_malloc(reinterpret_cast<void**>(&arena->base), nb, dev, s) == cudaSuccess) arena->cap = nb;
      else cudaGetLastError();
    }
    if (!backs.empty() && g_host_sync.load(std::memory_order_relaxed)) {
      cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess && st == FMOE_OK) st = cuda_fail(e, "stream sync");
    }
    return st;
  }
};

int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Sharded stores: a public call dispatches to its collective version, which
// runs the same public call on the local shard inside a LocalScope (no
// re-dispatch) with device outputs, then exchanges and merges.
thread_local int g_local_depth = 0;
struct LocalScope {
  LocalScope() { ++g_local_depth; }
  ~LocalScope() { --g_local_depth; }
};
bool sharded(const fmoe_store* st) { return st && st->dist && g_local_depth == 0; }
fmoe_status sharded_search(const fmoe_store* st, int64_t B, const float* q_emb, const float* q_prefix, int32_t ell,
                           float w, int32_t k, float* out_score, int64_t* out_id, void* stream, float* out_cos,
                           int64_t cos_stride);
fmoe_status sharded_blend_cos(const fmoe_store* st, int64_t B, const float* sem_cos, int64_t cos_stride,
                              const float* q_prefix, int32_t ell, float w_sem, int32_t k, float* out_score,
                              int64_t* out_id, void* stream);
fmoe_status sharded_select(const fmoe_store* st, int64_t B, const int64_t* map_id, const float* score, float delta,
                           int32_t lb, int32_t le, uint64_t* out_mask, int32_t* out_count, void* stream);
fmoe_status sharded_insert(fmoe_store* st, int64_t B, const float* emb, const float* maps, const float* sem_cos,
                           int64_t cos_stride, int64_t* out_slot, int64_t* out_replaced, void* stream);

fmoe_status check_cfg(const fmoe_store_config* c) {
  if (!c) return fail(FMOE_ERR_INVALID_ARG, "null config");
  if (c->L < 1 || c->E < 1 || c->E > FMOE_MAX_E || c->D < 1 || c->K < 1 || c->K > c->E)
    return fail(FMOE_ERR_SHAPE, "need L>=1, 1<=E<=64, 1<=K<=E, D>=1");
  if (c->d < 1 || c->d >= c->L) return fail(FMOE_ERR_SHAPE, "need 1 <= d < L");
  if (c->dtype != FMOE_F32 && c->dtype != FMOE_BF16) return fail(FMOE_ERR_SHAPE, "dtype");
  if (c->capacity < 1 || c->id_offset < 0 || c->capacity + c->id_offset > 0xffffffffll)
    return fail(FMOE_ERR_SHAPE, "capacity/id_offset: global ids must fit in 32 bits");
  if (c->L * int64_t(round_up(c->E, 8)) * 4 > 200 * 1024)
    return fail(FMOE_ERR_SHAPE, "L*E too large for the staged trajectory query");
  if (int64_t(round_up(c->D, 8)) * 4 > 200 * 1024) return fail(FMOE_ERR_SHAPE, "D too large");
  return FMOE_OK;
}

fmoe_status stream_scratch(const fmoe_store* st, cudaStream_t s, size_t bytes, int ncount, int nbest, char** buf,
                           unsigned** ctr, unsigned long long** best) {
  std::lock_guard<std::mutex> lk(st->mu);
  StreamScratch& sc = st->scratch[s];
  cudaError_t e;
  if (sc.bytes < bytes) {
    if (sc.buf) cudaFreeAsync(sc.buf, s);
    sc.buf = nullptr;
    sc.bytes = 0;
    const size_t nb = bytes + bytes / 2 + 4096;
    if ((e = pool_malloc(reinterpret_cast<void**>(&sc.buf), nb, st->device, s)) != cudaSuccess) return cuda_fail(e, "scratch");
    sc.bytes = nb;
  }
  if (sc.ncounters < ncount) {
    if (sc.counters) cudaFreeAsync(sc.counters, s);
    sc.counters = nullptr;
    sc.ncounters = 0;
    const int nc = ncount < 64 ? 64 : ncount;
    if ((e = pool_malloc(reinterpret_cast<void**>(&sc.counters), size_t(nc) * 4, st->device, s)) != cudaSuccess)
      return cuda_fail(e, "counters");
    if ((e = cudaMemsetAsync(sc.counters, 0, size_t(nc) * 4, s)) != cudaSuccess) return cuda_fail(e, "counters");
    sc.ncounters = nc;
  }
  if (sc.nbest < nbest) {
    if (sc.best) cudaFreeAsync(sc.best, s);
    sc.best = nullptr;
    sc.nbest = 0;
    const int nb = nbest < 256 ? 256 : nbest;
    if ((e = pool_malloc(reinterpret_cast<void**>(&sc.best), size_t(nb) * 8, st->device, s)) != cudaSuccess)
      return cuda_fail(e, "best keys");
    if ((e = cudaMemsetAsync(sc.best, 0, size_t(nb) * 8, s)) != cudaSuccess) return cuda_fail(e, "best keys");
    sc.nbest = nb;
  }
  *buf = sc.buf;
  *ctr = sc.counters;
  *best = sc.best;
  return FMOE_OK;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Batches of at least this many queries go to the tensor cores (bf16 stores).
int umma_min_batch() {
  static const int b = getenv("FMOE_UMMA_MIN_B") ? atoi(getenv("FMOE_UMMA_MIN_B")) : 5;
  return b;
}

// RDY insert: candidates kept per row by the first pass (see fmoe_store_insert_cos)
constexpr int kRdyFirst = 8;

// The claimed-slot bitmap of an insert's sub-batches, allocated zeroed on the
// first insert that needs more than one sub-batch.
fmoe_status ensure_excl(fmoe_store* st, int64_t nrep) {
  if (nrep <= FMOE_MAX_K || st->excl) return FMOE_OK;
  const size_t words = size_t(st->cfg.capacity + 31) / 32 + 1;
  cudaError_t e = cudaMalloc(&st->excl, words * 4);
  if (e == cudaSuccess) e = cudaMemset(st->excl, 0, words * 4);
  return e == cudaSuccess ? FMOE_OK : cuda_fail(e, "insert bitmap");
}

// Whether a search of B queries with list length k runs on the tensor cores
// (fills *in when it does).
bool umma_plan(const fmoe_store* st, int64_t B, int k, int ell, float w, int64_t n_rows, uint32_t id_offset,
               UmmaPlanIn* in) {
  if (!st->bf16 || B < umma_min_batch()) return false;
  UmmaPlanIn& u = *in;
  u = UmmaPlanIn{};
  u.bf16 = 1; u.nq = int(B < 256 ? B : 256); u.k = k; u.D = st->cfg.D; u.Dp = st->Dp; u.E = st->cfg.E;
  u.Ep = st->Ep; u.L = st->cfg.L; u.ell = ell; u.w_sem = w; u.n_rows = n_rows; u.cap = st->cfg.capacity;
  u.id_offset = id_offset; u.emb = st->emb; u.maps = st->maps; u.r_e = st->r_e; u.psq = st->psq;
  return umma_supported(u);
}

// Batched call on the tensor cores: passes of <= 128 queries (CTAs) or <= 256
// (CTA pairs, cta_group::2), per-CTA(-pair) lists, then one merge kernel over
// all passes.
struct CosArgs {
  float* out = nullptr;          // semantic scans: write the cosines
  const float* in = nullptr;     // RDY / blend scans: blend these instead of re-reading embeddings
  int64_t stride = 0;
  const uint32_t* excl = nullptr;   // RDY scans of a later insert sub-batch: rows already claimed
};

fmoe_status run_search_umma(const fmoe_store* st, UmmaPlanIn in, int64_t B, const float* dq, const float* dp,
                            int64_t q_stride, cudaStream_t s, float* ds, int64_t* di, uint64_t* dkeys,
                            bool check_queries, const CosArgs& cos, const int64_t* seed_ids, int seed_stride,
                            int seed_n, int k_out, const int* gate) {
  in.cg = umma_cg(in);                                // from the first (largest) pass
  const int grid = umma_grid(in);
  in.rep = umma_rep(in);
  const int pass = in.cg * 128;
  const int n_lists = grid / in.cg;                   // one list per (query, CTA or CTA pair)
  const size_t cand_b = align_up(size_t(B) * n_lists * in.k * 8);
  const size_t valid_b = align_up(size_t(B) * 4);
  const size_t prep_b = align_up(umma_scratch_bytes(in));
  char* buf = nullptr;
  unsigned* counters = nullptr;
  unsigned long long* best = nullptr;
  const size_t gthr_b = align_up(size_t(B) * 8);
  fmoe_status cs = stream_scratch(st, s, cand_b + valid_b + prep_b + gthr_b, 1, 1, &buf, &counters, &best);
  if (cs != FMOE_OK) return cs;
  uint64_t* cand = reinterpret_cast<uint64_t*>(buf);
  float* valid = reinterpret_cast<float*>(buf + cand_b);
  unsigned long long* gthr = reinterpret_cast<unsigned long long*>(buf + cand_b + valid_b + prep_b);
  for (int64_t q0 = 0; q0 < B; q0 += pass) {
    UmmaLaunch L{};
    L.in = in;
    L.in.nq = int(B - q0 < pass ? B - q0 : pass);
    L.q_emb = dq ? dq + q0 * in.D : nullptr;
    L.q_prefix = dp ? dp + q0 * q_stride : nullptr;
    L.q_stride = q_stride;
    L.scratch = buf + cand_b + valid_b;
    L.valid = valid + q0;
    L.gthr = gthr + q0;
    L.seed_ids = seed_ids ? seed_ids + q0 * seed_stride : nullptr;
    L.seed_stride = seed_stride;
    L.seed_n = seed_n;
    L.gate = gate;
    L.cand = cand;
    L.cand_q0 = int(q0);
    L.grid = grid;
    L.trace = trace_buffer();
    L.out_cos = cos.out ? cos.out + q0 * cos.stride : nullptr;
    L.sem_cos = cos.in ? cos.in + q0 * cos.stride : nullptr;
    L.cos_stride = cos.stride;
    L.excl = cos.excl;
    cudaError_t e = launch_umma(L, s);
    if (e != cudaSuccess) return cuda_fail(e, "umma scan launch");
  }
  cudaError_t e = launch_merge_keys(int(B), n_lists, in.k, cand, k_out > in.k ? k_out : in.k,
                                    check_queries ? valid : nullptr, ds, di, dkeys, s, gate);
  return e == cudaSuccess ? FMOE_OK : cuda_fail(e, "merge launch");
}

// Approximate tensor-core semantic scan + exact re-rank (rerank.cu): the scan
// keeps ke > k candidates per query from ONE TMEM accumulator (double-buffered
// tiles), the merge keeps the best ke, rerank_kernel recomputes Eq. 1 exactly
// for them and verifies the margin; queries that fail it are rescanned exactly
// by gated GEMV passes (none in practice) whose results are scattered back.
constexpr int kApproxMaxK = 48;
int approx_list_len(int k) {
  // candidates kept per query for the exact re-rank (FMOE_APPROX_EXTRA: k + extra, measurement knob)
  static const int extra = getenv("FMOE_APPROX_EXTRA") ? atoi(getenv("FMOE_APPROX_EXTRA")) : -1;
  if (extra >= 1) return k + extra < kMaxK ? k + extra : kMaxK;
  const int a = k + 8 > 2 * k ? k + 8 : 2 * k;
  return a < kMaxK ? a : kMaxK;
}

fmoe_status run_search_umma_approx(const fmoe_store* st, UmmaPlanIn in, int64_t B, const float* dq, cudaStream_t s,
                                   float* ds, int64_t* di, uint64_t* dkeys, const CosArgs& cos, int k) {
  const int ke = in.k;
  in.cg = umma_cg(in);
  const int grid = umma_grid(in);
  in.rep = umma_rep(in);
  const int pass = in.cg * 128;
  const int n_lists = grid / in.cg;
  const int D = st->cfg.D;
  // fallback GEMV geometry
  ScanArgs g{};
  g.st = st->view();
  g.n_rows = in.n_rows;
  g.ell = 0;
  g.w_sem = 1.f;
  g.k = k;
  g.nq = 4;
  g.id_offset = in.id_offset;
  g.grid = scan_gemv_grid(g);
  const int npass_g = int((B + 3) / 4);
  const size_t cand_b = align_up(size_t(B) * n_lists * ke * 8), valid_b = align_up(size_t(B) * 4);
  const size_t prep_b = align_up(umma_scratch_bytes(in)), gthr_b = align_up(size_t(B) * 8);
  const size_t mk_b = align_up(size_t(B) * ke * 8), qc_b = align_up(size_t(B) * D * 4), qmap_b = align_up(size_t(B) * 4);
  const size_t fbs_b = align_up(size_t(B) * k * 4), fbi_b = align_up(size_t(B) * k * 8);
  const size_t gc_b = align_up(size_t(4) * g.grid * k * 8);
  char* buf = nullptr;
  unsigned* counters = nullptr;
  unsigned long long* best = nullptr;
  fmoe_status cs = stream_scratch(st, s, cand_b + valid_b + prep_b + gthr_b + mk_b + qc_b + qmap_b + fbs_b + 2 * fbi_b +
                                  size_t(npass_g) * gc_b, npass_g + 1, int(B), &buf, &counters, &best);
  if (cs != FMOE_OK) return cs;
  char* c = buf;
  uint64_t* cand = reinterpret_cast<uint64_t*>(c); c += cand_b;
  float* valid = reinterpret_cast<float*>(c); c += valid_b;
  char* prep = c; c += prep_b;
  unsigned long long* gthr = reinterpret_cast<unsigned long long*>(c); c += gthr_b;
  uint64_t* mkeys = reinterpret_cast<uint64_t*>(c); c += mk_b;
  float* qc = reinterpret_cast<float*>(c); c += qc_b;
  int* qmap = reinterpret_cast<int*>(c); c += qmap_b;
  float* fb_s = reinterpret_cast<float*>(c); c += fbs_b;
  int64_t* fb_i = reinterpret_cast<int64_t*>(c); c += fbi_b;
  uint64_t* fb_k = reinterpret_cast<uint64_t*>(c); c += fbi_b;
  uint64_t* gcand = reinterpret_cast<uint64_t*>(c);
  int* nfail = reinterpret_cast<int*>(counters + npass_g);    // zero between calls (the scatter resets it)
  // Sample pass: the same scan over rows [0, S), S ~ n/32, seeds every query's
  // admission threshold with the ke-th best approximate key of the sample (a
  // valid bound: the full scan gives those rows bit-identical keys).  Without
  // it each list starts at -inf and the per-thread heap inserts of the first
  // tiles (warp-divergent, ~450 cycles each) cost ~7% of the scan.  Measured
  // (2M / 8M rows, B = 256): the sample pass costs what it saves -- opt-in
  // knob FMOE_SAMPLE_SEED=1.
  static const bool want_seed = getenv("FMOE_SAMPLE_SEED") != nullptr && atoi(getenv("FMOE_SAMPLE_SEED")) != 0;
  const int64_t S_rows = in.n_rows / 32 / 4096 * 4096;
  const bool seeded = want_seed && S_rows >= 65536;
  if (seeded) {
    UmmaPlanIn si = in;
    si.n_rows = S_rows;
    const int sgrid = umma_grid(si);
    const int s_lists = sgrid / si.cg;
    if (size_t(B) * s_lists * ke * 8 > cand_b) return fail(FMOE_ERR_UNSUPPORTED, "sample pass scratch");
    for (int64_t q0 = 0; q0 < B; q0 += pass) {
      UmmaLaunch L{};
      L.in = si;
      L.in.nq = int(B - q0 < pass ? B - q0 : pass);
      L.q_emb = dq + q0 * D;
      L.scratch = prep;
      L.valid = valid + q0;
      L.gthr = gthr + q0;
      L.cand = cand;
      L.cand_q0 = int(q0);
      L.grid = sgrid;
      L.trace = nullptr;
      cudaError_t e = launch_umma(L, s);
      if (e != cudaSuccess) return cuda_fail(e, "umma sample scan launch");
    }
    cudaError_t e = launch_merge_keys(int(B), s_lists, ke, cand, ke, nullptr, nullptr, nullptr, mkeys, s);
    if (e == cudaSuccess) e = launch_seed_from_sample(int(B), ke, mkeys, gthr, s);
    if (e != cudaSuccess) return cuda_fail(e, "sample seed launch");
  }
  for (int64_t q0 = 0; q0 < B; q0 += pass) {
    UmmaLaunch L{};
    L.in = in;
    L.keep_gthr = seeded ? 1 : 0;
    L.in.nq = int(B - q0 < pass ? B - q0 : pass);
    L.q_emb = dq + q0 * D;
    L.scratch = prep;
    L.valid = valid + q0;
    L.gthr = gthr + q0;
    L.cand = cand;
    L.cand_q0 = int(q0);
    L.grid = grid;
    L.trace = trace_buffer();
    L.out_cos = cos.out ? cos.out + q0 * cos.stride : nullptr;
    L.cos_stride = cos.stride;
    cudaError_t e = launch_umma(L, s);
    if (e != cudaSuccess) return cuda_fail(e, "umma scan launch");
  }
  cudaError_t e = launch_merge_keys(int(B), n_lists, ke, cand, ke, nullptr, nullptr, nullptr, mkeys, s);
  if (e != cudaSuccess) return cuda_fail(e, "merge launch");
  RerankArgs r{};
  r.B = int(B); r.ke = ke; r.k = k; r.keys = mkeys; r.q_emb = dq; r.D = D; r.Dp = st->Dp; r.emb = st->emb;
  r.r_e = st->r_e; r.id_offset = in.id_offset; r.valid = valid;
  // |approx - exact| <= (MMAs per dot) * 4 ulp of the largest partial sum
  // (relative to ||q|| ||e||, P:461-466 cosine scale) + epilogue roundings
  r.eps = float(double((st->Dp + 15) / 16) * std::ldexp(1.0, -21) + std::ldexp(1.0, -20));
  r.out_score = ds; r.out_id = di; r.out_keys = dkeys; r.nfail = nfail; r.qmap = qmap; r.qc = qc;
  if ((e = launch_rerank(r, s)) != cudaSuccess) return cuda_fail(e, "rerank launch");
  g.q_emb = qc;
  g.out_score = fb_s;
  g.out_id = fb_i;
  g.out_keys = fb_k;
  g.best = best;
  g.check_valid = 1;
  g.trace = trace_buffer();
  g.run_if_gt = nfail;
  for (int p = 0; p < npass_g; ++p) {
    g.q0 = 4 * p;
    g.counter = counters + p;
    g.cand = gcand + size_t(p) * (gc_b / 8);
    if ((e = launch_scan_gemv(g, s)) != cudaSuccess) return cuda_fail(e, "fallback scan launch");
  }
  e = launch_rerank_scatter(nfail, qmap, k, fb_s, fb_i, fb_k, ds, di, dkeys, nfail, s);
  return e == cudaSuccess ? FMOE_OK : cuda_fail(e, "rerank scatter launch");
}

// One scoring call: GEMV scan passes of <= 4 queries, each merging its

// fp32 store, B >= 5: passes of <= 64 queries on the FFMA batched scan
// (scan_f32mm.cu), each reading the store once, then one merge.
fmoe_status run_search_f32mm(const fmoe_store* st, int64_t B, const float* dq, const float* dp, int64_t q_stride,
                             int ell, float w, int k, int64_t n_rows, uint32_t id_offset, cudaStream_t s, float* ds,
                             int64_t* di, uint64_t* dkeys, bool check_queries, const CosArgs& cos, int k_out) {
  const bool sem = w != 0.f && !cos.in, traj = w != 1.f;
  const int nq0 = int(B < 64 ? B : 64);
  const int grid = f32mm_grid(n_rows, nq0, sem && traj);
  const int n_lists = grid * f32mm_lists_per_cta(nq0);
  const int n_sem_ch = sem ? (st->Dp + 31) / 32 : 0;
  const int n_traj_ch = traj ? (ell * st->Ep + 31) / 32 : 0;
  const int qpitch = (n_sem_ch + n_traj_ch) * 32;
  const size_t cand_b = align_up(size_t(B) * n_lists * k * 8);
  const size_t vec_b = align_up(size_t(B) * 4);
  const size_t qop_b = align_up(size_t(64) * qpitch * 4);
  char* buf = nullptr;
  unsigned* counters = nullptr;
  unsigned long long* best = nullptr;
  fmoe_status cs = stream_scratch(st, s, cand_b + 3 * vec_b + qop_b, 1, 1, &buf, &counters, &best);
  if (cs != FMOE_OK) return cs;
  uint64_t* cand = reinterpret_cast<uint64_t*>(buf);
  float* valid = reinterpret_cast<float*>(buf + cand_b);
  float* rq_s = reinterpret_cast<float*>(buf + cand_b + vec_b);
  float* rq_t = reinterpret_cast<float*>(buf + cand_b + 2 * vec_b);
  float* qop = reinterpret_cast<float*>(buf + cand_b + 3 * vec_b);
  for (int64_t q0 = 0; q0 < B; q0 += 64) {
    const int nq = int(B - q0 < 64 ? B - q0 : 64);
    F32mmPrep p{};
    p.q_emb = sem ? dq + q0 * st->cfg.D : nullptr;
    p.q_prefix = traj ? dp + q0 * q_stride : nullptr;
    p.q_stride = q_stride;
    p.D = st->cfg.D; p.E = st->cfg.E; p.Ep = st->Ep; p.ell = traj ? ell : 0;
    p.n_sem_ch = n_sem_ch; p.n_traj_ch = n_traj_ch; p.qpitch = qpitch;
    p.sem = sem; p.traj = traj;
    p.qop = qop; p.rq_s = rq_s + q0; p.rq_t = rq_t + q0; p.valid = valid + q0;
    cudaError_t e = launch_f32mm_prep(p, nq, s);
    if (e != cudaSuccess) return cuda_fail(e, "f32mm prep launch");
    F32mmArgs a{};
    a.st = st->view();
    a.n_rows = n_rows;
    a.ell = traj ? ell : 0;
    a.w = w;
    a.k = k;
    a.nq = nq;
    a.wq = f32mm_wq(nq0);          // uniform over the passes (the cand layout)
    a.qop = qop;
    a.qpitch = qpitch;
    a.n_sem_ch = n_sem_ch;
    a.n_traj_ch = n_traj_ch;
    a.rq_s = rq_s + q0;
    a.rq_t = rq_t + q0;
    a.id_offset = id_offset;
    a.cand = cand;
    a.cand_q0 = int(q0);
    // every pass writes n_lists lists per query: a smaller last pass uses the
    // first pass's grid and lists-per-CTA so the cand layout stays uniform
    a.grid = grid;
    a.out_cos = cos.out ? cos.out + q0 * cos.stride : nullptr;
    a.sem_cos = cos.in ? cos.in + q0 * cos.stride : nullptr;
    a.cos_stride = cos.stride;
    a.excl = cos.excl;
    e = launch_f32mm(a, s);
    if (e != cudaSuccess) return cuda_fail(e, "f32mm scan launch");
  }
  cudaError_t e = launch_merge_keys(int(B), n_lists, k, cand, k_out > k ? k_out : k,
                                    check_queries ? valid : nullptr, ds, di, dkeys, s);
  return e == cudaSuccess ? FMOE_OK : cuda_fail(e, "merge launch");
}

// candidates in its last block.  `extra` bytes of scratch are reserved after
// the candidate lists (returned in *extra_ptr) for the caller.
fmoe_status run_search(const fmoe_store* st, int64_t B, const float* dq, const float* dp, int64_t q_stride, int ell,
                       float w, int k, int64_t n_rows, uint32_t id_offset, cudaStream_t s, float* ds, int64_t* di,
                       uint64_t* dkeys, bool check_queries, const CosArgs& cos = CosArgs(),
                       const int64_t* seed_ids = nullptr, int seed_stride = 0, int seed_n = 0, int k_out = 0,
                       int* out_stride = nullptr, const int* gate = nullptr) {
  // k_out > k (tensor-core path only): the merge writes k_out keys per query,
  // the exact top-k first; *out_stride receives the row stride written
  if (out_stride) *out_stride = k;
  if (n_rows == 0) {
    cudaError_t e = launch_merge_keys(int(B), 0, k, nullptr, k, nullptr, ds, di, dkeys, s);
    return e == cudaSuccess ? FMOE_OK : cuda_fail(e, "merge launch");
  }
  UmmaPlanIn in{};
  static const bool no_approx = getenv("FMOE_NO_APPROX") != nullptr;   // knob: the K-split precise scan
  if (!no_approx && w == 1.f && !cos.in && !seed_ids && !gate && k <= kApproxMaxK &&
      umma_plan(st, B, approx_list_len(k), 0, 1.f, n_rows, id_offset, &in)) {
    in.approx = 1;
    // FMOE_COS_DIRECT=1: the cosine side output by direct stores (no smem staging; measurement knob)
    static const bool cos_direct = getenv("FMOE_COS_DIRECT") != nullptr && atoi(getenv("FMOE_COS_DIRECT")) != 0;
    in.cos_out = cos.out != nullptr && !cos_direct;
    if (umma_supported(in)) return run_search_umma_approx(st, in, B, dq, s, ds, di, dkeys, cos, k);
  }
  if (umma_plan(st, B, k, ell, w, n_rows, id_offset, &in)) {
    in.cos_out = cos.out != nullptr && w == 1.f;
    // the bounded reads of the cached cosines need no TMA ring (umma_cos_bound)
    in.cos_in = cos.in != nullptr && w != 1.f && !umma_cos_bound();
    if (in.cos_out && !umma_supported(in)) in.cos_out = 0;   // no room for the staging: direct stores
    if (in.cos_in && !umma_supported(in)) in.cos_in = 0;     // no room for the ring: direct loads
    if (out_stride && k_out > k) *out_stride = k_out;
    return run_search_umma(st, in, B, dq, dp, q_stride, s, ds, di, dkeys, check_queries, cos, seed_ids, seed_stride,
                           seed_n, k_out, gate);
  }
  if (gate) return fail(FMOE_ERR_UNSUPPORTED, "gated search needs the tensor-core path");
  static const bool no_f32mm = getenv("FMOE_NO_F32MM") != nullptr;   // knob: GEMV passes of 4 queries
  if (!st->bf16 && B > 4 && !seed_ids && !no_f32mm)
    return run_search_f32mm(st, B, dq, dp, q_stride, ell, w, k, n_rows, id_offset, s, ds, di, dkeys, check_queries,
                            cos, k_out);
  ScanArgs a{};
  a.st = st->view();
  a.n_rows = n_rows;
  a.ell = ell;
  a.w_sem = w;
  a.k = k;
  a.q_emb = dq;
  a.q_prefix = dp;
  a.q_stride = q_stride;
  a.id_offset = id_offset;
  a.q0 = 0;
  a.nq = int(B < 4 ? B : 4);
  // The TMA bulk-copy ring (scan_tma.cu) measured slower than register
  // streaming in steady state (5.4 vs 6.3 TB/s at ell = 31, K2t);
  // it stays selectable for measurements with FMOE_TMA=1.
  static const bool use_tma = getenv("FMOE_TMA") != nullptr;
  const bool tma = use_tma && scan_tma_supported(a);
  a.grid = tma ? scan_tma_grid(a) : scan_gemv_grid(a);
  const int npass = int((B + 3) / 4);
  char* buf = nullptr;
  unsigned* counters = nullptr;
  unsigned long long* best = nullptr;
  fmoe_status cs = stream_scratch(st, s, size_t(B) * a.grid * k * 8, npass, int(B), &buf, &counters, &best);
  if (cs != FMOE_OK) return cs;
  a.best = best;
  a.cand = reinterpret_cast<uint64_t*>(buf);
  a.out_score = ds;
  a.out_id = di;
  a.out_keys = dkeys;
  a.check_valid = check_queries ? 1 : 0;
  a.trace = trace_buffer();
  a.out_cos = cos.out;
  a.sem_cos = cos.in;
  a.cos_stride = cos.stride;
  a.excl = cos.excl;
  for (int p = 0; p < npass; ++p) {
    a.q0 = 4 * p;
    a.nq = int(B - a.q0 < 4 ? B - a.q0 : 4);
    a.counter = counters + p;
    cudaError_t e = tma ? launch_scan_tma(a, s) : launch_scan_gemv(a, s);
    if (e != cudaSuccess) return cuda_fail(e, "scan launch");
  }
  return FMOE_OK;
}

fmoe_status search_common(const fmoe_store* st, int64_t B, const float* q_emb, const float* q_prefix, int32_t ell,
                          float w, int32_t k, float* out_score, int64_t* out_id, void* stream,
                          float* out_cos = nullptr, int64_t cos_stride = 0) {
  if (!st) return fail(FMOE_ERR_INVALID_ARG, "null store");
  if (B < 0) return fail(FMOE_ERR_INVALID_ARG, "B < 0");
  if (k < 1 || k > FMOE_MAX_K) return fail(FMOE_ERR_INVALID_ARG, "k must be in [1, 64]");
  if (!out_score && !out_id) return fail(FMOE_ERR_INVALID_ARG, "no output");
  const bool sem = w != 0.f, traj = w != 1.f;
  if (sem && !q_emb) return fail(FMOE_ERR_INVALID_ARG, "null q_emb");
  if (traj && (!q_prefix || ell < 1 || ell > st->cfg.L)) return fail(FMOE_ERR_INVALID_ARG, "need q_prefix and 1 <= ell <= L");
  if (!(w >= 0.f && w <= 1.f)) return fail(FMOE_ERR_INVALID_ARG, "w_sem");
  if (B == 0) return FMOE_OK;
  if (sharded(st)) return sharded_search(st, B, q_emb, q_prefix, ell, w, k, out_score, out_id, stream, out_cos, cos_stride);
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device);
  const int E = st->cfg.E, D = st->cfg.D;
  const float* dq = sem ? S.in(q_emb, size_t(B) * D) : nullptr;
  const float* dp = traj ? S.in(q_prefix, size_t(B) * ell * E) : nullptr;
  float* ds = S.out(out_score, size_t(B) * k);
  int64_t* di = S.out(out_id, size_t(B) * k);
  CosArgs cos;
  cos.out = out_cos ? S.out(out_cos, size_t(B) * cos_stride) : nullptr;
  cos.stride = cos_stride;
  fmoe_status r = S.check();
  if (r == FMOE_OK)
    r = run_search(st, B, dq, dp, int64_t(ell) * E, traj ? ell : 0, w, k, st->n, uint32_t(st->cfg.id_offset), s, ds,
                   di, nullptr, true, cos);
  return S.finish(r);
}

}  // namespace

extern "C" {

const char* fmoe_status_string(fmoe_status s) {
  switch (s) {
    case FMOE_OK: return "ok";
    case FMOE_ERR_INVALID_ARG: return "invalid argument";
    case FMOE_ERR_SHAPE: return "unsupported shape";
    case FMOE_ERR_OOM: return "out of device memory";
    case FMOE_ERR_CUDA: return "CUDA error";
    case FMOE_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

const char* fmoe_last_error(void) { return g_err.c_str(); }

int64_t fmoe_kernel_launch_count(void) { return fmoe::launch_count(); }

int32_t fmoe_set_host_sync(int32_t enable) { return g_host_sync.exchange(enable != 0 ? 1 : 0); }

fmoe_status fmoe_store_create(const fmoe_store_config* cfg, int device, fmoe_store** out) {
  if (!out) return fail(FMOE_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  fmoe_status cs = check_cfg(cfg);
  if (cs != FMOE_OK) return cs;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return fail(FMOE_ERR_INVALID_ARG, "no such CUDA device");
  }
  DeviceGuard g(device);
  scratch_pool(device);
  fmoe_store* st = new fmoe_store();
  st->cfg = *cfg;
  st->device = device;
  st->bf16 = cfg->dtype == FMOE_BF16;
  st->esz = st->bf16 ? 2 : 4;
  const int per16 = 16 / st->esz;
  st->Dp = round_up(cfg->D, per16);
  st->Ep = round_up(cfg->E, per16);
  const size_t cap = size_t(cfg->capacity);
  cudaError_t e;
  if ((e = cudaMalloc(&st->emb, cap * st->Dp * st->esz)) != cudaSuccess ||
      (e = cudaMalloc(&st->r_e, cap * 4)) != cudaSuccess ||
      (e = cudaMalloc(&st->maps, cap * size_t(cfg->L) * st->Ep * st->esz)) != cudaSuccess ||
      (e = cudaMalloc(&st->psq, cap * size_t(cfg->L) * 4)) != cudaSuccess) {
    fmoe_store_destroy(st);
    return cuda_fail(e, "cudaMalloc store tiles");
  }
  *out = st;
  return FMOE_OK;
}

void fmoe_store_destroy(fmoe_store* st) {
  if (!st) return;
  DeviceGuard g(st->device);
  // Scratch is stream-ordered: freed on the stream that used it (no device-wide
  // synchronisation; the caller guarantees no other work on the store is
  // pending, the usual rule for freeing memory).  cudaFree of the tiles waits
  // for the device only as the runtime itself requires.
  if (st->dist) {
    st->dist->comm.destroy();
    delete st->dist;
    st->dist = nullptr;
  }
  for (auto& kv : st->scratch) {
    cudaFreeAsync(kv.second.buf, kv.first);
    cudaFreeAsync(kv.second.counters, kv.first);
    cudaFreeAsync(kv.second.best, kv.first);
    cudaStreamSynchronize(kv.first);
  }
  cudaGetLastError();
  cudaFree(st->excl);
  cudaFree(st->emb);
  cudaFree(st->r_e);
  cudaFree(st->maps);
  cudaFree(st->psq);
  delete st;
}

fmoe_status fmoe_store_size(const fmoe_store* st, int64_t* out_n) {
  if (!st || !out_n) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  *out_n = st->dist ? st->dist->n_total : st->n;
  return FMOE_OK;
}

fmoe_status fmoe_store_get_config(const fmoe_store* st, fmoe_store_config* out_cfg) {
  if (!st || !out_cfg) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  *out_cfg = st->cfg;
  return FMOE_OK;
}

fmoe_status fmoe_store_insert(fmoe_store* st, int64_t B, const float* emb, const float* maps, int64_t* out_slot,
                              int64_t* out_replaced, void* stream) {
  return fmoe_store_insert_cos(st, B, emb, maps, nullptr, 0, out_slot, out_replaced, stream);
}

fmoe_status fmoe_store_insert_cos(fmoe_store* st, int64_t B, const float* emb, const float* maps,
                                  const float* sem_cos, int64_t cos_stride, int64_t* out_slot,
                                  int64_t* out_replaced, void* stream) {
  if (!st) return fail(FMOE_ERR_INVALID_ARG, "null store");
  if (sem_cos && cos_stride < st->n) return fail(FMOE_ERR_INVALID_ARG, "cos_stride < store size");
  if (B < 0 || B > (int64_t(1) << 30)) return fail(FMOE_ERR_INVALID_ARG, "B");
  if (B == 0) return FMOE_OK;
  if (!emb || !maps) return fail(FMOE_ERR_INVALID_ARG, "null emb/maps");
  if (sharded(st)) return sharded_insert(st, B, emb, maps, sem_cos, cos_stride, out_slot, out_replaced, stream);
  const int64_t cap = st->cfg.capacity, n0 = st->n;
  const int64_t a = B < cap - n0 ? B : cap - n0;   // appended rows
  const int64_t nrep = B - a;                        // rows needing a victim
  const int L = st->cfg.L, E = st->cfg.E, D = st->cfg.D;
  fmoe_status xs = ensure_excl(st, nrep);
  if (xs != FMOE_OK) return xs;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device);
  const float* de = S.in(emb, size_t(B) * D);
  const float* dm = S.in(maps, size_t(B) * L * E);
  const float* dcos = sem_cos && nrep > 0 ? S.in(sem_cos, size_t(B) * cos_stride) : nullptr;
  int64_t* dslot = S.out(out_slot, size_t(B));
  int64_t* drep = S.out(out_replaced, size_t(B));
  int64_t* slots_all = nrep > 0 ? static_cast<int64_t*>(S.scratch(size_t(B) * 8)) : nullptr;
  fmoe_status r = S.check();
  const uint32_t off = uint32_t(st->cfg.id_offset);
  if (r == FMOE_OK && nrep > 0) {
    // Row j (batch order) takes its best candidate not claimed by rows < j.
    // Rows go in sub-batches of <= 64 (the candidate lists' length); every
    // RDY scan is against the contexts present before the call (rows [0, n0),
    // P:552-553 computes one RDY matrix) and a later sub-batch's scan skips
    // the slots earlier sub-batches claimed (a device bitmap), so the result
    // is the sequential rule of Reading R8 for any batch size.  Within a
    // sub-batch kk = min(rows, n0) candidates per row always suffice; a first
    // pass keeps kRdyFirst, and only when some row finds all of them claimed
    // does a second, gated pass (device flag, no host sync) rescan with kk.
    const float w = float(st->cfg.d) / float(L);
    const int64_t nsub_rows = FMOE_MAX_K;
    for (int64_t sb = 0; sb < nrep && r == FMOE_OK; sb += nsub_rows) {
      const int64_t nb = nrep - sb < nsub_rows ? nrep - sb : nsub_rows;
      const int kk = int(nb < n0 ? nb : n0);
      const int k1 = kk < kRdyFirst ? kk : kRdyFirst;
      UmmaPlanIn p1{}, p2{};
      const bool two = k1 < kk && umma_plan(st, nb, k1, L, w, n0, 0u, &p1) && umma_plan(st, nb, kk, L, w, n0, 0u, &p2);
      uint64_t* keys = static_cast<uint64_t*>(S.scratch(size_t(nb) * (kk > 0 ? kk : 1) * 8));
      uint64_t* keys1 = two ? static_cast<uint64_t*>(S.scratch(size_t(nb) * k1 * 8)) : nullptr;
      int* need = two ? static_cast<int*>(S.scratch(sizeof(int))) : nullptr;
      r = S.check();
      // RDY_{x,y} = d/L sem + (L-d)/L traj over full maps, against
      // the contexts present before this call: rows [0, n0).
      CosArgs cos;
      cos.in = dcos ? dcos + (a + sb) * cos_stride : nullptr;     // cos(emb_x, sem_y) from the semantic search
      cos.stride = cos_stride;
      cos.excl = sb > 0 ? st->excl : nullptr;
      const float* qe = de + (a + sb) * D;
      const float* qm = dm + (a + sb) * int64_t(L) * E;
      const int x0 = int(a + sb), mark = sb == 0 ? int(a) : 0;
      if (r == FMOE_OK && two) {
        r = run_search(st, nb, qe, qm, int64_t(L) * E, L, w, k1, n0, 0u, s, nullptr, nullptr, keys1, false, cos);
        if (r == FMOE_OK) {
          cudaError_t e = launch_resolve(int(nb), k1, keys1, off, slots_all, x0, n0, dslot, drep, s, need, kk,
                                         nullptr, mark);
          if (e != cudaSuccess) r = cuda_fail(e, "resolve launch");
        }
      }
      if (r == FMOE_OK && kk > 0)
        r = run_search(st, nb, qe, qm, int64_t(L) * E, L, w, kk, n0, 0u, s, nullptr, nullptr, keys, false, cos,
                       nullptr, 0, 0, 0, nullptr, need);
      if (r == FMOE_OK) {
        cudaError_t e = launch_resolve(int(nb), kk, keys, off, slots_all, x0, n0, dslot, drep, s, nullptr, 0, need,
                                       mark);
        if (e == cudaSuccess && sb + nb < nrep)       // claimed: no candidate of later sub-batches
          e = launch_excl(st->excl, slots_all + x0, int(nb), 0, cap, 1, s);
        if (e != cudaSuccess) r = cuda_fail(e, "resolve launch");
      }
    }
    if (r == FMOE_OK && nrep > nsub_rows) {         // leave the bitmap zero for the next call
      cudaError_t e = launch_excl(st->excl, slots_all + a, int(nrep - nsub_rows), 0, cap, 0, s);
      if (e != cudaSuccess) r = cuda_fail(e, "bitmap reset launch");
    }
  } else if (r == FMOE_OK) {
    cudaError_t e = launch_append_ids(int(a), n0, off, dslot, drep, s);
    if (e != cudaSuccess) r = cuda_fail(e, "append ids launch");
  }
  if (r == FMOE_OK) {
    WriteArgs w{};
    w.emb = st->emb; w.r_e = st->r_e; w.maps = st->maps; w.psq = st->psq;
    w.cap = cap; w.L = L; w.E = E; w.D = D; w.Dp = st->Dp; w.Ep = st->Ep; w.bf16 = st->bf16;
    w.in_emb = de; w.in_maps = dm;
    w.B = int(nrep > 0 ? B : a);
    w.slots = slots_all;
    w.first_slot = n0;
    w.slot_offset = 0;
    w.slot_limit = cap;
    cudaError_t e = launch_write_rows(w, s);
    if (e != cudaSuccess) r = cuda_fail(e, "write launch");
  }
  // (the size counts enqueued inserts: calls are asynchronous; a failed call
  // leaves the store and its generation unchanged)
  if (r == FMOE_OK) {
    st->n = n0 + a;
    ++st->gen;
  }
  return S.finish(r);
}

fmoe_status fmoe_store_write(fmoe_store* st, int64_t B, const float* emb, const float* maps, const int64_t* slot,
                             void* stream) {
  if (!st) return fail(FMOE_ERR_INVALID_ARG, "null store");
  if (B < 0) return fail(FMOE_ERR_INVALID_ARG, "B");
  if (B == 0) return FMOE_OK;
  if (!emb || !maps || !slot) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  const int L = st->cfg.L, E = st->cfg.E, D = st->cfg.D;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device);
  const float* de = S.in(emb, size_t(B) * D);
  const float* dm = S.in(maps, size_t(B) * L * E);
  const int64_t* dsl = S.in(slot, size_t(B));
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    WriteArgs w{};
    w.emb = st->emb; w.r_e = st->r_e; w.maps = st->maps; w.psq = st->psq;
    w.cap = st->cfg.capacity; w.L = L; w.E = E; w.D = D; w.Dp = st->Dp; w.Ep = st->Ep; w.bf16 = st->bf16;
    w.in_emb = de; w.in_maps = dm;
    w.B = int(B);
    w.slots = dsl;
    w.slot_offset = st->cfg.id_offset;
    w.slot_limit = st->n;
    cudaError_t e = launch_write_rows(w, s);
    if (e != cudaSuccess) r = cuda_fail(e, "write launch");
  }
  if (r == FMOE_OK) ++st->gen;
  return S.finish(r);
}

}  // extern "C"

// Two implementations behind one API:
//  * incremental (B below the tensor-core threshold, or an f32 store): the
//    running per-row dot products acc [B][cap] (traj_session.cu);
//  * batched (bf16 store, B >= FMOE_UMMA_MIN_B): the session keeps the query
//    prefixes [B][L][E] and each step runs the tcgen05 scan over the whole
//    prefix, seeded with the previous step's top-k ids -- k distinct rows
//    whose scores at the new prefix bound the k-th best key from below, so
//    the scan's per-query admission threshold starts near its final value
//    instead of at -inf (the fused top-k otherwise dominates short prefixes).
constexpr int kSessionSeeds = 32;

struct fmoe_traj_session {
  const fmoe_store* st;
  int64_t B;
  bool batched = false;
  float* acc = nullptr;      // [B][cap] (incremental)
  double* qn = nullptr;      // [2][B]   (incremental)
  float* prefix = nullptr;   // [B][L][E] (batched)
  int64_t* prev = nullptr;   // [B][kk] the last step's top-kk ids, kk = max(k, 32) (batched)
  float* sctmp = nullptr;    // [B][kk] its scores
  int prev_k = 0;
  int layer = 0;
  int qslot = 0;             // qn slot holding the running norm (incremental); the next
                             // step writes the other slot, so a launch never reads and
                             // writes the same word
  unsigned* abort = nullptr; // device word: a sweep abandoned on a layer_ready timeout
                             // poisons the session until reset (incremental)
  bool clear_abort = false;  // reset() asked: zero `abort` on the next call's stream
  uint64_t gen = 0;
  void* sweep_scratch = nullptr;   // [L] u64 best keys + [L] u32 tickets (fmoe_traj_session_sweep)
};

extern "C" {

fmoe_status fmoe_traj_session_create(const fmoe_store* st, int64_t B, fmoe_traj_session** out) {
  if (!st || !out) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  if (B < 1 || B > FMOE_MAX_K) return fail(FMOE_ERR_INVALID_ARG, "1 <= B <= 64");
  *out = nullptr;
  DeviceGuard g(st->device);
  fmoe_traj_session* s = new fmoe_traj_session();
  s->st = st;
  s->B = B;
  s->gen = st->gen;
  s->batched = st->bf16 && B >= umma_min_batch();
  cudaError_t e = cudaSuccess;
  if (s->batched ? ((e = cudaMalloc(&s->prefix, size_t(B) * st->cfg.L * st->cfg.E * 4)) != cudaSuccess ||
                    (e = cudaMalloc(&s->prev, size_t(B) * FMOE_MAX_K * 8)) != cudaSuccess ||
                    (e = cudaMalloc(&s->sctmp, size_t(B) * FMOE_MAX_K * 4)) != cudaSuccess)
                 : ((e = cudaMalloc(&s->acc, size_t(B) * st->cfg.capacity * 4)) != cudaSuccess ||
                    (e = cudaMalloc(&s->qn, size_t(2) * B * 8)) != cudaSuccess ||
                    (e = cudaMalloc(&s->abort, 4)) != cudaSuccess ||
                    (e = cudaMemset(s->abort, 0, 4)) != cudaSuccess)) {
    fmoe_traj_session_destroy(s);
    return cuda_fail(e, "session memory");
  }
  *out = s;
  return FMOE_OK;
}

void fmoe_traj_session_destroy(fmoe_traj_session* s) {
  if (!s) return;
  DeviceGuard g(s->st->device);
  // (the caller guarantees no step of the session is pending, as for any free)
  cudaFree(s->abort);
  cudaFree(s->acc);
  cudaFree(s->qn);
  cudaFree(s->prefix);
  cudaFree(s->prev);
  cudaFree(s->sctmp);
  cudaFree(s->sweep_scratch);
  delete s;
}

fmoe_status fmoe_traj_session_reset(fmoe_traj_session* s) {
  if (!s) return fail(FMOE_ERR_INVALID_ARG, "null session");
  s->layer = 0;
  s->prev_k = 0;
  s->qslot = 0;
  s->clear_abort = s->abort != nullptr;
  s->gen = s->st->gen;
  return FMOE_OK;
}

fmoe_status fmoe_traj_session_abandoned(const fmoe_traj_session* s, int32_t* out_abandoned) {
  if (!s || !out_abandoned) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  *out_abandoned = 0;
  if (!s->abort || s->clear_abort) return FMOE_OK;
  DeviceGuard g(s->st->device);
  unsigned v = 0;
  cudaError_t e = cudaMemcpy(&v, s->abort, 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "session status read");
  *out_abandoned = v != 0 ? 1 : 0;
  return FMOE_OK;
}

}  // extern "C"

namespace {
// Optional selection fused into a session step (fmoe_traj_session_step_select).
struct StepSelect {
  float delta = -1.f;
  int lb = 0, le = 0;                 // layers [lb, le); le == lb: none
  uint64_t* mask = nullptr;
  int32_t* count = nullptr;
};

fmoe_status session_step(fmoe_traj_session* ss, const float* q_layer, int32_t k, float* out_score, int64_t* out_id,
                         const StepSelect& sel, void* stream) {
  if (!ss || !q_layer) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  const fmoe_store* st = ss->st;
  if (ss->gen != st->gen) return fail(FMOE_ERR_INVALID_ARG, "store changed since the session was reset");
  if (ss->layer >= st->cfg.L) return fail(FMOE_ERR_INVALID_ARG, "all L layers consumed; reset the session");
  if (k < 1 || k > FMOE_MAX_K) return fail(FMOE_ERR_INVALID_ARG, "k must be in [1, 64]");
  if (!out_score && !out_id) return fail(FMOE_ERR_INVALID_ARG, "no output");
  const int64_t B = ss->B;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device);
  const int T = sel.le - sel.lb;
  const float* dq = S.in(q_layer, size_t(B) * st->cfg.E);
  float* ds = S.out(out_score, size_t(B) * k);
  int64_t* di = S.out(out_id, size_t(B) * k);
  uint64_t* dm = T > 0 ? S.out(sel.mask, size_t(B) * T) : nullptr;
  int32_t* dc = T > 0 ? S.out(sel.count, size_t(B) * T) : nullptr;
  fmoe_status r = S.check();
  // selection by the select kernel on (ids, scores) with row stride `stride`
  auto select_after = [&](const int64_t* ids, const float* sc, int stride) {
    if (r != FMOE_OK || T <= 0) return;
    cudaError_t e = launch_select(st->view(), int(B), ids, sc, sel.delta, st->cfg.K, sel.lb, sel.le,
                                  st->cfg.id_offset, st->n, dm, dc, s, stride);
    if (e != cudaSuccess) r = cuda_fail(e, "select launch");
  };
  if (r == FMOE_OK && st->n == 0) {
    cudaError_t e = launch_merge_keys(int(B), 0, k, nullptr, k, nullptr, ds, di, nullptr, s);
    if (e != cudaSuccess) r = cuda_fail(e, "merge launch");
    select_after(di, ds, k);
  } else if (r == FMOE_OK && ss->batched) {
    const int L = st->cfg.L, E = st->cfg.E, ell = ss->layer + 1;
    cudaError_t e = cudaMemcpy2DAsync(ss->prefix + int64_t(ss->layer) * E, size_t(L) * E * 4, dq, size_t(E) * 4,
                                      size_t(E) * 4, size_t(B), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) r = cuda_fail(e, "session prefix copy");
    // The session keeps kk = max(k, 32) rows per query from the merge: the
    // exact top-k followed by the next best keys of the per-CTA lists --
    // distinct rows with high scores, which seed the next step (their k-th
    // best score at the next prefix is a tight lower bound on its k-th best).
    // The caller gets the first k.  The seeds are read by the query
    // preparation kernel before this step's merge rewrites prev (stream order).
    int kk = k > kSessionSeeds ? k : kSessionSeeds;
    if (r == FMOE_OK) {
      const bool seeded = ss->prev_k >= k;
      r = run_search(st, B, nullptr, ss->prefix, int64_t(L) * E, ell, 0.f, k, st->n, uint32_t(st->cfg.id_offset), s,
                     ss->sctmp, ss->prev, nullptr, true, CosArgs(), seeded ? ss->prev : nullptr, ss->prev_k,
                     ss->prev_k, kk, &kk);
    }
    if (r == FMOE_OK && ds) {
      e = cudaMemcpy2DAsync(ds, size_t(k) * 4, ss->sctmp, size_t(kk) * 4, size_t(k) * 4, size_t(B),
                            cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) r = cuda_fail(e, "session score copy");
    }
    if (r == FMOE_OK && di) {
      e = cudaMemcpy2DAsync(di, size_t(k) * 8, ss->prev, size_t(kk) * 8, size_t(k) * 8, size_t(B),
                            cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) r = cuda_fail(e, "session id copy");
    }
    select_after(ss->prev, ss->sctmp, kk);
    if (r == FMOE_OK) {
      ss->prev_k = kk;      // == k when the search ran without extra keys
      ++ss->layer;
    }
  } else if (r == FMOE_OK) {
    ScanArgs a{};
    a.st = st->view();
    a.n_rows = st->n;
    a.ell = ss->layer + 1;
    a.k = k;
    a.id_offset = uint32_t(st->cfg.id_offset);
    a.nq = int(B < 4 ? B : 4);
    a.grid = traj_session_grid(a);
    const int npass = int((B + 3) / 4);
    char* buf = nullptr;
    unsigned* counters = nullptr;
    unsigned long long* best = nullptr;
    r = stream_scratch(st, s, size_t(B) * a.grid * k * 8, npass, int(B), &buf, &counters, &best);
    if (r == FMOE_OK) {
      a.cand = reinterpret_cast<uint64_t*>(buf);
      a.best = best;
      a.out_score = ds;
      a.out_id = di;
      a.check_valid = 1;
      a.trace = trace_buffer();
      if (ss->clear_abort) {
        cudaError_t e = cudaMemsetAsync(ss->abort, 0, 4, s);
        if (e != cudaSuccess) r = cuda_fail(e, "session status reset");
        else ss->clear_abort = false;
      }
      SessionArgs sa{};
      sa.q_layer = dq;
      sa.layer = ss->layer;
      sa.acc = ss->acc;
      sa.abort = ss->abort;
      sa.qn_prev = ss->qn + ss->qslot * B;
      sa.qn_next = ss->qn + (ss->qslot ^ 1) * B;
      // the selection runs in each pass's last block, on that pass's queries
      sa.sel_delta = sel.delta;
      sa.sel_K = st->cfg.K;
      sa.sel_lb = sel.lb;
      sa.sel_T = T > 0 ? T : 0;
      sa.sel_mask = dm;
      sa.sel_count = dc;
      for (int p = 0; p < npass && r == FMOE_OK; ++p) {
        a.q0 = 4 * p;
        a.nq = int(B - a.q0 < 4 ? B - a.q0 : 4);
        a.counter = counters + p;
        cudaError_t e = launch_traj_session(a, sa, s);
        if (e != cudaSuccess) r = cuda_fail(e, "session launch");
      }
      if (r == FMOE_OK) {
        ++ss->layer;
        ss->qslot ^= 1;
      }
    }
  }
  return S.finish(r);
}
fmoe_status sharded_session_step(fmoe_traj_session* ss, const float* q_layer, int32_t k, float* out_score,
                                 int64_t* out_id, const StepSelect& sel, void* stream);
fmoe_status sharded_sweep(fmoe_traj_session* ss, const float* q_layers, int32_t n_steps, float* out_score,
                          int64_t* out_id, float delta, int32_t sel_d, uint64_t* out_mask, int32_t* out_count,
                          void* stream);
}  // namespace

extern "C" {

fmoe_status fmoe_traj_session_step(fmoe_traj_session* ss, const float* q_layer, int32_t k, float* out_score,
                                   int64_t* out_id, void* stream) {
  if (ss && sharded(ss->st) && q_layer && k >= 1 && k <= FMOE_MAX_K && (out_score || out_id))
    return sharded_session_step(ss, q_layer, k, out_score, out_id, StepSelect(), stream);
  return session_step(ss, q_layer, k, out_score, out_id, StepSelect(), stream);
}

fmoe_status fmoe_traj_session_step_select(fmoe_traj_session* ss, const float* q_layer, int32_t k, float* out_score,
                                          int64_t* out_id, float delta, int32_t layer_begin, int32_t layer_end,
                                          uint64_t* out_mask, int32_t* out_count, void* stream) {
  if (!ss) return fail(FMOE_ERR_INVALID_ARG, "null session");
  const int L = ss->st->cfg.L;
  if (layer_begin < 0 || layer_end > L || layer_begin >= layer_end)
    return fail(FMOE_ERR_INVALID_ARG, "0 <= layer_begin < layer_end <= L");
  if (!(delta <= 1.f)) return fail(FMOE_ERR_INVALID_ARG, "delta must be <= 1 (negative: dynamic)");
  if (!out_score || !out_id || !out_mask || !out_count) return fail(FMOE_ERR_INVALID_ARG, "null output");
  StepSelect sel;
  sel.delta = delta;
  sel.lb = layer_begin;
  sel.le = layer_end;
  sel.mask = out_mask;
  sel.count = out_count;
  if (sharded(ss->st) && q_layer && k >= 1 && k <= FMOE_MAX_K)
    return sharded_session_step(ss, q_layer, k, out_score, out_id, sel, stream);
  return session_step(ss, q_layer, k, out_score, out_id, sel, stream);
}

fmoe_status fmoe_search_blend_cos(const fmoe_store* st, int64_t B, const float* sem_cos, int64_t cos_stride,
                                  const float* q_prefix, int32_t ell, float w_sem, int32_t k, float* out_score,
                                  int64_t* out_id, void* stream) {
  if (!st) return fail(FMOE_ERR_INVALID_ARG, "null store");
  if (B < 0) return fail(FMOE_ERR_INVALID_ARG, "B < 0");
  if (k < 1 || k > FMOE_MAX_K) return fail(FMOE_ERR_INVALID_ARG, "k must be in [1, 64]");
  if (!out_score && !out_id) return fail(FMOE_ERR_INVALID_ARG, "no output");
  if (!q_prefix || ell < 1 || ell > st->cfg.L) return fail(FMOE_ERR_INVALID_ARG, "need q_prefix and 1 <= ell <= L");
  const float w = w_sem < 0.f ? float(st->cfg.d) / float(st->cfg.L) : w_sem;
  if (!(w >= 0.f && w < 1.f)) return fail(FMOE_ERR_INVALID_ARG, "0 <= w_sem < 1 (w = 1: the semantic search itself)");
  if (B > 0 && (!sem_cos || cos_stride < st->n)) return fail(FMOE_ERR_INVALID_ARG, "sem_cos [B][cos_stride >= n]");
  if (B == 0) return FMOE_OK;
  if (sharded(st)) return sharded_blend_cos(st, B, sem_cos, cos_stride, q_prefix, ell, w_sem, k, out_score, out_id, stream);
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device);
  const int E = st->cfg.E;
  const float* dp = S.in(q_prefix, size_t(B) * ell * E);
  const float* dc = S.in(sem_cos, size_t(B) * cos_stride);
  float* ds = S.out(out_score, size_t(B) * k);
  int64_t* di = S.out(out_id, size_t(B) * k);
  CosArgs cos;
  cos.in = dc;
  cos.stride = cos_stride;
  fmoe_status r = S.check();
  if (r == FMOE_OK)
    r = run_search(st, B, nullptr, dp, int64_t(ell) * E, ell, w, k, st->n, uint32_t(st->cfg.id_offset), s, ds, di,
                   nullptr, true, cos);
  return S.finish(r);
}

fmoe_status fmoe_traj_session_sweep(fmoe_traj_session* ss, const float* q_layers, int32_t n_steps,
                                    float* out_score, int64_t* out_id, float delta, int32_t sel_d,
                                    uint64_t* out_mask, int32_t* out_count, const uint32_t* layer_ready,
                                    uint32_t* guidance_ready, void* stream) {
  if (!ss || !q_layers || !out_score || !out_id) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  const fmoe_store* st = ss->st;
  const int L = st->cfg.L, E = st->cfg.E;
  if (n_steps < 1 || ss->layer + n_steps > L) return fail(FMOE_ERR_INVALID_ARG, "1 <= n_steps <= L - layer");
  if (ss->gen != st->gen) return fail(FMOE_ERR_INVALID_ARG, "store changed since the session was reset");
  if (!(delta <= 1.f)) return fail(FMOE_ERR_INVALID_ARG, "delta must be <= 1 (negative: dynamic)");
  if (out_mask && (!out_count || sel_d < 0)) return fail(FMOE_ERR_INVALID_ARG, "selection needs out_count, sel_d >= 0");
  if (sharded(st)) {
    if (layer_ready || guidance_ready) return fail(FMOE_ERR_UNSUPPORTED, "ready flags on a sharded store");
    return sharded_sweep(ss, q_layers, n_steps, out_score, out_id, delta, sel_d, out_mask, out_count, stream);
  }
  const int esz = st->bf16 ? 2 : 4;
  int grid = 1;
  // without ready flags the row-major sweep takes any store size; with them the
  // step-major kernel keeps its rows in registers (n <= 8 * 4 * SMs * 256)
  const bool fused = ss->B == 1 && !ss->batched && st->view().Ep * esz == 16 && st->n > 0 && n_steps <= 64 &&
                     ((!layer_ready && !guidance_ready) || traj_sweep_rows(st->n, &grid) != 0);
  if (!fused) {
    // same results through one step call per layer; device flags cannot gate host-issued steps
    if (layer_ready || guidance_ready)
      return fail(FMOE_ERR_UNSUPPORTED, "ready flags need the fused sweep (B = 1, 16-byte slab rows, n <= 8 * 4 * SMs * 256)");
    const int64_t B = ss->B;
    for (int s2 = 0; s2 < n_steps; ++s2) {
      const int layer = ss->layer, tgt = layer + sel_d;
      StepSelect sel;
      if (out_mask && tgt < L) {
        sel.delta = delta; sel.lb = tgt; sel.le = tgt + 1;
        sel.mask = out_mask + int64_t(s2) * B; sel.count = out_count + int64_t(s2) * B;
      }
      fmoe_status r = session_step(ss, q_layers + int64_t(s2) * B * E, 1, out_score + int64_t(s2) * B,
                                   out_id + int64_t(s2) * B, sel, stream);
      if (r != FMOE_OK) return r;
      if (out_mask && tgt >= L) {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const bool dev = ptr_kind(out_mask, st->device) == 1;
        if (dev) {
          DeviceGuard g(st->device);
          cudaMemsetAsync(out_mask + int64_t(s2) * B, 0, size_t(B) * 8, s);
          cudaMemsetAsync(out_count + int64_t(s2) * B, 0, size_t(B) * 4, s);
        } else {
          memset(out_mask + int64_t(s2) * B, 0, size_t(B) * 8);
          memset(out_count + int64_t(s2) * B, 0, size_t(B) * 4);
        }
      }
    }
    return FMOE_OK;
  }
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((layer_ready && ptr_kind(layer_ready, st->device) != 1) ||
      (guidance_ready && ptr_kind(guidance_ready, st->device) != 1))
    return fail(FMOE_ERR_INVALID_ARG, "ready flags must be device memory of the store's device");
  if (!ss->sweep_scratch) {
    cudaError_t e = cudaMalloc(&ss->sweep_scratch, size_t(L) * 12);
    if (e != cudaSuccess) return cuda_fail(e, "sweep scratch");
  }
  Staging S(s, st->device);
  const float* dq = S.in(q_layers, size_t(n_steps) * E);
  float* ds = S.out(out_score, size_t(n_steps));
  int64_t* di = S.out(out_id, size_t(n_steps));
  uint64_t* dm = out_mask ? S.out(out_mask, size_t(n_steps)) : nullptr;
  int32_t* dc = out_mask ? S.out(out_count, size_t(n_steps)) : nullptr;
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    cudaError_t e = cudaMemsetAsync(ss->sweep_scratch, 0, size_t(L) * 12, s);
    if (e == cudaSuccess && ss->clear_abort) {
      e = cudaMemsetAsync(ss->abort, 0, 4, s);
      if (e == cudaSuccess) ss->clear_abort = false;
    }
    SweepArgs a{};
    a.st = st->view();
    a.n_rows = st->n;
    a.id_offset = uint32_t(st->cfg.id_offset);
    a.q_layers = dq;
    a.layer0 = ss->layer;
    a.n_steps = n_steps;
    a.acc = ss->acc;
    // B = 1: slot q holds the norm; input and output never alias (ADVICE r1:
    // a block starting after block 0 exits must still read the input norm)
    a.qn_in = ss->qn + ss->qslot;
    a.qn_out = ss->qn + (ss->qslot ^ 1);
    a.abort = ss->abort;
    a.best = reinterpret_cast<unsigned long long*>(ss->sweep_scratch);
    a.tickets = reinterpret_cast<unsigned*>(static_cast<char*>(ss->sweep_scratch) + size_t(L) * 8);
    a.out_score = ds;
    a.out_id = di;
    a.sel_delta = delta;
    a.sel_K = st->cfg.K;
    a.sel_d = sel_d;
    a.sel_mask = dm;
    a.sel_count = dc;
    a.layer_ready = layer_ready;
    a.guidance_ready = guidance_ready;
    a.timeout_ns = 10ull * 1000 * 1000 * 1000;
    if (e == cudaSuccess) e = launch_traj_sweep(a, s);
    if (e != cudaSuccess) r = cuda_fail(e, "sweep launch");
    else {
      ss->layer += n_steps;
      ss->qslot ^= 1;
    }
  }
  return S.finish(r);
}

fmoe_status fmoe_resolve_victims(int64_t B, int32_t k, const int64_t* ids, int64_t* out_victim, int device,
                                 void* stream) {
  if (B < 0 || k < 1 || k > FMOE_MAX_K || B > FMOE_MAX_K) return fail(FMOE_ERR_INVALID_ARG, "sizes");
  if (!ids || !out_victim) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  if (B == 0) return FMOE_OK;
  DeviceGuard g(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, device);
  const int64_t* di = S.in(ids, size_t(B) * k);
  int64_t* dv = S.out(out_victim, size_t(B));
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    cudaError_t e = launch_resolve_ids(int(B), k, di, dv, s);
    if (e != cudaSuccess) r = cuda_fail(e, "resolve launch");
  }
  return S.finish(r);
}

fmoe_status fmoe_store_read(const fmoe_store* st, int64_t slot_begin, int64_t count, float* out_emb, float* out_maps,
                            void* stream) {
  if (!st) return fail(FMOE_ERR_INVALID_ARG, "null store");
  if (st->dist) slot_begin -= st->cfg.id_offset;     // sharded: global slots of this rank's shard
  if (slot_begin < 0 || count < 0 || slot_begin + count > st->n) return fail(FMOE_ERR_INVALID_ARG, "slot range");
  if (count == 0) return FMOE_OK;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device);
  float* de = S.out(out_emb, size_t(count) * st->cfg.D);
  float* dm = S.out(out_maps, size_t(count) * st->cfg.L * st->cfg.E);
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    cudaError_t e = launch_read_rows(st->view(), slot_begin, count, de, dm, s);
    if (e != cudaSuccess) r = cuda_fail(e, "read launch");
  }
  return S.finish(r);
}

fmoe_status fmoe_search_semantic(const fmoe_store* st, int64_t B, const float* q_emb, int32_t k, float* out_score,
                                 int64_t* out_id, void* stream) {
  return search_common(st, B, q_emb, nullptr, 0, 1.f, k, out_score, out_id, stream);
}

fmoe_status fmoe_search_semantic_cos(const fmoe_store* st, int64_t B, const float* q_emb, int32_t k, float* out_score,
                                     int64_t* out_id, float* out_cos, int64_t cos_stride, void* stream) {
  if (!st) return fail(FMOE_ERR_INVALID_ARG, "null store");
  if (out_cos && cos_stride < st->n) return fail(FMOE_ERR_INVALID_ARG, "cos_stride < store size");
  return search_common(st, B, q_emb, nullptr, 0, 1.f, k, out_score, out_id, stream, out_cos, cos_stride);
}

fmoe_status fmoe_search_trajectory(const fmoe_store* st, int64_t B, const float* q_prefix, int32_t ell, int32_t k,
                                   float* out_score, int64_t* out_id, void* stream) {
  return search_common(st, B, nullptr, q_prefix, ell, 0.f, k, out_score, out_id, stream);
}

fmoe_status fmoe_search_blend(const fmoe_store* st, int64_t B, const float* q_emb, const float* q_prefix, int32_t ell,
                              float w_sem, int32_t k, float* out_score, int64_t* out_id, void* stream) {
  if (!st) return fail(FMOE_ERR_INVALID_ARG, "null store");
  if (w_sem < 0.f) w_sem = float(st->cfg.d) / float(st->cfg.L);
  return search_common(st, B, q_emb, q_prefix, ell, w_sem, k, out_score, out_id, stream);
}

fmoe_status fmoe_select_experts(const fmoe_store* st, int64_t B, const int64_t* map_id, const float* score, float delta,
                                int32_t layer_begin, int32_t layer_end, uint64_t* out_mask, int32_t* out_count,
                                void* stream) {
  if (!st) return fail(FMOE_ERR_INVALID_ARG, "null store");
  if (B < 0 || !map_id || !out_mask || !out_count) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  if (layer_begin < 0 || layer_begin >= layer_end || layer_end > st->cfg.L)
    return fail(FMOE_ERR_INVALID_ARG, "need 0 <= layer_begin < layer_end <= L");
  if (!(delta <= 1.f)) return fail(FMOE_ERR_INVALID_ARG, "delta must be <= 1 (negative = dynamic)");
  if (delta < 0.f && !score) return fail(FMOE_ERR_INVALID_ARG, "dynamic delta needs score");
  if (B == 0) return FMOE_OK;
  if (sharded(st)) return sharded_select(st, B, map_id, score, delta, layer_begin, layer_end, out_mask, out_count, stream);
  const int T = layer_end - layer_begin;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device);
  const int64_t* did = S.in(map_id, size_t(B));
  const float* dsc = delta < 0.f ? S.in(score, size_t(B)) : nullptr;
  uint64_t* dm = S.out(out_mask, size_t(B) * T);
  int32_t* dc = S.out(out_count, size_t(B) * T);
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    cudaError_t e = launch_select(st->view(), int(B), did, dsc, delta, st->cfg.K, layer_begin, layer_end,
                                  st->cfg.id_offset, st->n, dm, dc, s);
    if (e != cudaSuccess) r = cuda_fail(e, "select launch");
  }
  return S.finish(r);
}

fmoe_status fmoe_prefetch_plan(const fmoe_store* st, int64_t B, const int64_t* map_id, const float* score, float delta,
                               int32_t l_now, int32_t layer_begin, int32_t layer_end, int32_t max_jobs,
                               int32_t* out_layer, int32_t* out_expert, double* out_priority, int32_t* out_njobs,
                               void* stream) {
  if (!st || !map_id || !out_layer || !out_expert || !out_priority || !out_njobs)
    return fail(FMOE_ERR_INVALID_ARG, "null argument");
  if (st->dist) return fail(FMOE_ERR_UNSUPPORTED, "prefetch plan on a sharded store");
  if (B < 0 || max_jobs < 1) return fail(FMOE_ERR_INVALID_ARG, "B / max_jobs");
  if (layer_begin < 0 || layer_begin >= layer_end || layer_end > st->cfg.L || l_now >= layer_begin)
    return fail(FMOE_ERR_INVALID_ARG, "need l_now < layer_begin < layer_end <= L");
  if ((layer_end - layer_begin) * st->cfg.E > 2048) return fail(FMOE_ERR_INVALID_ARG, "too many (layer, expert) jobs");
  if (!(delta <= 1.f)) return fail(FMOE_ERR_INVALID_ARG, "delta must be <= 1 (negative = dynamic)");
  if (delta < 0.f && !score) return fail(FMOE_ERR_INVALID_ARG, "dynamic delta needs score");
  if (B == 0) return FMOE_OK;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device);
  const int64_t* did = S.in(map_id, size_t(B));
  const float* dsc = delta < 0.f ? S.in(score, size_t(B)) : nullptr;
  int32_t* dl = S.out(out_layer, size_t(B) * max_jobs);
  int32_t* de = S.out(out_expert, size_t(B) * max_jobs);
  double* dp = S.out(out_priority, size_t(B) * max_jobs);
  int32_t* dn = S.out(out_njobs, size_t(B));
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    cudaError_t e = launch_prefetch_plan(st->view(), int(B), did, dsc, delta, st->cfg.K, l_now, layer_begin,
                                         layer_end, st->cfg.id_offset, st->n, max_jobs, dl, de, dp, dn, s);
    if (e != cudaSuccess) r = cuda_fail(e, "plan launch");
  }
  return S.finish(r);
}

fmoe_status fmoe_prefetch_issue(const fmoe_store* st, int64_t B, const int64_t* map_id, const float* score,
                                float delta, int32_t l_now, int32_t layer_begin, int32_t layer_end, int32_t max_jobs,
                                const void* const* host_expert, void* const* dev_expert, int64_t expert_bytes,
                                uint64_t* resident_mask, const uint32_t* wait_flag, void* copy_stream,
                                int32_t* out_layer, int32_t* out_expert, int32_t* out_njobs) {
  if (!st || !map_id || !host_expert || !dev_expert || expert_bytes < 1)
    return fail(FMOE_ERR_INVALID_ARG, "null argument / expert_bytes");
  if (st->dist) return fail(FMOE_ERR_UNSUPPORTED, "prefetch copies on a sharded store");
  if (B < 0 || max_jobs < 1) return fail(FMOE_ERR_INVALID_ARG, "B / max_jobs");
  if (layer_begin < 0 || layer_begin >= layer_end || layer_end > st->cfg.L || l_now >= layer_begin)
    return fail(FMOE_ERR_INVALID_ARG, "need l_now < layer_begin < layer_end <= L");
  if ((layer_end - layer_begin) * st->cfg.E > 2048) return fail(FMOE_ERR_INVALID_ARG, "too many (layer, expert) jobs");
  if (!(delta <= 1.f)) return fail(FMOE_ERR_INVALID_ARG, "delta must be <= 1 (negative = dynamic)");
  if (delta < 0.f && !score) return fail(FMOE_ERR_INVALID_ARG, "dynamic delta needs score");
  if (B == 0) return FMOE_OK;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(copy_stream);
  if (ptr_kind(map_id, st->device) != 1 || (score && ptr_kind(score, st->device) != 1) ||
      (wait_flag && ptr_kind(wait_flag, st->device) != 1))
    return fail(FMOE_ERR_INVALID_ARG, "map_id / score / wait_flag must be device memory of the store's device");
  // pinned plan buffer, allocated before the stream waits (an allocation may
  // synchronise)
  thread_local int32_t* pin = nullptr;
  thread_local size_t pin_n = 0;
  const size_t need = 2 * size_t(B) * max_jobs + size_t(B);
  if (pin_n < need) {
    if (pin) cudaFreeHost(pin);
    pin = nullptr;
    pin_n = 0;
    cudaError_t ea = cudaMallocHost(&pin, need * 4);
    if (ea != cudaSuccess) return cuda_fail(ea, "pinned plan buffer");
    pin_n = need;
  }
  if (wait_flag) {
    // the guidance is published by a device flag: the copy stream waits on the
    // device (no host polling), then reads the plan
    using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    static WaitFn wait = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        wait = reinterpret_cast<WaitFn>(fn);
    });
    if (!wait) return fail(FMOE_ERR_UNSUPPORTED, "cuStreamWaitValue32 unavailable");
    if (wait(s, reinterpret_cast<CUdeviceptr>(wait_flag), 1u, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return fail(FMOE_ERR_UNSUPPORTED, "stream memory operations unsupported on this device");
  }
  const size_t nj = size_t(B) * max_jobs;
  Staging S(s, st->device, true);
  int32_t* dl = static_cast<int32_t*>(S.scratch(nj * 4));
  int32_t* de = static_cast<int32_t*>(S.scratch(nj * 4));
  double* dp = static_cast<double*>(S.scratch(nj * 8));
  int32_t* dn = static_cast<int32_t*>(S.scratch(size_t(B) * 4));
  fmoe_status r = S.check();
  if (r != FMOE_OK) return S.finish(r);
  cudaError_t e = launch_prefetch_plan(st->view(), int(B), map_id, delta < 0.f ? score : nullptr, delta, st->cfg.K,
                                       l_now, layer_begin, layer_end, st->cfg.id_offset, st->n, max_jobs, dl, de, dp,
                                       dn, s);
  // the plan comes back through PINNED memory: a copy into pageable memory
  // would block inside the runtime (holding its locks) until the device wait
  // on the guidance flag resolves, stalling every other thread's CUDA calls --
  // including the ones that will eventually raise the flag
  int32_t* hl = pin;
  int32_t* he = pin + nj;
  int32_t* hn = pin + 2 * nj;
  if (e == cudaSuccess) e = cudaMemcpyAsync(hl, dl, nj * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(he, de, nj * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hn, dn, size_t(B) * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);           // the plan is on the host
  if (e != cudaSuccess) return S.finish(cuda_fail(e, "prefetch plan"));
  const int E = st->cfg.E;
  // plan order per query (priority descending); queries in batch order
  for (int64_t x = 0; x < B && r == FMOE_OK; ++x) {
    int issued = 0;
    for (int j = 0; j < hn[x] && j < max_jobs; ++j) {
      const int t = hl[x * max_jobs + j], ex = he[x * max_jobs + j];
      if (t < 0 || ex < 0) continue;
      const uint64_t bit = uint64_t(1) << ex;
      if (resident_mask && (resident_mask[t] & bit)) continue;   // already resident (or copied for an earlier query)
      const size_t idx = size_t(t) * E + ex;
      e = cudaMemcpyAsync(dev_expert[idx], host_expert[idx], size_t(expert_bytes), cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) { r = cuda_fail(e, "expert copy"); break; }
      if (resident_mask) resident_mask[t] |= bit;
      if (out_layer) out_layer[x * max_jobs + issued] = t;
      if (out_expert) out_expert[x * max_jobs + issued] = ex;
      ++issued;
    }
    for (int j = issued; j < max_jobs; ++j) {
      if (out_layer) out_layer[x * max_jobs + j] = -1;
      if (out_expert) out_expert[x * max_jobs + j] = -1;
    }
    if (out_njobs) out_njobs[x] = issued;
  }
  return S.finish(r);
}

fmoe_status fmoe_eviction_order(int64_t n, const float* p, const float* freq, float eps, double* out_priority,
                                int32_t* out_order, int device, void* stream) {
  if (n < 1 || n > 8192) return fail(FMOE_ERR_INVALID_ARG, "1 <= n <= 8192");
  if (!p || !freq || !out_priority || !out_order) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  if (!(eps > 0.f)) return fail(FMOE_ERR_INVALID_ARG, "eps > 0");
  DeviceGuard g(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, device);
  const float* dp = S.in(p, size_t(n));
  const float* df = S.in(freq, size_t(n));
  double* dpr = S.out(out_priority, size_t(n));
  int32_t* dor = S.out(out_order, size_t(n));
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    cudaError_t e = launch_eviction_order(int(n), dp, df, eps, dpr, dor, s);
    if (e != cudaSuccess) r = cuda_fail(e, "eviction launch");
  }
  return S.finish(r);
}

fmoe_status fmoe_expert_hits(int64_t B, int32_t T, int32_t E, int32_t K, const float* gate,
                             const uint64_t* prefetch_mask, uint64_t* out_active, int32_t* out_hits, int device,
                             void* stream) {
  if (B < 0 || T < 1 || E < 1 || E > 64 || K < 1 || K > E) return fail(FMOE_ERR_INVALID_ARG, "sizes");
  if (B == 0) return FMOE_OK;
  if (!gate || !prefetch_mask || !out_hits) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  DeviceGuard g(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, device);
  const size_t rows = size_t(B) * size_t(T);
  const float* dg = S.in(gate, rows * size_t(E));
  const uint64_t* dm = S.in(prefetch_mask, rows);
  uint64_t* da = out_active ? S.out(out_active, rows) : nullptr;
  int32_t* dh = S.out(out_hits, rows);
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    cudaError_t e = launch_expert_hits(int64_t(rows), E, K, dg, dm, da, dh, s);
    if (e != cudaSuccess) r = cuda_fail(e, "hits launch");
  }
  return S.finish(r);
}

fmoe_status fmoe_topk_merge(int64_t B, int32_t n_lists, int32_t k_in, const float* scores, const int64_t* ids,
                            int32_t k, float* out_score, int64_t* out_id, int device, void* stream) {
  if (B < 0 || n_lists < 0 || k_in < 1 || k_in > FMOE_MAX_K || k < 1 || k > FMOE_MAX_K)
    return fail(FMOE_ERR_INVALID_ARG, "sizes");
  if ((n_lists > 0 && (!scores || !ids)) || !out_score || !out_id) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  if (B == 0) return FMOE_OK;
  DeviceGuard g(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, device);
  const size_t nin = size_t(n_lists) * B * k_in;
  const float* dsc = S.in(scores, nin);
  const int64_t* did = S.in(ids, nin);
  float* ds = S.out(out_score, size_t(B) * k);
  int64_t* di = S.out(out_id, size_t(B) * k);
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    cudaError_t e = launch_merge_lists(int(B), n_lists, k_in, dsc, did, k, ds, di, s);
    if (e != cudaSuccess) r = cuda_fail(e, "merge launch");
  }
  return S.finish(r);
}

}  // extern "C"

// ============================================================================
// Sharded store: collective versions of the calls.  Each runs
// the single-GPU call on the local shard (LocalScope: no re-dispatch) with
// device outputs, then ONE all-gather of a packed payload and a merge kernel.
// ============================================================================
namespace {

// local top-k (score, id) [B][k] device -> replicated global top-k
fmoe_status exchange_topk(const fmoe_store* st, Staging& S, int64_t B, int k, const float* ls, const int64_t* li,
                          float* ds, int64_t* di, uint64_t* dkeys, cudaStream_t s) {
  const int G = st->dist->comm.world;
  const size_t pay_b = size_t(B) * (k + 1) * 8;
  uint64_t* pay = static_cast<uint64_t*>(S.scratch(pay_b));
  uint64_t* gat = static_cast<uint64_t*>(S.scratch(pay_b * G));
  fmoe_status r = S.check();
  if (r != FMOE_OK) return r;
  cudaError_t e = launch_pack_topk(int(B), k, ls, li, pay, s);
  if (e != cudaSuccess) return cuda_fail(e, "pack launch");
  std::string err;
  if (!st->dist->comm.allgather(pay, gat, pay_b, s, &err)) return fail(FMOE_ERR_CUDA, err);
  e = launch_merge_gathered(G, int(B), k, k, gat, ds, di, dkeys, s);
  return e == cudaSuccess ? FMOE_OK : cuda_fail(e, "merge launch");
}

// the owner's Eq. 4-6 selection (other ranks contribute mask 0, count 0) -> replicated
fmoe_status exchange_select(const fmoe_store* st, Staging& S, int64_t B, const int64_t* did, const float* dsc,
                            int stride, float delta, int lb, int le, int layer_step, uint64_t* dm, int32_t* dc,
                            cudaStream_t s) {
  const int G = st->dist->comm.world;
  const int64_t n = B * (le - lb);
  uint64_t* lm = static_cast<uint64_t*>(S.scratch(size_t(n) * 8));
  int32_t* lc = static_cast<int32_t*>(S.scratch(size_t(n) * 4));
  uint64_t* pay = static_cast<uint64_t*>(S.scratch(size_t(n) * 16));
  uint64_t* gat = static_cast<uint64_t*>(S.scratch(size_t(n) * 16 * G));
  fmoe_status r = S.check();
  if (r != FMOE_OK) return r;
  cudaError_t e = launch_select(st->view(), int(B), did, dsc, delta, st->cfg.K, lb, le, st->cfg.id_offset, st->n, lm,
                                lc, s, stride, layer_step);
  if (e == cudaSuccess) e = launch_pack_select(int(n), lm, lc, pay, s);
  if (e != cudaSuccess) return cuda_fail(e, "select launch");
  std::string err;
  if (!st->dist->comm.allgather(pay, gat, size_t(n) * 16, s, &err)) return fail(FMOE_ERR_CUDA, err);
  e = launch_combine_select(G, int(n), gat, dm, dc, s);
  return e == cudaSuccess ? FMOE_OK : cuda_fail(e, "combine launch");
}

// run `local(ls, li)` (device [B][k]) then exchange into the caller's outputs
template <class F>
fmoe_status sharded_topk(const fmoe_store* st, int64_t B, int k, float* out_score, int64_t* out_id, void* stream,
                         F&& local) {
  if (B == 0) return FMOE_OK;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device, true);
  float* ds = S.out(out_score, size_t(B) * k);
  int64_t* di = S.out(out_id, size_t(B) * k);
  float* ls = static_cast<float*>(S.scratch(size_t(B) * k * 4));
  int64_t* li = static_cast<int64_t*>(S.scratch(size_t(B) * k * 8));
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    LocalScope ls_scope;
    r = local(ls, li, s);
  }
  if (r == FMOE_OK) r = exchange_topk(st, S, B, k, ls, li, ds, di, nullptr, s);
  return S.finish(r);
}

fmoe_status sharded_search(const fmoe_store* st, int64_t B, const float* q_emb, const float* q_prefix, int32_t ell,
                           float w, int32_t k, float* out_score, int64_t* out_id, void* stream, float* out_cos,
                           int64_t cos_stride) {
  return sharded_topk(st, B, k, out_score, out_id, stream, [&](float* ls, int64_t* li, cudaStream_t s) {
    return search_common(st, B, q_emb, q_prefix, ell, w, k, ls, li, s, out_cos, cos_stride);
  });
}

fmoe_status sharded_blend_cos(const fmoe_store* st, int64_t B, const float* sem_cos, int64_t cos_stride,
                              const float* q_prefix, int32_t ell, float w_sem, int32_t k, float* out_score,
                              int64_t* out_id, void* stream) {
  return sharded_topk(st, B, k, out_score, out_id, stream, [&](float* ls, int64_t* li, cudaStream_t s) {
    return fmoe_search_blend_cos(st, B, sem_cos, cos_stride, q_prefix, ell, w_sem, k, ls, li, s);
  });
}

fmoe_status sharded_select(const fmoe_store* st, int64_t B, const int64_t* map_id, const float* score, float delta,
                           int32_t lb, int32_t le, uint64_t* out_mask, int32_t* out_count, void* stream) {
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device, true);
  const int T = le - lb;
  const int64_t* did = S.in(map_id, size_t(B));
  const float* dsc = delta < 0.f ? S.in(score, size_t(B)) : nullptr;
  uint64_t* dm = S.out(out_mask, size_t(B) * T);
  int32_t* dc = S.out(out_count, size_t(B) * T);
  fmoe_status r = S.check();
  if (r == FMOE_OK) r = exchange_select(st, S, B, did, dsc, 1, delta, lb, le, 0, dm, dc, s);
  return S.finish(r);
}

// Insert (Reading R8) on a sharded store: appends go to the ranks
// owning slots n0, n0+1, ...; once full, every rank finds its local RDY top-kk
// over the contexts present before the call, the lists are all-gathered and
// merged, the victims are resolved in batch order on every rank (same result
// everywhere), and each rank writes the rows whose slot it owns.
fmoe_status sharded_insert(fmoe_store* st, int64_t B, const float* emb, const float* maps, const float* sem_cos,
                           int64_t cos_stride, int64_t* out_slot, int64_t* out_replaced, void* stream) {
  fmoe_store::Dist& ds_ = *st->dist;
  const int64_t C = ds_.cap_total, n0 = ds_.n_total, off = st->cfg.id_offset, capl = st->cfg.capacity;
  const int64_t a = B < C - n0 ? B : C - n0, nrep = B - a;
  fmoe_status xs = ensure_excl(st, nrep);
  if (xs != FMOE_OK) return xs;
  const int L = st->cfg.L, E = st->cfg.E, D = st->cfg.D;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device, true);
  const int64_t n_loc0 = n0 - off < 0 ? 0 : (n0 - off > capl ? capl : n0 - off);   // local rows before the call
  const float* de = S.in(emb, size_t(B) * D);
  const float* dm = S.in(maps, size_t(B) * L * E);
  const float* dcos = sem_cos && nrep > 0 && n_loc0 > 0 ? S.in(sem_cos, size_t(B) * cos_stride) : nullptr;
  int64_t* dslot = S.out(out_slot, size_t(B));
  int64_t* drep = S.out(out_replaced, size_t(B));
  int64_t* slots_all = static_cast<int64_t*>(S.scratch(size_t(B) * 8));
  fmoe_status r = S.check();
  // sub-batches of <= 64 rows, as the single-GPU insert (later ones skip the
  // slots earlier ones claimed; every rank marks the victims it owns)
  const int64_t nsub_rows = FMOE_MAX_K;
  for (int64_t sb = 0; r == FMOE_OK && (sb < nrep || (sb == 0 && nrep == 0)); sb += nsub_rows) {
    const int64_t nb = nrep - sb < nsub_rows ? nrep - sb : nsub_rows;
    const int kk = int(nb < n0 ? nb : n0) > 0 ? int(nb < n0 ? nb : n0) : 1;
    float* ls = static_cast<float*>(S.scratch(size_t(nb > 0 ? nb : 1) * kk * 4));
    int64_t* li = static_cast<int64_t*>(S.scratch(size_t(nb > 0 ? nb : 1) * kk * 8));
    uint64_t* mkeys = static_cast<uint64_t*>(S.scratch(size_t(nb > 0 ? nb : 1) * kk * 8));
    r = S.check();
    if (r == FMOE_OK && nb > 0) {
      if (n_loc0 > 0) {
        CosArgs cos;
        cos.in = dcos ? dcos + (a + sb) * cos_stride : nullptr;
        cos.stride = cos_stride;
        cos.excl = sb > 0 ? st->excl : nullptr;
        // RDY = d/L sem + (L-d)/L traj over full maps, unchecked queries
        r = run_search(st, nb, de + (a + sb) * D, dm + (a + sb) * int64_t(L) * E, int64_t(L) * E, L,
                       float(st->cfg.d) / float(L), kk, n_loc0, uint32_t(off), s, ls, li, nullptr, false, cos);
      } else {
        cudaError_t e = launch_merge_keys(int(nb), 0, kk, nullptr, kk, nullptr, ls, li, nullptr, s);
        if (e != cudaSuccess) r = cuda_fail(e, "merge launch");
      }
      if (r == FMOE_OK) r = exchange_topk(st, S, nb, kk, ls, li, nullptr, nullptr, mkeys, s);
    }
    if (r == FMOE_OK) {
      // keys hold global ids; appended rows get global slots n0 + x
      cudaError_t e = launch_resolve(int(nb > 0 ? nb : 0), kk, mkeys, 0u, slots_all, int(a + sb), n0, dslot, drep, s,
                                     nullptr, 0, nullptr, sb == 0 ? int(a) : 0);
      if (e == cudaSuccess && sb + nb < nrep) e = launch_excl(st->excl, slots_all + a + sb, int(nb), off, capl, 1, s);
      if (e != cudaSuccess) r = cuda_fail(e, "resolve launch");
    }
    if (nrep == 0) break;
  }
  if (r == FMOE_OK && nrep > nsub_rows) {
    cudaError_t e = launch_excl(st->excl, slots_all + a, int(nrep - nsub_rows), off, capl, 0, s);
    if (e != cudaSuccess) r = cuda_fail(e, "bitmap reset launch");
  }
  if (r == FMOE_OK) {
    WriteArgs w{};
    w.emb = st->emb; w.r_e = st->r_e; w.maps = st->maps; w.psq = st->psq;
    w.cap = capl; w.L = L; w.E = E; w.D = D; w.Dp = st->Dp; w.Ep = st->Ep; w.bf16 = st->bf16;
    w.in_emb = de; w.in_maps = dm;
    w.B = int(B);
    w.slots = slots_all;
    w.slot_offset = off;
    w.slot_limit = capl;          // this rank's rows: appends and victims it owns
    cudaError_t e = launch_write_rows(w, s);
    if (e != cudaSuccess) r = cuda_fail(e, "write launch");
  }
  if (r == FMOE_OK) {
    ds_.n_total = n0 + a;
    const int64_t nl = ds_.n_total - off;
    st->n = nl < 0 ? 0 : (nl > capl ? capl : nl);
    ++st->gen;
  }
  return S.finish(r);
}

fmoe_status sharded_session_step(fmoe_traj_session* ss, const float* q_layer, int32_t k, float* out_score,
                                 int64_t* out_id, const StepSelect& sel, void* stream) {
  const fmoe_store* st = ss->st;
  const int64_t B = ss->B;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device, true);
  const int T = sel.le - sel.lb;
  float* ds = S.out(out_score, size_t(B) * k);
  int64_t* di = S.out(out_id, size_t(B) * k);
  uint64_t* dm = T > 0 ? S.out(sel.mask, size_t(B) * T) : nullptr;
  int32_t* dc = T > 0 ? S.out(sel.count, size_t(B) * T) : nullptr;
  float* ls = static_cast<float*>(S.scratch(size_t(B) * k * 4));
  int64_t* li = static_cast<int64_t*>(S.scratch(size_t(B) * k * 8));
  // merged outputs in device memory (the selection reads the merged top-1)
  float* ms = static_cast<float*>(S.scratch(size_t(B) * k * 4));
  int64_t* mi = static_cast<int64_t*>(S.scratch(size_t(B) * k * 8));
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    LocalScope scope;
    r = session_step(ss, q_layer, k, ls, li, StepSelect(), s);
  }
  if (r == FMOE_OK) r = exchange_topk(st, S, B, k, ls, li, ms, mi, nullptr, s);
  if (r == FMOE_OK && T > 0)
    r = exchange_select(st, S, B, mi, ms, k, sel.delta, sel.lb, sel.le, 0, dm, dc, s);
  if (r == FMOE_OK) {
    cudaError_t e = cudaSuccess;
    if (ds) e = cudaMemcpyAsync(ds, ms, size_t(B) * k * 4, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && di) e = cudaMemcpyAsync(di, mi, size_t(B) * k * 8, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) r = cuda_fail(e, "session output copy");
  }
  return S.finish(r);
}

fmoe_status sharded_sweep(fmoe_traj_session* ss, const float* q_layers, int32_t n_steps, float* out_score,
                          int64_t* out_id, float delta, int32_t sel_d, uint64_t* out_mask, int32_t* out_count,
                          void* stream) {
  const fmoe_store* st = ss->st;
  const int64_t B = ss->B, n = int64_t(n_steps) * B;
  const int layer0 = ss->layer;
  DeviceGuard g(st->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Staging S(s, st->device, true);
  float* ds = S.out(out_score, size_t(n));
  int64_t* di = S.out(out_id, size_t(n));
  uint64_t* dm = out_mask ? S.out(out_mask, size_t(n)) : nullptr;
  int32_t* dc = out_mask ? S.out(out_count, size_t(n)) : nullptr;
  float* ls = static_cast<float*>(S.scratch(size_t(n) * 4));
  int64_t* li = static_cast<int64_t*>(S.scratch(size_t(n) * 8));
  float* ms = static_cast<float*>(S.scratch(size_t(n) * 4));
  int64_t* mi = static_cast<int64_t*>(S.scratch(size_t(n) * 8));
  fmoe_status r = S.check();
  if (r == FMOE_OK) {
    LocalScope scope;
    r = fmoe_traj_session_sweep(ss, q_layers, n_steps, ls, li, delta, sel_d, nullptr, nullptr, nullptr, nullptr, s);
  }
  // every (step, query) row is a top-1 search: one exchange for the whole sweep
  if (r == FMOE_OK) r = exchange_topk(st, S, n, 1, ls, li, ms, mi, nullptr, s);
  // row (step s, query x) selects target layer layer0 + s + sel_d (none past L)
  if (r == FMOE_OK && dm) {
    if (B == 1) r = exchange_select(st, S, n, mi, ms, 1, delta, layer0 + sel_d, layer0 + sel_d + 1, 1, dm, dc, s);
    else
      for (int st2 = 0; st2 < n_steps && r == FMOE_OK; ++st2) {
        const int tgt = layer0 + st2 + sel_d;
        r = exchange_select(st, S, B, mi + int64_t(st2) * B, ms + int64_t(st2) * B, 1, delta, tgt, tgt + 1, 0,
                            dm + int64_t(st2) * B, dc + int64_t(st2) * B, s);
      }
  }
  if (r == FMOE_OK) {
    cudaError_t e = cudaMemcpyAsync(ds, ms, size_t(n) * 4, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(di, mi, size_t(n) * 8, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) r = cuda_fail(e, "sweep output copy");
  }
  return S.finish(r);
}

}  // namespace

extern "C" {

fmoe_status fmoe_get_nccl_unique_id(void* out_128_bytes) {
  if (!out_128_bytes) return fail(FMOE_ERR_INVALID_ARG, "null out");
  std::string err;
  if (!nccl_unique_id(out_128_bytes, &err)) return fail(FMOE_ERR_UNSUPPORTED, err);
  return FMOE_OK;
}

fmoe_status fmoe_store_create_sharded(const fmoe_store_config* cfg, const fmoe_dist_config* dist, int device,
                                      fmoe_store** out) {
  if (!out || !cfg || !dist) return fail(FMOE_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world)
    return fail(FMOE_ERR_INVALID_ARG, "need 0 <= rank < world");
  if (dist->transport != FMOE_TRANSPORT_NCCL && dist->transport != FMOE_TRANSPORT_HOST)
    return fail(FMOE_ERR_INVALID_ARG, "transport");
  if (cfg->id_offset != 0) return fail(FMOE_ERR_INVALID_ARG, "sharded: cfg->id_offset must be 0");
  if (cfg->capacity < dist->world) return fail(FMOE_ERR_SHAPE, "sharded: capacity < world");
  const int64_t per = (cfg->capacity + dist->world - 1) / dist->world;
  const int64_t off = per * dist->rank;
  const int64_t capl = cfg->capacity - off < per ? cfg->capacity - off : per;
  if (capl < 1) return fail(FMOE_ERR_SHAPE, "sharded: a rank would hold no slots (capacity too small)");
  fmoe_store_config lc = *cfg;
  lc.capacity = capl;
  lc.id_offset = off;
  fmoe_store* st = nullptr;
  fmoe_status r = fmoe_store_create(&lc, device, &st);
  if (r != FMOE_OK) return r;
  st->dist = new fmoe_store::Dist();
  st->dist->cap_total = cfg->capacity;
  st->dist->per = per;
  std::string err;
  {
    DeviceGuard g(device);
    if (!st->dist->comm.init(dist->rank, dist->world, dist->transport, dist->nccl_unique_id,
                             reinterpret_cast<AllGatherFn>(dist->allgather), dist->allgather_user, &err)) {
      fmoe_store_destroy(st);
      return fail(FMOE_ERR_CUDA, err);
    }
  }
  *out = st;
  return FMOE_OK;
}

}  // extern "C"
