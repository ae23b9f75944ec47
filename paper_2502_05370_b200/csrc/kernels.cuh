// kernels.cuh -- launch interface of the fMoE sm_100a kernels (internal, not ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <string>
#include <utility>

namespace fmoe {

// Launch with programmatic stream serialization (PDL): the grid may start
// while the previous grid on the stream drains; kernels call pdl_wait()
// before reading dependent memory.
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Device view of a store's HBM tiles.
struct StoreView {
  const void* emb;     // [cap][Dp] dtype, row-major
  const float* r_e;    // [cap] 1/||quantised embedding|| (0 for a zero row)
  const void* maps;    // [L][cap][Ep] dtype, layer-major slabs
  const float* psq;    // [L][cap] prefix squared norms sum_{l'<=l} ||P_l'||^2
  int64_t cap;         // slab stride (rows)
  int L, E, D, Dp, Ep;
  int bf16;            // 1 = bf16 tiles, 0 = fp32
};

// One scoring pass: queries [q0, q0+nq) of the batch against rows [0, n_rows).
struct ScanArgs {
  StoreView st;
  int64_t n_rows;
  int ell;                   // prefix layers used by the trajectory part
  float w_sem;               // blend weight: 1 semantic only, 0 trajectory only
  int k;                     // list length (<= kMaxK)
  const float* q_emb;        // [B][D]  (may be null when w_sem == 0)
  const float* q_prefix;     // [B][*] rows of q_stride floats, layer l at l*E
  int64_t q_stride;
  int q0, nq;                // query slice of this pass (nq <= 4)
  uint32_t id_offset;        // global id of row 0
  uint64_t* cand;            // [B][grid][k] per-block candidate keys
  int grid;                  // blocks of the launch (cand stride)
  unsigned* counter;         // zeroed ticket counter of this pass (last block merges)
  // outputs of the fused grid merge (queries q0..q0+nq): either (score, id) or raw keys
  float* out_score;          // [B][k]
  int64_t* out_id;           // [B][k]
  uint64_t* out_keys;        // [B][k]
  int check_valid;           // 1: zero-norm query -> (NaN, -1)
  unsigned long long* trace; // debug phase tracer [kTraceBlocks][8] or null
  unsigned long long* best;  // [B] zeroed keys for the k == 1 merge (reset by the last block)
  // semantic cosines: a semantic scan may write them (out_cos), a blend/RDY scan
  // may take them instead of re-reading the embeddings (sem_cos); [B][cos_stride]
  float* out_cos;
  const float* sem_cos;
  int64_t cos_stride;
  const int* run_if_gt;      // nullable device count: the pass runs only if *run_if_gt > q0 (re-rank fallback)
  const uint32_t* excl;      // nullable bitmap over local rows: set bits are no candidates (insert sub-batches)
};

// debug tracer buffer (null unless fmoe_debug_trace enabled it)
unsigned long long* trace_buffer();

// GEMV scan (B <= 4 per pass): bandwidth-bound warp-per-32-rows streaming.
cudaError_t launch_scan_gemv(const ScanArgs& a, cudaStream_t s);
int scan_gemv_grid(const ScanArgs& a);

// Trajectory-only scan fed by a TMA bulk-copy ring (one CTA per SM).
bool scan_tma_supported(const ScanArgs& a);
int scan_tma_grid(const ScanArgs& a);
cudaError_t launch_scan_tma(const ScanArgs& a, cudaStream_t s);

// Merge per-list candidate keys -> per-query top-k (also fills an empty
// result when n_lists == 0).  keys [B][n_lists][k_in]; writes (out_score,
// out_id) and/or out_keys [B][k]; valid (nullable) [B]: 0 -> (NaN, -1).
// gate (nullable, device): when it holds 0 the launch does nothing (see
// launch_resolve's need_full).
cudaError_t launch_merge_keys(int B, int n_lists, int k_in, const uint64_t* keys, int k, const float* valid,
                              float* out_score, int64_t* out_id, uint64_t* out_keys, cudaStream_t s,
                              const int* gate = nullptr);

// Incremental trajectory session (traj_session.cu): step `layer` consumes one
// layer of each query; acc [B][cap] running dots; qn [2][B] running norms.
struct SessionArgs {
  const float* q_layer;   // [B][E] fp32, this step's layer
  int layer;              // 0-based layer consumed by this step
  float* acc;             // [B][cap]
  int64_t rpw;            // rows per warp (a contiguous range; set by launch_traj_session)
  const double* qn_prev;  // [B]
  double* qn_next;        // [B]
  const unsigned* abort;  // device word: != 0 -> the session was abandoned; every query is invalid
  // optional fused Eq. 4-6 selection on each query's top-1 (sel_T = 0: none),
  // run by the step's last block: layers [sel_lb, sel_lb + sel_T)
  float sel_delta;        // < 0: dynamic Clip(1 - score, 0, 1)
  int sel_K, sel_lb, sel_T;
  uint64_t* sel_mask;     // [B][sel_T]
  int32_t* sel_count;     // [B][sel_T]
};
cudaError_t launch_traj_session(const ScanArgs& a, const SessionArgs& s, cudaStream_t stream);
int traj_session_grid(const ScanArgs& a);

// n session steps of one request (B = 1, k = 1, 16-byte slab rows) in one launch
struct SweepArgs {
  StoreView st;
  int64_t n_rows;
  uint32_t id_offset;
  const float* q_layers;            // [n_steps][E] fp32
  int layer0, n_steps;
  float* acc;                       // [cap] session accumulators (read if layer0 > 0, written at the end)
  const double* qn_in;              // running query norm before layer0
  double* qn_out;                   // after the last step
  unsigned long long* best;         // [n_steps] zeroed scratch (reset by the kernel)
  unsigned* tickets;                // [n_steps] zeroed scratch (reset by the kernel)
  float* out_score;                 // [n_steps]
  int64_t* out_id;                  // [n_steps]
  float sel_delta;
  int sel_K, sel_d;                 // target layer of step s = layer0 + s + sel_d (none if >= L)
  uint64_t* sel_mask;               // [n_steps] or null (no selection)
  int32_t* sel_count;               // [n_steps]
  const unsigned* layer_ready;      // [n_steps] or null: step s waits for layer_ready[s] != 0
  unsigned* guidance_ready;         // [n_steps] or null: 1 when step s's outputs are written, 2 if abandoned
  unsigned long long timeout_ns;    // give up waiting for a layer after this long
  unsigned* abort;                  // session status word: set on a timeout; a poisoned session
                                    // (word != 0 at start) writes (NaN, -1) and abandons every step
};
int traj_sweep_rows(int64_t n_rows, int* grid_out);   // 0: the store is too large for the register sweep
cudaError_t launch_traj_sweep(const SweepArgs& a, cudaStream_t stream);

// fp32 batched scan (scan_f32mm.cu): 5 <= nq <= 64 queries per pass, the store
// streamed once per pass, register-tiled FFMA, per-warp top-k lists.
struct F32mmPrep {
  const float* q_emb;      // [nq][D] (null: no semantic part)
  const float* q_prefix;   // [nq][q_stride] (null: no trajectory part)
  int64_t q_stride;
  int D, E, Ep, ell;
  int n_sem_ch, n_traj_ch, qpitch;
  int sem, traj;           // parts that decide validity (sem: embeddings scored)
  float* qop;              // [nq][qpitch]
  float* rq_s; float* rq_t; float* valid;   // [nq]
};
struct F32mmArgs {
  StoreView st;
  int64_t n_rows;
  int ell; float w; int k;
  int nq, wq;              // queries of this pass, query groups (f32mm_wq(nq))
  const float* qop; int qpitch;
  int n_sem_ch, n_traj_ch; // 32-float K chunks (semantic over Dp, trajectory over ell*Ep)
  const float* rq_s; const float* rq_t;
  uint32_t id_offset;
  uint64_t* cand; int cand_q0; int grid;    // cand [B][grid * lists_per_cta][k]
  float* out_cos; const float* sem_cos; int64_t cos_stride;   // this pass's first query row
  const uint32_t* excl;
};
int f32mm_wq(int nq);
int f32mm_grid(int64_t n_rows, int nq, bool blend);
int f32mm_lists_per_cta(int nq);
cudaError_t launch_f32mm_prep(const F32mmPrep& p, int nq, cudaStream_t s);
cudaError_t launch_f32mm(const F32mmArgs& a, cudaStream_t s);

// tcgen05 batched scan (scan_umma.cu)
struct UmmaPlanIn {
  int bf16, nq, k, D, Dp, E, Ep, L, ell;
  float w_sem;
  int64_t n_rows, cap;
  uint32_t id_offset;
  const void* emb; const void* maps; const float* r_e; const float* psq;
  int rep;                     // query replication (umma_rep), uniform over a call's passes
  int cg;                      // 1: CTAs, 2: CTA pairs (M = 256); 0 = by nq.  Uniform over a call's passes
  int approx;                  // semantic scan with one accumulator; an exact re-rank follows (rerank.cu)
  int cos_out;                 // the call writes the cosine side output (reserve the TMA staging smem)
  int cos_in;                  // the call blends cached cosines (reserve the TMA load ring)
};
struct UmmaLaunch {
  UmmaPlanIn in;
  const float* q_emb; const float* q_prefix; int64_t q_stride;   // this pass's first query
  void* scratch;               // umma_scratch_bytes(in)
  float* out_cos; const float* sem_cos; int64_t cos_stride;   // see ScanArgs
  float* valid;                // [nq] validity flags of this pass
  unsigned long long* gthr;    // [nq] scratch: shared per-query admission thresholds
  const int* gate;             // nullable device flag: 0 -> every kernel of the launch returns at once
  const int64_t* seed_ids;     // optional [nq][seed_stride] ids of seed_n distinct rows (trajectory only)
  int seed_stride, seed_n;
  uint64_t* cand; int cand_q0; int grid;
  unsigned long long* trace;
  int keep_gthr;               // 1: gthr already holds a valid admission bound (sample pass); prep keeps it
  const uint32_t* excl;        // nullable bitmap over rows: set bits are no candidates (insert sub-batches)
};
bool umma_supported(const UmmaPlanIn& in);
bool umma_cos_bound();
int umma_rep(const UmmaPlanIn& in);
size_t umma_scratch_bytes(const UmmaPlanIn& in);
int umma_grid(const UmmaPlanIn& in);   // CTAs to launch (a multiple of umma_cg)
int umma_cg(const UmmaPlanIn& in);
cudaError_t launch_umma(const UmmaLaunch& L, cudaStream_t s);
cudaError_t launch_seed_from_sample(int B, int ke, const uint64_t* keys, unsigned long long* gthr, cudaStream_t s);
// Exact re-rank of an approximate (single-accumulator) tensor-core semantic
// scan's merged candidates (rerank.cu): [B][ke] keys -> the exact top k, and
// the queries whose completeness margin fails, queued for the GEMV fallback.
struct RerankArgs {
  int B, ke, k;
  const uint64_t* keys;        // [B][ke] merged approximate keys (desc)
  const float* q_emb;          // [B][D] fp32 queries
  int D, Dp;
  const void* emb;             // store embeddings [cap][Dp] bf16
  const float* r_e;
  uint32_t id_offset;
  const float* valid;          // [B] query validity (prep)
  float eps;                   // bound on |approximate - exact| score
  float* out_score; int64_t* out_id; uint64_t* out_keys;   // [B][k] (any may be null)
  int* nfail; int* qmap; float* qc;                        // fallback queue: count, slot -> query, [B][D] queries
};
cudaError_t launch_rerank(const RerankArgs& r, cudaStream_t s);
cudaError_t launch_rerank_scatter(const int* nfail, const int* qmap, int k, const float* fb_s, const int64_t* fb_i,
                                  const uint64_t* fb_keys, float* out_score, int64_t* out_id, uint64_t* out_keys,
                                  int* nfail_w, cudaStream_t s);
// Merge (score, id) lists from an all-gather: [n_lists][B][k_in].
cudaError_t launch_merge_lists(int B, int n_lists, int k_in, const float* scores,
                               const int64_t* ids, int k, float* out_score, int64_t* out_id,
                               cudaStream_t s);

// Eq. 4-6 selection, one warp per (query, layer).
cudaError_t launch_select(const StoreView& st, int B, const int64_t* map_id, const float* score,
                          float delta, int K, int layer_begin, int layer_end, int64_t id_offset,
                          int64_t n_rows, uint64_t* out_mask, int32_t* out_count, cudaStream_t s,
                          int stride = 1,    // map_id[q * stride], score[q * stride]
                          int layer_step = 0);   // row q selects layers + q * layer_step (>= L: none)

// Expert-cache priorities: prefetch plan per query, eviction order.
cudaError_t launch_prefetch_plan(const StoreView& st, int B, const int64_t* map_id, const float* score, float delta,
                                 int K, int l_now, int lb, int le, int64_t id_offset, int64_t n_rows, int max_jobs,
                                 int32_t* out_layer, int32_t* out_expert, double* out_pri, int32_t* out_njobs,
                                 cudaStream_t s);
cudaError_t launch_eviction_order(int n, const float* p, const float* freq, float eps, double* out_pri,
                                  int32_t* out_order, cudaStream_t s);
// Expert hits of prefetch guidance: top-K of each gate row vs the prefetched mask.
cudaError_t launch_expert_hits(int64_t rows, int E, int K, const float* gate, const uint64_t* pmask,
                               uint64_t* out_active, int32_t* out_hits, cudaStream_t s);

// Quantise + write rows (append or replace) and their norm tables.
//  slot of new row x: slots ? slots[x] (skip if < 0) : first_slot + x.
struct WriteArgs {
  void* emb; float* r_e; void* maps; float* psq;
  int64_t cap; int L, E, D, Dp, Ep, bf16;
  const float* in_emb; const float* in_maps;   // [B][D], [B][L][E]
  int B;
  const int64_t* slots; int64_t first_slot;
  int64_t slot_offset;   // slots[] hold global ids: local = slot - slot_offset
  int64_t slot_limit;    // rows whose local slot is outside [0, slot_limit) are skipped
};
cudaError_t launch_write_rows(const WriteArgs& w, cudaStream_t s);

// Victim resolution (Reading R8): rows j in batch order take their best
// candidate not claimed by an earlier row.  keys [nrep][kk] (from merge).
//  victims [nrep] (local slot or -1); also scatters to out_slot/out_replaced
//  at positions x0 + j, and marks appended rows [0, x0) in out_slot/out_replaced.
//  need_full (nullable): set to 1 when some row found every one of its kk
//  candidates claimed while its list was full and k_full > kk -- its victim
//  may lie beyond the kk kept keys (the call's results are then provisional),
//  else 0.  gate (nullable): skip the launch when *gate == 0.
cudaError_t launch_resolve(int nrep, int kk, const uint64_t* keys, uint32_t id_offset,
                           int64_t* victims, int x0, int64_t first_append_slot,
                           int64_t* out_slot, int64_t* out_replaced, cudaStream_t s,
                           int* need_full = nullptr, int k_full = 0, const int* gate = nullptr,
                           int mark_append = -1);   // rows [0, mark_append) are appends (-1: x0)
// Exclusion bitmap of an insert's sub-batches: set / clear the bits of the
// victims slots[x] (global ids; local bit = id - offset if in [0, limit)).
cudaError_t launch_excl(uint32_t* excl, const int64_t* slots, int n, int64_t offset, int64_t limit, int set,
                        cudaStream_t s);
// Victim resolution from merged candidate ids [B][k] (best first).
cudaError_t launch_resolve_ids(int B, int k, const int64_t* ids, int64_t* out_victim, cudaStream_t s);
cudaError_t launch_append_ids(int n, int64_t first_slot, uint32_t id_offset, int64_t* out_slot,
                              int64_t* out_replaced, cudaStream_t s);

// Read back rows as fp32.
cudaError_t launch_read_rows(const StoreView& st, int64_t slot0, int64_t count, float* out_emb,
                             float* out_maps, cudaStream_t s);

// ---- sharded store: the exchange step (dist.cu)
constexpr int kTransportNccl = 0;
constexpr int kTransportHost = 1;
using AllGatherFn = int32_t (*)(const void* send, void* recv, int64_t bytes, void* user);
struct Comm {
  int rank = 0, world = 1, transport = kTransportNccl;
  void* comm = nullptr;                 // ncclComm_t
  AllGatherFn host_fn = nullptr;
  void* host_user = nullptr;
  void* h_send = nullptr;               // HOST transport: pinned staging
  void* h_recv = nullptr;
  size_t h_bytes = 0;
  bool init(int rank, int world, int transport, const void* nccl_uid, AllGatherFn fn, void* user, std::string* err);
  void destroy();
  // recv [world][bytes] <- every rank's send [bytes], rank order (stream-ordered for NCCL)
  bool allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s, std::string* err);
};
bool nccl_unique_id(void* out128, std::string* err);
// local top-k [B][k] -> payload [B*k keys | B validity flags]
cudaError_t launch_pack_topk(int B, int k, const float* sc, const int64_t* id, uint64_t* payload, cudaStream_t s);
// gathered payloads [G][B*k_in + B] -> global top k (NaN, -1 where a rank flags the query invalid)
cudaError_t launch_merge_gathered(int G, int B, int k_in, int k, const uint64_t* g, float* out_score,
                                  int64_t* out_id, uint64_t* out_keys, cudaStream_t s);
// selection payload [2][n] (masks, counts) and its OR / sum over [G] ranks
cudaError_t launch_pack_select(int n, const uint64_t* mask, const int32_t* count, uint64_t* payload, cudaStream_t s);
cudaError_t launch_combine_select(int G, int n, const uint64_t* g, uint64_t* out_mask, int32_t* out_count,
                                  cudaStream_t s);

// launch counter (for the bench's gpu_launches)
void count_launch(int n = 1);

}  // namespace fmoe
