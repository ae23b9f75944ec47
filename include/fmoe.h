/*
 * fmoe.h -- C ABI of the B200-native fMoE expert-map search (arXiv 2502.05370).
 *
 * Citations: P:n = PAPER.md line n (paper section / equation named), S:n =
 * SPEC.md line n.  Readings R1..R12 of ambiguous passages are listed in
 * DESIGN.md §"Readings".
 *
 * The store holds N historical iteration contexts ("Expert Map
 * Store"): a semantic embedding sem_y in R^D and an expert map
 * map_y = {P_1..P_L}, P_l in R^E the gate probability distribution of layer l
 * (P:410-421).  Searches score a batch of B live queries against every stored
 * context and return the top-k contexts per query; selection turns
 * a matched map into per-layer prefetch sets; insertion appends or
 * replaces the most redundant context.
 *
 * ---------------------------------------------------------------------------
 * Conventions (apply to every call)
 *  - Layouts are C row-major, fp32 inputs, int64 ids.  Layer indices are
 *    0-based (the paper is 1-based): ABI layer t = paper layer t+1.
 *  - Pointers: every array argument may be DEVICE memory on the store's device
 *    or HOST memory (pageable or pinned).  Host arrays are staged through
 *    stream-ordered device buffers; if any OUTPUT array is host memory the call
 *    synchronises `stream` before returning, otherwise the call is
 *    asynchronous and stream-ordered.  The caller owns all arrays; the store
 *    owns its device tiles.  Device arrays on another device -> INVALID_ARG.
 *  - `stream` is a cudaStream_t (NULL = the legacy default stream).
 *  - Host-side argument checks return an error synchronously with no device
 *    work enqueued.  Data-dependent conditions are reported in-band per row
 *    (e.g. a zero-norm query gets id -1 and score NaN, R3).
 *  - Ids are slot indices: a context keeps its id until it is replaced, and the
 *    replacing context takes the same id.  With a sharded store (id_offset !=
 *    0) every id in/out of this ABI is the GLOBAL id id_offset + slot.
 *  - Ordering of results: score descending, ties -> lowest id (R5).
 *    If k > |store| the tail is id -1, score -inf.
 *  - Concurrency: single writer, multiple readers.  Searches on
 *    different streams may overlap; an insert must be stream-ordered after the
 *    searches that should not observe it.
 * ---------------------------------------------------------------------------
 */
#ifndef FMOE_H_
#define FMOE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMOE_ABI_VERSION 1
#define FMOE_MAX_K 64        /* largest k of one search call                    */
#define FMOE_MAX_E 64        /* experts per layer: a prefetch set is a uint64 mask */

typedef struct fmoe_store fmoe_store;   /* opaque; owns all device tiles */

typedef enum {
  FMOE_OK = 0,
  FMOE_ERR_INVALID_ARG = 1,   /* null pointer, k/ell/layer range out of bounds, wrong device */
  FMOE_ERR_SHAPE = 2,         /* configuration shape unsupported (E > 64, D < 1, ...)      */
  FMOE_ERR_OOM = 3,           /* device allocation failed                                  */
  FMOE_ERR_CUDA = 4,          /* a CUDA runtime call or launch failed (see fmoe_last_error) */
  FMOE_ERR_UNSUPPORTED = 5    /* legal request this build does not implement               */
} fmoe_status;

typedef enum { FMOE_F32 = 0, FMOE_BF16 = 1 } fmoe_dtype;

typedef struct {
  int32_t L;          /* MoE layers (paper L)                                         */
  int32_t E;          /* experts per layer (paper J), 1..64                             */
  int32_t K;          /* experts activated per layer (Constraint 6), 1..E       */
  int32_t D;          /* semantic embedding dimension (paper h), >= 1           */
  int32_t d;          /* prefetch distance (d = 3 at P:672), 1 <= d < L         */
  int32_t dtype;      /* fmoe_dtype of the stored embedding and map tiles              */
  int64_t capacity;   /* slots held by THIS store object (paper C)  <= 2^32-1  */
  int64_t id_offset;  /* global id of slot 0 (sharded store); 0 if unsharded */
} fmoe_store_config;

/* ---- lifetime ---------------------------------------------------------- */

/* Create an empty store on CUDA device `device`.  Allocates the tiles of
 * capacity contexts: bytes = capacity*(D'*s + 4 + L*E'*s + 4*L) with
 * s = 2 (bf16) or 4 (fp32), D' and E' rounded up to 16-byte rows (DESIGN.md
 * "HBM layout").  Errors: SHAPE for an illegal config, OOM, CUDA. */
fmoe_status fmoe_store_create(const fmoe_store_config* cfg, int device, fmoe_store** out);

/* Free the store and its tiles.  The caller guarantees that no work on the
 * store is pending (as for any free); the store's scratch is released on the
 * streams that used it.  NULL is a no-op. */
void fmoe_store_destroy(fmoe_store* store);

/* Number of occupied slots |S| (host counter; inserts update it when enqueued,
 * a call that fails leaves it unchanged).  Sharded store: the GLOBAL size. */
fmoe_status fmoe_store_size(const fmoe_store* store, int64_t* out_n);

/* ---- sharded store over several GPUs ----------------------
 * Rank r of G holds the global slots [r*P, min((r+1)*P, C)), P = ceil(C/G);
 * store rows are independent, so every call is the single-GPU kernels on the
 * local slots followed by ONE all-gather of a packed per-rank result and a
 * merge on every rank: outputs are replicated on every rank and bit-identical
 * to the unsharded store (a row's score does not depend on its rank; ties
 * break by global id).  On a sharded store every call below is COLLECTIVE:
 * every rank calls it, in the same order, with the same arguments (replicated
 * queries / contexts, same k, ell, delta ...), except the cosine side outputs
 * and inputs (fmoe_search_semantic_cos, fmoe_search_blend_cos,
 * fmoe_store_insert_cos), which hold this rank's LOCAL columns
 * [0, local size), and fmoe_store_read / fmoe_store_write, which are local
 * (global slots; read needs a range inside this rank's shard).
 * fmoe_prefetch_plan returns FMOE_ERR_UNSUPPORTED on a sharded store. */
typedef enum {
  FMOE_TRANSPORT_NCCL = 0,   /* ncclAllGather on the call's stream (NVLink / NVSwitch; CUDA-graph capturable) */
  FMOE_TRANSPORT_HOST = 1    /* the caller's host all-gather (synchronous; e.g. gloo, or ranks sharing one GPU) */
} fmoe_transport;

/* HOST transport: gather `bytes` bytes of every rank's send (host memory) into
 * recv [world][bytes] in rank order; return 0 on success. */
typedef int32_t (*fmoe_allgather_fn)(const void* send, void* recv, int64_t bytes, void* user);

typedef struct {
  int32_t rank, world;            /* 0 <= rank < world                                       */
  int32_t transport;              /* fmoe_transport                                          */
  const void* nccl_unique_id;     /* NCCL: the 128 bytes of fmoe_get_nccl_unique_id, the same
                                     on every rank (the caller distributes them)             */
  fmoe_allgather_fn allgather;    /* HOST: the exchange                                       */
  void* allgather_user;
} fmoe_dist_config;

/* 128 bytes identifying a new NCCL communicator (call on one rank, share). */
fmoe_status fmoe_get_nccl_unique_id(void* out_128_bytes);

/* Create this rank's shard of a store of cfg->capacity GLOBAL slots
 * (cfg->id_offset must be 0; capacity >= world).  Collective (NCCL: every rank
 * initialises the communicator).  Errors: as fmoe_store_create; FMOE_ERR_CUDA
 * with the NCCL message when the communicator cannot be created. */
fmoe_status fmoe_store_create_sharded(const fmoe_store_config* cfg, const fmoe_dist_config* dist, int device,
                                      fmoe_store** out);

/* Copy the configuration the store was created with. */
fmoe_status fmoe_store_get_config(const fmoe_store* store, fmoe_store_config* out_cfg);

/* ---- insertion with RDY de-duplication ------------ */

/* Insert B new contexts: emb [B][D] fp32, maps [B][L][E] fp32 (gate rows).
 * The store quantises each row to its dtype (round-to-nearest-even) and keeps
 * 1/||row|| of the quantised embedding and the prefix norms of the map.
 * Rule (Reading R8): while |S| < capacity the context is appended to the next
 * slot; afterwards each remaining context x (batch order) replaces the old
 * context y* = argmax_y RDY_{x,y} (RDY = d/L*score^sem + (L-d)/L*score^map over
 * full maps) among the contexts that existed before this call and
 * are not yet claimed by an earlier row of the batch (ties -> lowest id).
 * Outputs: out_slot[B] = the slot (id) written, or -1 if no unclaimed slot was
 * left; out_replaced[B] = the id that was evicted (== out_slot) or -1 if the
 * row was appended.  Either output may be NULL.
 * Any number of rows may need replacement: they are resolved in sub-batches
 * of FMOE_MAX_K rows, each scanned against the pre-call store with the slots
 * earlier sub-batches claimed excluded (a device bitmap), which is the same
 * rule as one pass over the batch.  A zero-norm embedding is stored and
 * scores 0 against every query (Reading R3). */
fmoe_status fmoe_store_insert(fmoe_store* store, int64_t B, const float* emb, const float* maps,
                              int64_t* out_slot, int64_t* out_replaced, void* stream);

/* As fmoe_store_insert, with the semantic half of RDY supplied by the caller:
 * sem_cos [B][cos_stride] fp32 holds cos(emb_x, sem_y) for every context y
 * currently in the store (columns [0, size)), e.g. the out_cos of
 * fmoe_search_semantic_cos run on the same embeddings since the last insert.
 * An iteration's context carries the embedding its semantic search used
 * (P:459-461), so the RDY scan then reads only the maps instead of
 * the embeddings again.  Results are identical to fmoe_store_insert when
 * sem_cos holds those cosines; the caller guarantees that.  sem_cos NULL =
 * fmoe_store_insert.  cos_stride >= size. */
fmoe_status fmoe_store_insert_cos(fmoe_store* store, int64_t B, const float* emb, const float* maps,
                                  const float* sem_cos, int64_t cos_stride, int64_t* out_slot,
                                  int64_t* out_replaced, void* stream);

/* Overwrite existing contexts at explicit slots (the write half of an insert;
 * used by the sharded insert, SURVEY §8(e), and to restore a snapshot).
 * emb [B][D], maps [B][L][E] fp32, slot [B] int64 GLOBAL ids.  Rows whose slot
 * is -1 or lies outside [id_offset, id_offset + size) are skipped (that is how
 * each shard ignores the other shards' rows); appends go through
 * fmoe_store_insert.  Rows are quantised exactly as by fmoe_store_insert. */
fmoe_status fmoe_store_write(fmoe_store* store, int64_t B, const float* emb, const float* maps,
                             const int64_t* slot, void* stream);

/* Read back `count` slots from `slot_begin` as the fp32 values the store holds
 * (the quantised rows): out_emb [count][D], out_maps [count][L][E]; either
 * may be NULL.  (SPEC snapshot.) */
fmoe_status fmoe_store_read(const fmoe_store* store, int64_t slot_begin, int64_t count,
                            float* out_emb, float* out_maps, void* stream);

/* ---- search ------------------------------------------------- */

/* Semantic search, Eq. 1: score_{x,y} = cos(q_emb_x, sem_y).
 * q_emb [B][D] fp32.  Outputs out_score [B][k] fp32, out_id [B][k] int64.
 * 1 <= k <= FMOE_MAX_K.  A zero-norm query row gets (NaN, -1). */
fmoe_status fmoe_search_semantic(const fmoe_store* store, int64_t B, const float* q_emb, int32_t k,
                                 float* out_score, int64_t* out_id, void* stream);

/* fmoe_search_semantic that also writes every cosine: out_cos [B][cos_stride]
 * fp32, column y = score_{x,y} of Eq. 1 for the contexts y in [0, size);
 * cos_stride >= size (a multiple of 4 keeps the writes vectorised).  Feeds
 * fmoe_store_insert_cos. */
fmoe_status fmoe_search_semantic_cos(const fmoe_store* store, int64_t B, const float* q_emb, int32_t k,
                                     float* out_score, int64_t* out_id, float* out_cos, int64_t cos_stride,
                                     void* stream);

/* Trajectory search, Eq. 2: score_{x,y} = cos(flat(q_x[0:ell]),
 * flat(map_y[0:ell])) over the ell*E entries of the observed prefix (Reading
 * R1: ell = number of observed layers, 1 <= ell <= L; stored maps truncated).
 * q_prefix [B][ell][E] fp32 (row stride ell*E).  Outputs as semantic. */
fmoe_status fmoe_search_trajectory(const fmoe_store* store, int64_t B, const float* q_prefix,
                                   int32_t ell, int32_t k, float* out_score, int64_t* out_id,
                                   void* stream);

/* Blended search (Reading R4): score = w*score^sem + (1-w)*score^traj(ell),
 * the RDY weighting of P:544-551 with a caller weight; w_sem < 0 selects the
 * paper's d/L.  q_emb [B][D], q_prefix [B][ell][E]; 0 <= w_sem <= 1 or < 0. */
fmoe_status fmoe_search_blend(const fmoe_store* store, int64_t B, const float* q_emb,
                              const float* q_prefix, int32_t ell, float w_sem, int32_t k,
                              float* out_score, int64_t* out_id, void* stream);

/* fmoe_search_blend with the semantic half taken from the cosines a
 * semantic search of the same queries wrote (fmoe_search_semantic_cos:
 * sem_cos [B][cos_stride], cos_stride >= store size) instead of re-reading
 * the embeddings (P:544-551 blend): S = w*sem_cos +
 * (1-w)*S_traj(ell), w = w_sem (< 0 => d/L), 0 <= w < 1.  Equal to
 * fmoe_search_blend(q_emb, ...) when sem_cos came from
 * fmoe_search_semantic_cos(q_emb) on the unchanged store.  Query validity is
 * judged on the trajectory prefix only (a zero-norm embedding was reported by
 * the semantic search).  Pointers device or host, caller-owned. */
fmoe_status fmoe_search_blend_cos(const fmoe_store* store, int64_t B, const float* sem_cos, int64_t cos_stride,
                                  const float* q_prefix, int32_t ell, float w_sem, int32_t k, float* out_score,
                                  int64_t* out_id, void* stream);

/* ---- incremental trajectory search ---------------- */

/* A session follows B requests through the layers of one inference iteration:
 * step t (t = 0, 1, ...) consumes layer t of each query and returns the
 * trajectory search (Eq. 2) at prefix ell = t+1 -- the same result as
 * fmoe_search_trajectory on the prefix (summation order aside), but step t
 * reads only slab t of the store plus a running per-row dot product
 * (4 bytes per query and row, kept in the session), instead of t+1 slabs.
 * The session owns B*capacity*4 bytes of device memory.  Any insert/write to
 * the store invalidates it (the next step returns INVALID_ARG until reset).
 * Batched sessions (bf16 store, B >= 5) instead keep the query prefixes
 * (B*L*E*4 bytes) and run the tensor-core scan over the whole prefix each
 * step, seeded with the previous step's top-k ids (k distinct stored rows
 * whose scores bound the k-th best from below); results are identical to
 * fmoe_search_trajectory on the prefix.
 * 1 <= B <= 64. */
typedef struct fmoe_traj_session fmoe_traj_session;
fmoe_status fmoe_traj_session_create(const fmoe_store* store, int64_t B, fmoe_traj_session** out);
/* q_layer [B][E] fp32: layer t of every query.  Outputs as fmoe_search_trajectory. */
fmoe_status fmoe_traj_session_step(fmoe_traj_session* session, const float* q_layer, int32_t k,
                                   float* out_score, int64_t* out_id, void* stream);
/* A step followed by the selection of fmoe_select_experts on each
 * query's top-1 of this step (id out_id[x][0], score out_score[x][0]) for the
 * layers [layer_begin, layer_end): out_mask/out_count [B][layer_end -
 * layer_begin] exactly as fmoe_select_experts would write them.  Incremental
 * sessions run the selection in the step kernel's last block (no extra
 * launch, no dependent round trip); batched sessions launch the select kernel
 * after the scan.  All four outputs are required; delta, layer range and the
 * error cases as fmoe_select_experts; otherwise as fmoe_traj_session_step. */
fmoe_status fmoe_traj_session_step_select(fmoe_traj_session* session, const float* q_layer, int32_t k,
                                          float* out_score, int64_t* out_id, float delta, int32_t layer_begin,
                                          int32_t layer_end, uint64_t* out_mask, int32_t* out_count,
                                          void* stream);
/* n_steps consecutive steps of the session in ONE call: step s consumes layer
 * ell0 + s (ell0 = layers consumed so far) from q_layers [n_steps][B][E] fp32,
 * writes the top-1 (k = 1, "the highest score is selected") to
 * out_score / out_id [n_steps][B] and, when out_mask is non-NULL, the Eq. 4-6
 * selection (delta as in fmoe_select_experts) of target layer
 * ell0 + s + sel_d to out_mask / out_count [n_steps][B] (mask 0, count 0 when
 * the target is >= L).  Results are bit-identical to n_steps calls of
 * fmoe_traj_session_step_select(k = 1).  Fused path (B = 1, 16-byte slab rows
 * -- bf16 E <= 8 or fp32 E <= 4 -- and n <= 8 * 4 * SMs * 256 rows): one
 * kernel keeps the running dot products in registers across the steps.
 * Optional DEVICE flags (fused path only, else FMOE_ERR_UNSUPPORTED):
 * layer_ready [n_steps] -- step s starts once layer_ready[s] != 0 (written by
 * the producer of the gates, e.g. the MoE forward; the kernel waits, so the
 * producer must not need this kernel's SMs to make progress); guidance_ready
 * [n_steps] -- set to 1 (release) once step s's outputs are written: the
 * device-side publisher/subscriber of P:528-533.  A layer not ready within
 * 10 s abandons the sweep: the steps not finished publish guidance_ready = 2
 * (so a subscriber never waits forever), the session is poisoned until reset
 * (fmoe_traj_session_abandoned).  Sharded store: ready flags are unsupported. */
fmoe_status fmoe_traj_session_sweep(fmoe_traj_session* session, const float* q_layers, int32_t n_steps,
                                    float* out_score, int64_t* out_id, float delta, int32_t sel_d,
                                    uint64_t* out_mask, int32_t* out_count, const uint32_t* layer_ready,
                                    uint32_t* guidance_ready, void* stream);
/* Start a new prefix (next step consumes layer 0); re-validates against the store. */
fmoe_status fmoe_traj_session_reset(fmoe_traj_session* session);
void fmoe_traj_session_destroy(fmoe_traj_session* session);

/* ---- similarity-aware expert selection ----------------------- */

/* For each query x with matched context map_id[x] (-1 = none) and its score:
 * delta_x = Clip(1 - score[x], 0, 1) (score clamped to [-1,1], NaN
 * -> 1) when delta < 0, else the fixed threshold delta in [0,1].  For each
 * layer t in [layer_begin, layer_end): sort P_{map_id,t} by (p desc, index asc),
 * accumulate in float64 in that order and stop at the first count with
 * cum >= delta and count >= K; all E if never reached (Eq. 4-6, Reading R7).
 * Outputs out_mask [B][T] uint64 (bit j = expert j prefetched), out_count
 * [B][T] int32, T = layer_end - layer_begin.  A map_id outside this store
 * (-1, or another shard's id) gives mask 0, count 0.  score may be NULL when
 * delta >= 0. */
fmoe_status fmoe_select_experts(const fmoe_store* store, int64_t B, const int64_t* map_id,
                                const float* score, float delta, int32_t layer_begin,
                                int32_t layer_end, uint64_t* out_mask, int32_t* out_count,
                                void* stream);

/* ---- expert-cache priorities ------------ */

/* Prefetch plan: for each query, every expert of the Eq. 4-6 prefetch set of
 * each target layer t in [layer_begin, layer_end) of its matched map
 * (selection exactly as fmoe_select_experts, same delta rule), with
 * PRI^prefetch = p_{t,j} / (t - l_now) in float64, ordered by
 * priority descending, ties -> lower layer, then lower expert.
 * Outputs [B][max_jobs]: out_layer, out_expert (int32, -1 past the end),
 * out_priority (float64); out_njobs [B] (jobs beyond max_jobs are dropped).
 * Requires l_now < layer_begin and (layer_end - layer_begin) * E <= 2048. */
fmoe_status fmoe_prefetch_plan(const fmoe_store* store, int64_t B, const int64_t* map_id, const float* score,
                               float delta, int32_t l_now, int32_t layer_begin, int32_t layer_end,
                               int32_t max_jobs, int32_t* out_layer, int32_t* out_expert, double* out_priority,
                               int32_t* out_njobs, void* stream);

/* Expert prefetch copies driven by the guidance (P:528-533 publisher/
 * subscriber, P:573-580 PRI^prefetch, P:595-597 loading the experts of the
 * next layers, P:618-619 expert management through the CUDA runtime).  On
 * `copy_stream`: optionally wait (on the device, cuStreamWaitValue32) until
 * the DEVICE flag `wait_flag` >= 1 -- e.g. guidance_ready[s] of a session
 * sweep --, run fmoe_prefetch_plan for queries [B] (map_id, score: DEVICE
 * arrays the guidance wrote, read after the wait), bring the jobs to the host,
 * then issue ONE cudaMemcpyAsync per job, in plan order (priority descending),
 * host_expert[t*E + j] -> dev_expert[t*E + j] of expert_bytes bytes, skipping
 * experts whose bit j is set in resident_mask[t] (host, [L], may be NULL; the
 * call sets the bits of the experts it copies).  The calling thread blocks
 * until the plan is known (the copies themselves are asynchronous on
 * copy_stream): a copy-manager thread of a serving system.  host_expert must
 * be pinned for the copies to overlap.  Outputs (host, may be NULL):
 * out_layer / out_expert [B][max_jobs] of the jobs issued (-1 past the end),
 * out_njobs [B].  Same argument rules as fmoe_prefetch_plan; not for sharded
 * stores.  FMOE_ERR_UNSUPPORTED if the device lacks stream memory operations
 * (wait_flag given).  A device-side wait blocks the hardware queue copy_stream
 * maps to: the flag's producer must already be enqueued (or run on a stream
 * that cannot share that queue), else the two wait on each other -- a
 * copy-manager thread that learns of the guidance later waits on the host
 * (an event) and passes wait_flag = NULL. */
fmoe_status fmoe_prefetch_issue(const fmoe_store* store, int64_t B, const int64_t* map_id, const float* score,
                                float delta, int32_t l_now, int32_t layer_begin, int32_t layer_end, int32_t max_jobs,
                                const void* const* host_expert, void* const* dev_expert, int64_t expert_bytes,
                                uint64_t* resident_mask, const uint32_t* wait_flag, void* copy_stream,
                                int32_t* out_layer, int32_t* out_expert, int32_t* out_njobs);

/* Eviction order of n cached experts: PRI^evict = 1 / (max(p, eps)
 * * freq) in float64 (p floored at eps, Reading R13), and out_order [n]
 * = cache indices by priority descending, ties -> lower index (= earlier
 * inserted).  p, freq [n] fp32; out_priority [n] float64.  1 <= n <= 8192. */
fmoe_status fmoe_eviction_order(int64_t n, const float* p, const float* freq, float eps, double* out_priority,
                                int32_t* out_order, int device, void* stream);

/* ---- expert hit count of prefetch guidance -------- */

/* For each row r = (query x, layer t) of gate [B][T][E] fp32 (the query's own
 * observed gate probabilities, finite), the activated experts A_r = the K
 * largest probabilities, ties -> lower index (top-K routing, Table 1 K,
 * Reading R14), and out_hits [B][T] int32 = popcount(A_r & prefetch_mask[r])
 * (prefetch_mask [B][T] uint64, bit j = expert j prefetched, e.g. the output
 * of fmoe_select_experts).  out_active [B][T] uint64 (may be NULL) receives
 * A_r.  Hit rate = sum(out_hits) / (B*T*K) (every layer activates K).
 * 1 <= K <= E <= 64, T >= 1; B == 0 is a no-op.  Pointers device (stream-
 * ordered) or host (staged), caller-owned. */
fmoe_status fmoe_expert_hits(int64_t B, int32_t T, int32_t E, int32_t K, const float* gate,
                             const uint64_t* prefetch_mask, uint64_t* out_active, int32_t* out_hits, int device,
                             void* stream);

/* ---- sharded merge ---------------------------------------- */

/* Merge n_lists candidate lists per query into the global top-k: scores
 * [n_lists][B][k_in] fp32, ids [n_lists][B][k_in] int64 (the layout of an
 * all-gather of per-rank search outputs), ordered (score desc, id asc); a NaN
 * anywhere in a query's lists marks the query invalid -> (NaN, -1).  Entries
 * with id -1 are ignored.  1 <= k <= FMOE_MAX_K, 1 <= k_in <= FMOE_MAX_K. */
fmoe_status fmoe_topk_merge(int64_t B, int32_t n_lists, int32_t k_in, const float* scores,
                            const int64_t* ids, int32_t k, float* out_score, int64_t* out_id,
                            int device, void* stream);

/* Victim resolution of the RDY insert (Reading R8): ids [B][k] are
 * each new row's candidate old contexts, best first (e.g. the merged output of
 * per-shard RDY searches).  Row j, in batch order, takes its first id not taken
 * by an earlier row; -1 if none.  out_victim [B].  1 <= k <= FMOE_MAX_K,
 * B <= FMOE_MAX_K. */
fmoe_status fmoe_resolve_victims(int64_t B, int32_t k, const int64_t* ids, int64_t* out_victim,
                                 int device, void* stream);

/* ---- host-buffer completion ---------------------------------------------- */
/* Calls may take host arrays (staged through device buffers on the call's
 * stream).  enable != 0 (the default): a call with a host OUTPUT synchronises
 * its stream before returning, so the output is ready on return.  enable == 0:
 * the H2D/D2H copies are only enqueued (stream order), the call returns at
 * once, and the caller synchronises the stream before reading host outputs
 * and keeps host inputs unchanged until then (pinned memory makes the copies
 * truly asynchronous; with pageable memory the copies themselves block).  A
 * host output of one call may be passed as a host input of a later call on
 * the same stream: the copies are stream-ordered.  Process-wide; returns the
 * previous setting. */
int32_t fmoe_set_host_sync(int32_t enable);

/* Whether a session sweep with device flags was abandoned (a layer_ready flag
 * not set within 10 s) since the session's last reset: the steps it did not
 * finish published guidance_ready = 2, and every later step of the session
 * reports (NaN, -1) until fmoe_traj_session_reset.  Reads a device word: call
 * after synchronising the sweep's stream. */
fmoe_status fmoe_traj_session_abandoned(const fmoe_traj_session* session, int32_t* out_abandoned);

/* ---- diagnostics --------------------------------------------------------- */
const char* fmoe_status_string(fmoe_status s);
/* Message of the last error on the calling thread ("" if none). */
const char* fmoe_last_error(void);
/* Number of kernels this library has launched in this process (a counter the
 * bench reports as gpu_launches). */
int64_t fmoe_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FMOE_H_ */
