/* SPDX-License-Identifier: Apache-2.0
 *
 * pikv_b200.h — C-ABI of the B200-native PiKV decode engine.
 *
 * This is the drop-in boundary for the reference's decode path
 * (`pikv::Engine::step`, /root/reference/proj/src/pipeline.cpp:213-351) and
 * the free functions it is built from.  Every entry point names the reference
 * interface it replaces.  Signatures use plain pointers and sizes only; all
 * device buffers are caller-owned CUDA device pointers unless the name ends
 * in `_host`.  Store memory (paged KV pool, slot metadata) is owned by the
 * engine.
 *
 * Error convention: every call returns an int status.  0 is success; the
 * non-zero codes map 1:1 onto the reference's exception classes
 * (/root/reference/proj/include/pikv/errors.hpp:9-47) plus CUDA/NCCL/OOM.
 * `pikv_last_error()` returns the message of the last failure on the calling
 * thread.  A failing step leaves no partial state (pipeline.cpp:153-154).
 *
 * Threading: an engine is single-writer; calls are
 * stream-ordered on the engine's CUDA stream and not thread-safe per engine.
 */
#ifndef PIKV_B200_H
#define PIKV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:9-47) ---------------------------------- */
#define PIKV_OK 0
#define PIKV_ERR_INVALID_ARGUMENT 1        /* pikv::InvalidArgument  errors.hpp:13 */
#define PIKV_ERR_INVALID_CONFIG 2          /* pikv::InvalidConfig    errors.hpp:17 */
#define PIKV_ERR_INVALID_ENTRY 3           /* pikv::InvalidEntry     errors.hpp:21 */
#define PIKV_ERR_NUMERICAL 4               /* pikv::NumericalError   errors.hpp:25 */
#define PIKV_ERR_CODEC_MISMATCH 5          /* pikv::CodecMismatch    errors.hpp:29 */
#define PIKV_ERR_NOT_FITTED 6              /* pikv::NotFitted        errors.hpp:33 */
#define PIKV_ERR_INSUFFICIENT_CALIBRATION 7
#define PIKV_ERR_INVALID_COMPARISON 8
#define PIKV_ERR_IO 9
#define PIKV_ERR_CUDA 10
#define PIKV_ERR_NCCL 11
#define PIKV_ERR_OUT_OF_MEMORY 12          /* KV page pool exhausted */

/* ---- enums (same order as the reference enums) ------------------------ */
/* RouterStrategy, router.hpp:11-19 */
#define PIKV_ROUTER_BASE 0
#define PIKV_ROUTER_TOPK 1
#define PIKV_ROUTER_LOAD_BALANCED 2
#define PIKV_ROUTER_CACHE_AWARE 3
#define PIKV_ROUTER_ENTROPY_LB 4
#define PIKV_ROUTER_ADAPTIVE 5
#define PIKV_ROUTER_HIERARCHICAL 6
/* SchedStrategy, scheduler.hpp:16-25 (QUEST is out of scope: needs an Eigen fit) */
#define PIKV_SCHED_H2O 0
#define PIKV_SCHED_SL 1
#define PIKV_SCHED_QUEST 2
#define PIKV_SCHED_FLEX 3
#define PIKV_SCHED_LRU 4
#define PIKV_SCHED_LRU_PLUS 5
#define PIKV_SCHED_ADAKV 6
#define PIKV_SCHED_DUO 7
/* EvictReason, scheduler.hpp:87 */
#define PIKV_EVICT_BUDGET 0
#define PIKV_EVICT_THRESHOLD 1
#define PIKV_EVICT_OVERWRITE 2
/* Stored-entry codecs.  IDENTITY/LOWRANK/LORAPLUS/FASTV/PRUNE follow the
 * reference's projection schemes (compressor.cpp:318-474) with one basis per
 * head; INT8/INT4 are this engine's quantizers (not in the reference,
 * SPEC.md:331). */
#define PIKV_CODEC_IDENTITY 0
#define PIKV_CODEC_LOWRANK 1   /* Scheme::SVD / Scheme::LoRA: y = B^T x     */
#define PIKV_CODEC_LORAPLUS 2  /* Scheme::LoRAPlus: y = B^T (x - bias)      */
#define PIKV_CODEC_FASTV 3     /* Scheme::FastV: keep the first r coords     */
#define PIKV_CODEC_PRUNE 4     /* Scheme::Prune: keep sorted coords `kept`   */
#define PIKV_CODEC_INT8 5      /* symmetric absmax per (entry, head)         */
#define PIKV_CODEC_INT4 6      /* symmetric absmax per (entry, head), packed */
/* input / storage dtypes */
#define PIKV_DTYPE_F32 0
#define PIKV_DTYPE_BF16 1

/* ---- configuration ------------------------------------------------------
 * One flat POD mirroring EngineConfig (pipeline.hpp:87-98) and the configs
 * it aggregates.  Field meanings follow the reference; extra fields are the
 * batch/multi-head/runtime knobs the reference does not have.             */
typedef struct pikv_config {
    /* ModelConfig, config.hpp:23-55 */
    int32_t d;            /* query/key/value width before compression       */
    int32_t head_width;   /* h: fetch-cost model only (pipeline.cpp:22-26)  */
    int32_t E;            /* experts                                         */
    int32_t k;            /* active experts per token (RouterConfig.k too)   */
    int64_t L;            /* token budget (cost model only)                  */
    int32_t G;            /* devices of shard_assign (kvstore.cpp:14-30)     */
    int32_t S;            /* shard ring capacity                             */
    int32_t K;            /* ModelConfig.K (cost model only)                 */
    int32_t elem_bytes;   /* bytes per stored scalar for memory_bytes()      */
    double rho;           /* d / d'                                          */
    /* multi-head convention: H independent heads of width
     * d/H; attention is per head, attn_mass += mean over heads of alpha.   */
    int32_t n_heads;
    /* StoreConfig, kvstore.hpp:63-72 */
    int32_t n_tok, n_exp, additive, shards_per_device;
    /* RouterConfig, router.hpp:24-37 */
    int32_t router_strategy, groups, stride;
    double alpha, lambda_miss, beta_ent, bandit_step, bias_cap, load_decay;
    /* SchedulerConfig, scheduler.hpp:30-47 */
    int32_t sched_strategy, budget_pages, page_size, sink, flex_bucket;
    int32_t n_adakv_weights, n_flex_plan;
    double tau, lambda_freq, adakv_step, target_hit, gamma_sim, theta0, hit_decay;
    double adakv_weights[8];
    double flex_plan[32];
    /* CompressorConfig, compressor.hpp:28-41 (runtime part only) */
    int32_t codec;        /* PIKV_CODEC_*                                    */
    int32_t rank;         /* r per head for LOWRANK/LORAPLUS/FASTV/PRUNE     */
    /* EngineConfig, pipeline.hpp:87-98 */
    int32_t unbounded_budget;
    int32_t n_layers;     /* width of per_layer_scores (TokenInput.layer_saliency) */
    /* B200 runtime (no reference counterpart) */
    int32_t batch;        /* B independent decode streams     */
    int32_t kv_dtype;     /* PIKV_DTYPE_*: dtype of q/k/v inputs and of the
                             stored identity/low-rank payload               */
    int32_t world_size;   /* ranks; rank r owns devices g with g % world == r */
    int32_t rank_id;
    int64_t pool_entries; /* KV page pool capacity in entries (0 = auto)     */
    uint64_t seed;        /* EngineConfig.seed: W_r = Rng(seed ^ kRouterSalt) */
    /* PIKV_ROUTE_EXACT: logits as the reference's sequential fp64 sum
     * (router.cpp:224-229, bit-exact routing); PIKV_ROUTE_FAST: the same fp64
     * products reduced as a tree (FMA) -- rounding-order differences only,
     * routing flips only on near-ties (tests report the rate), ~10x lower
     * route latency. */
    int32_t route_mode;
    int32_t reserved0;
} pikv_config;

#define PIKV_ROUTE_EXACT 0
#define PIKV_ROUTE_FAST 1

/* One eviction record, scheduler.hpp:90-98 (+ the stream it belongs to). */
typedef struct pikv_evict_record {
    uint64_t step;
    uint64_t entry_id;
    int64_t token_id;
    int32_t expert_id;
    int32_t device;
    double score;
    int32_t reason;     /* PIKV_EVICT_* */
    int32_t stream;
} pikv_evict_record;

/* One KV entry's identity and metadata: KVEntry (types.hpp:27-34) minus its
 * key/value vectors, with EntryMeta (types.hpp:11-24) inlined.  id and
 * shard_seq are assigned by the store on insert (kvstore.cpp:114-115). */
typedef struct pikv_entry {
    uint64_t id;
    uint64_t shard_seq;
    int64_t token_id;
    int32_t expert_id;
    int32_t has_layers;        /* per_layer_scores non-empty (n_layers values) */
    uint64_t insert_step;
    uint64_t last_access_step;
    uint64_t freq;
    double attn_mass;
} pikv_entry;

/* One live entry of the store, KVStore::snapshot (kvstore.hpp:89-96). */
typedef struct pikv_snapshot_record {
    int32_t device;
    int32_t shard;      /* shard index within the device */
    int64_t token_id;
    int32_t expert_id;
    int32_t reserved;
    uint64_t age;       /* now - insert_step (0 when negative), types.hpp:19-21 */
    uint64_t freq;
} pikv_snapshot_record;

/* Per-stream summary of the last step (StepResult, pipeline.hpp:68-80). */
typedef struct pikv_step_summary {
    uint64_t step;
    int32_t inserts;
    int32_t hits;
    int32_t lookups;
    int32_t n_attended;      /* attn.retrieved                              */
    int64_t fetch_elements;  /* pipeline.cpp:262-264                         */
    int32_t n_evictions;     /* overwrite + scheduled                         */
    int32_t pages_before;    /* EvictionReport, scheduler.hpp:100-104        */
    int32_t pages_after;
    int32_t error;           /* per-stream PIKV_ERR_* raised on device        */
} pikv_step_summary;

typedef struct pikv_engine pikv_engine;

/* ---- library --------------------------------------------------------- */
const char* pikv_version(void);
const char* pikv_last_error(void);
int pikv_config_size(void);                 /* sizeof(pikv_config) for FFI checks */
/* Fills `cfg` with the reference defaults (config.hpp, kvstore.hpp:63-72,
 * router.hpp:24-37, scheduler.hpp:30-47, compressor.hpp:28-41). */
void pikv_config_default(pikv_config* cfg);

/* ---- pure functions (device kernels over arrays) ----------------------- */
/* shard_assign, kvstore.cpp:14-30, for n (t, e) pairs; outputs device/shard/raw. */
int pikv_shard_assign(const int64_t* t, const int32_t* e, int32_t n, int32_t n_tok,
                      int32_t n_exp, int32_t devices, int32_t additive,
                      int32_t* device_out, int32_t* shard_out, int32_t* raw_out);
/* select_evictions, scheduler.cpp:231-260, on one device's page list.
 * Writes up to n victims (page index, reason) in eviction order. */
int pikv_select_evictions(const double* aggregate, const uint64_t* oldest_id,
                          int32_t n, int32_t budget_pages, int32_t use_theta,
                          double theta, int32_t* idx_out, int32_t* reason_out,
                          int32_t* n_out);
/* attention, pipeline.cpp:59-85, for `n_queries` independent single-head
 * problems of width w over n entries each (fp32 in/out; fp64 not used). */
int pikv_attention(const float* q, const float* keys, const float* values,
                   int32_t n_queries, int32_t n, int32_t w, float* y_out,
                   float* weights_out);
/* int8/int4 codes (this engine's quantizer; oracle/pikv_oracle.c restates it). */
int pikv_quantize(const void* x, int32_t dtype, int32_t rows, int32_t width,
                  int32_t bits, uint8_t* codes_out, float* scales_out);
int pikv_dequantize(const uint8_t* codes, const float* scales, int32_t rows,
                    int32_t width, int32_t bits, float* x_out);
/* Codec::project_encode / project_decode, compressor.cpp:318-340, per head:
 * x [rows][H*hd] -> y [rows][H*r] with basis [H][r][hd] (column j of the
 * reference's col-major d x r basis is basis[h][j][:]). */
int pikv_lowrank_encode(const float* x, const float* basis, const float* bias,
                        int32_t rows, int32_t heads, int32_t hd, int32_t r, float* y_out);
int pikv_lowrank_decode(const float* y, const float* basis, const float* bias,
                        int32_t rows, int32_t heads, int32_t hd, int32_t r, float* x_out);

/* Host-buffer variants of the above (copy in, run the same kernels, copy
 * out); used by the C++ facade include/pikv_b200.hpp. */
int pikv_shard_assign_host(const int64_t* t, const int32_t* e, int32_t n, int32_t n_tok,
                           int32_t n_exp, int32_t devices, int32_t additive,
                           int32_t* device_out, int32_t* shard_out, int32_t* raw_out);
int pikv_select_evictions_host(const double* aggregate, const uint64_t* oldest_id, int32_t n,
                               int32_t budget_pages, int32_t use_theta, double theta,
                               int32_t* idx_out, int32_t* reason_out, int32_t* n_out);
int pikv_attention_host(const float* q, const float* keys, const float* values,
                        int32_t n_queries, int32_t n, int32_t w, float* y_out,
                        float* weights_out);

/* ---- engine (Engine, pipeline.hpp:101-145) ------------------------------ */
int pikv_engine_create(const pikv_config* cfg, int32_t cuda_device, pikv_engine** out);
int pikv_engine_destroy(pikv_engine* eng);
/* The engine's CUDA stream (cudaStream_t) all calls are ordered on. */
void* pikv_engine_stream(pikv_engine* eng);
/* RouterState::init(E, d, seed ^ kRouterSalt) (router.cpp:54-67,
 * pipeline.cpp:16,91) is done at create; this overrides W_r (E x d, fp64,
 * host, row-major) for all streams. */
int pikv_set_router_matrix_host(pikv_engine* eng, const double* w_r);
/* Codec parameters (host): basis [H][r][hd] fp32, bias [d] fp32 (LoRAPlus),
 * kept [H][r] int32 (Prune). Pass NULL for unused ones. */
int pikv_set_codec_host(pikv_engine* eng, const float* basis, const float* bias,
                        const int32_t* kept);

/* Engine::step for all B streams.  q/k/v: device [B][d] in cfg.kv_dtype;
 * saliency: device [B][n_layers] fp64 or NULL; y_out: device [B][d'] fp32
 * (attention output in compressed space, pipeline.cpp:295-299).  Enqueued on
 * the engine stream; no host synchronisation. */
int pikv_step(pikv_engine* eng, const void* q, const void* k, const void* v,
              const double* saliency, float* y_out);
/* Same step through HOST buffers (pinned or pageable): copies the inputs in,
 * runs the step and copies y back, synchronising before returning. */
int pikv_step_host(pikv_engine* eng, const void* q, const void* k, const void* v,
                   const double* saliency, float* y_out);
/* Engine::step(TokenInput) from the tokens' embeddings, pipeline.cpp:213-351
 * including the encode at :222: the QueryEncoder (pipeline.cpp:29-57; seeded
 * like the reference, cfg.seed ^ 0x71c9de52ae0aef, unless replaced by
 * pikv_set_encoder_host) runs on the GPU in fp64 with the reference's
 * summation order, so routing is bit-exact; K/V are stored in cfg.kv_dtype.
 * emb: device [B][d] fp64 (pikv_step_embed) or host (pikv_step_embed_host). */
int pikv_step_embed(pikv_engine* eng, const double* emb, const double* saliency, float* y_out);
int pikv_step_embed_host(pikv_engine* eng, const double* emb, const double* saliency,
                         float* y_out);
/* Replace the QueryEncoder's matrices (each [d][d] row-major fp64, host). */
int pikv_set_encoder_host(pikv_engine* eng, const double* w_query, const double* w_key,
                          const double* w_value);
/* ---- multi-GPU (expert-sharded store, SURVEY 8 e) ---------------------
 * Rank r of world_size owns the logical devices g with g % world == r.
 * With NCCL attached, pikv_step / pikv_step_host / pikv_prefill_synthetic /
 * the group run the whole sharded step, the all-gather of the per-stream LSE
 * records (B x pikv_exchange_bytes()/B bytes) enqueued on the engine stream
 * inside the captured step graph, then the cross-rank merge on every rank.
 * pikv_nccl_unique_id: rank 0 creates the id, the caller broadcasts its
 * PIKV_NCCL_ID_BYTES bytes; pikv_engine_attach_nccl is collective over the
 * ranks (ncclCommInitRank with world_size / rank_id of the config).
 * pikv_engine_set_nccl_comm takes a caller-owned ncclComm_t instead (NULL
 * detaches).  A one-rank communicator runs the same exchange path. */
#define PIKV_NCCL_ID_BYTES 128
int pikv_nccl_unique_id(uint8_t* id_out);
int pikv_engine_attach_nccl(pikv_engine* eng, const uint8_t* id);
int pikv_engine_set_nccl_comm(pikv_engine* eng, void* nccl_comm);
/* Attended entries of this rank's last step, summed over streams (the KV this
 * rank's attention kernel read; the summaries carry the global counts). */
int64_t pikv_local_attended(pikv_engine* eng);
/* Without NCCL: the rank-local part, an all-gather the caller provides (any
 * transport) into [world][exchange] device memory, then the finish.  The
 * exchange buffer is device memory of pikv_exchange_bytes() per rank. */
int64_t pikv_exchange_bytes(pikv_engine* eng);
int pikv_step_local(pikv_engine* eng, const void* q, const void* k, const void* v,
                    const double* saliency, void** exchange_out);
int pikv_step_finish(pikv_engine* eng, const void* gathered /* [world][exchange] */,
                     float* y_out);
/* Prefill `tokens` decode steps without attention (store synthesis for
 * benchmarks): synthetic q/k/v ~ N(0,1) rounded to kv_dtype, generated on the
 * device from `seed`.  Route/insert/evict/retrieve all run as in step(). */
int pikv_prefill_synthetic(pikv_engine* eng, int64_t tokens, uint64_t seed);
/* Device-side synthetic inputs for one step ([B][d] each, kv_dtype). */
int pikv_fill_synthetic(pikv_engine* eng, void* q, void* k, void* v, uint64_t seed);
int pikv_sync(pikv_engine* eng);

/* ---- results / state readback (host) -------------------------------- */
/* experts [B][k] int32, gates [B][k] f64, logits [B][E] f64, summary [B].
 * Any pointer may be NULL.  Synchronises. */
int pikv_read_step_host(pikv_engine* eng, int32_t* experts, double* gates,
                        double* logits, pikv_step_summary* summary);
/* Eviction records of the last step for all streams, reference order per
 * stream (overwrites, then per device the scheduled victims): at most cap
 * written, *n_out = the step's total (cap 0 queries the count). */
int pikv_read_evictions_host(pikv_engine* eng, pikv_evict_record* out, int32_t cap,
                             int32_t* n_out);
/* Attended entries of the last step of `stream`: (token, expert, alpha) in
 * this engine's (ring, slot) order; the reference orders by (token, expert). */
int pikv_read_attended_host(pikv_engine* eng, int32_t stream, int64_t* token,
                            int32_t* expert, double* alpha, int32_t cap,
                            int32_t* n_out);
/* The store build of a prefill: T tokens of `stream` with
 * their experts given (experts [T][k], selection order) -- token t is step
 * now + t -- are encoded with the engine's codec and inserted exactly as T
 * Engine::step inserts would (pipeline.cpp:148-211, kvstore.cpp:107-120:
 * ids in order, ring overwrite, metadata insert_step = last_access = step),
 * without routing, eviction or retrieval; now advances by T.  Runs as bulk
 * kernels: entries placed straight at their final ring slots, pages built
 * once, LowRank/LoRAPlus projections as one GEMM over all T rows (tcgen05 on
 * sm_100a).  k, v: [T][d] in kv_dtype; saliency [T][n_layers] fp64 or NULL;
 * *n_displaced = KVStore::insert displacements.  Device buffers
 * (pikv_insert_bulk) or host buffers (pikv_insert_bulk_host). */
int pikv_insert_bulk(pikv_engine* eng, int32_t stream, int64_t T, const void* k, const void* v,
                     const int32_t* experts, const double* saliency, int64_t* n_displaced);
int pikv_insert_bulk_host(pikv_engine* eng, int32_t stream, int64_t T, const void* k, const void* v,
                          const int32_t* experts, const double* saliency, int64_t* n_displaced);
/* generate_trace (trace.cpp:54-82) with TraceSpec{steps, width, vocab,
 * zipf_skew, seed, layers} (trace.hpp:12-21; errors per TraceSpec::validate):
 * the vocabulary [vocab][width] fp64, each step's embedding id [steps] and
 * per-layer saliency [steps][layers].  Any output pointer may be NULL. */
int pikv_generate_trace(uint64_t steps, int32_t width, int32_t vocab, double zipf_skew,
                        uint64_t seed, int32_t layers, double* vocab_out, uint32_t* embed_ids,
                        float* saliency);
/* KVStore::snapshot(now) (kvstore.cpp:206-221) of `stream`: its live entries
 * on this rank's devices, sorted by (device, shard, token, expert), computed
 * on the GPU.  now < 0 takes the stream's current step.  *n_out = number of
 * live entries; at most cap records are written. */
int pikv_snapshot_host(pikv_engine* eng, int32_t stream, int64_t now, pikv_snapshot_record* out,
                       int64_t cap, int64_t* n_out);
/* Slot metadata of `stream` for its owned devices:
 * [G_local][SPD][S] arrays; id 0 marks an empty slot.  Any pointer may be NULL. */
int64_t pikv_slot_count(pikv_engine* eng);
int pikv_read_slots_host(pikv_engine* eng, int32_t stream, uint64_t* id,
                         uint64_t* shard_seq, int64_t* token, int32_t* expert,
                         uint64_t* insert_step, uint64_t* last_access,
                         uint64_t* freq, double* attn_mass, double* per_layer);
/* Stored K and V of n slots of `stream` (stream-local slot index, the
 * pikv_read_slots_host order) decoded to fp32 -- the values attention reads:
 * KVEntry::key / value (types.hpp:27-34) in the stored width d'.  Empty
 * slots read as zeros.  key_out / value_out: [n][d'] host. */
int pikv_read_entries_host(pikv_engine* eng, int32_t stream, const int64_t* slots, int32_t n,
                           float* key_out, float* value_out);
/* Overwrite attn_mass (and optionally per_layer) of `stream`'s slots, to
 * inject identical metadata for step-local parity of H2O/AdaKV/Duo. */
int pikv_write_attn_mass_host(pikv_engine* eng, int32_t stream,
                              const double* attn_mass, const double* per_layer);
/* RouterState (router.hpp:41-56) and SchedulerState (scheduler.hpp:49-56). */
int pikv_read_router_state_host(pikv_engine* eng, int32_t stream, double* load,
                                uint64_t* usage, uint64_t* miss, double* bias,
                                uint64_t* step, uint64_t* total_usage);
int pikv_read_sched_state_host(pikv_engine* eng, int32_t stream, double* theta,
                               double* running_hit, uint64_t* step);
/* KVStore::live_entries / memory_bytes (kvstore.cpp:187-196) per stream,
 * and the pool's allocated page count. */
int pikv_store_stats_host(pikv_engine* eng, int32_t stream, uint64_t* live,
                          uint64_t* memory_bytes, uint64_t* inserts,
                          uint64_t* overwrites);
int64_t pikv_pool_pages_in_use(pikv_engine* eng);
/* Bytes of one stored entry (K + V payload + scales) and entries per page. */
int64_t pikv_entry_bytes(pikv_engine* eng);
/* Launch statistics: number of kernels this engine enqueued so far. */
int64_t pikv_kernel_launches(pikv_engine* eng);
/* Profiling mode: steps run eagerly (no graph) with CUDA events on the engine
 * stream between kernels.  pikv_read_profile_host returns the summed ms of
 * each kernel over the profiled steps: [route, insert, sched_pages,
 * sched_select, retr_count, retr_scan, retr_write, attend, combine,
 * finish_merge, foldback, feedback] (n_phases <= 12) and resets them. */
int pikv_set_profiling(pikv_engine* eng, int32_t on);
int pikv_read_profile_host(pikv_engine* eng, float* phase_ms, int32_t n_phases,
                           int32_t* n_steps);

/* ---- component API: the reference's free functions and classes ----------
 * The reference exposes its pieces individually (kvstore.hpp, router.hpp,
 * scheduler.hpp, compressor.hpp, pipeline.hpp:46-47); these entry points run
 * them on the GPU against ONE stream of an engine -- the same HBM store,
 * RouterState and SchedulerState Engine::step uses.  Host buffers,
 * synchronous, world_size 1.  Vectors in the stored space are fp32 of width
 * d' (KVEntry::key/value, types.hpp:27-34); slots are stream-local indices
 * (the pikv_read_slots_host order). */

/* Router / scheduler coefficients and strategies of later calls (route(q,
 * state, cfg) takes its RouterConfig per call, router.hpp:64-66); structural
 * fields (d, E, k, G, S, heads, store/codec layout, batch) must be unchanged. */
int pikv_update_config(pikv_engine* eng, const pikv_config* cfg);
/* route (router.cpp:216-234): exact fp64 W_r q, penalty, selection, gates,
 * note_selection.  query [d] fp64 (NULL allowed for Base).  experts [k],
 * gates [k], logits [E] (RoutingDecision, router.hpp:58-62); any out may be
 * NULL.  NaN logits -> PIKV_ERR_NUMERICAL with the state unchanged. */
int pikv_route_host(pikv_engine* eng, int32_t stream, const double* query, int32_t* experts,
                    double* gates, double* logits);
/* route_logits (router.cpp:122-214) on caller logits [E]. */
int pikv_route_logits_host(pikv_engine* eng, int32_t stream, const double* logits_in,
                           int32_t* experts, double* gates, double* logits);
int pikv_record_miss(pikv_engine* eng, int32_t stream, int32_t expert);     /* router.cpp:236-241 */
int pikv_router_adapt(pikv_engine* eng, int32_t stream, const int32_t* experts, int32_t n,
                      double reward);                                       /* router.cpp:243-255 */
/* RouterState / SchedulerState overwrite (any pointer NULL = keep). */
int pikv_write_router_state_host(pikv_engine* eng, int32_t stream, const double* load,
                                 const uint64_t* usage, const uint64_t* miss, const double* bias,
                                 const uint64_t* step, const uint64_t* total_usage);
int pikv_write_sched_state_host(pikv_engine* eng, int32_t stream, const double* theta,
                                const double* running_hit, const uint64_t* step);
/* KVStore::insert (kvstore.cpp:107-120) of n entries in order: entries[j]
 * carries (token, expert, EntryMeta); key/value [n][d'] fp32 in the stored
 * space (kv_dtype values, or quantized for INT8/INT4); per_layer [n][n_layers]
 * or NULL.  Displaced entries (full ring, kvstore.cpp:41-43) come back in
 * displaced[j] / displaced_key/value[j] / displaced_layers[j] with
 * displaced_flag[j] = 1.  Any output may be NULL. */
int pikv_store_insert_host(pikv_engine* eng, int32_t stream, int32_t n, const pikv_entry* entries,
                           const float* key, const float* value, const double* per_layer,
                           pikv_entry* displaced, float* displaced_key, float* displaced_value,
                           double* displaced_layers, int32_t* displaced_flag);
/* KVStore::retrieve (kvstore.cpp:122-178): live entries with expert in the
 * set and token < since, ordered by (token, expert); freq += 1 and
 * last_access = now for each; *n_out = count, slots_out = their slots (at
 * most cap), missed_out = experts with no hit (given order). */
int pikv_store_retrieve_host(pikv_engine* eng, int32_t stream, const int32_t* experts,
                             int32_t n_experts, int64_t since, uint64_t now, int64_t* slots_out,
                             int32_t cap, int32_t* n_out, int32_t* missed_out, int32_t* n_missed);
/* KVStore::erase (kvstore.cpp:180-185); *erased = 1 when the id was live. */
int pikv_store_erase_host(pikv_engine* eng, int32_t stream, uint64_t entry_id, int32_t* erased);
/* StoreStats retrievals / misses (kvstore.hpp:74-79; inserts and overwrites:
 * pikv_store_stats_host). */
int pikv_store_counters_host(pikv_engine* eng, int32_t stream, uint64_t* retrievals, uint64_t* misses);
/* ShardBuffer::live_count of every local (device, shard): live [G_local][SPD]. */
int pikv_ring_live_host(pikv_engine* eng, int32_t stream, int32_t* live);
/* score_entry (scheduler.cpp:181-229) of n entries' metadata under cfg's
 * scheduler strategy at `now`; per_layer [n][cfg->n_layers] or NULL. */
int pikv_score_entries_host(const pikv_config* cfg, const pikv_entry* entries, const double* per_layer,
                            int32_t n, uint64_t now, double* out);
/* evict (scheduler.cpp:262-330) on the stream's store at `now` (also the
 * stream's clock from here on): page scores, select_evictions per device,
 * erase in id order, state.step++.  Records as pikv_read_evictions_host
 * (at most cap); pages summed over the devices (EvictionReport). */
int pikv_evict_host(pikv_engine* eng, int32_t stream, uint64_t now, pikv_evict_record* out, int32_t cap,
                    int32_t* n_out, int32_t* pages_before, int32_t* pages_after);
int pikv_observe_hits(pikv_engine* eng, int32_t stream, uint64_t hits, uint64_t lookups); /* :332-338 */
int pikv_adakv_update(pikv_engine* eng, int32_t stream);                                 /* :340-342 */
/* attention (pipeline.cpp:59-85) of a stored-space query [d'] over stored
 * entries (slots [n]) per head, multi-head convention: y [d'], alpha [n] =
 * mean over heads of the weights (NULL allowed). */
int pikv_attend_host(pikv_engine* eng, int32_t stream, const float* query, const int64_t* slots, int32_t n,
                     float* y_out, float* alpha_out);
/* Codec::encode_vector / decode_vector (compressor.cpp:364-474) for
 * IDENTITY / LOWRANK / LORAPLUS / FASTV / PRUNE, per head of width hd ->
 * r: x [rows][heads*hd] <-> y [rows][heads*r]; basis [heads][r][hd], bias
 * [heads*hd], kept [heads][r] (sorted).  Device buffers, or host (_host). */
int pikv_codec_encode(int32_t codec, int32_t rows, int32_t heads, int32_t hd, int32_t r, const float* basis,
                      const float* bias, const int32_t* kept, const float* x, float* y);
int pikv_codec_decode(int32_t codec, int32_t rows, int32_t heads, int32_t hd, int32_t r, const float* basis,
                      const float* bias, const int32_t* kept, const float* y, float* x);
int pikv_codec_encode_host(int32_t codec, int32_t rows, int32_t heads, int32_t hd, int32_t r,
                           const float* basis, const float* bias, const int32_t* kept, const float* x,
                           float* y);
int pikv_codec_decode_host(int32_t codec, int32_t rows, int32_t heads, int32_t hd, int32_t r,
                           const float* basis, const float* bias, const int32_t* kept, const float* y,
                           float* x);
/* Column variances of n calibration rows [n][d] (Prune's fit statistic,
 * compressor.cpp:250-255). */
int pikv_column_variance_host(const double* rows, int32_t n, int32_t d, double* var);

/* ---- micro-batch pipeline (no reference counterpart) ------------------
 * The reference's Engine is one stream; B streams are B independent
 * Engine::step calls.  A group splits them into n_micro
 * engines of B / n_micro streams, each on its own CUDA stream, and orders
 * only their attention kernels (micro-batch m's attention starts after
 * micro-batch m-1's): the latency-bound control plane (route, insert, evict,
 * retrieve) and merge/fold-back of one micro-batch run while another one's
 * attention streams the KV pool from HBM.  Every stream still executes
 * exactly the reference's step sequence; results equal those of the
 * micro-batch engines stepped one after another.
 * attend_sms > 0 limits the persistent attention grid to that many SMs so
 * the other micro-batch's control kernels find free SMs (0 = auto when
 * n_micro > 1: all but 44 SMs for bf16 / f32 heads, 12 for int8, 32 for the
 * int4 IMMA kernel, 40 for the HMMA kernel of 32-wide bf16 slices; measured
 * on B200). */
typedef struct pikv_group pikv_group;
int pikv_group_create(const pikv_config* cfg, int32_t n_micro, int32_t attend_sms,
                      int32_t cuda_device, pikv_group** out);
int pikv_group_destroy(pikv_group* grp);
int pikv_group_size(pikv_group* grp);
/* Micro-batch m's engine (its streams are the group's streams
 * [m B/n, (m+1) B/n)); all per-engine calls apply (readback, codec, ...). */
pikv_engine* pikv_group_engine(pikv_group* grp, int32_t m);
/* Enqueue one step of micro-batch m: q/k/v [B/n][d], saliency [B/n][n_layers]
 * or NULL, y_out [B/n][d'].  host != 0: pinned host buffers (copied in and
 * out on the micro-batch's stream); host == 0: device buffers.  Returns
 * without waiting; pikv_group_wait(m) blocks until y_out is written. */
int pikv_group_submit(pikv_group* grp, int32_t m, const void* q, const void* k, const void* v,
                      const double* saliency, float* y_out, int32_t host);
int pikv_group_wait(pikv_group* grp, int32_t m);
/* world_size > 1: one NCCL communicator per micro-batch (ids
 * [n_micro][PIKV_NCCL_ID_BYTES], each from pikv_nccl_unique_id on rank 0);
 * micro-batch m's all-gather overlaps micro-batch m+1's attention. */
int pikv_group_attach_nccl(pikv_group* grp, const uint8_t* ids);
/* One step of all B streams from full-batch device buffers (q/k/v [B][d],
 * y [B][d']): pikv_group_submit for every micro-batch, no host wait. */
int pikv_group_step(pikv_group* grp, const void* q, const void* k, const void* v,
                    const double* saliency, float* y_out);
/* Make micro-batch 0's stream wait for all work submitted so far. */
int pikv_group_join(pikv_group* grp);
int pikv_group_sync(pikv_group* grp);
/* Attention timing: when on, every submit brackets its attention kernel with
 * CUDA events; *ms = summed attention time since the last read, *n = count
 * (at most 8192 launches per micro-batch are kept between reads). */
int pikv_group_set_timing(pikv_group* grp, int32_t on);
int pikv_group_read_timing(pikv_group* grp, double* ms, int32_t* n);
/* The same launches as intervals on one time axis: *sum_ms = summed launch
 * times, *union_ms = the time any attention launch was in flight (launches of
 * different micro-batches overlap in the attention SM partition). */
int pikv_group_read_timing_union(pikv_group* grp, double* sum_ms, double* union_ms, int32_t* n);
/* 1 when the group's attention runs in its own green-context SM partition
 * (default for the two-CTA CUDA-core attention kernel; PIKV_GREEN=0 / 1). */
int pikv_group_attention_partition(pikv_group* grp);
/* Debug probe (PIKV_GROUP_TIMELINE=1 when the group is created; device-pointer
 * submits): rows of 6 doubles (micro-batch, control start, control end, cross-
 * micro-batch wait satisfied, attention end, tail end) in ms relative to the
 * first recorded submit; at most cap rows, clears the record. */
int pikv_group_read_timeline(pikv_group* grp, double* out, int32_t cap, int32_t* n);

#ifdef __cplusplus
}
#endif
#endif /* PIKV_B200_H */
