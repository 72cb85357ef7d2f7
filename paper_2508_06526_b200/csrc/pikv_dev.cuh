// SPDX-License-Identifier: Apache-2.0
//
// Device-side state and helpers of the B200 PiKV engine.
//
// HBM layout (per GPU = per rank):
//   * stores: B streams x G_local logical devices x SPD shards; each shard is
//     a ring of S slots (kvstore.hpp:31-61).  ring index
//     r = (stream * G_local + g_local) * SPD + shard, slot index r * S + slot.
//     Slot metadata is SoA (id, shard_seq, token, expert, insert_step,
//     last_access, freq, attn_mass, per_layer[n_layers]); id 0 = empty.
//   * KV payload: a paged pool shared by all streams.  A ring's slot range
//     [p*spg, (p+1)*spg) maps through page_table[r][p] to a pool page of spg
//     entries; pages are taken on first write and returned when their last
//     live entry is erased, so HBM use follows live entries (kvstore.cpp:
//     193-196's M = 2 d' elem live) instead of ring capacity.
//   * entry = [K payload H*dph][V payload H*dph][K scales H][V scales H]
//     (scales only for INT8/INT4), padded to 16 B so one cp.async.bulk moves
//     it; payload element = bf16 / f32 / int8 / packed int4.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pikv_b200.h"

namespace pikv_dev {

constexpr int kMaxK = 64;
constexpr int kMaxE = 256;

struct EvictRec {  // == pikv_evict_record
    uint64_t step;
    uint64_t entry_id;
    int64_t token_id;
    int32_t expert_id;
    int32_t device;
    double score;
    int32_t reason;
    int32_t stream;
};
static_assert(sizeof(EvictRec) == sizeof(pikv_evict_record), "record layout");

// Per-stream exchange record for the cross-rank merge (one per stream per
// rank; world==1 uses it directly).  o is unnormalised w.r.t. m (base-2).
struct ExchangeLayout {
    int64_t o_off, m_off, l_off, found_off, stats_off, bytes_per_stream;
};

struct Dims {
    int B, Gl, SPD, R, S, H, dph, dp, d, E, k, n_layers;
    int G, world, rank;
    int spg, ppr;            // storage page entries, pages per ring
    int entry_bytes, payload_bytes, elem_bits;
    int codec, kv_dtype;
    int n_tok, n_exp, additive;
    int page_size, ppr_sched;  // scheduler pages per ring (candidates)
    int max_cand, nch, chunk_slots;  // retrieval grid
    int sel_stride;                  // pow2 >= SPD * ppr_sched
    int64_t pool_entries, pool_pages, att_cap, item_cap;
    int64_t att_stride;  // attended-list region per stream: min(max_cand * S, pool_entries)
    int attend_ctas;
    int items_per_cta;  // split-K work items per attention CTA (PIKV_ITEMS, default 4)
    int route_ch;       // router columns per W ring stage (pick_route_chunk)
    int q_f64;          // the step's q is fp64 (QueryEncoder output), not kv_dtype
    int ctl_cl, ctl_smem;  // k_control cluster size and dynamic smem (control_geometry)
    int att_eps;           // k_attend entries per ring stage (item sizes are multiples)
    int att_share;         // work items as equal static shares per attention CTA (cta_first), not tickets
    int dbg_ctl;        // k_control phase timestamps into dbg[64 + 8 s + p] (PIKV_DEBUG_CTL=1)
    int dbg_att;        // k_attend per-CTA (start, end, items, entries, smid) into dbg[64 + 8 B + 8 cta] (PIKV_DEBUG_ATT=1)
    int only_s;         // >= 0: the scheduler kernels evict this stream only (pikv_evict_host)
    int holes;          // an arbitrary KVStore::erase happened: page members are not a
                        // contiguous range, membership is checked per slot
};

struct Cfg {  // scalar config needed on device (copied by value into kernels)
    int router_strategy, groups, stride;
    double alpha, lambda_miss, beta_ent, bandit_step, bias_cap, load_decay;
    int sched_strategy, budget_pages, page_size, sink, flex_bucket, n_adakv_weights, n_flex_plan;
    double tau, lambda_freq, adakv_step, target_hit, theta0, hit_decay;
    double adakv_weights[8];
    double flex_plan[32];
    int unbounded_budget, head_width;
    int exact_sum;  // page aggregates are exact in any order (see capi.cu)
    int route_mode; // PIKV_ROUTE_EXACT (sequential fp64 chain) / PIKV_ROUTE_FAST (fp64 tree)
    int record_agg; // LRU / LRU+ with exact sums: aggregates from page records
};

struct State {
    // router (router.hpp:41-56), per stream
    const double* W;  // W_r, shared by all streams (same seed), chunk-major:
                      // [ceil(d / route_ch)][E][route_ch + 2] (zero-padded rows)
    double* load;
    uint64_t* usage;
    uint64_t* total_usage;
    uint64_t* miss;
    double* bias;
    uint64_t* rstep;
    // scheduler (scheduler.hpp:49-56), per stream
    double* theta;
    double* running_hit;
    uint64_t* sstep;
    // engine
    uint64_t* now;      // per stream
    uint64_t* next_id;  // per stream (KVStore::next_id_)
    int32_t* err;       // per stream
    uint64_t* st_inserts;
    uint64_t* st_overwrites;
    uint64_t* st_retrievals;  // StoreStats (kvstore.hpp:74-79): retrieve calls
    uint64_t* st_misses;      // and missed experts
    // rings
    int32_t* head;
    int32_t* live;
    uint64_t* seq;
    int32_t* page_table;  // [B*R][ppr]
    // slots
    uint64_t* id;
    uint64_t* shard_seq;
    int64_t* token;
    int32_t* expert;
    uint64_t* insert_step;
    uint64_t* last_access;
    uint64_t* freq;
    double* attn_mass;
    double* per_layer;
    uint8_t* has_pl;  // per_layer_scores non-empty (the insert carried saliency;
                      // pipeline.cpp:307, scheduler.cpp:222-226)
    // pool
    uint8_t* pool;
    int32_t* page_live;
    int32_t* free_stack;
    int32_t* free_top;
    // codec params
    const float* basis;  // [H][r][hd]
    const float* cbias;  // [d]
    const int32_t* kept; // [H][r]
    // step scratch
    int32_t* experts;  // [B][k]
    double* gates;     // [B][k]
    double* logits;    // [B][E]
    float* q_attn;     // [B][dp]
    float* proj;       // [2][B][dp] LowRank/LoRAPlus encoded k, v of the step
    int32_t* cand;     // [B][max_cand] local ring ids
    int32_t* ncand;    // [B]
    EvictRec* rec_ow;  // [B][k]
    int32_t* n_ow;     // [B]
    EvictRec* rec_ev;  // [B*Gl][SPD*S]
    int32_t* n_ev;     // [B*Gl]
    int32_t* pages_before;  // [B*Gl]
    int32_t* pages_after;   // [B*Gl]
    // per-page records, [B*R][ppr_sched] indexed by page_no % ppr_sched:
    // live members of a scheduler page are the contiguous shard_seq range
    // [q*ps + pr_first, q*ps + pr_first + pr_cnt) (erasure is whole pages or a
    // ring overwrite of the page's front member)
    int32_t* pr_cnt;
    int32_t* pr_first;
    uint64_t* pr_sla;       // sum of last_access over live members
    uint64_t* pr_sf;        // sum of freq over live members
    int32_t* pages_live;    // [B*Gl] scheduler pages with >= 1 live member (EvictionReport.pages_before)
    double* pg_agg;         // [B*R][ppr_sched]
    uint64_t* pg_oldest;
    int32_t* pg_cnt;
    int32_t* sel_idx;       // [B*Gl][R_dev*ppr_sched] scratch for selection
    int32_t* chunk_cnt;     // [B][max_cand][nch]
    int32_t* chunk_off;     // same, exclusive within stream
    int32_t* found;         // [B][k]
    int32_t* att_cnt;       // [B] attended entries of each stream (this rank)
    int32_t* att_slot;      // [B][att_stride] global slot index (ring*S+slot)
    int32_t* att_entry;     // [B][att_stride] pool entry index
    float* scores;          // [B][att_stride][H]  (base-2 logits)
    int32_t* item_stream;   // [item_cap]
    int32_t* item_begin;
    int32_t* item_end;
    int32_t* n_items;       // [2]: item count, k_attend's dynamic item ticket
    int32_t* item_first;    // [B+1] first work item of each stream
    int32_t* cta_first;     // [attend_ctas+1] first work item of each attention CTA (att_share)
    float* part_m;          // [item_cap][H]
    float* part_l;
    float* part_o;          // [item_cap][H][dph]
    uint8_t* exchange;      // [B][bytes_per_stream]
    float* gM;              // [B][H] global max (base 2): k_combine (one rank) / k_finish_merge
    float* gL;              // [B][H]
    pikv_step_summary* summary;  // [B]
    long long* dbg;              // [64] debug timestamps (k_route, stream 0)
    unsigned* done_ctr;          // last-block counter (k_foldback)
    unsigned* ctl_ctr;           // [4] last-block counter (k_control); [1] ticket, [2] done (k_retr_fused)
};

// ---- helpers -------------------------------------------------------------
// t, e >= 0 and n_tok, n_exp powers of two (validated on the host,
// kvstore.cpp:17-22), so the moduli are masks (no 64-bit division)
__device__ __forceinline__ int shard_raw(int64_t t, int e, int n_tok, int n_exp, int additive) {
    int lhs = (int)(t & (int64_t)(n_tok - 1));
    int rhs = e & (n_exp - 1);
    return additive ? lhs + rhs : (lhs ^ rhs);
}

// Does local ring (g_local, shard) possibly hold expert e?  Under xor mode
// raw = (t mod n_tok) ^ (e mod n_exp) for some t  <=>  raw ^ (e mod n_exp) < n_tok.
__device__ __forceinline__ bool ring_can_hold(int raw, int e, int n_tok, int n_exp, int additive) {
    int rhs = e % n_exp;
    int lhs = additive ? raw - rhs : (raw ^ rhs);
    return lhs >= 0 && lhs < n_tok;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int smid() {
    int r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

// Orderable 64-bit key of a double (ascending numeric order; no NaNs here).
__device__ __forceinline__ uint64_t dkey(double x) {
    uint64_t u = (uint64_t)__double_as_longlong(x);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// score_entry, scheduler.cpp:181-229 (QUEST rejected at create).  `m`
// reads one entry's EntryMeta fields (types.hpp:11-24) lazily: each
// strategy loads only what it scores.
template <class Meta>
__device__ __forceinline__ double score_impl(const Cfg& c, const Meta& m, int n_layers, uint64_t now) {
    switch (c.sched_strategy) {
        case PIKV_SCHED_H2O:
            return m.mass();
        case PIKV_SCHED_SL: {
            const uint64_t ins = m.ins(), age = now >= ins ? now - ins : 0;
            double u = (double)age <= c.tau ? 1.0 : 0.0;
            if (m.token() < c.sink) u = __dadd_rn(u, 2.0);
            return u;
        }
        case PIKV_SCHED_FLEX: {
            const uint64_t ins = m.ins(), age = now >= ins ? now - ins : 0;
            uint64_t bucket = age / (uint64_t)c.flex_bucket;
            if (bucket >= (uint64_t)c.n_flex_plan) bucket = (uint64_t)c.n_flex_plan - 1;
            return c.flex_plan[bucket];
        }
        case PIKV_SCHED_LRU: {
            const uint64_t la = m.la();
            return -(double)(now >= la ? now - la : 0);
        }
        case PIKV_SCHED_LRU_PLUS: {
            const uint64_t la = m.la();
            return __dadd_rn(-(double)(now >= la ? now - la : 0), __dmul_rn(c.lambda_freq, (double)m.freq()));
        }
        case PIKV_SCHED_ADAKV: {
            const uint64_t ins = m.ins(), age = now >= ins ? now - ins : 0;
            double phi0 = m.mass(), phi1 = (double)m.freq();
            double phi2 = __ddiv_rn(1.0, __dadd_rn(1.0, (double)age));
            double u = 0.0;
            if (c.n_adakv_weights > 0) u = __dadd_rn(u, __dmul_rn(c.adakv_weights[0], phi0));
            if (c.n_adakv_weights > 1) u = __dadd_rn(u, __dmul_rn(c.adakv_weights[1], phi1));
            if (c.n_adakv_weights > 2) u = __dadd_rn(u, __dmul_rn(c.adakv_weights[2], phi2));
            return u;
        }
        case PIKV_SCHED_DUO: {
            double u = 0.0;
            if (!m.has_pl()) return u;  // empty per_layer_scores
            const double* pl = m.pl();
            for (int l = 0; l < n_layers; ++l) u = __dadd_rn(u, pl[l]);
            return u;
        }
    }
    return 0.0;
}

struct SlotMeta {  // stored slot gi
    const State& st;
    int64_t gi;
    int n_layers;
    __device__ uint64_t ins() const { return st.insert_step[gi]; }
    __device__ uint64_t la() const { return st.last_access[gi]; }
    __device__ uint64_t freq() const { return st.freq[gi]; }
    __device__ double mass() const { return st.attn_mass[gi]; }
    __device__ int64_t token() const { return st.token[gi]; }
    __device__ bool has_pl() const { return st.has_pl[gi] != 0; }
    __device__ const double* pl() const { return st.per_layer + gi * (int64_t)n_layers; }
};

__device__ __forceinline__ double score_entry(const Cfg& c, const State& st, int64_t gi,
                                              uint64_t now, int n_layers) {
    return score_impl(c, SlotMeta{st, gi, n_layers}, n_layers, now);
}

// page-record maintenance (see State::pr_*)
__device__ __forceinline__ int64_t page_rec(const Dims& D, int64_t ring, uint64_t shard_seq) {
    return ring * D.ppr_sched + (int64_t)((shard_seq / (uint64_t)D.page_size) % (uint64_t)D.ppr_sched);
}
__device__ __forceinline__ void rec_append(const Dims& D, const State& S, int64_t ring, uint64_t sq,
                                           uint64_t now) {
    const int64_t r = page_rec(D, ring, sq);
    if (S.pr_cnt[r] == 0) {
        atomicAdd(&S.pages_live[ring / D.SPD], 1);  // a page comes to life
        S.pr_cnt[r] = 1;
        S.pr_first[r] = (int)(sq % (uint64_t)D.page_size);
        S.pr_sla[r] = now;
        S.pr_sf[r] = 0;
    } else {
        S.pr_cnt[r] += 1;
        S.pr_sla[r] += now;
    }
}
// Is offset i of scheduler page q of `ring` a live member (slot holds that shard_seq)?
__device__ __forceinline__ bool page_member(const Dims& D, const State& S, int64_t ring, uint64_t q, int i) {
    const uint64_t sq = q * (uint64_t)D.page_size + (uint64_t)i;
    const int64_t gi = ring * D.S + (int64_t)(sq % (uint64_t)D.S);
    return S.id[gi] != 0 && S.shard_seq[gi] == sq;
}
// First live member offset >= `from` of page q (after the previous first
// left): from itself unless arbitrary erases left holes (D.holes).
__device__ __forceinline__ int next_member(const Dims& D, const State& S, int64_t ring, uint64_t q, int from) {
    if (!D.holes) return from;
    while (from < D.page_size && !page_member(D, S, ring, q, from)) ++from;
    return from;
}
__device__ __forceinline__ void rec_drop_front(const Dims& D, const State& S, int64_t ring, uint64_t sq,
                                               uint64_t la, uint64_t fr) {
    const int64_t r = page_rec(D, ring, sq);
    if (--S.pr_cnt[r] == 0) atomicSub(&S.pages_live[ring / D.SPD], 1);  // last member displaced
    S.pr_first[r] += 1;
    if (D.holes && S.pr_cnt[r] > 0)
        S.pr_first[r] = next_member(D, S, ring, sq / (uint64_t)D.page_size, S.pr_first[r]);
    S.pr_sla[r] -= la;
    S.pr_sf[r] -= fr;
}

__device__ __forceinline__ float load_in(const void* p, int dtype, int64_t i) {
    if (dtype == PIKV_DTYPE_BF16) return __uint_as_float(((uint32_t)((const uint16_t*)p)[i]) << 16);
    return ((const float*)p)[i];
}

// ---- mbarrier / TMA bulk-copy helpers (sm_90+ PTX; SASS SYNCS.* / UBLKCP) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    }
}
// Same wait with a suspend-time hint: the warp sleeps in hardware until the
// phase completes (or the hint expires) instead of re-issuing try_wait --
// spinning producer / consumer warps otherwise take issue slots from the
// warps doing the math on the same SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity, uint32_t hint_ns = 20000) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity), "r"(hint_ns)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes,
                                               uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ---- programmatic dependent launch ------------------------------------------
// Every step kernel is launched with programmatic stream serialization and
// starts with griddep_enter(): wait for the predecessor grid (and therefore,
// transitively, every earlier kernel of the step) to complete and flush.  The wait must precede any early
// return so that a kernel's completion still implies its predecessors'.
__device__ __forceinline__ void griddep_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // No explicit launch_dependents: the successor is released as this grid's
    // CTAs exit (an early trigger let successor CTAs take SM slots the
    // current kernel still needed: +26 us per step measured).
}

bool pdl_enabled();  // PIKV_PDL=1 env (default off), read once (capi.cu)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Launch with thread-block clusters of `cl` CTAs along x (grid.x % cl == 0).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                  cudaStream_t st, int cl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- launch wrappers (defined in the .cu files) ----------------------------
void launch_route(const Dims& D, const Cfg& C, const State& S, const void* q, cudaStream_t st);
void launch_project(const Dims& D, const State& S, const void* q, const void* k, const void* v,
                    cudaStream_t st);
void launch_insert(const Dims& D, const Cfg& C, const State& S, const void* q, const void* k,
                   const void* v, const double* saliency, cudaStream_t st);
void launch_sched_pages(const Dims& D, const Cfg& C, const State& S, cudaStream_t st);
void launch_sched_select(const Dims& D, const Cfg& C, const State& S, cudaStream_t st);

bool control_supported(const Dims& D, const Cfg& C);
void control_geometry(Dims& D);
int pick_route_chunk(const Dims& D);
void launch_control(const Dims& D, const Cfg& C, const State& S, const void* q, const void* k, const void* v,
                    const double* saliency, cudaStream_t st);  // route+insert+evict+retrieve per stream
void launch_retr_fused(const Dims& D, const Cfg& C, const State& S, cudaStream_t st);  // count+scan+write
void launch_retr_count(const Dims& D, const State& S, cudaStream_t st);
void launch_retr_scan(const Dims& D, const Cfg& C, const State& S, cudaStream_t st);
void launch_retr_write(const Dims& D, const State& S, cudaStream_t st);
void launch_attend(const Dims& D, const State& S, cudaStream_t st);
bool attend_i4tc_applies(const Dims& D);  // int4 / 128-dim heads: the tensor-core kernel (attend_i4tc.cu)
void launch_attend_i4tc(const Dims& D, const State& S, cudaStream_t st);
int attend_i4tc_eps();
int attend_i4tc_stages(const Dims& D);
bool attend_bf16tc_applies(const Dims& D);  // 32-wide bf16 head slices: tensor cores (attend_bf16tc.cu)
void launch_attend_bf16tc(const Dims& D, const State& S, cudaStream_t st);
int attend_bf16tc_stages(const Dims& D);
int attend_bf16tc_eps();
void launch_combine(const Dims& D, const Cfg& C, const State& S, const ExchangeLayout& X, float* y,
                    int direct, int attended, cudaStream_t st);
void launch_finish_merge(const Dims& D, const Cfg& C, const State& S, const ExchangeLayout& X,
                         const uint8_t* gathered, float* y, int granks, cudaStream_t st);
void launch_foldback(const Dims& D, const Cfg& C, const State& S, cudaStream_t st);  // + feedback
void launch_feedback(const Dims& D, const Cfg& C, const State& S, cudaStream_t st);
// bulk store build of a prefill (engine_kernels.cu); dst [T*k] int64 scratch,
// proj [2][T][dp] + [H][r] fp32 (LowRank/LoRAPlus), counters [2 + Gl],
// sort_buf bulk_sort_ints(D, T) int32 for the ring counting sort (or null)
size_t bulk_sort_ints(const Dims& D, int64_t T);
int bulk_insert(const Dims& D, const State& S, int s, int64_t T, const void* k, const void* v,
                const int32_t* experts, const double* saliency, int64_t* dst, float* proj,
                unsigned long long* counters, int use_tc, cudaStream_t st, int32_t* sort_buf);
// tcgen05 projection GEMM (bulk_tc.cu); nonzero when the shape is unsupported
// fuse_dst != null: may write the bf16 projections straight into the pool
// entries dst (returns 2 then; 0 = fp32 projections in proj; 1 = unsupported)
int launch_bulk_project_tc(const Dims& D, const State& S, int64_t T, const void* k, const void* v, float* proj,
                           float* bias_scratch, cudaStream_t st, const int64_t* fuse_dst = nullptr);
int encode_chunk(const Dims& D, int nb);
void launch_encode(const Dims& D, const double* wt, const double* emb, double* q64, void* kout, void* vout,
                   cudaStream_t st);  // QueryEncoder (pipeline.cpp:29-57) for all streams
void launch_snapshot(const Dims& D, const State& S, int s, uint64_t now, const int64_t* ring_off,
                     pikv_snapshot_record* out, int64_t n, cudaStream_t st);
void launch_synth(const Dims& D, void* q, void* k, void* v, uint64_t seed, uint64_t step,
                  cudaStream_t st);
int attend_max_smem();
// ---- component API (components.cu; pikv_route_host / pikv_store_* / ...) ----
void launch_route_one(const Dims& D, const Cfg& C, const State& S, int s, const double* q, const double* logits,
                      cudaStream_t st);
void launch_store_insert(const Dims& D, const State& S, int s, int n, const pikv_entry* in, const float* kv,
                         const double* layers, pikv_entry* disp, float* disp_kv, double* disp_layers,
                         int32_t* disp_flag, int32_t* status, cudaStream_t st);
void launch_store_erase(const Dims& D, const State& S, int s, uint64_t id, int32_t* status, cudaStream_t st);
size_t retrieve_scratch_bytes(const Dims& D);
int launch_retrieve(const Dims& D, const State& S, int s, int64_t since, uint64_t now, const uint32_t* want,
                    void* scratch, int32_t** sorted_out, int32_t** cnt_out, uint32_t** found_out, cudaStream_t st);
void launch_score_meta(const Cfg& C, const pikv_entry* m, const double* layers, int n_layers, int n, uint64_t now,
                       double* out, cudaStream_t st);
void launch_state_op(const Dims& D, const Cfg& C, const State& S, int s, int op, uint64_t a, uint64_t b,
                     const int32_t* experts, int n, double reward, cudaStream_t st);
void launch_read_heads(const Dims& D, const State& S, int s, const int64_t* slots, int n, float* kh, float* vh,
                       cudaStream_t st);
void launch_head_mean(const float* w, int H, int n, float* out, cudaStream_t st);
void launch_codec_select(int decode, int codec, int64_t rows, int heads, int hd, int r, const int32_t* kept,
                         const float* x, float* y, cudaStream_t st);
void launch_col_var(const double* x, int n, int d, double* var, cudaStream_t st);
// stored K/V of n stream-local slots decoded to fp32 (readback)
void launch_read_entries(const Dims& D, const State& S, int s, const int64_t* slots, int n, float* k, float* v,
                         cudaStream_t st);
// token / expert of n slots (global slot indices) -> out arrays (readback)
void launch_gather_slots(const State& S, const int32_t* slot, int n, int64_t* token, int32_t* expert,
                         cudaStream_t st);

}  // namespace pikv_dev
