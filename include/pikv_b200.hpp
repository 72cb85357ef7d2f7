// SPDX-License-Identifier: Apache-2.0
//
// pikv_b200.hpp -- header-only C++ facade of the B200 engine with the
// reference's API (/root/reference/proj/include/pikv) over the C-ABI
// (pikv_b200.h).  Names, argument meanings and exception types follow the
// reference so a caller of pikv::Engine / pikv::shard_assign / ... switches by
// changing the namespace to pikv::b200:
//
//   reference                               this facade
//   pikv::shard_assign (kvstore.hpp:25)     pikv::b200::shard_assign
//   pikv::select_evictions (scheduler.hpp:114) pikv::b200::select_evictions
//   pikv::attention (pipeline.hpp:46)       pikv::b200::attention
//   pikv::Engine (pipeline.hpp:101)         pikv::b200::Engine (B streams; step,
//                                           flush, StepResult.inserted)
//   pikv::KVStore (kvstore.hpp:100-159)     pikv::b200::KVStore (in HBM)
//   pikv::RouterState, route, route_logits, record_miss, adapt (router.hpp:41-79)
//                                           same names (state in HBM)
//   pikv::score_entry, evict, observe_hits, adakv_update (scheduler.hpp:83-129)
//                                           score_entry / KVStore::evict / ...
//   pikv::Codec encode/decode_vector (compressor.hpp:57-80)  pikv::b200::Codec
//   pikv::Error tree (errors.hpp:9-47)      pikv::b200::Error tree
//
// Differences, all from the reference's own scope notes: the engine takes the
// token's q/k/v directly (QueryEncoder is a desk-scale stand-in for the host
// model, pipeline.hpp:17-18); codecs take a caller basis (fitting is offline,
// PAPER.md:499); heads/batch/dtype are extra config.
// No CUDA headers are needed: link with libpikv_b200.so.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pikv_b200.h"

namespace pikv::b200 {

// ---- errors.hpp:9-47 ----------------------------------------------------
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InvalidArgument : Error { using Error::Error; };
struct InvalidConfig : Error { using Error::Error; };
struct InvalidEntry : Error { using Error::Error; };
struct NumericalError : Error { using Error::Error; };
struct CodecMismatch : Error { using Error::Error; };
struct NotFitted : Error { using Error::Error; };
struct InsufficientCalibration : Error { using Error::Error; };
struct InvalidComparison : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA / NCCL / pool exhaustion

inline void check(int rc) {
    if (rc == PIKV_OK) return;
    const std::string msg = pikv_last_error();
    switch (rc) {
        case PIKV_ERR_INVALID_ARGUMENT: throw InvalidArgument(msg);
        case PIKV_ERR_INVALID_CONFIG: throw InvalidConfig(msg);
        case PIKV_ERR_INVALID_ENTRY: throw InvalidEntry(msg);
        case PIKV_ERR_NUMERICAL: throw NumericalError(msg);
        case PIKV_ERR_CODEC_MISMATCH: throw CodecMismatch(msg);
        case PIKV_ERR_NOT_FITTED: throw NotFitted(msg);
        case PIKV_ERR_INSUFFICIENT_CALIBRATION: throw InsufficientCalibration(msg);
        case PIKV_ERR_INVALID_COMPARISON: throw InvalidComparison(msg);
        case PIKV_ERR_IO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}

// ---- free functions ----------------------------------------------------
struct ShardId {  // kvstore.hpp:14-20
    int device = 0;
    int shard_index = 0;
    int raw = 0;
    bool operator==(const ShardId&) const = default;
};

inline ShardId shard_assign(std::int64_t t, int e, int n_tok, int n_exp, int devices,
                            bool additive = false) {
    std::int32_t d = 0, s = 0, r = 0, ee = e;
    check(pikv_shard_assign_host(&t, &ee, 1, n_tok, n_exp, devices, additive ? 1 : 0, &d, &s, &r));
    return {d, s, r};
}

enum class EvictReason { Budget, Threshold, Overwrite };  // scheduler.hpp:87

struct PageScore {  // scheduler.hpp:106-109
    double aggregate = 0.0;
    std::uint64_t oldest_id = 0;
};

inline std::vector<std::pair<std::size_t, EvictReason>> select_evictions(
    const std::vector<PageScore>& pages, int budget_pages, bool use_theta, double theta) {
    const int n = static_cast<int>(pages.size());
    std::vector<double> agg(n);
    std::vector<std::uint64_t> old(n);
    for (int i = 0; i < n; ++i) agg[i] = pages[i].aggregate, old[i] = pages[i].oldest_id;
    std::vector<std::int32_t> idx(n + 1), why(n + 1);
    std::int32_t m = 0;
    check(pikv_select_evictions_host(agg.data(), old.data(), n, budget_pages, use_theta ? 1 : 0,
                                     theta, idx.data(), why.data(), &m));
    std::vector<std::pair<std::size_t, EvictReason>> out;
    for (int i = 0; i < m; ++i)
        out.emplace_back(static_cast<std::size_t>(idx[i]), static_cast<EvictReason>(why[i]));
    return out;
}

struct AttentionOutput {  // pipeline.hpp:39-43
    std::vector<double> output;
    std::vector<double> weights;
    std::size_t retrieved = 0;
};

// attention(query, entries) with entries given as key/value rows.
inline AttentionOutput attention(const std::vector<double>& query,
                                 const std::vector<std::vector<double>>& keys,
                                 const std::vector<std::vector<double>>& values) {
    AttentionOutput out;
    const int w = static_cast<int>(query.size()), n = static_cast<int>(keys.size());
    out.retrieved = static_cast<std::size_t>(n);
    if (n == 0) {
        out.output.assign(query.size(), 0.0);
        return out;
    }
    std::vector<float> q(query.begin(), query.end()), k, v, y(w), wt(n);
    for (int i = 0; i < n; ++i) {
        if (static_cast<int>(keys[i].size()) != w)
            throw InvalidArgument("attention: key/query width mismatch");  // pipeline.cpp:71-73
        k.insert(k.end(), keys[i].begin(), keys[i].end());
        v.insert(v.end(), values[i].begin(), values[i].end());
    }
    check(pikv_attention_host(q.data(), k.data(), v.data(), 1, n, w, y.data(), wt.data()));
    out.output.assign(y.begin(), y.end());
    out.weights.assign(wt.begin(), wt.end());
    return out;
}

// ---- configuration (config.hpp, kvstore.hpp, router.hpp, scheduler.hpp,
//      compressor.hpp, pipeline.hpp) -------------------------------------
enum class RouterStrategy { Base, TopK, LoadBalanced, CacheAware, EntropyLB, Adaptive, Hierarchical };
enum class SchedStrategy { H2O, SL, QUEST, Flex, LRU, LRUPlus, AdaKV, Duo };
// compressor.hpp:14-23 (Scheme; SVD / LoRA are LowRank here), plus this engine's quantizers
enum class Scheme { Identity, LowRank, LoRAPlus, FastV, Prune, Int8, Int4 };
enum class DType { F32, BF16 };

struct ModelConfig { int d = 64, head_width = 16, E = 8, k = 2; long long L = 1024; int G = 2, S = 16, K = 4;
                     double rho = 1.0; int elem_bytes = 2; };
struct StoreConfig { int n_tok = 64, n_exp = 64; bool additive = false; int shards_per_device = 0; };
struct RouterConfig { RouterStrategy strategy = RouterStrategy::TopK; int k = 2; double alpha = 1.0,
                      lambda_miss = 1.0, beta_ent = 1.0, bandit_step = 0.05; int groups = 1, stride = 1;
                      double bias_cap = 5.0, load_decay = 0.99; };
struct SchedulerConfig { SchedStrategy strategy = SchedStrategy::LRU; int budget_pages = 4, page_size = 16;
                         double tau = 64.0; int sink = 4; double lambda_freq = 0.5, adakv_step = 0.05,
                         target_hit = 0.9, gamma_sim = 0.5, theta0 = -1e18, hit_decay = 0.9;
                         std::vector<double> adakv_weights{1.0, 0.5, 0.25};
                         std::vector<double> flex_plan{1.0}; int flex_bucket = 16; };
struct CompressorConfig { Scheme scheme = Scheme::Identity; int rank = 8; };

struct EngineConfig {  // pipeline.hpp:87-98 (+ B200 runtime fields)
    ModelConfig model;
    StoreConfig store;
    RouterConfig router;
    SchedulerConfig scheduler;
    CompressorConfig compressor;
    bool unbounded_budget = false;
    std::uint64_t seed = 1;
    int n_heads = 1, n_layers = 0, batch = 1;
    DType kv_dtype = DType::F32;
    long long pool_entries = 0;
    int cuda_device = 0;
    bool fast_routing = false;  // PIKV_ROUTE_FAST (tree-reduced fp64 logits)

    pikv_config to_c() const {
        pikv_config c;
        pikv_config_default(&c);
        c.d = model.d, c.head_width = model.head_width, c.E = model.E, c.k = router.k;
        c.L = model.L, c.G = model.G, c.S = model.S, c.K = model.K, c.elem_bytes = model.elem_bytes;
        c.rho = model.rho, c.n_heads = n_heads;
        c.n_tok = store.n_tok, c.n_exp = store.n_exp, c.additive = store.additive;
        c.shards_per_device = store.shards_per_device;
        c.router_strategy = static_cast<int>(router.strategy), c.groups = router.groups;
        c.stride = router.stride, c.alpha = router.alpha, c.lambda_miss = router.lambda_miss;
        c.beta_ent = router.beta_ent, c.bandit_step = router.bandit_step, c.bias_cap = router.bias_cap;
        c.load_decay = router.load_decay;
        c.sched_strategy = static_cast<int>(scheduler.strategy);
        c.budget_pages = scheduler.budget_pages, c.page_size = scheduler.page_size;
        c.sink = scheduler.sink, c.flex_bucket = scheduler.flex_bucket, c.tau = scheduler.tau;
        c.lambda_freq = scheduler.lambda_freq, c.adakv_step = scheduler.adakv_step;
        c.target_hit = scheduler.target_hit, c.gamma_sim = scheduler.gamma_sim;
        c.theta0 = scheduler.theta0, c.hit_decay = scheduler.hit_decay;
        if (scheduler.adakv_weights.size() > 8 || scheduler.flex_plan.size() > 32)
            throw InvalidConfig("SchedulerConfig: at most 8 adakv weights / 32 flex buckets");
        c.n_adakv_weights = static_cast<int>(scheduler.adakv_weights.size());
        for (std::size_t i = 0; i < scheduler.adakv_weights.size(); ++i) c.adakv_weights[i] = scheduler.adakv_weights[i];
        c.n_flex_plan = static_cast<int>(scheduler.flex_plan.size());
        for (std::size_t i = 0; i < scheduler.flex_plan.size(); ++i) c.flex_plan[i] = scheduler.flex_plan[i];
        c.codec = static_cast<int>(compressor.scheme), c.rank = compressor.rank;
        c.unbounded_budget = unbounded_budget, c.n_layers = n_layers, c.batch = batch;
        c.kv_dtype = kv_dtype == DType::BF16 ? PIKV_DTYPE_BF16 : PIKV_DTYPE_F32;
        c.world_size = 1, c.rank_id = 0, c.pool_entries = pool_entries, c.seed = seed;
        c.route_mode = fast_routing ? PIKV_ROUTE_FAST : PIKV_ROUTE_EXACT;
        return c;
    }
};

// ---- step I/O (pipeline.hpp:59-85) ----------------------------------------
struct TokenInput {
    // The reference's TokenInput (pipeline.hpp:59-62): the token's embedding
    // (width d); the step runs the QueryEncoder on the GPU (pipeline.cpp:222).
    std::vector<double> embedding;
    std::vector<double> layer_saliency;     // n_layers (Duo)
    // Alternatively the already-encoded q/k/v (width d, rounded to kv_dtype
    // by the engine): used when `embedding` is empty.
    std::vector<double> query, key, value;
};

struct EvictionRecord {  // scheduler.hpp:90-98
    std::uint64_t step = 0, entry_id = 0;
    std::int64_t token_id = 0;
    int expert_id = 0, device = 0;
    double score = 0.0;
    EvictReason reason = EvictReason::Budget;
};

struct AttendedEntry {
    std::int64_t token_id = 0;
    int expert_id = 0;
    double weight = 0.0;
};

struct StepResult {  // pipeline.hpp:68-80
    std::uint64_t step = 0;
    std::vector<int> experts;
    std::vector<double> gates;
    int inserts = 0;
    std::vector<std::pair<std::int64_t, int>> inserted;  // (token, expert) per stored entry
    std::vector<EvictionRecord> evictions;  // overwrite + scheduled
    std::uint64_t fetch_elements = 0;
    std::uint64_t hits = 0, lookups = 0;
    AttentionOutput attn;                   // output; weights in (token, expert) order
    std::vector<AttendedEntry> attended;    // (token, expert) order (kvstore.cpp:144-163)
};

struct SnapshotRecord {  // kvstore.hpp:89-96
    int device = 0, shard = 0;
    std::int64_t token_id = 0;
    int expert_id = 0;
    std::uint64_t age = 0, freq = 0;
};

struct StoreStats { std::uint64_t live = 0, memory_bytes = 0, inserts = 0, overwrites = 0; };
using pikv_store_stats_view = StoreStats;
struct RouterStateView { std::vector<double> load, bandit_bias; std::vector<std::uint64_t> usage_counts,
                         miss_counts; std::uint64_t total_usage = 0, step = 0; };
struct SchedulerStateView { double theta = 0.0, running_hit = 0.0; std::uint64_t step = 0; };

// B independent decode streams of pikv::Engine on one GPU.
class Engine {
  public:
    explicit Engine(const EngineConfig& cfg) : cfg_(cfg) {
        pikv_config c = cfg.to_c();
        check(pikv_engine_create(&c, cfg.cuda_device, &h_));
    }
    ~Engine() { if (h_) pikv_engine_destroy(h_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // Codec basis [H][r][hd], LoRAPlus bias [d], Prune kept [H][r].
    void set_codec(const std::vector<float>& basis, const std::vector<float>& bias = {},
                   const std::vector<std::int32_t>& kept = {}) {
        check(pikv_set_codec_host(h_, basis.empty() ? nullptr : basis.data(),
                                  bias.empty() ? nullptr : bias.data(), kept.empty() ? nullptr : kept.data()));
    }
    void set_router_matrix(const std::vector<double>& w_r) { check(pikv_set_router_matrix_host(h_, w_r.data())); }

    // Engine::step (pipeline.cpp:213-351) for all streams, one token each.
    std::vector<StepResult> step(const std::vector<TokenInput>& tokens) {
        const int B = cfg_.batch, d = cfg_.model.d, k = cfg_.router.k, E = cfg_.model.E;
        if (static_cast<int>(tokens.size()) != B) throw InvalidArgument("Engine::step: one token per stream");
        const bool bf16 = cfg_.kv_dtype == DType::BF16;
        const bool embed = !tokens.empty() && !tokens[0].embedding.empty();
        std::vector<std::uint16_t> qb, kb, vb;
        std::vector<float> qf, kf, vf;
        std::vector<double> emb;
        std::vector<double> sal(static_cast<std::size_t>(B) * (cfg_.n_layers > 0 ? cfg_.n_layers : 1));
        for (int s = 0; s < B; ++s) {
            const TokenInput& t = tokens[s];
            for (int l = 0; l < cfg_.n_layers; ++l)
                sal[static_cast<std::size_t>(s) * cfg_.n_layers + l] =
                    l < static_cast<int>(t.layer_saliency.size()) ? t.layer_saliency[l] : 0.0;
            if (embed) {
                if (static_cast<int>(t.embedding.size()) != d)
                    throw InvalidArgument("Engine::step: embedding width mismatch");  // pipeline.cpp:214-216
                emb.insert(emb.end(), t.embedding.begin(), t.embedding.end());
                continue;
            }
            if (static_cast<int>(t.query.size()) != d || static_cast<int>(t.key.size()) != d ||
                static_cast<int>(t.value.size()) != d)
                throw InvalidArgument("Engine::step: embedding width mismatch");  // pipeline.cpp:214-216
            for (int i = 0; i < d; ++i) {
                if (bf16) {
                    qb.push_back(to_bf16(t.query[i])), kb.push_back(to_bf16(t.key[i]));
                    vb.push_back(to_bf16(t.value[i]));
                } else {
                    qf.push_back(static_cast<float>(t.query[i])), kf.push_back(static_cast<float>(t.key[i]));
                    vf.push_back(static_cast<float>(t.value[i]));
                }
            }
        }
        const int dp = stored_width();
        std::vector<float> y(static_cast<std::size_t>(B) * dp);
        if (embed) {
            check(pikv_step_embed_host(h_, emb.data(), cfg_.n_layers > 0 ? sal.data() : nullptr, y.data()));
        } else {
            const void* q = bf16 ? static_cast<const void*>(qb.data()) : qf.data();
            const void* kk = bf16 ? static_cast<const void*>(kb.data()) : kf.data();
            const void* v = bf16 ? static_cast<const void*>(vb.data()) : vf.data();
            check(pikv_step_host(h_, q, kk, v, cfg_.n_layers > 0 ? sal.data() : nullptr, y.data()));
        }
        check(pikv_sync(h_));
        std::vector<std::int32_t> ex(static_cast<std::size_t>(B) * k);
        std::vector<double> gates(static_cast<std::size_t>(B) * k);
        std::vector<pikv_step_summary> sm(B);
        check(pikv_read_step_host(h_, ex.data(), gates.data(), nullptr, sm.data()));
        std::int32_t nrec = 0;
        check(pikv_read_evictions_host(h_, nullptr, 0, &nrec));  // count, then the records
        std::vector<pikv_evict_record> recs(nrec > 0 ? nrec : 1);
        check(pikv_read_evictions_host(h_, recs.data(), nrec, &nrec));
        std::vector<StepResult> out(B);
        for (int s = 0; s < B; ++s) {
            StepResult& r = out[s];
            r.step = sm[s].step;
            r.experts.assign(ex.begin() + s * k, ex.begin() + (s + 1) * k);
            r.gates.assign(gates.begin() + s * k, gates.begin() + (s + 1) * k);
            r.inserts = sm[s].inserts;
            // Engine::insert_compressed (pipeline.cpp:197-199): one entry per
            // selected expert, token = the step, in selection order
            for (int j = 0; j < r.inserts && j < k; ++j)
                r.inserted.emplace_back(static_cast<std::int64_t>(r.step), r.experts[j]);
            r.fetch_elements = static_cast<std::uint64_t>(sm[s].fetch_elements);
            r.hits = static_cast<std::uint64_t>(sm[s].hits);
            r.lookups = static_cast<std::uint64_t>(sm[s].lookups);
            r.attn.output.assign(y.begin() + static_cast<std::size_t>(s) * dp,
                                 y.begin() + static_cast<std::size_t>(s + 1) * dp);
            for (int i = 0; i < nrec && i < static_cast<int>(recs.size()); ++i) {
                if (recs[i].stream != s) continue;
                r.evictions.push_back({recs[i].step, recs[i].entry_id, recs[i].token_id, recs[i].expert_id,
                                       recs[i].device, recs[i].score, static_cast<EvictReason>(recs[i].reason)});
            }
            std::int32_t n = 0;
            check(pikv_read_attended_host(h_, s, nullptr, nullptr, nullptr, 0, &n));
            std::vector<std::int64_t> tok(n > 0 ? n : 1);
            std::vector<std::int32_t> exp(n > 0 ? n : 1);
            std::vector<double> al(n > 0 ? n : 1);
            check(pikv_read_attended_host(h_, s, tok.data(), exp.data(), al.data(), n, &n));
            std::vector<AttendedEntry> att(n);
            for (int i = 0; i < n; ++i) att[i] = {tok[i], exp[i], al[i]};
            sort_attended(att);
            r.attended = att;
            r.attn.retrieved = static_cast<std::size_t>(n);
            for (const auto& a : att) r.attn.weights.push_back(a.weight);
        }
        (void)E;
        return out;
    }

    // Engine::flush (pipeline.hpp:108): inserts a Chunk codec's pending
    // entries.  No codec here buffers entries (Chunk is out of scope), so
    // nothing is pending: an empty result per stream, as the reference
    // returns for non-Chunk codecs.
    std::vector<StepResult> flush() { return std::vector<StepResult>(cfg_.batch); }

    // KVStore::snapshot(now) (kvstore.cpp:206-221), computed on the GPU;
    // now < 0: the stream's current step.
    std::vector<SnapshotRecord> snapshot(int stream = 0, std::int64_t now = -1) const {
        std::int64_t n = 0;
        check(pikv_snapshot_host(h_, stream, now, nullptr, 0, &n));
        std::vector<pikv_snapshot_record> raw(static_cast<std::size_t>(n));
        if (n) check(pikv_snapshot_host(h_, stream, now, raw.data(), n, &n));
        std::vector<SnapshotRecord> out;
        out.reserve(raw.size());
        for (const auto& r : raw) out.push_back({r.device, r.shard, r.token_id, r.expert_id, r.age, r.freq});
        return out;
    }

    StoreStats store_stats(int stream = 0) const {
        StoreStats st;
        check(pikv_store_stats_host(h_, stream, &st.live, &st.memory_bytes, &st.inserts, &st.overwrites));
        return st;
    }
    RouterStateView router_state(int stream = 0) const {
        const int E = cfg_.model.E;
        RouterStateView r;
        r.load.resize(E), r.bandit_bias.resize(E), r.usage_counts.resize(E), r.miss_counts.resize(E);
        check(pikv_read_router_state_host(h_, stream, r.load.data(), r.usage_counts.data(), r.miss_counts.data(),
                                          r.bandit_bias.data(), &r.step, &r.total_usage));
        return r;
    }
    SchedulerStateView scheduler_state(int stream = 0) const {
        SchedulerStateView v;
        check(pikv_read_sched_state_host(h_, stream, &v.theta, &v.running_hit, &v.step));
        return v;
    }
    int stored_width() const {
        const int hd = cfg_.model.d / cfg_.n_heads;
        const bool proj = cfg_.compressor.scheme == Scheme::LowRank || cfg_.compressor.scheme == Scheme::LoRAPlus ||
                          cfg_.compressor.scheme == Scheme::FastV || cfg_.compressor.scheme == Scheme::Prune;
        return (proj ? cfg_.compressor.rank : hd) * cfg_.n_heads;
    }
    pikv_engine* handle() { return h_; }

  private:
    static std::uint16_t to_bf16(double x) {
        float f = static_cast<float>(x);
        std::uint32_t u;
        std::memcpy(&u, &f, 4);
        if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
        return static_cast<std::uint16_t>(u >> 16);
    }
    static void sort_attended(std::vector<AttendedEntry>& a) {
        // (token, expert) order of KVStore::retrieve (kvstore.cpp:144-163)
        std::sort(a.begin(), a.end(), [](const AttendedEntry& x, const AttendedEntry& y) {
            return x.token_id != y.token_id ? x.token_id < y.token_id : x.expert_id < y.expert_id;
        });
    }
    EngineConfig cfg_;
    pikv_engine* h_ = nullptr;
};

// ---- component classes (kvstore.hpp, router.hpp, scheduler.hpp,
//      compressor.hpp) over the component C-ABI: one-stream engines whose
//      HBM state is the store / RouterState / SchedulerState -----------------
struct EntryMeta {  // types.hpp:11-24
    std::uint64_t insert_step = 0, last_access_step = 0, freq = 0;
    double attn_mass = 0.0;
    std::vector<double> per_layer_scores;
};
struct KVEntry {  // types.hpp:27-34
    std::uint64_t id = 0, shard_seq = 0;
    std::int64_t token_id = 0;
    int expert_id = 0;
    std::vector<double> key, value;
    EntryMeta meta;
};
// kvstore.hpp:81-87; entries are host copies (the store lives in HBM), with
// their stream-local slots for attention over stored entries
struct RetrievalResult {
    std::vector<KVEntry> entries;
    std::vector<int> missed_experts;
    std::vector<std::int64_t> slots;
};
struct StoreCounters { std::uint64_t inserts = 0, overwrites = 0, retrievals = 0, misses = 0; };
struct EvictionReport {  // scheduler.hpp:100-104
    std::vector<EvictionRecord> evicted;
    int pages_before = 0, pages_after = 0;
};

namespace detail {
inline pikv_entry to_c(const KVEntry& e) {
    pikv_entry c{};
    c.token_id = e.token_id, c.expert_id = e.expert_id;
    c.has_layers = e.meta.per_layer_scores.empty() ? 0 : 1;
    c.insert_step = e.meta.insert_step, c.last_access_step = e.meta.last_access_step;
    c.freq = e.meta.freq, c.attn_mass = e.meta.attn_mass;
    return c;
}
}  // namespace detail

// KVStore (kvstore.hpp:100-159) in HBM.  The store is built for the
// scheduler's page size (its page records are maintained on every insert).
class KVStore {
  public:
    KVStore(const ModelConfig& model, const StoreConfig& store, int page_size = 16, int n_layers = 0,
            DType kv_dtype = DType::F32, int cuda_device = 0)
        : n_layers_(n_layers) {
        EngineConfig c;
        c.model = model;
        c.model.d = d_prime_of(model);
        c.model.rho = 1.0;
        c.model.head_width = std::min(model.head_width, c.model.d);
        c.store = store;
        c.router.k = 1;
        c.scheduler.page_size = page_size;
        c.n_layers = n_layers, c.kv_dtype = kv_dtype, c.batch = 1, c.cuda_device = cuda_device;
        cfg_ = c;
        pikv_config pc = c.to_c();
        check(pikv_engine_create(&pc, cuda_device, &h_));
    }
    ~KVStore() { if (h_) pikv_engine_destroy(h_); }
    KVStore(const KVStore&) = delete;
    KVStore& operator=(const KVStore&) = delete;

    ShardId locate(std::int64_t token_id, int expert_id) const {  // kvstore.hpp:105
        return shard_assign(token_id, expert_id, cfg_.store.n_tok, cfg_.store.n_exp, cfg_.model.G,
                            cfg_.store.additive);
    }
    // KVStore::insert (kvstore.cpp:107-120): the displaced entry, if any
    std::optional<KVEntry> insert(const KVEntry& e) {
        const int dp = stored_width();
        if (static_cast<int>(e.key.size()) != dp || static_cast<int>(e.value.size()) != dp)
            throw InvalidEntry("KVStore::insert: entry width != d'");  // kvstore.cpp:108-111
        pikv_entry in = detail::to_c(e), out{};
        std::vector<float> k(e.key.begin(), e.key.end()), v(e.value.begin(), e.value.end());
        std::vector<double> layers(n_layers_ > 0 ? n_layers_ : 1, 0.0), dl(layers.size());
        for (int l = 0; l < n_layers_ && l < static_cast<int>(e.meta.per_layer_scores.size()); ++l)
            layers[l] = e.meta.per_layer_scores[l];
        if (n_layers_ == 0) in.has_layers = 0;
        std::vector<float> dk(dp), dv(dp);
        std::int32_t flag = 0;
        check(pikv_store_insert_host(h_, 0, 1, &in, k.data(), v.data(), in.has_layers ? layers.data() : nullptr,
                                     &out, dk.data(), dv.data(), dl.data(), &flag));
        if (!flag) return std::nullopt;
        KVEntry r;
        r.id = out.id, r.shard_seq = out.shard_seq, r.token_id = out.token_id, r.expert_id = out.expert_id;
        r.key.assign(dk.begin(), dk.end()), r.value.assign(dv.begin(), dv.end());
        r.meta = {out.insert_step, out.last_access_step, out.freq, out.attn_mass, {}};
        if (out.has_layers) r.meta.per_layer_scores.assign(dl.begin(), dl.begin() + n_layers_);
        return r;
    }
    // KVStore::retrieve (kvstore.cpp:122-178)
    RetrievalResult retrieve(const std::vector<int>& experts, std::int64_t since, std::uint64_t now) {
        std::vector<std::int32_t> ex(experts.begin(), experts.end()), missed(experts.size() + 1);
        const std::int64_t cap = pikv_slot_count(h_);
        std::vector<std::int64_t> slots(cap > 0 ? cap : 1);
        std::int32_t n = 0, nm = 0;
        check(pikv_store_retrieve_host(h_, 0, ex.data(), static_cast<std::int32_t>(ex.size()), since, now,
                                       slots.data(), static_cast<std::int32_t>(cap), &n, missed.data(), &nm));
        RetrievalResult r;
        r.slots.assign(slots.begin(), slots.begin() + n);
        r.entries = entries_at(r.slots);
        r.missed_experts.assign(missed.begin(), missed.begin() + nm);
        return r;
    }
    bool erase(std::uint64_t entry_id) {  // kvstore.cpp:180-185
        std::int32_t ok = 0;
        check(pikv_store_erase_host(h_, 0, entry_id, &ok));
        return ok != 0;
    }
    std::uint64_t memory_bytes() const { return stats_raw().memory_bytes; }
    std::uint64_t live_entries() const { return stats_raw().live; }
    StoreCounters stats() const {
        StoreCounters c;
        const auto s = stats_raw();
        c.inserts = s.inserts, c.overwrites = s.overwrites;
        check(pikv_store_counters_host(h_, 0, &c.retrievals, &c.misses));
        return c;
    }
    int devices() const { return cfg_.model.G; }
    int shards_per_device() const { return static_cast<int>(pikv_slot_count(h_) / cfg_.model.S / cfg_.model.G); }
    int stored_width() const { return cfg_.model.d; }
    int shard_capacity() const { return cfg_.model.S; }
    // buffer(device, shard).live_count() (kvstore.hpp:41)
    int live_count(int device, int shard) const {
        std::vector<std::int32_t> live(static_cast<std::size_t>(devices()) * shards_per_device());
        check(pikv_ring_live_host(h_, 0, live.data()));
        return live[static_cast<std::size_t>(device) * shards_per_device() + shard];
    }
    // for_each_live (kvstore.hpp:136-144): fn(device, shard, entry) in slot order
    template <typename Fn>
    void for_each_live(Fn&& fn) const {
        const std::int64_t n = pikv_slot_count(h_);
        std::vector<std::uint64_t> id(n);
        check(pikv_read_slots_host(h_, 0, id.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                   nullptr));
        std::vector<std::int64_t> live;
        for (std::int64_t i = 0; i < n; ++i)
            if (id[i]) live.push_back(i);
        const auto es = entries_at(live);
        const int S = cfg_.model.S, spd = shards_per_device();
        for (std::size_t i = 0; i < live.size(); ++i)
            fn(static_cast<int>(live[i] / S) / spd, static_cast<int>(live[i] / S) % spd, es[i]);
    }
    std::vector<SnapshotRecord> snapshot(std::uint64_t now) const {
        std::int64_t n = 0;
        check(pikv_snapshot_host(h_, 0, static_cast<std::int64_t>(now), nullptr, 0, &n));
        std::vector<pikv_snapshot_record> raw(static_cast<std::size_t>(n));
        if (n) check(pikv_snapshot_host(h_, 0, static_cast<std::int64_t>(now), raw.data(), n, &n));
        std::vector<SnapshotRecord> out;
        for (const auto& r : raw) out.push_back({r.device, r.shard, r.token_id, r.expert_id, r.age, r.freq});
        return out;
    }
    // attention (pipeline.cpp:59-85) of a stored-space query over retrieved entries
    AttentionOutput attention(const std::vector<double>& query, const std::vector<std::int64_t>& slots) {
        if (static_cast<int>(query.size()) != stored_width())
            throw InvalidArgument("attention: key/query width mismatch");
        std::vector<float> q(query.begin(), query.end()), y(stored_width()), a(slots.size() + 1);
        check(pikv_attend_host(h_, 0, q.data(), slots.data(), static_cast<std::int32_t>(slots.size()), y.data(),
                               a.data()));
        AttentionOutput o;
        o.output.assign(y.begin(), y.end());
        o.weights.assign(a.begin(), a.begin() + slots.size());
        o.retrieved = slots.size();
        return o;
    }
    std::vector<KVEntry> entries_at(const std::vector<std::int64_t>& slots) const {
        std::vector<KVEntry> out;
        if (slots.empty()) return out;
        const std::int64_t n = pikv_slot_count(h_);
        std::vector<std::uint64_t> id(n), sq(n), ins(n), la(n), fr(n);
        std::vector<std::int64_t> tok(n);
        std::vector<std::int32_t> ex(n);
        std::vector<double> mass(n), pl(static_cast<std::size_t>(n) * (n_layers_ > 0 ? n_layers_ : 1));
        check(pikv_read_slots_host(h_, 0, id.data(), sq.data(), tok.data(), ex.data(), ins.data(), la.data(),
                                   fr.data(), mass.data(), n_layers_ > 0 ? pl.data() : nullptr));
        const int dp = stored_width();
        std::vector<float> k(slots.size() * dp), v(slots.size() * dp);
        check(pikv_read_entries_host(h_, 0, slots.data(), static_cast<std::int32_t>(slots.size()), k.data(),
                                     v.data()));
        for (std::size_t i = 0; i < slots.size(); ++i) {
            const std::int64_t s = slots[i];
            KVEntry e;
            e.id = id[s], e.shard_seq = sq[s], e.token_id = tok[s], e.expert_id = ex[s];
            e.key.assign(k.begin() + i * dp, k.begin() + (i + 1) * dp);
            e.value.assign(v.begin() + i * dp, v.begin() + (i + 1) * dp);
            e.meta = {ins[s], la[s], fr[s], mass[s], {}};
            if (n_layers_ > 0) e.meta.per_layer_scores.assign(pl.begin() + s * n_layers_, pl.begin() + (s + 1) * n_layers_);
            out.push_back(std::move(e));
        }
        return out;
    }

    // scheduler on this store (scheduler.hpp:118-129), with its SchedulerState
    EvictionReport evict(const SchedulerConfig& cfg, std::uint64_t now) {
        set_scheduler(cfg);
        const std::int64_t cap = pikv_slot_count(h_);
        std::vector<pikv_evict_record> recs(cap > 0 ? cap : 1);
        std::int32_t n = 0, pb = 0, pa = 0;
        check(pikv_evict_host(h_, 0, now, recs.data(), static_cast<std::int32_t>(cap), &n, &pb, &pa));
        EvictionReport r;
        r.pages_before = pb, r.pages_after = pa;
        for (int i = 0; i < n; ++i)
            r.evicted.push_back({recs[i].step, recs[i].entry_id, recs[i].token_id, recs[i].expert_id,
                                 recs[i].device, recs[i].score, static_cast<EvictReason>(recs[i].reason)});
        return r;
    }
    void observe_hits(const SchedulerConfig& cfg, std::uint64_t hits, std::uint64_t lookups) {
        set_scheduler(cfg);
        check(pikv_observe_hits(h_, 0, hits, lookups));
    }
    void adakv_update(const SchedulerConfig& cfg) {
        set_scheduler(cfg);
        check(pikv_adakv_update(h_, 0));
    }
    SchedulerStateView scheduler_state() const {
        SchedulerStateView v;
        check(pikv_read_sched_state_host(h_, 0, &v.theta, &v.running_hit, &v.step));
        return v;
    }
    void set_scheduler_state(double theta, double running_hit) {
        check(pikv_write_sched_state_host(h_, 0, &theta, &running_hit, nullptr));
    }
    pikv_engine* handle() { return h_; }

  private:
    static int d_prime_of(const ModelConfig& m) {  // config.hpp:37-40
        const long long dp = std::llround(m.d / m.rho);
        return dp < 1 ? 1 : static_cast<int>(dp);
    }
    void set_scheduler(const SchedulerConfig& cfg) {
        if (cfg.page_size != cfg_.scheduler.page_size)
            throw InvalidConfig("evict: the store was built for another page_size");
        cfg_.scheduler = cfg;
        pikv_config pc = cfg_.to_c();
        check(pikv_update_config(h_, &pc));
    }
    pikv_store_stats_view stats_raw() const {
        pikv_store_stats_view s{};
        check(pikv_store_stats_host(h_, 0, &s.live, &s.memory_bytes, &s.inserts, &s.overwrites));
        return s;
    }
    EngineConfig cfg_;
    int n_layers_ = 0;
    pikv_engine* h_ = nullptr;
};

// score_entry (scheduler.cpp:181-229) of one entry's metadata, on the GPU.
inline double score_entry(const KVEntry& e, const SchedulerConfig& cfg, std::uint64_t now) {
    EngineConfig ec;
    ec.scheduler = cfg;
    ec.n_layers = static_cast<int>(e.meta.per_layer_scores.size());
    pikv_config pc = ec.to_c();
    pikv_entry in = detail::to_c(e);
    double out = 0.0;
    check(pikv_score_entries_host(&pc, &in, e.meta.per_layer_scores.empty() ? nullptr : e.meta.per_layer_scores.data(),
                                  1, now, &out));
    return out;
}

struct RoutingDecision {  // router.hpp:58-62
    std::vector<int> experts;
    std::vector<double> gates;
    std::vector<double> logits;
};

// RouterState::init(experts, width, seed) (router.cpp:54-67): W_r =
// Rng(seed) N(0, 1/d) and the load / usage / miss / bias estimators in HBM.
// Sized for one k at a time; a call with another k moves the state over.
class RouterState {
  public:
    static RouterState init(int experts, int width, std::uint64_t seed) { return RouterState(experts, width, seed); }
    RouterState(int experts, int width, std::uint64_t seed) : E_(experts), d_(width), seed_(seed) {}
    ~RouterState() { if (h_) pikv_engine_destroy(h_); }
    RouterState(RouterState&& o) noexcept { *this = std::move(o); }
    RouterState& operator=(RouterState&& o) noexcept {
        std::swap(E_, o.E_), std::swap(d_, o.d_), std::swap(seed_, o.seed_), std::swap(h_, o.h_);
        std::swap(cfg_, o.cfg_);
        return *this;
    }
    RouterStateView view() const {
        RouterStateView r;
        r.load.assign(E_, 0.0), r.bandit_bias.assign(E_, 0.0), r.usage_counts.assign(E_, 0), r.miss_counts.assign(E_, 0);
        if (h_)
            check(pikv_read_router_state_host(h_, 0, r.load.data(), r.usage_counts.data(), r.miss_counts.data(),
                                              r.bandit_bias.data(), &r.step, &r.total_usage));
        return r;
    }
    void set_load(const std::vector<double>& v) { bind(cfg_.router); write(v.data(), nullptr); }
    void set_bias(const std::vector<double>& v) { bind(cfg_.router); write(nullptr, v.data()); }
    int experts() const { return E_; }
    int width() const { return d_; }

    pikv_engine* bind(const RouterConfig& rc) {
        if (h_ && rc.k == cfg_.router.k) {
            cfg_.router = rc;
            pikv_config pc = cfg_.to_c();
            check(pikv_update_config(h_, &pc));
            return h_;
        }
        const bool carry = h_ != nullptr;
        const RouterStateView old = view();
        if (h_) pikv_engine_destroy(h_), h_ = nullptr;
        cfg_ = EngineConfig{};
        cfg_.model.d = d_, cfg_.model.head_width = 1, cfg_.model.E = E_, cfg_.model.G = 1, cfg_.model.S = 1;
        cfg_.store.n_tok = 1, cfg_.store.n_exp = 1;
        cfg_.router = rc;
        cfg_.unbounded_budget = true;
        cfg_.seed = seed_ ^ 0x2545f4914f6cdd1dULL;  // the engine seeds W_r with seed ^ kRouterSalt
        cfg_.pool_entries = 16;
        pikv_config pc = cfg_.to_c();
        check(pikv_engine_create(&pc, 0, &h_));
        if (carry)
            check(pikv_write_router_state_host(h_, 0, old.load.data(), old.usage_counts.data(), old.miss_counts.data(),
                                               old.bandit_bias.data(), &old.step, &old.total_usage));
        return h_;
    }

  private:
    void write(const double* load, const double* bias) {
        check(pikv_write_router_state_host(h_, 0, load, nullptr, nullptr, bias, nullptr, nullptr));
    }
    int E_ = 0, d_ = 0;
    std::uint64_t seed_ = 0;
    EngineConfig cfg_;
    pikv_engine* h_ = nullptr;
};

namespace detail {
inline RoutingDecision decision(pikv_engine* h, int k, int E, const double* q, const double* logits) {
    RoutingDecision d;
    d.experts.resize(k), d.gates.resize(k), d.logits.resize(E);
    std::vector<std::int32_t> ex(k);
    if (logits) check(pikv_route_logits_host(h, 0, logits, ex.data(), d.gates.data(), d.logits.data()));
    else check(pikv_route_host(h, 0, q, ex.data(), d.gates.data(), d.logits.data()));
    d.experts.assign(ex.begin(), ex.end());
    return d;
}
}  // namespace detail

// route (router.cpp:216-234): exact fp64 logits W_r q, penalty, selection
inline RoutingDecision route(const std::vector<double>& query, RouterState& st, const RouterConfig& cfg) {
    if (cfg.strategy != RouterStrategy::Base && static_cast<int>(query.size()) != st.width())
        throw InvalidArgument("route: query width != d");
    return detail::decision(st.bind(cfg), cfg.k, st.experts(), query.data(), nullptr);
}
// route_logits (router.cpp:122-214)
inline RoutingDecision route_logits(const std::vector<double>& logits, RouterState& st, const RouterConfig& cfg) {
    if (static_cast<int>(logits.size()) != st.experts()) throw InvalidArgument("route_logits: logit width != E");
    return detail::decision(st.bind(cfg), cfg.k, st.experts(), nullptr, logits.data());
}
inline void record_miss(RouterState& st, int expert, const RouterConfig& cfg = {}) {  // router.cpp:236-241
    check(pikv_record_miss(st.bind(cfg), 0, expert));
}
inline void adapt(RouterState& st, const RoutingDecision& d, double reward, const RouterConfig& cfg) {
    std::vector<std::int32_t> ex(d.experts.begin(), d.experts.end());  // router.cpp:243-255
    check(pikv_router_adapt(st.bind(cfg), 0, ex.data(), static_cast<std::int32_t>(ex.size()), reward));
}

// Codec (compressor.hpp:57-80): encode_vector / decode_vector on the GPU for
// Identity / LowRank (SVD, LoRA) / LoRAPlus / FastV / Prune.  Projection
// bases come from the caller (fitting is offline); FastV and Prune fit here.
class Codec {
  public:
    static Codec identity(int d) { return Codec(PIKV_CODEC_IDENTITY, d, d); }
    static Codec lowrank(int d, int r, std::vector<float> basis /* [r][d] */, std::vector<float> bias = {}) {
        Codec c(bias.empty() ? PIKV_CODEC_LOWRANK : PIKV_CODEC_LORAPLUS, d, r);
        c.basis_ = std::move(basis), c.bias_ = std::move(bias);
        return c;
    }
    static Codec fastv(int d, int r) { return Codec(PIKV_CODEC_FASTV, d, r); }
    // Prune fit (compressor.cpp:250-262): keep the d - ceil(frac d) highest-
    // variance coordinates (ties by index), sorted
    static Codec fit_prune(const std::vector<std::vector<double>>& rows, double prune_frac) {
        if (rows.empty()) throw InsufficientCalibration("Prune: no calibration rows");
        const int d = static_cast<int>(rows[0].size()), n = static_cast<int>(rows.size());
        std::vector<double> flat, var(d);
        for (const auto& r : rows) flat.insert(flat.end(), r.begin(), r.end());
        check(pikv_column_variance_host(flat.data(), n, d, var.data()));
        int keep = d - static_cast<int>(std::ceil(prune_frac * d));
        if (keep < 1) keep = 1;
        std::vector<int> order(d);
        for (int i = 0; i < d; ++i) order[i] = i;
        std::sort(order.begin(), order.end(), [&](int a, int b) { return var[a] != var[b] ? var[a] > var[b] : a < b; });
        Codec c(PIKV_CODEC_PRUNE, d, keep);
        c.kept_.assign(order.begin(), order.begin() + keep);
        std::sort(c.kept_.begin(), c.kept_.end());
        return c;
    }
    int stored_width() const { return r_; }
    std::vector<int> zero_set() const {
        std::vector<int> z;
        for (int i = 0; i < d_; ++i)
            if (codec_ == PIKV_CODEC_PRUNE && !std::binary_search(kept_.begin(), kept_.end(), i)) z.push_back(i);
        return z;
    }
    std::vector<double> encode_vector(const std::vector<double>& x) const {
        if (static_cast<int>(x.size()) != d_) throw InvalidEntry("encode: width mismatch");
        return run(false, x, r_);
    }
    std::vector<double> decode_vector(const std::vector<double>& y) const {
        if (static_cast<int>(y.size()) != r_) throw CodecMismatch("decode: payload width mismatch");
        return run(true, y, d_);
    }
    double reconstruction_error(const std::vector<double>& x) const {  // compressor.cpp:551-572
        const auto xr = decode_vector(encode_vector(x));
        double num = 0, den = 0;
        for (std::size_t i = 0; i < x.size(); ++i) num += (x[i] - xr[i]) * (x[i] - xr[i]), den += x[i] * x[i];
        if (den == 0.0) throw InvalidArgument("reconstruction_error: zero-norm input");
        return std::sqrt(num / den);
    }

  private:
    Codec(int codec, int d, int r) : codec_(codec), d_(d), r_(r) {}
    std::vector<double> run(bool decode, const std::vector<double>& in, int wout) const {
        std::vector<float> x(in.begin(), in.end()), y(wout);
        const int r = codec_ == PIKV_CODEC_IDENTITY ? d_ : r_;
        const float* b = basis_.empty() ? nullptr : basis_.data();
        const float* bi = bias_.empty() ? nullptr : bias_.data();
        const std::int32_t* k = kept_.empty() ? nullptr : kept_.data();
        check(decode ? pikv_codec_decode_host(codec_, 1, 1, d_, r, b, bi, k, x.data(), y.data())
                     : pikv_codec_encode_host(codec_, 1, 1, d_, r, b, bi, k, x.data(), y.data()));
        return std::vector<double>(y.begin(), y.end());
    }
    int codec_ = PIKV_CODEC_IDENTITY, d_ = 0, r_ = 0;
    std::vector<float> basis_, bias_;
    std::vector<std::int32_t> kept_;
};

// Micro-batch pipeline (include/pikv_b200.h, pikv_group_*; no reference
// counterpart): the B streams split into n_micro engines whose control plane
// overlaps each other's attention.  Serving loop per micro-batch m:
// wait(m) -> the caller's next-token inputs -> submit(m, ...).  Host buffers
// (pinned for asynchronous copies): q/k/v [B/n][d] in the kv dtype (uint16
// bf16 bits or float), y [B/n][d'] fp32, valid after the next wait(m).
class EngineGroup {
  public:
    explicit EngineGroup(const EngineConfig& cfg, int n_micro = 2, int attend_sms = 0) : cfg_(cfg) {
        pikv_config c = cfg.to_c();
        check(pikv_group_create(&c, n_micro, attend_sms, cfg.cuda_device, &g_));
    }
    ~EngineGroup() { if (g_) pikv_group_destroy(g_); }
    EngineGroup(const EngineGroup&) = delete;
    EngineGroup& operator=(const EngineGroup&) = delete;

    int size() const { return pikv_group_size(g_); }
    int streams_per_micro() const { return cfg_.batch / size(); }
    void set_codec(const std::vector<float>& basis, const std::vector<float>& bias = {},
                   const std::vector<std::int32_t>& kept = {}) {
        for (int m = 0; m < size(); ++m)
            check(pikv_set_codec_host(pikv_group_engine(g_, m), basis.empty() ? nullptr : basis.data(),
                                      bias.empty() ? nullptr : bias.data(), kept.empty() ? nullptr : kept.data()));
    }
    void submit(int m, const void* q, const void* k, const void* v, float* y) {
        check(pikv_group_submit(g_, m, q, k, v, nullptr, y, 1));
    }
    void wait(int m) { check(pikv_group_wait(g_, m)); }
    void sync() { check(pikv_group_sync(g_)); }
    pikv_engine* engine(int m) { return pikv_group_engine(g_, m); }

  private:
    EngineConfig cfg_;
    pikv_group* g_ = nullptr;
};

// ---- wire formats of the reference's run output (runner.cpp) --------------
// nlohmann::json dump(): keys sorted, compact, doubles as nlohmann's grisu2
// digits in its layout (fixed for decimal exponents -4 < n <= 15).
namespace wire {

// Grisu2 (Loitsch 2010) digits d1..dk and exponent (value = d1..dk 10^exp)
// exactly as nlohmann's dtoa_impl generates them, including the doubles
// where grisu2 is not the shortest form (1e23 -> 9.999999999999999e+22).
inline void grisu2(double v, std::string& digits, int& dec_exp) {
    struct Fp { std::uint64_t f; int e; };
    struct Cached { std::uint64_t f; int e; int k; };
    static const Cached pow10[] = {
        {0xAB70FE17C79AC6CAULL, -1060, -300}, {0xFF77B1FCBEBCDC4FULL, -1034, -292}, {0xBE5691EF416BD60CULL, -1007, -284},
        {0x8DD01FAD907FFC3CULL, -980, -276}, {0xD3515C2831559A83ULL, -954, -268}, {0x9D71AC8FADA6C9B5ULL, -927, -260},
        {0xEA9C227723EE8BCBULL, -901, -252}, {0xAECC49914078536DULL, -874, -244}, {0x823C12795DB6CE57ULL, -847, -236},
        {0xC21094364DFB5637ULL, -821, -228}, {0x9096EA6F3848984FULL, -794, -220}, {0xD77485CB25823AC7ULL, -768, -212},
        {0xA086CFCD97BF97F4ULL, -741, -204}, {0xEF340A98172AACE5ULL, -715, -196}, {0xB23867FB2A35B28EULL, -688, -188},
        {0x84C8D4DFD2C63F3BULL, -661, -180}, {0xC5DD44271AD3CDBAULL, -635, -172}, {0x936B9FCEBB25C996ULL, -608, -164},
        {0xDBAC6C247D62A584ULL, -582, -156}, {0xA3AB66580D5FDAF6ULL, -555, -148}, {0xF3E2F893DEC3F126ULL, -529, -140},
        {0xB5B5ADA8AAFF80B8ULL, -502, -132}, {0x87625F056C7C4A8BULL, -475, -124}, {0xC9BCFF6034C13053ULL, -449, -116},
        {0x964E858C91BA2655ULL, -422, -108}, {0xDFF9772470297EBDULL, -396, -100}, {0xA6DFBD9FB8E5B88FULL, -369, -92},
        {0xF8A95FCF88747D94ULL, -343, -84}, {0xB94470938FA89BCFULL, -316, -76}, {0x8A08F0F8BF0F156BULL, -289, -68},
        {0xCDB02555653131B6ULL, -263, -60}, {0x993FE2C6D07B7FACULL, -236, -52}, {0xE45C10C42A2B3B06ULL, -210, -44},
        {0xAA242499697392D3ULL, -183, -36}, {0xFD87B5F28300CA0EULL, -157, -28}, {0xBCE5086492111AEBULL, -130, -20},
        {0x8CBCCC096F5088CCULL, -103, -12}, {0xD1B71758E219652CULL, -77, -4}, {0x9C40000000000000ULL, -50, 4},
        {0xE8D4A51000000000ULL, -24, 12}, {0xAD78EBC5AC620000ULL, 3, 20}, {0x813F3978F8940984ULL, 30, 28},
        {0xC097CE7BC90715B3ULL, 56, 36}, {0x8F7E32CE7BEA5C70ULL, 83, 44}, {0xD5D238A4ABE98068ULL, 109, 52},
        {0x9F4F2726179A2245ULL, 136, 60}, {0xED63A231D4C4FB27ULL, 162, 68}, {0xB0DE65388CC8ADA8ULL, 189, 76},
        {0x83C7088E1AAB65DBULL, 216, 84}, {0xC45D1DF942711D9AULL, 242, 92}, {0x924D692CA61BE758ULL, 269, 100},
        {0xDA01EE641A708DEAULL, 295, 108}, {0xA26DA3999AEF774AULL, 322, 116}, {0xF209787BB47D6B85ULL, 348, 124},
        {0xB454E4A179DD1877ULL, 375, 132}, {0x865B86925B9BC5C2ULL, 402, 140}, {0xC83553C5C8965D3DULL, 428, 148},
        {0x952AB45CFA97A0B3ULL, 455, 156}, {0xDE469FBD99A05FE3ULL, 481, 164}, {0xA59BC234DB398C25ULL, 508, 172},
        {0xF6C69A72A3989F5CULL, 534, 180}, {0xB7DCBF5354E9BECEULL, 561, 188}, {0x88FCF317F22241E2ULL, 588, 196},
        {0xCC20CE9BD35C78A5ULL, 614, 204}, {0x98165AF37B2153DFULL, 641, 212}, {0xE2A0B5DC971F303AULL, 667, 220},
        {0xA8D9D1535CE3B396ULL, 694, 228}, {0xFB9B7CD9A4A7443CULL, 720, 236}, {0xBB764C4CA7A44410ULL, 747, 244},
        {0x8BAB8EEFB6409C1AULL, 774, 252}, {0xD01FEF10A657842CULL, 800, 260}, {0x9B10A4E5E9913129ULL, 827, 268},
        {0xE7109BFBA19C0C9DULL, 853, 276}, {0xAC2820D9623BF429ULL, 880, 284}, {0x80444B5E7AA7CF85ULL, 907, 292},
        {0xBF21E44003ACDD2DULL, 933, 300}, {0x8E679C2F5E44FF8FULL, 960, 308}, {0xD433179D9C8CB841ULL, 986, 316},
        {0x9E19DB92B4E31BA9ULL, 1013, 324}};
    auto normalize = [](Fp x) {
        while (!(x.f >> 63)) x.f <<= 1, --x.e;
        return x;
    };
    auto mul = [](Fp a, Fp b) {  // high 64 bits of the product, rounded half up
        const unsigned __int128 p = (unsigned __int128)a.f * b.f + ((unsigned __int128)1 << 63);
        return Fp{(std::uint64_t)(p >> 64), a.e + b.e + 64};
    };
    std::uint64_t bits;
    std::memcpy(&bits, &v, 8);
    const std::uint64_t E = bits >> 52, F = bits & ((1ULL << 52) - 1);
    const Fp w0 = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (1ULL << 52), static_cast<int>(E) - 1075};
    const bool closer = F == 0 && E > 1;
    const Fp mp = normalize(Fp{2 * w0.f + 1, w0.e - 1});
    Fp mm = closer ? Fp{4 * w0.f - 1, w0.e - 2} : Fp{2 * w0.f - 1, w0.e - 1};
    mm = Fp{mm.f << (mm.e - mp.e), mp.e};
    const Fp w = normalize(w0);
    const int fx = -60 - mp.e - 1;
    const int k = fx * 78913 / (1 << 18) + (fx > 0);
    const Cached c = pow10[(300 + k + 7) / 8];
    const Fp cw = mul(w, {c.f, c.e}), cmm = mul(mm, {c.f, c.e}), cmp = mul(mp, {c.f, c.e});
    const Fp Mm{cmm.f + 1, cmm.e}, Mp{cmp.f - 1, cmp.e};
    dec_exp = -c.k;
    std::uint64_t delta = Mp.f - Mm.f, dist = Mp.f - cw.f;
    const int shift = -Mp.e;
    const std::uint64_t one = 1ULL << shift;
    std::uint32_t p1 = static_cast<std::uint32_t>(Mp.f >> shift);
    std::uint64_t p2 = Mp.f & (one - 1);
    digits.clear();
    auto round = [&](std::uint64_t rest, std::uint64_t ten_k) {
        while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
            --digits.back();
            rest += ten_k;
        }
    };
    int n = 1;
    std::uint32_t p10 = 1;
    while (p10 <= p1 / 10) p10 *= 10, ++n;
    while (n > 0) {
        digits.push_back(static_cast<char>('0' + p1 / p10));
        p1 %= p10;
        --n;
        const std::uint64_t rest = (static_cast<std::uint64_t>(p1) << shift) + p2;
        if (rest <= delta) {
            dec_exp += n;
            round(rest, static_cast<std::uint64_t>(p10) << shift);
            return;
        }
        p10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10, delta *= 10, dist *= 10;
        digits.push_back(static_cast<char>('0' + (p2 >> shift)));
        p2 &= one - 1;
        ++m;
        if (p2 <= delta) break;
    }
    dec_exp -= m;
    round(p2, one);
}

inline std::string json_double(double x) {
    if (x != x || x - x != 0.0) return "null";  // NaN, inf
    if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
    std::string ds;
    int ex = 0;
    grisu2(x < 0 ? -x : x, ds, ex);
    const int k = static_cast<int>(ds.size());
    const int n = k + ex;  // value = 0.d1..dk * 10^n
    std::string out = x < 0 ? "-" : "";
    if (k <= n && n <= 15) return out + ds + std::string(n - k, '0') + ".0";
    if (0 < n && n <= 15) return out + ds.substr(0, n) + "." + ds.substr(n);
    if (-4 < n && n <= 0) return out + "0." + std::string(-n, '0') + ds;
    const int e = n - 1;
    std::string es = std::to_string(e < 0 ? -e : e);
    if (es.size() < 2) es = "0" + es;
    out += ds.substr(0, 1);
    if (k > 1) out += "." + ds.substr(1);
    return out + "e" + (e < 0 ? "-" : "+") + es;
}

inline const char* reason_name(EvictReason r) {  // scheduler.cpp:40-46
    return r == EvictReason::Budget ? "budget" : r == EvictReason::Threshold ? "threshold" : "overwrite";
}

// runner.cpp:215-222 (store dump line)
inline std::string store_dump_line(const SnapshotRecord& r) {
    return "{\"age\":" + std::to_string(r.age) + ",\"device\":" + std::to_string(r.device) +
           ",\"expert\":" + std::to_string(r.expert_id) + ",\"freq\":" + std::to_string(r.freq) +
           ",\"shard\":" + std::to_string(r.shard) + ",\"token\":" + std::to_string(r.token_id) + "}";
}

// runner.cpp:58-65 (eviction_json)
inline std::string eviction_line(const EvictionRecord& r) {
    return "{\"device\":" + std::to_string(r.device) + ",\"expert\":" + std::to_string(r.expert_id) +
           ",\"id\":" + std::to_string(r.entry_id) + ",\"reason\":\"" + reason_name(r.reason) +
           "\",\"score\":" + json_double(r.score) + ",\"token\":" + std::to_string(r.token_id) + "}";
}

}  // namespace wire

}  // namespace pikv::b200
