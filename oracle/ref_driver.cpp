// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — step driver over the reference's OWN objects.
//
// Linked (by oracle/build.py) against the reference translation units
// compiled from /root/reference/proj unchanged (mathops.cpp, kvstore.cpp,
// router.cpp) and hash-verified line extracts of scheduler.cpp (49-80,
// 162-350: SchedulerConfig/State, score_entry, select_evictions, evict,
// observe_hits, adakv_update) and pipeline.cpp (59-85: attention), which are
// the Eigen-free parts of those files.  Output: oracle/_ref/libpikv_ref.so.
//
// `ref_step` follows Engine::step (pipeline.cpp:213-351) with an Identity
// codec and caller-supplied q/k/v in place of QueryEncoder: route ->
// insert (+overwrite records) -> evict -> retrieve -> attention -> fold-back
// -> adapt/observe_hits/adakv_update -> now++.  Multi-head: each head is an
// independent reference attention() call on its d/H slice and attn_mass
// gains the mean over heads; at H = 1 this IS Engine::step.
#include <chrono>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "pikv/errors.hpp"
#include "pikv/costmodel.hpp"
#include "pikv/kvstore.hpp"
#include "pikv/trace.hpp"
#include "pikv/pipeline.hpp"
#include "pikv/rng.hpp"
#include "pikv/router.hpp"
#include "pikv/scheduler.hpp"
#include "pikv_oracle.h"  // pikv_config / po_step_out layouts only

using namespace pikv;

namespace {

constexpr std::uint64_t kRouterSalt = 0x2545f4914f6cdd1dULL;  // pipeline.cpp:16

int code_of(const std::exception& ex) {
    if (dynamic_cast<const InvalidArgument*>(&ex)) return PIKV_ERR_INVALID_ARGUMENT;
    if (dynamic_cast<const InvalidConfig*>(&ex)) return PIKV_ERR_INVALID_CONFIG;
    if (dynamic_cast<const InvalidEntry*>(&ex)) return PIKV_ERR_INVALID_ENTRY;
    if (dynamic_cast<const NumericalError*>(&ex)) return PIKV_ERR_NUMERICAL;
    if (dynamic_cast<const NotFitted*>(&ex)) return PIKV_ERR_NOT_FITTED;
    return PIKV_ERR_INVALID_ARGUMENT;
}

ModelConfig model_of(const pikv_config& c) {
    ModelConfig m;
    m.d = c.d;
    m.head_width = c.head_width;
    m.E = c.E;
    m.k = c.k;
    m.L = c.L;
    m.G = c.G;
    m.S = c.S;
    m.K = c.K;
    m.rho = c.rho;
    m.elem_bytes = c.elem_bytes;
    return m;
}

StoreConfig store_of(const pikv_config& c) {
    StoreConfig s;
    s.n_tok = c.n_tok;
    s.n_exp = c.n_exp;
    s.additive = c.additive != 0;
    s.shards_per_device = c.shards_per_device;
    return s;
}

RouterConfig router_of(const pikv_config& c) {
    RouterConfig r;
    r.strategy = static_cast<RouterStrategy>(c.router_strategy);
    r.k = c.k;
    r.alpha = c.alpha;
    r.lambda_miss = c.lambda_miss;
    r.beta_ent = c.beta_ent;
    r.bandit_step = c.bandit_step;
    r.groups = c.groups;
    r.stride = c.stride;
    r.bias_cap = c.bias_cap;
    r.load_decay = c.load_decay;
    return r;
}

SchedulerConfig sched_of(const pikv_config& c) {
    SchedulerConfig s;
    s.strategy = static_cast<SchedStrategy>(c.sched_strategy);
    s.budget_pages = c.budget_pages;
    s.page_size = c.page_size;
    s.tau = c.tau;
    s.sink = c.sink;
    s.lambda_freq = c.lambda_freq;
    s.adakv_step = c.adakv_step;
    s.target_hit = c.target_hit;
    s.gamma_sim = c.gamma_sim;
    s.theta0 = c.theta0;
    s.hit_decay = c.hit_decay;
    s.adakv_weights.assign(c.adakv_weights, c.adakv_weights + c.n_adakv_weights);
    s.flex_plan.assign(c.flex_plan, c.flex_plan + c.n_flex_plan);
    s.flex_bucket = c.flex_bucket;
    return s;
}

}  // namespace

struct ref_engine {
    pikv_config c;
    ModelConfig model;
    RouterConfig router;
    SchedulerConfig sched;
    KVStore store;
    RouterState rs;
    SchedulerState ss;
    std::uint64_t now = 0;

    explicit ref_engine(const pikv_config& cfg)
        : c(cfg),
          model(model_of(cfg)),
          router(router_of(cfg)),
          sched(sched_of(cfg)),
          store(model, store_of(cfg)),
          rs(RouterState::init(cfg.E, cfg.d, cfg.seed ^ kRouterSalt)),
          ss(SchedulerState::init(sched)) {
        model.validate();
        router.validate(model.E);
    }
};

extern "C" {

ref_engine* ref_create(const pikv_config* cfg, const double* w_r, int* err) {
    try {
        if (cfg->codec != PIKV_CODEC_IDENTITY) throw InvalidConfig("ref: identity codec only");
        if (cfg->n_heads < 1 || cfg->d % cfg->n_heads) throw InvalidConfig("ref: heads");
        auto* e = new ref_engine(*cfg);
        if (w_r) std::memcpy(e->rs.routing_matrix.data(), w_r, sizeof(double) * cfg->E * cfg->d);
        if (err) *err = 0;
        return e;
    } catch (const std::exception& ex) {
        if (err) *err = code_of(ex);
        return nullptr;
    }
}

void ref_destroy(ref_engine* e) { delete e; }

int ref_shards_per_device(ref_engine* e) { return e->store.shards_per_device(); }

static int step_impl(ref_engine* e, const double* q, const double* k, const double* v,
                     const double* saliency, po_step_out* out, bool attend) {
    try {
        const pikv_config& c = e->c;
        const int d = c.d;
        out->inserts = out->hits = out->lookups = out->n_attended = 0;
        out->fetch_elements = 0;
        out->pages_before = out->pages_after = 0;
        out->n_evictions = 0;
        auto token_id = static_cast<std::int64_t>(e->now);
        std::vector<double> query(q, q + d), key(k, k + d), value(v, v + d);
        std::vector<double> sal;
        if (c.n_layers > 0 && saliency) sal.assign(saliency, saliency + c.n_layers);

        auto emit = [&](const EvictionRecord& r) {
            if (out->evictions && out->n_evictions < out->evict_cap) {
                po_evict& o = out->evictions[out->n_evictions];
                o.step = r.step;
                o.id = r.entry_id;
                o.token = r.token_id;
                o.expert = r.expert_id;
                o.device = r.device;
                o.score = r.score;
                o.reason = static_cast<int>(r.reason);
                o.stream = 0;
            }
            out->n_evictions += 1;
        };

        // pipeline.cpp:223
        auto decision = route(query, e->rs, e->router);
        for (int j = 0; j < c.k; ++j) {
            out->experts[j] = decision.experts[j];
            out->gates[j] = decision.gates[j];
        }
        if (out->logits)
            for (int i = 0; i < c.E; ++i) out->logits[i] = decision.logits[i];
        // pipeline.cpp:228-246 + 148-211 (Identity codec)
        for (int ex : decision.experts) {
            KVEntry en;
            en.token_id = token_id;
            en.expert_id = ex;
            en.key = key;
            en.value = value;
            en.meta.insert_step = e->now;
            en.meta.last_access_step = e->now;
            en.meta.per_layer_scores = sal;
            auto displaced = e->store.insert(std::move(en));
            if (displaced.has_value()) {
                emit({e->now, displaced->id, displaced->token_id, displaced->expert_id,
                      e->store.locate(displaced->token_id, displaced->expert_id).device, 0.0,
                      EvictReason::Overwrite});
            }
            out->inserts += 1;
        }
        // pipeline.cpp:249-254
        if (!c.unbounded_budget) {
            auto report = evict(e->store, e->ss, e->sched, nullptr, e->now);
            for (const auto& r : report.evicted) emit(r);
            out->pages_before = report.pages_before;
            out->pages_after = report.pages_after;
        }
        // pipeline.cpp:257-264
        auto retrieval = e->store.retrieve(decision.experts, token_id, e->now);
        for (int ex : retrieval.missed_experts) record_miss(e->rs, ex);
        out->lookups = static_cast<int>(decision.experts.size());
        out->hits = out->lookups - static_cast<int>(retrieval.missed_experts.size());
        const int dp = e->store.stored_width();
        out->fetch_elements = static_cast<std::int64_t>(retrieval.entries.size()) *
                              (2 * std::min(c.head_width, dp) + dp);
        const int n = static_cast<int>(retrieval.entries.size());
        out->n_attended = n;
        if (attend) {
            // pipeline.cpp:295-312, per head
            const int H = c.n_heads, w = d / H;
            std::vector<double> alpha(n, 0.0);
            for (int h = 0; h < H; ++h) {
                std::vector<KVEntry> view(n);
                std::vector<const KVEntry*> ptrs(n);
                for (int i = 0; i < n; ++i) {
                    const KVEntry* src = retrieval.entries[i];
                    view[i].key.assign(src->key.begin() + h * w, src->key.begin() + (h + 1) * w);
                    view[i].value.assign(src->value.begin() + h * w,
                                         src->value.begin() + (h + 1) * w);
                    ptrs[i] = &view[i];
                }
                std::span<const double> qh(query.data() + h * w, w);
                auto att = attention(qh, ptrs);
                for (int j = 0; j < w; ++j) out->y[h * w + j] = att.output[j];
                for (int i = 0; i < n; ++i) alpha[i] += att.weights[i];
            }
            for (int i = 0; i < n; ++i) {
                KVEntry* en = retrieval.entries[i];
                double a = alpha[i] / H;
                en->meta.attn_mass += a;
                if (!en->meta.per_layer_scores.empty()) {
                    en->meta.per_layer_scores[e->now % en->meta.per_layer_scores.size()] += a;
                }
                if (i < out->att_cap) {
                    if (out->att_token) out->att_token[i] = en->token_id;
                    if (out->att_expert) out->att_expert[i] = en->expert_id;
                    if (out->att_weight) out->att_weight[i] = a;
                }
            }
        }
        // pipeline.cpp:337-347
        if (e->router.strategy == RouterStrategy::Adaptive) {
            double reward =
                out->lookups == 0 ? 0.0 : static_cast<double>(out->hits) / out->lookups;
            adapt(e->rs, decision, reward, e->router);
        }
        observe_hits(e->ss, e->sched, out->hits, out->lookups);
        if (e->sched.strategy == SchedStrategy::AdaKV && !c.unbounded_budget) {
            adakv_update(e->ss, e->sched);
        }
        e->now += 1;
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

int ref_step(ref_engine* e, const double* q, const double* k, const double* v,
             const double* saliency, po_step_out* out) {
    return step_impl(e, q, k, v, saliency, out, true);
}

int ref_step_noattend(ref_engine* e, const double* q, const double* k, const double* v,
                      const double* saliency, po_step_out* out) {
    return step_impl(e, q, k, v, saliency, out, false);
}

// Slot dump in (device, shard, slot) order like po_engine_dump_slots.  The
// reference grows slots lazily; absent slots read as empty (id 0).
int ref_dump_slots(ref_engine* e, uint64_t* id, uint64_t* shard_seq, int64_t* token,
                   int32_t* expert, uint64_t* insert_step, uint64_t* last_access, uint64_t* freq,
                   double* attn_mass) {
    const int G = e->store.devices(), spd = e->store.shards_per_device(), S = e->c.S;
    const std::size_t n = static_cast<std::size_t>(G) * spd * S;
    if (id) std::memset(id, 0, n * sizeof(uint64_t));
    for (int dev = 0; dev < G; ++dev) {
        for (int sh = 0; sh < spd; ++sh) {
            // for_each_live visits slots in slot order; recover slot indices
            // from shard_seq (slot == shard_seq % S for this ring).
            e->store.buffer(dev, sh).for_each_live([&](const KVEntry& en) {
                std::size_t gi = (static_cast<std::size_t>(dev) * spd + sh) * S + en.shard_seq % S;
                if (id) id[gi] = en.id;
                if (shard_seq) shard_seq[gi] = en.shard_seq;
                if (token) token[gi] = en.token_id;
                if (expert) expert[gi] = en.expert_id;
                if (insert_step) insert_step[gi] = en.meta.insert_step;
                if (last_access) last_access[gi] = en.meta.last_access_step;
                if (freq) freq[gi] = en.meta.freq;
                if (attn_mass) attn_mass[gi] = en.meta.attn_mass;
            });
        }
    }
    return 0;
}

// The reference's own cost_report (costmodel.cpp:123-135), flattened:
// out[0..2] memory, [3..5] memory_bytes, [6..10] shard (exact, floor, ceil,
// best_integer, best_cost), [11..13] latency, [14..21] roofline (io_dense,
// io_sparse, rd_dense, rd_sparse, hit_rate, arith_intensity,
// throughput_scaling, compute_bound), [22..24] utilization (eta, threshold,
// pass), [25] mem_total_optimal, [26] speedup(1, rho).  hw = beta, gamma,
// eta, peak_compute, peak_mem_bw.
int ref_cost_report(const pikv_config* c, const double* hw, double batch, int active, double thr,
                    double* out) {
    try {
        const ModelConfig m = model_of(*c);
        HardwareProfile h;
        h.hbm_bandwidth = hw[0];
        h.core_throughput = hw[1];
        h.decode_factor = hw[2];
        h.peak_compute = hw[3];
        h.peak_mem_bw = hw[4];
        const CostReport r = cost_report(m, h, batch, active, thr);
        const double v[] = {r.memory.token, r.memory.page, r.memory.total,
                            r.memory_bytes.token, r.memory_bytes.page, r.memory_bytes.total,
                            r.shard.exact, (double)r.shard.floor_candidate, (double)r.shard.ceil_candidate,
                            (double)r.shard.best_integer, r.shard.best_cost,
                            r.latency.read, r.latency.decode, r.latency.step,
                            r.roofline.io_dense, r.roofline.io_sparse, r.roofline.rd_dense,
                            r.roofline.rd_sparse, r.roofline.hit_rate, r.roofline.arith_intensity,
                            r.roofline.throughput_scaling, r.roofline.compute_bound ? 1.0 : 0.0,
                            r.utilization.eta_util, r.utilization.threshold, r.utilization.pass ? 1.0 : 0.0,
                            mem_total_optimal(m), speedup(1.0, m.rho)};
        std::memcpy(out, v, sizeof(v));
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

// The reference's own QueryEncoder (pipeline.cpp:29-57): construct from the
// seed and encode one embedding.
int ref_encode(int width, uint64_t seed, const double* x, double* q, double* k, double* v) {
    try {
        QueryEncoder enc(width, seed);
        const auto r = enc.encode(std::span<const double>(x, static_cast<std::size_t>(width)));
        std::memcpy(q, r.query.data(), sizeof(double) * width);
        std::memcpy(k, r.key.data(), sizeof(double) * width);
        std::memcpy(v, r.value.data(), sizeof(double) * width);
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

// The reference's own generate_trace (trace.cpp:54-82) and trace file I/O
// (save_trace / load_trace, trace.cpp:84-134).
int ref_generate_trace(uint64_t steps, int width, int vocab, double skew, uint64_t seed, int layers,
                       double* vocab_out, uint32_t* embed_ids, float* saliency, const char* save_path) {
    try {
        TraceSpec spec;
        spec.steps = steps, spec.width = width, spec.vocab = vocab, spec.zipf_skew = skew;
        spec.seed = seed, spec.layers = layers;
        Trace tr = generate_trace(spec);
        for (int v = 0; v < vocab; ++v)
            std::memcpy(vocab_out + (size_t)v * width, tr.vocabulary[v].data(), sizeof(double) * width);
        for (uint64_t t = 0; t < steps; ++t) {
            embed_ids[t] = tr.events[t].embed_id;
            for (int l = 0; l < layers; ++l) saliency[t * layers + l] = tr.events[t].layer_saliency[l];
        }
        if (save_path) save_trace(tr, save_path);
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

// The reference's own KVStore::snapshot (kvstore.cpp:206-221).
int ref_snapshot(ref_engine* e, uint64_t now, pikv_snapshot_record* out, int64_t cap, int64_t* n_out) {
    const auto recs = e->store.snapshot(now);
    const int64_t n = static_cast<int64_t>(recs.size());
    for (int64_t i = 0; i < n && i < cap; ++i) {
        out[i].device = recs[i].device;
        out[i].shard = recs[i].shard;
        out[i].token_id = recs[i].token_id;
        out[i].expert_id = recs[i].expert_id;
        out[i].reserved = 0;
        out[i].age = recs[i].age;
        out[i].freq = recs[i].freq;
    }
    *n_out = n;
    return 0;
}

void ref_router_state(ref_engine* e, double* load, uint64_t* usage, uint64_t* miss, double* bias,
                      uint64_t* step, uint64_t* total_usage) {
    const auto& s = e->rs;
    for (int i = 0; i < s.experts; ++i) {
        if (load) load[i] = s.load[i];
        if (usage) usage[i] = s.usage_counts[i];
        if (miss) miss[i] = s.miss_counts[i];
        if (bias) bias[i] = s.bandit_bias[i];
    }
    if (step) *step = s.step;
    if (total_usage) *total_usage = s.total_usage;
}

void ref_sched_state(ref_engine* e, double* theta, double* running_hit, uint64_t* step) {
    if (theta) *theta = e->ss.theta;
    if (running_hit) *running_hit = e->ss.running_hit;
    if (step) *step = e->ss.step;
}

// Reference free functions for the known-answer tests.
int ref_shard_assign(int64_t t, int e, int n_tok, int n_exp, int devices, int additive,
                     int* device, int* shard, int* raw) {
    try {
        auto s = shard_assign(t, e, n_tok, n_exp, devices, additive != 0);
        *device = s.device;
        *shard = s.shard_index;
        *raw = s.raw;
        return 0;
    } catch (const std::exception& ex) {
        return code_of(ex);
    }
}

int ref_select_evictions(const double* agg, const uint64_t* oldest, int n, int budget,
                         int use_theta, double theta, int* idx_out, int* reason_out) {
    std::vector<PageScore> pages(n);
    for (int i = 0; i < n; ++i) pages[i] = {agg[i], oldest[i]};
    auto out = select_evictions(pages, budget, use_theta != 0, theta);
    for (std::size_t i = 0; i < out.size(); ++i) {
        idx_out[i] = static_cast<int>(out[i].first);
        reason_out[i] = static_cast<int>(out[i].second);
    }
    return static_cast<int>(out.size());
}

int ref_attention(const double* q, const double* keys, const double* values, int n, int w,
                  double* y, double* weights) {
    std::vector<KVEntry> view(n);
    std::vector<const KVEntry*> ptrs(n);
    for (int i = 0; i < n; ++i) {
        view[i].key.assign(keys + static_cast<std::size_t>(i) * w, keys + static_cast<std::size_t>(i + 1) * w);
        view[i].value.assign(values + static_cast<std::size_t>(i) * w,
                             values + static_cast<std::size_t>(i + 1) * w);
        ptrs[i] = &view[i];
    }
    auto att = attention(std::span<const double>(q, w), ptrs);
    for (int j = 0; j < w; ++j) y[j] = att.output[j];
    for (int i = 0; i < n; ++i) weights[i] = att.weights[i];
    return 0;
}

// Timed CPU baseline: `threads` independent streams, one
// std::thread each, every stream its own reference engine.  Setup (untimed):
// `prefill` tokens are routed and inserted with the reference's route() and
// KVStore::insert() (no evict/retrieve/attention, to bound setup time).
// Timed: `steps` full ref_step calls per stream.  Inputs are N(0,1) from
// pikv::Rng(seed ^ stream) rounded to cfg->kv_dtype.  Returns the max over
// threads of the timed wall seconds.
static double round_dtype(double x, int dtype) {
    float f = static_cast<float>(x);
    if (dtype == PIKV_DTYPE_BF16) {
        std::uint32_t u;
        std::memcpy(&u, &f, 4);
        if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
        std::memcpy(&f, &u, 4);
    }
    return static_cast<double>(f);
}

double ref_time_streams(const pikv_config* cfg, int threads, long prefill, int steps,
                        std::uint64_t seed, double* seconds_per_thread, long* attended_out) {
    std::vector<std::thread> pool;
    std::vector<double> secs(threads, 0.0);
    std::vector<long> att(threads, 0);
    const int d = cfg->d;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t]() {
            int err = 0;
            std::unique_ptr<ref_engine> e(ref_create(cfg, nullptr, &err));
            if (!e) return;
            Rng rng(seed ^ static_cast<std::uint64_t>(t));
            auto draw = [&](std::vector<double>& x) {
                for (auto& v : x) v = round_dtype(rng.normal(), cfg->kv_dtype);
            };
            std::vector<double> q(d), k(d), v(d), y(d);
            for (long s = 0; s < prefill; ++s) {
                draw(q), draw(k), draw(v);
                auto decision = route(q, e->rs, e->router);
                for (int ex : decision.experts) {
                    KVEntry en;
                    en.token_id = static_cast<std::int64_t>(e->now);
                    en.expert_id = ex;
                    en.key = k;
                    en.value = v;
                    en.meta.insert_step = e->now;
                    en.meta.last_access_step = e->now;
                    e->store.insert(std::move(en));
                }
                e->now += 1;
            }
            po_step_out out{};
            out.y = y.data();
            auto t0 = std::chrono::steady_clock::now();
            for (int s = 0; s < steps; ++s) {
                draw(q), draw(k), draw(v);
                step_impl(e.get(), q.data(), k.data(), v.data(), nullptr, &out, true);
                att[t] += out.n_attended;
            }
            auto t1 = std::chrono::steady_clock::now();
            secs[t] = std::chrono::duration<double>(t1 - t0).count();
        });
    }
    for (auto& th : pool) th.join();
    double mx = 0.0;
    long total_att = 0;
    for (int t = 0; t < threads; ++t) {
        if (seconds_per_thread) seconds_per_thread[t] = secs[t];
        mx = std::max(mx, secs[t]);
        total_att += att[t];
    }
    if (attended_out) *attended_out = total_att;
    return mx;
}

}  // extern "C"

extern "C" void ref_normal_vector(std::uint64_t seed, std::int64_t n, double scale, double* out) {
    Rng rng(seed);  // rng.hpp:54-58
    auto v = rng.normal_vector(static_cast<std::size_t>(n), scale);
    for (std::int64_t i = 0; i < n; ++i) out[i] = v[i];
}
