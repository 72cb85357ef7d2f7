// SPDX-License-Identifier: Apache-2.0
// The reference's own known-answer tests, restated against the C++ facade
// (include/pikv_b200.hpp) that a reference caller would switch to.  Each check
// cites the reference test it mirrors.  Exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include <tuple>

#include "pikv_b200.hpp"

using namespace pikv::b200;

static int failures = 0;
#define CHECK(c)                                                       \
    do {                                                               \
        if (!(c)) {                                                    \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);   \
            ++failures;                                                \
        }                                                              \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                       \
    do {                                                               \
        bool ok_ = false;                                              \
        try { expr; } catch (const T&) { ok_ = true; } catch (...) {}  \
        CHECK(ok_);                                                    \
    } while (0)

static EngineConfig engine_config(RouterStrategy strat, int S = 256) {  // test_pipeline.cpp:16-48
    EngineConfig cfg;
    cfg.model.d = 16, cfg.model.head_width = 4, cfg.model.E = 8, cfg.model.k = 2;
    cfg.model.S = S, cfg.model.G = 2, cfg.model.L = 1024, cfg.model.K = 4;
    cfg.store.n_tok = 16, cfg.store.n_exp = 8;
    cfg.router.strategy = strat, cfg.router.k = 2;
    cfg.router.groups = strat == RouterStrategy::Hierarchical ? 4 : 1;
    cfg.scheduler.strategy = SchedStrategy::LRU, cfg.scheduler.budget_pages = 64, cfg.scheduler.page_size = 4;
    cfg.seed = 7;
    cfg.unbounded_budget = true;
    return cfg;
}

static std::vector<TokenInput> make_stream(int T, int d, unsigned seed) {
    std::mt19937_64 g(seed);
    std::normal_distribution<double> n(0.0, 1.0);
    std::vector<TokenInput> out(T);
    for (auto& t : out) {
        t.query.resize(d), t.key.resize(d), t.value.resize(d);
        for (int i = 0; i < d; ++i) t.query[i] = n(g), t.key[i] = n(g), t.value[i] = n(g);
    }
    return out;
}

int main() {
    // test_kvstore.cpp:42-57
    auto s = shard_assign(5, 3, 4, 4, 2);
    CHECK(s.raw == 2 && s.device == 0 && s.shard_index == 1);
    CHECK(shard_assign(0, 0, 8, 8, 4).raw == 0);
    CHECK(shard_assign(7, 2, 8, 4, 4).raw == 5);
    CHECK(shard_assign(5, 3, 4, 4, 2, true).raw == 4);
    CHECK_THROWS_AS(shard_assign(1, 1, 3, 4, 2), InvalidConfig);
    CHECK_THROWS_AS(shard_assign(1, 1, 4, 6, 2), InvalidConfig);
    CHECK_THROWS_AS(shard_assign(-1, 1, 4, 4, 2), InvalidArgument);

    // test_scheduler.cpp:178-207
    CHECK(select_evictions({{1, 1}, {2, 2}, {3, 3}}, 5, false, 0).empty());
    {
        auto out = select_evictions({{5, 1}, {1, 2}, {3, 3}, {2, 4}}, 2, false, 0);
        CHECK(out.size() == 2 && out[0].first == 1 && out[1].first == 3);
        CHECK(out[0].second == EvictReason::Budget);
    }
    {
        auto out = select_evictions({{5, 1}, {1, 2}, {3, 3}}, 10, true, 4.0);
        CHECK(out.size() == 2 && out[0].first == 1 && out[1].first == 2);
        CHECK(out[1].second == EvictReason::Threshold);
    }
    {
        auto out = select_evictions({{1, 9}, {1, 2}, {1, 5}}, 1, false, 0);
        CHECK(out.size() == 2 && out[0].first == 1 && out[1].first == 2);
    }

    // test_pipeline.cpp:80-119
    {
        auto out = attention({1, 0}, {}, {});
        CHECK(out.output == (std::vector<double>{0, 0}) && out.retrieved == 0 && out.weights.empty());
        auto one = attention({0.2, 0.9}, {{1.0, 0.0}}, {{3.0, 4.0}});
        CHECK(one.weights.size() == 1 && one.weights[0] == 1.0);
        CHECK(std::fabs(one.output[0] - 3.0) < 1e-6 && std::fabs(one.output[1] - 4.0) < 1e-6);
        auto two = attention({2.0, 1.0}, {{0.3, -0.7}, {0.3, -0.7}}, {{1, 0}, {0, 1}});
        CHECK(std::fabs(two.weights[0] - 0.5) < 1e-6 && std::fabs(two.weights[1] - 0.5) < 1e-6);
        auto orth = attention({0, 0, 5}, {{1, 0, 0}, {0, 1, 0}}, {{2, 0, 0}, {0, 4, 0}});
        CHECK(std::fabs(orth.output[0] - 1.0) < 1e-6 && std::fabs(orth.output[1] - 2.0) < 1e-6);
        CHECK_THROWS_AS(attention({1, 0}, {{1, 0, 0}}, {{1, 0, 0}}), InvalidArgument);
    }

    // test_pipeline.cpp:121-130: first token sees an empty prefix
    {
        Engine engine(engine_config(RouterStrategy::TopK));
        auto r = engine.step(make_stream(1, 16, 3))[0];
        CHECK(r.attn.retrieved == 0 && r.hits == 0 && r.lookups == 2);
        for (double y : r.attn.output) CHECK(y == 0.0);
        CHECK(engine.router_state().miss_counts[r.experts[0]] == 1);
    }
    // test_pipeline.cpp:138-152: failed step leaves no partial state
    {
        Engine engine(engine_config(RouterStrategy::TopK));
        auto stream = make_stream(2, 16, 5);
        engine.step({stream[0]});
        auto live = engine.store_stats().live;
        TokenInput bad;
        bad.query.assign(7, 0.0), bad.key.assign(7, 0.0), bad.value.assign(7, 0.0);
        CHECK_THROWS_AS(engine.step({bad}), InvalidArgument);
        CHECK(engine.store_stats().live == live);
        auto r = engine.step({stream[1]})[0];
        CHECK(r.step == 1);
    }
    // test_pipeline.cpp:154-168: deterministic replay; every router
    for (int st = 0; st <= 6; ++st) {
        auto cfg = engine_config(static_cast<RouterStrategy>(st));
        cfg.unbounded_budget = false, cfg.scheduler.budget_pages = 2;
        Engine a(cfg), b(cfg);
        for (const auto& tok : make_stream(40, 16, 11)) {
            auto ra = a.step({tok})[0];
            auto rb = b.step({tok})[0];
            CHECK(ra.attn.output == rb.attn.output);
            CHECK(ra.experts == rb.experts);
            CHECK(ra.fetch_elements == rb.fetch_elements);
            CHECK(ra.evictions.size() == rb.evictions.size());
            if (ra.attn.retrieved > 0) {  // test_pipeline.cpp:194-207 normalization
                double total = 0.0;
                for (double w : ra.attn.weights) total += w;
                CHECK(std::fabs(total - 1.0) < 1e-5);
            }
        }
    }
    // the reference's TokenInput{embedding}: the QueryEncoder runs on the GPU
    // (pipeline.cpp:222); width check before any state change (:214-216)
    {
        auto cfg = engine_config(RouterStrategy::Adaptive);
        Engine a(cfg), b(cfg);
        std::mt19937_64 g(17);
        std::normal_distribution<double> n(0.0, 1.0);
        for (int t = 0; t < 30; ++t) {
            TokenInput tok;
            tok.embedding.resize(16);
            for (auto& x : tok.embedding) x = n(g);
            auto ra = a.step({tok})[0];
            auto rb = b.step({tok})[0];
            CHECK(ra.experts == rb.experts && ra.attn.output == rb.attn.output);
            CHECK(ra.step == static_cast<std::uint64_t>(t));
        }
        TokenInput bad;
        bad.embedding.assign(15, 0.0);
        const auto live = a.store_stats().live;
        CHECK_THROWS_AS(a.step({bad}), InvalidArgument);
        CHECK(a.store_stats().live == live);
        // KVStore::snapshot (kvstore.cpp:206-221): one record per live entry, sorted
        const auto snap = a.snapshot();
        CHECK(snap.size() == live);
        for (std::size_t i = 1; i < snap.size(); ++i)
            CHECK(std::tie(snap[i - 1].device, snap[i - 1].shard, snap[i - 1].token_id, snap[i - 1].expert_id) <
                  std::tie(snap[i].device, snap[i].shard, snap[i].token_id, snap[i].expert_id));
        CHECK(!snap.empty() && wire::store_dump_line(snap[0]).find("\"age\":") == 1);
    }
    // micro-batch pipeline (pikv_group_*): a group of 2 x 2 streams submitted
    // without waiting between micro-batches equals two engines stepped one
    // call at a time (experts exactly; y to fp32 rounding: the attention grids
    // differ, so the split-K partials merge in another order)
    {
        auto cfg = engine_config(RouterStrategy::TopK);
        cfg.batch = 4;
        EngineGroup grp(cfg, 2);
        CHECK(grp.size() == 2 && grp.streams_per_micro() == 2);
        auto one = cfg;
        one.batch = 2;
        Engine e0(one), e1(one);
        Engine* ref[2] = {&e0, &e1};
        std::mt19937_64 g(23);
        std::normal_distribution<double> n(0.0, 1.0);
        const int d = cfg.model.d, T = 20;
        std::vector<float> in(static_cast<std::size_t>(T) * 4 * 3 * d), y(static_cast<std::size_t>(T) * 4 * d);
        for (auto& x : in) x = static_cast<float>(n(g));
        auto at = [&](int t, int s, int which) { return &in[((static_cast<std::size_t>(t) * 4 + s) * 3 + which) * d]; };
        // packed per micro-batch: [q of its 2 streams][k][v]
        std::vector<float> packed(static_cast<std::size_t>(T) * 2 * 3 * 2 * d);
        for (int t = 0; t < T; ++t)
            for (int m = 0; m < 2; ++m)
                for (int w = 0; w < 3; ++w)
                    for (int s = 0; s < 2; ++s)
                        std::memcpy(&packed[((((static_cast<std::size_t>(t) * 2 + m) * 3 + w) * 2 + s) * d)],
                                    at(t, 2 * m + s, w), sizeof(float) * d);
        for (int t = 0; t < T; ++t)
            for (int m = 0; m < 2; ++m) {
                if (t) grp.wait(m);
                const float* b = &packed[((static_cast<std::size_t>(t) * 2 + m) * 3) * 2 * d];
                grp.submit(m, b, b + 2 * d, b + 4 * d, &y[(static_cast<std::size_t>(t) * 4 + 2 * m) * d]);
            }
        grp.sync();
        double err = 0.0, nrm = 0.0;
        for (int t = 0; t < T; ++t)
            for (int m = 0; m < 2; ++m) {
                std::vector<TokenInput> toks(2);
                for (int s = 0; s < 2; ++s) {
                    toks[s].query.assign(at(t, 2 * m + s, 0), at(t, 2 * m + s, 0) + d);
                    toks[s].key.assign(at(t, 2 * m + s, 1), at(t, 2 * m + s, 1) + d);
                    toks[s].value.assign(at(t, 2 * m + s, 2), at(t, 2 * m + s, 2) + d);
                }
                auto r = ref[m]->step(toks);
                for (int s = 0; s < 2; ++s)
                    for (int i = 0; i < d; ++i) {
                        const double a = y[(static_cast<std::size_t>(t) * 4 + 2 * m + s) * d + i];
                        const double b = r[s].attn.output[i];
                        err += (a - b) * (a - b), nrm += b * b;
                    }
            }
        CHECK(std::sqrt(err / (nrm > 0 ? nrm : 1.0)) <= 2e-5);
        for (int m = 0; m < 2; ++m) {  // last step's routing, both streams of the micro-batch
            std::vector<std::int32_t> ea(4), eb(4);
            CHECK(pikv_read_step_host(grp.engine(m), ea.data(), nullptr, nullptr, nullptr) == 0);
            CHECK(pikv_read_step_host(ref[m]->handle(), eb.data(), nullptr, nullptr, nullptr) == 0);
            CHECK(ea == eb);
        }
    }
    // QUEST needs a fitted scorer (test_scheduler.cpp:142-153)
    {
        auto cfg = engine_config(RouterStrategy::TopK);
        cfg.scheduler.strategy = SchedStrategy::QUEST;
        CHECK_THROWS_AS(Engine{cfg}, NotFitted);
    }
    // ---- component classes (kvstore / router / scheduler / compressor) ----
    {  // test_kvstore.cpp:72-88: ring fill then FIFO overwrite (one shard)
        ModelConfig m;
        m.d = 2, m.head_width = 1, m.E = 8, m.k = 1, m.S = 4, m.G = 1;
        KVStore st(m, StoreConfig{1, 1, false, 0});
        auto mk = [](std::int64_t t) { KVEntry e; e.token_id = t; e.key.assign(2, 1.0); e.value.assign(2, 1.0); return e; };
        CHECK(!st.insert(mk(0)).has_value());
        CHECK(st.live_count(0, 0) == 1);
        for (int t = 1; t < 4; ++t) st.insert(mk(t));
        auto fifth = st.insert(mk(4));
        CHECK(fifth.has_value() && fifth->token_id == 0);
        for (int t = 5; t < 7; ++t) st.insert(mk(t));
        auto eighth = st.insert(mk(7));
        CHECK(eighth.has_value() && eighth->token_id == 3);
        CHECK(st.live_count(0, 0) == 4);
        KVEntry bad = mk(9);
        bad.key.assign(3, 1.0);
        CHECK_THROWS_AS(st.insert(bad), InvalidEntry);  // test_kvstore.cpp:109-112
    }
    {  // test_kvstore.cpp:114-160, 220-230
        ModelConfig m;
        m.d = 4, m.head_width = 1, m.E = 8, m.k = 1, m.S = 16, m.G = 1;
        KVStore st(m, StoreConfig{8, 8, false, 0});
        auto r0 = st.retrieve({2}, 100, 100);
        CHECK(r0.entries.empty() && r0.missed_experts == std::vector<int>{2} && st.stats().misses == 1);
        for (std::int64_t t = 0; t < 12; ++t) {
            KVEntry e;
            e.token_id = t, e.expert_id = static_cast<int>(t % 3);
            e.key.assign(4, 1.0), e.value.assign(4, 1.0);
            st.insert(e);
        }
        auto r = st.retrieve({0, 2}, 12, 12);
        std::vector<std::int64_t> got, want;
        for (const auto& e : r.entries) got.push_back(e.token_id);
        for (std::int64_t t = 0; t < 12; ++t)
            if (t % 3 != 1) want.push_back(t);
        CHECK(got == want);
        CHECK(r.entries[0].meta.freq == 1 && r.entries[0].meta.last_access_step == 12);
        const auto id = r.entries[0].id;
        CHECK(st.erase(id));
        CHECK(!st.erase(id));
        CHECK(st.live_entries() == 11);
        auto snap = st.snapshot(12);
        CHECK(snap.size() == 11);
    }
    {  // test_kvstore.cpp:178-205: memory accounting
        ModelConfig m;
        m.d = 16, m.head_width = 1, m.E = 8, m.k = 1, m.S = 8, m.G = 1, m.elem_bytes = 2;
        KVStore st(m, StoreConfig{2, 1, false, 0});
        auto mk = [](std::int64_t t) { KVEntry e; e.token_id = t; e.key.assign(16, 1.0); e.value.assign(16, 1.0); return e; };
        for (std::int64_t t : {0, 2, 4}) st.insert(mk(t));
        for (std::int64_t t : {1, 3, 5, 7, 9}) st.insert(mk(t));
        CHECK(st.live_count(0, 0) == 3 && st.live_count(0, 1) == 5 && st.memory_bytes() == 512);
    }
    {  // test_router.cpp:34-117, 281-291
        RouterState base = RouterState::init(4, 8, 1);
        RouterConfig rb;
        rb.strategy = RouterStrategy::Base, rb.k = 1;
        for (int t = 0; t < 4; ++t) {
            auto d = route(std::vector<double>(8, 0.0), base, rb);
            CHECK(d.experts.size() == 1 && d.experts[0] == t && std::fabs(d.gates[0] - 1.0) < 1e-12);
        }
        RouterState st = RouterState::init(4, 4, 1);
        RouterConfig top;
        top.strategy = RouterStrategy::TopK, top.k = 2;
        auto d = route_logits({2, 1, 0, -1}, st, top);
        CHECK((d.experts == std::vector<int>{0, 1}));
        CHECK(std::fabs(d.gates[0] - 0.7310585786300049) <= 1e-12 && std::fabs(d.gates[1] - 0.2689414213699951) <= 1e-12);
        RouterState lb = RouterState::init(4, 4, 1);
        RouterConfig lbc;
        lbc.strategy = RouterStrategy::LoadBalanced, lbc.k = 1, lbc.alpha = 0.5;
        lb.bind(lbc);
        lb.set_load({10, 0, 0, 0});
        CHECK(route_logits({1, 1, 1, 1}, lb, lbc).experts[0] == 1);
        record_miss(st, 2, top);
        record_miss(st, 2, top);
        CHECK(st.view().miss_counts[2] == 2);
        CHECK_THROWS_AS(record_miss(st, 4, top), InvalidArgument);
        RouterConfig ad;
        ad.strategy = RouterStrategy::Adaptive, ad.k = 2, ad.bandit_step = 0.1;
        RouterState sa = RouterState::init(4, 4, 1);
        RoutingDecision dec;
        dec.experts = {0, 2};
        adapt(sa, dec, 1.0, ad);
        auto v = sa.view();
        CHECK(std::fabs(v.bandit_bias[0] - 0.1) < 1e-12 && std::fabs(v.bandit_bias[2] - 0.1) < 1e-12 && v.bandit_bias[1] == 0.0);
        CHECK_THROWS_AS(adapt(sa, dec, 1.5, ad), InvalidArgument);
        CHECK_THROWS_AS(route_logits({0.0, std::nan(""), 1.0, 2.0}, st, top), NumericalError);
    }
    {  // test_scheduler.cpp:75-104, 236-259, 277-292
        KVEntry e;
        e.meta.attn_mass = 0.37;
        SchedulerConfig h2o;
        h2o.strategy = SchedStrategy::H2O;
        CHECK(std::fabs(score_entry(e, h2o, 5) - 0.37) < 1e-15);
        KVEntry l;
        l.meta.last_access_step = 3, l.meta.freq = 3;
        SchedulerConfig lp;
        lp.strategy = SchedStrategy::LRUPlus, lp.lambda_freq = 0.5;
        CHECK(score_entry(l, lp, 5) == -0.5);
        ModelConfig m;
        m.d = 2, m.head_width = 1, m.E = 4, m.k = 1, m.S = 16, m.G = 1;
        KVStore st(m, StoreConfig{1, 1, false, 0}, /*page_size=*/1);
        const double attn[4] = {5.0, 1.0, 3.0, 2.0};
        for (int t = 0; t < 4; ++t) {
            KVEntry x;
            x.token_id = t, x.key.assign(2, 1.0), x.value.assign(2, 1.0), x.meta.attn_mass = attn[t];
            st.insert(x);
        }
        SchedulerConfig c;
        c.strategy = SchedStrategy::H2O, c.page_size = 1, c.budget_pages = 2;
        auto rep = st.evict(c, 4);
        CHECK(rep.pages_before == 4 && rep.pages_after == 2 && rep.evicted.size() == 2);
        CHECK(rep.evicted.size() == 2 && rep.evicted[0].token_id == 1 && rep.evicted[1].token_id == 3);
        CHECK(st.live_entries() == 2 && st.evict(c, 5).evicted.empty());
        SchedulerConfig ak;
        ak.strategy = SchedStrategy::AdaKV, ak.adakv_step = 0.1, ak.target_hit = 0.9, ak.theta0 = 0.5, ak.hit_decay = 0.0;
        ak.page_size = 1;
        st.set_scheduler_state(0.5, 0.0);
        st.observe_hits(ak, 7, 10);
        st.adakv_update(ak);
        CHECK(std::fabs(st.scheduler_state().theta - 0.52) < 1e-12);
    }
    {  // test_compressor.cpp:130-161; test_pipeline.cpp:80-119 on stored entries
        Codec fv = Codec::fastv(2, 1);
        CHECK(fv.encode_vector({3, 4}) == std::vector<double>{3});
        CHECK((fv.decode_vector(fv.encode_vector({3, 4})) == std::vector<double>{3, 0}));
        CHECK(std::fabs(fv.reconstruction_error({3, 4}) - 0.8) < 1e-6);
        Codec pr = Codec::fit_prune({{1, 7}, {-3, 7}, {2, 7}, {-1, 7}}, 0.5);
        CHECK(pr.zero_set() == std::vector<int>{1});
        CHECK((pr.decode_vector(pr.encode_vector({3, 4})) == std::vector<double>{3, 0}));
        ModelConfig m;
        m.d = 2, m.head_width = 1, m.E = 4, m.k = 1, m.S = 8, m.G = 1;
        KVStore st(m, StoreConfig{1, 1, false, 0});
        CHECK(st.attention({1.0, 0.0}, {}).output == (std::vector<double>{0.0, 0.0}));
        for (int t = 0; t < 2; ++t) {
            KVEntry x;
            x.token_id = t, x.key = {1.0, 0.0}, x.value = {3.0 + 2 * t, 4.0 + 2 * t};
            st.insert(x);
        }
        auto a = st.attention({1.0, 0.0}, {0, 1});  // identical keys: 0.5 / 0.5
        CHECK(std::fabs(a.weights[0] - 0.5) < 1e-6 && std::fabs(a.output[0] - 4.0) < 1e-5);
    }
    {  // Engine::flush / StepResult.inserted (pipeline.hpp:79, 108)
        EngineConfig cfg = engine_config(RouterStrategy::TopK, 64);
        Engine eng(cfg);
        auto toks = make_stream(2, cfg.model.d, 5);
        auto r = eng.step({toks[0]});
        CHECK(r[0].inserted.size() == 2 && r[0].inserted[0].first == 0 && r[0].inserted[0].second == r[0].experts[0]);
        CHECK(eng.flush().size() == 1 && eng.flush()[0].inserted.empty());
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
    return failures;
}
