// SPDX-License-Identifier: Apache-2.0
// The reference's own known-answer tests, restated against the C++ facade
// (include/pikv_b200.hpp) that a reference caller would switch to.  Each check
// cites the reference test it mirrors.  Exit code = number of failures.
#include <cmath>
#include <cstdio>
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
    // QUEST needs a fitted scorer (test_scheduler.cpp:142-153)
    {
        auto cfg = engine_config(RouterStrategy::TopK);
        cfg.scheduler.strategy = SchedStrategy::QUEST;
        CHECK_THROWS_AS(Engine{cfg}, NotFitted);
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
    return failures;
}
