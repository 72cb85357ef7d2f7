/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — CPU oracle (restatement) of the PiKV decode path.
 * See pikv_oracle.h for scope and how it is pinned.  Only tests/, smoke()
 * and bench.py's cpu_baseline leg load this; the product never does.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off keeps every a*b+c a separate multiply and add, as in the
 * reference built by g++ for baseline x86-64 (no FMA).
 */
#define _GNU_SOURCE
#include "pikv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PO_ROUTER_SALT 0x2545f4914f6cdd1dULL /* pipeline.cpp:16 */

/* ======================================================================
 * Rng: mt19937_64 (the standard engine the reference wraps) plus the
 * reference's own transforms, rng.hpp:15-70.
 * ==================================================================== */
void po_rng_init(po_rng* r, uint64_t seed) {
    r->seed = seed;
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
    r->has_spare = 0;
    r->spare = 0.0;
}

uint64_t po_rng_next(po_rng* r) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (r->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag01[x & 1ULL];
        }
        for (; i < 311; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[x & 1ULL];
        }
        x = (r->mt[311] & UM) | (r->mt[0] & LM);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag01[x & 1ULL];
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* rng.hpp:24-26 */
double po_rng_uniform(po_rng* r) { return (double)(po_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:38-52 */
double po_rng_normal(po_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = po_rng_uniform(r);
    double u2 = po_rng_uniform(r);
    while (u1 <= 0.0) u1 = po_rng_uniform(r);
    double radius = sqrt(-2.0 * log(u1));
    double angle = 2.0 * M_PI * u2;
    r->spare = radius * sin(angle);
    r->has_spare = 1;
    return radius * cos(angle);
}

/* rng.hpp:54-58 */
void po_normal_vector(uint64_t seed, int64_t n, double scale, double* out) {
    po_rng r;
    po_rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = scale * po_rng_normal(&r);
}

/* ======================================================================
 * mathops.cpp
 * ==================================================================== */
/* mathops.cpp:11-30 */
int po_softmax(const double* logits, int n, double* out) {
    if (n <= 0) return PIKV_ERR_INVALID_ARGUMENT;
    double mx = logits[0];
    for (int i = 0; i < n; ++i) {
        if (isnan(logits[i])) return PIKV_ERR_INVALID_ARGUMENT;
        mx = (mx < logits[i]) ? logits[i] : mx; /* std::max(a,b) */
    }
    double total = 0.0;
    for (int i = 0; i < n; ++i) {
        out[i] = exp(logits[i] - mx);
        total += out[i];
    }
    for (int i = 0; i < n; ++i) out[i] /= total;
    return PIKV_OK;
}

/* mathops.cpp:48-55 */
double po_dot(const double* a, const double* b, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* ======================================================================
 * shard_assign, kvstore.cpp:14-30
 * ==================================================================== */
static int is_pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }

int po_shard_assign(int64_t t, int e, int n_tok, int n_exp, int devices, int additive,
                    int* device, int* shard, int* raw) {
    if (!is_pow2(n_tok) || !is_pow2(n_exp)) return PIKV_ERR_INVALID_CONFIG;
    if (t < 0 || e < 0) return PIKV_ERR_INVALID_ARGUMENT;
    int lhs = (int)(t % n_tok);
    int rhs = e % n_exp;
    int rw = additive ? lhs + rhs : (lhs ^ rhs);
    if (raw) *raw = rw;
    if (device) *device = rw % devices;
    if (shard) *shard = rw / devices;
    return PIKV_OK;
}

/* ======================================================================
 * attention, pipeline.cpp:59-85 (one head)
 * ==================================================================== */
int po_attention(const double* q, const double* keys, const double* values, int n, int w,
                 double* y, double* weights) {
    for (int j = 0; j < w; ++j) y[j] = 0.0;
    if (n == 0) return PIKV_OK;
    double scale = 1.0 / sqrt((double)w);
    double* scores = (double*)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) scores[i] = po_dot(q, keys + (size_t)i * w, w) * scale;
    int rc = po_softmax(scores, n, weights);
    free(scores);
    if (rc) return rc;
    for (int i = 0; i < n; ++i) {
        const double* v = values + (size_t)i * w;
        for (int j = 0; j < w; ++j) y[j] += weights[i] * v[j];
    }
    return PIKV_OK;
}

/* ======================================================================
 * select_evictions, scheduler.cpp:231-260
 * ==================================================================== */
static const double* g_sel_agg;
static const uint64_t* g_sel_old;
static int sel_cmp(const void* pa, const void* pb) {
    int a = *(const int*)pa, b = *(const int*)pb;
    if (g_sel_agg[a] != g_sel_agg[b]) return g_sel_agg[a] < g_sel_agg[b] ? -1 : 1;
    if (g_sel_old[a] != g_sel_old[b]) return g_sel_old[a] < g_sel_old[b] ? -1 : 1;
    return 0;
}

int po_select_evictions(const double* agg, const uint64_t* oldest, int n, int budget,
                        int use_theta, double theta, int* idx_out, int* reason_out) {
    int* order = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) order[i] = i;
    g_sel_agg = agg;
    g_sel_old = oldest;
    qsort(order, (size_t)n, sizeof(int), sel_cmp);
    int out = 0, remaining = n, cursor = 0;
    if (use_theta) {
        while (cursor < n && agg[order[cursor]] < theta) {
            idx_out[out] = order[cursor];
            reason_out[out] = PIKV_EVICT_THRESHOLD;
            ++out, ++cursor, --remaining;
        }
    }
    while (remaining > budget) {
        idx_out[out] = order[cursor];
        reason_out[out] = PIKV_EVICT_BUDGET;
        ++out, ++cursor, --remaining;
    }
    free(order);
    return out;
}

/* ======================================================================
 * quantizer (this engine's; no reference counterpart)
 *   amax = max|x|; scale = amax / qmax; inv = qmax / amax (fp32 divides);
 *   code = clamp(rint(x * inv), -qmax, qmax); qmax = 127 (int8) / 7 (int4).
 *   int4 packs code[2j] in the low nibble of byte j, code[2j+1] high.
 * ==================================================================== */
void po_quantize_row(const float* x, int width, int bits, uint8_t* codes, float* scale) {
    const float qmax = bits == 8 ? 127.0f : 7.0f;
    float amax = 0.0f;
    for (int i = 0; i < width; ++i) {
        float a = fabsf(x[i]);
        amax = a > amax ? a : amax;
    }
    float inv = 0.0f;
    if (amax > 0.0f) {
        *scale = amax / qmax;
        inv = qmax / amax;
    } else {
        *scale = 0.0f;
    }
    if (bits == 4) memset(codes, 0, (size_t)width / 2);
    for (int i = 0; i < width; ++i) {
        volatile float prod = x[i] * inv; /* one fp32 rounding, no contraction */
        float c = rintf(prod);
        if (c > qmax) c = qmax;
        if (c < -qmax) c = -qmax;
        int ci = (int)c;
        if (bits == 8) {
            codes[i] = (uint8_t)(int8_t)ci;
        } else {
            uint8_t nib = (uint8_t)(ci & 0xF);
            codes[i >> 1] |= (uint8_t)((i & 1) ? (nib << 4) : nib);
        }
    }
}

void po_dequantize_row(const uint8_t* codes, float scale, int width, int bits, float* x) {
    for (int i = 0; i < width; ++i) {
        int ci;
        if (bits == 8) {
            ci = (int)(int8_t)codes[i];
        } else {
            int nib = (codes[i >> 1] >> ((i & 1) * 4)) & 0xF;
            ci = nib >= 8 ? nib - 16 : nib;
        }
        x[i] = (float)ci * scale;
    }
}

/* ======================================================================
 * Router, router.cpp
 * ==================================================================== */
struct po_router {
    int experts, width;
    double* w;     /* E x d row-major */
    double* load;  /* mu_e */
    uint64_t* usage;
    uint64_t total_usage;
    uint64_t* miss;
    double* bias;
    uint64_t step;
};

/* RouterState::init, router.cpp:54-67 */
po_router* po_router_create(int experts, int width, uint64_t seed) {
    po_router* r = (po_router*)calloc(1, sizeof(po_router));
    r->experts = experts;
    r->width = width;
    r->w = (double*)malloc(sizeof(double) * (size_t)experts * (size_t)width);
    po_normal_vector(seed, (int64_t)experts * width, 1.0 / sqrt((double)width), r->w);
    r->load = (double*)calloc((size_t)experts, sizeof(double));
    r->usage = (uint64_t*)calloc((size_t)experts, sizeof(uint64_t));
    r->miss = (uint64_t*)calloc((size_t)experts, sizeof(uint64_t));
    r->bias = (double*)calloc((size_t)experts, sizeof(double));
    return r;
}

void po_router_destroy(po_router* r) {
    if (!r) return;
    free(r->w), free(r->load), free(r->usage), free(r->miss), free(r->bias);
    free(r);
}

void po_router_set_matrix(po_router* r, const double* w) {
    memcpy(r->w, w, sizeof(double) * (size_t)r->experts * (size_t)r->width);
}

void po_router_state(const po_router* r, double* load, uint64_t* usage, uint64_t* miss,
                     double* bias, uint64_t* step, uint64_t* total_usage) {
    size_t E = (size_t)r->experts;
    if (load) memcpy(load, r->load, E * sizeof(double));
    if (usage) memcpy(usage, r->usage, E * sizeof(uint64_t));
    if (miss) memcpy(miss, r->miss, E * sizeof(uint64_t));
    if (bias) memcpy(bias, r->bias, E * sizeof(double));
    if (step) *step = r->step;
    if (total_usage) *total_usage = r->total_usage;
}

void po_router_set_state(po_router* r, const double* load, const uint64_t* usage,
                         const uint64_t* miss, const double* bias, uint64_t step,
                         uint64_t total_usage) {
    size_t E = (size_t)r->experts;
    if (load) memcpy(r->load, load, E * sizeof(double));
    if (usage) memcpy(r->usage, usage, E * sizeof(uint64_t));
    if (miss) memcpy(r->miss, miss, E * sizeof(uint64_t));
    if (bias) memcpy(r->bias, bias, E * sizeof(double));
    r->step = step;
    r->total_usage = total_usage;
}

/* RouterConfig::validate, router.cpp:40-53 */
static int router_cfg_validate(const pikv_config* c, int experts) {
    if (c->k < 1 || c->k > experts) return PIKV_ERR_INVALID_CONFIG;
    if (c->alpha < 0 || c->lambda_miss < 0 || c->beta_ent < 0 || c->bandit_step < 0)
        return PIKV_ERR_INVALID_CONFIG;
    if (c->groups < 1 || c->groups > experts) return PIKV_ERR_INVALID_CONFIG;
    if (c->load_decay < 0 || c->load_decay >= 1.0) return PIKV_ERR_INVALID_CONFIG;
    return PIKV_OK;
}

/* top_k_of, router.cpp:82-90: order by (score desc, index asc), keep k. */
static void top_k_of(const double* scores, int* pool, int n, int k, int* out) {
    for (int i = 1; i < n; ++i) { /* insertion sort: strict total order */
        int v = pool[i], j = i - 1;
        while (j >= 0) {
            int a = v, b = pool[j];
            int before = scores[a] != scores[b] ? scores[a] > scores[b] : a < b;
            if (!before) break;
            pool[j + 1] = pool[j];
            --j;
        }
        pool[j + 1] = v;
    }
    for (int i = 0; i < k; ++i) out[i] = pool[i];
}

/* note_selection, router.cpp:92-105 */
static void note_selection(po_router* r, const int* sel, int k, const pikv_config* c) {
    for (int e = 0; e < r->experts; ++e) {
        int picked = 0;
        for (int j = 0; j < k; ++j) picked |= sel[j] == e;
        r->load[e] = c->load_decay * r->load[e] + (1.0 - c->load_decay) * (picked ? 1.0 : 0.0);
    }
    for (int j = 0; j < k; ++j) {
        r->usage[sel[j]] += 1;
        r->total_usage += 1;
    }
    r->step += 1;
}

/* base_round_robin, router.cpp:107-118 */
static void base_round_robin(po_router* r, const pikv_config* c, double* logits, int* experts,
                             double* gates) {
    int64_t t = (int64_t)r->step;
    for (int j = 0; j < c->k; ++j) experts[j] = (int)((t * c->stride + j) % r->experts);
    for (int j = 0; j < c->k; ++j) gates[j] = 1.0 / c->k;
    if (logits)
        for (int e = 0; e < r->experts; ++e) logits[e] = 0.0;
    note_selection(r, experts, c->k, c);
}

/* route_logits, router.cpp:122-214 */
int po_route_logits(po_router* r, const pikv_config* c, double* logits, int* experts,
                    double* gates) {
    int rc = router_cfg_validate(c, r->experts);
    if (rc) return rc;
    if (c->router_strategy == PIKV_ROUTER_BASE) {
        base_round_robin(r, c, logits, experts, gates);
        return PIKV_OK;
    }
    const int E = r->experts;
    for (int e = 0; e < E; ++e)
        if (isnan(logits[e])) return PIKV_ERR_NUMERICAL;
    switch (c->router_strategy) {
        case PIKV_ROUTER_LOAD_BALANCED: {
            double acc = 0.0;
            for (int e = 0; e < E; ++e) acc += r->load[e];
            double mean_load = acc / E;
            for (int e = 0; e < E; ++e) logits[e] -= c->alpha * (r->load[e] - mean_load);
            break;
        }
        case PIKV_ROUTER_CACHE_AWARE:
            for (int e = 0; e < E; ++e) logits[e] -= c->lambda_miss * log1p((double)r->miss[e]);
            break;
        case PIKV_ROUTER_ENTROPY_LB:
            for (int e = 0; e < E; ++e) {
                double p = r->total_usage == 0 ? 0.0
                                               : (double)r->usage[e] / (double)r->total_usage;
                double h = p > 0.0 ? -p * log(p) : 0.0;
                logits[e] -= c->beta_ent * h;
            }
            break;
        case PIKV_ROUTER_ADAPTIVE:
            for (int e = 0; e < E; ++e) logits[e] += r->bias[e];
            break;
        default:
            break;
    }
    int* pool = (int*)malloc(sizeof(int) * (size_t)E);
    int npool = 0;
    if (c->router_strategy == PIKV_ROUTER_HIERARCHICAL) {
        int cs = (E + c->groups - 1) / c->groups;
        double* cscore = (double*)malloc(sizeof(double) * (size_t)c->groups);
        int* corder = (int*)malloc(sizeof(int) * (size_t)c->groups);
        for (int g = 0; g < c->groups; ++g) cscore[g] = -INFINITY, corder[g] = g;
        for (int e = 0; e < E; ++e) {
            int g = e / cs;
            cscore[g] = (cscore[g] < logits[e]) ? logits[e] : cscore[g];
        }
        for (int i = 1; i < c->groups; ++i) {
            int v = corder[i], j = i - 1;
            while (j >= 0) {
                int a = v, b = corder[j];
                int before = cscore[a] != cscore[b] ? cscore[a] > cscore[b] : a < b;
                if (!before) break;
                corder[j + 1] = corder[j];
                --j;
            }
            corder[j + 1] = v;
        }
        for (int i = 0; i < c->groups; ++i) {
            int g = corder[i];
            int begin = g * cs, end = begin + cs < E ? begin + cs : E;
            for (int e = begin; e < end; ++e) pool[npool++] = e;
            if (npool >= c->k) break;
        }
        free(cscore), free(corder);
    } else {
        for (int e = 0; e < E; ++e) pool[npool++] = e;
    }
    top_k_of(logits, pool, npool, c->k, experts);
    free(pool);
    double sel[64];
    for (int j = 0; j < c->k; ++j) sel[j] = logits[experts[j]];
    po_softmax(sel, c->k, gates);
    note_selection(r, experts, c->k, c);
    return PIKV_OK;
}

/* route, router.cpp:216-234 */
int po_route(po_router* r, const pikv_config* c, const double* q, double* logits, int* experts,
             double* gates) {
    int rc = router_cfg_validate(c, r->experts);
    if (rc) return rc;
    if (c->router_strategy == PIKV_ROUTER_BASE) {
        base_round_robin(r, c, logits, experts, gates);
        return PIKV_OK;
    }
    for (int e = 0; e < r->experts; ++e) {
        const double* row = r->w + (size_t)e * (size_t)r->width;
        double s = 0.0;
        for (int i = 0; i < r->width; ++i) s += row[i] * q[i];
        logits[e] = s;
    }
    return po_route_logits(r, c, logits, experts, gates);
}

/* record_miss, router.cpp:236-241 */
int po_record_miss(po_router* r, int expert) {
    if (expert < 0 || expert >= r->experts) return PIKV_ERR_INVALID_ARGUMENT;
    r->miss[expert] += 1;
    return PIKV_OK;
}

/* adapt, router.cpp:243-255 */
int po_adapt(po_router* r, const pikv_config* c, const int* experts, int k, double reward) {
    if (reward < 0.0 || reward > 1.0) return PIKV_ERR_INVALID_ARGUMENT;
    double acc = 0.0;
    for (int e = 0; e < r->experts; ++e) acc += r->bias[e];
    double mean_bias = acc / r->experts;
    for (int j = 0; j < k; ++j) {
        int e = experts[j];
        double b = r->bias[e] + c->bandit_step * (reward - mean_bias);
        r->bias[e] = b < -c->bias_cap ? -c->bias_cap : (c->bias_cap < b ? c->bias_cap : b);
    }
    return PIKV_OK;
}

/* ======================================================================
 * Store, scheduler, engine
 * ==================================================================== */
typedef struct po_slot {
    uint64_t id; /* 0 = empty slot (ids start at 1, kvstore.hpp:157) */
    uint64_t shard_seq;
    int64_t token;
    int32_t expert;
    uint64_t insert_step, last_access, freq;
    double attn_mass;
    /* per_layer_scores non-empty: the TokenInput carried layer saliency
     * (pipeline.cpp:307 folds only into non-empty vectors; an empty vector
     * scores 0 under Duo, scheduler.cpp:222-226) */
    int32_t has_layers;
} po_slot;

struct po_engine {
    pikv_config c;
    int H, hd, dp, dph; /* heads, head dim, stored width d', stored per head */
    int spd, nrings;
    po_slot* slots;     /* [nrings][S] */
    /* K then V of each slot as attended (dequantized), [2][dp] floats per slot
     * in chunks of PO_CHUNK slots allocated on first write, so host memory
     * follows the slots ever written, not nrings * S (full-context parity
     * runs).  float is exact: every stored value is an f32/bf16-rounded input,
     * a dtype-rounded projection or an f32 dequantized code. */
    float** payload;
    size_t n_chunks;
    double* layers;     /* [nrings][S][n_layers] */
    int* head;
    int* live;
    uint64_t* seq;
    uint64_t next_id;
    uint64_t st_inserts, st_overwrites;
    po_router* router;
    /* SchedulerState, scheduler.hpp:49-56 */
    double theta, running_hit;
    uint64_t sched_step;
    uint64_t now;
    /* codec params */
    double* basis; /* [H][r][hd] */
    double* bias;  /* [d] */
    int32_t* kept; /* [H][r] */
    /* QueryEncoder (pipeline.cpp:29-57), generated on first embedding step */
    double* enc_w;  /* [3][d][d]: w_query, w_key, w_value row-major */
    /* scratch */
    double* stage_k;
    double* stage_v;
};

#define PO_CHUNK 64
/* K/V floats of slot gi (allocating its chunk when `write`). */
static float* slot_payload(po_engine* e, size_t gi, int write) {
    float** ch = &e->payload[gi / PO_CHUNK];
    if (!*ch) {
        if (!write) abort(); /* a live slot was never written */
        *ch = (float*)calloc((size_t)PO_CHUNK * 2 * (size_t)e->dp, sizeof(float));
        if (!*ch) abort();
    }
    return *ch + (gi % PO_CHUNK) * 2 * (size_t)e->dp;
}

static int model_validate(const pikv_config* c) { /* config.hpp:42-54 */
    if (c->d < 1) return PIKV_ERR_INVALID_CONFIG;
    if (c->head_width < 1 || c->head_width > c->d) return PIKV_ERR_INVALID_CONFIG;
    if (c->E < 1) return PIKV_ERR_INVALID_CONFIG;
    if (c->k < 1 || c->k > c->E) return PIKV_ERR_INVALID_CONFIG;
    if (c->L < 1 || c->G < 1 || c->S < 1 || c->K < 1) return PIKV_ERR_INVALID_CONFIG;
    if (!(c->rho >= 1.0)) return PIKV_ERR_INVALID_CONFIG;
    if (c->elem_bytes < 1) return PIKV_ERR_INVALID_CONFIG;
    return PIKV_OK;
}

static int sched_validate(const pikv_config* c) { /* scheduler.cpp:49-71 */
    if (c->budget_pages < 1 || c->page_size < 1) return PIKV_ERR_INVALID_CONFIG;
    if (c->lambda_freq < 0 || c->adakv_step < 0 || c->gamma_sim < 0)
        return PIKV_ERR_INVALID_CONFIG;
    if (c->target_hit < 0.0 || c->target_hit > 1.0) return PIKV_ERR_INVALID_CONFIG;
    if (c->hit_decay < 0.0 || c->hit_decay >= 1.0) return PIKV_ERR_INVALID_CONFIG;
    if (c->n_flex_plan < 1 || c->flex_bucket < 1) return PIKV_ERR_INVALID_CONFIG;
    if (c->sink < 0 || c->tau < 0) return PIKV_ERR_INVALID_CONFIG;
    return PIKV_OK;
}

static double round_to_dtype(double x, int dtype) {
    float f = (float)x;
    if (dtype == PIKV_DTYPE_BF16) {
        uint32_t u;
        memcpy(&u, &f, 4);
        if ((u & 0x7f800000u) != 0x7f800000u) {
            u += 0x7fffu + ((u >> 16) & 1u);
        }
        u &= 0xffff0000u;
        memcpy(&f, &u, 4);
    }
    return (double)f;
}

po_engine* po_engine_create(const pikv_config* c, const double* w_r, const double* basis,
                            const double* bias, const int32_t* kept, int* err) {
    int rc = model_validate(c);
    if (!rc && (!is_pow2(c->n_tok) || !is_pow2(c->n_exp) || c->shards_per_device < 0))
        rc = PIKV_ERR_INVALID_CONFIG;
    if (!rc) rc = router_cfg_validate(c, c->E);
    if (!rc) rc = sched_validate(c);
    if (!rc && (c->n_heads < 1 || c->d % c->n_heads)) rc = PIKV_ERR_INVALID_CONFIG;
    if (!rc && c->sched_strategy == PIKV_SCHED_QUEST) rc = PIKV_ERR_NOT_FITTED;
    if (rc) {
        if (err) *err = rc;
        return NULL;
    }
    po_engine* e = (po_engine*)calloc(1, sizeof(po_engine));
    e->c = *c;
    e->H = c->n_heads;
    e->hd = c->d / c->n_heads;
    int lowrank = c->codec == PIKV_CODEC_LOWRANK || c->codec == PIKV_CODEC_LORAPLUS ||
                  c->codec == PIKV_CODEC_FASTV || c->codec == PIKV_CODEC_PRUNE;
    e->dph = lowrank ? c->rank : e->hd;
    e->dp = e->dph * e->H;
    /* KVStore ctor, kvstore.cpp:82-100 */
    int spd = c->shards_per_device > 0 ? c->shards_per_device
                                       : ((c->n_tok > c->n_exp ? c->n_tok : c->n_exp) / c->G);
    if (spd < 1) spd = 1;
    int raw_span = c->additive ? c->n_tok + c->n_exp - 1 : (c->n_tok > c->n_exp ? c->n_tok : c->n_exp);
    int needed = (raw_span + c->G - 1) / c->G;
    if (spd < needed) spd = needed;
    e->spd = spd;
    e->nrings = c->G * spd;
    size_t ns = (size_t)e->nrings * (size_t)c->S;
    e->slots = (po_slot*)calloc(ns, sizeof(po_slot));
    e->n_chunks = (ns + PO_CHUNK - 1) / PO_CHUNK;
    e->payload = (float**)calloc(e->n_chunks, sizeof(float*));
    e->layers = (double*)calloc(ns * (size_t)(c->n_layers > 0 ? c->n_layers : 1), sizeof(double));
    e->head = (int*)calloc((size_t)e->nrings, sizeof(int));
    e->live = (int*)calloc((size_t)e->nrings, sizeof(int));
    e->seq = (uint64_t*)calloc((size_t)e->nrings, sizeof(uint64_t));
    e->next_id = 1;
    e->router = po_router_create(c->E, c->d, c->seed ^ PO_ROUTER_SALT);
    if (w_r) po_router_set_matrix(e->router, w_r);
    e->theta = c->theta0; /* SchedulerState::init, scheduler.cpp:73-80 */
    e->running_hit = 0.0;
    if (basis) {
        size_t nb = (size_t)e->H * (size_t)c->rank * (size_t)e->hd;
        e->basis = (double*)malloc(nb * sizeof(double));
        memcpy(e->basis, basis, nb * sizeof(double));
    }
    if (bias) {
        e->bias = (double*)malloc((size_t)c->d * sizeof(double));
        memcpy(e->bias, bias, (size_t)c->d * sizeof(double));
    }
    if (kept) {
        size_t nk = (size_t)e->H * (size_t)c->rank;
        e->kept = (int32_t*)malloc(nk * sizeof(int32_t));
        memcpy(e->kept, kept, nk * sizeof(int32_t));
    }
    e->stage_k = (double*)malloc((size_t)e->dp * sizeof(double));
    e->stage_v = (double*)malloc((size_t)e->dp * sizeof(double));
    if (err) *err = PIKV_OK;
    return e;
}

void po_engine_destroy(po_engine* e) {
    if (!e) return;
    if (e->payload)
        for (size_t i = 0; i < e->n_chunks; ++i) free(e->payload[i]);
    free(e->slots), free(e->payload), free(e->layers), free(e->head), free(e->live);
    free(e->seq), free(e->basis), free(e->bias), free(e->kept);
    free(e->stage_k), free(e->stage_v), free(e->enc_w);
    po_router_destroy(e->router);
    free(e);
}

po_router* po_engine_router(po_engine* e) { return e->router; }
int po_engine_stored_width(const po_engine* e) { return e->dp; }
int po_engine_shards_per_device(const po_engine* e) { return e->spd; }
int64_t po_engine_slot_count(const po_engine* e) { return (int64_t)e->nrings * e->c.S; }

void po_engine_sched_state(const po_engine* e, double* theta, double* running_hit,
                           uint64_t* step) {
    if (theta) *theta = e->theta;
    if (running_hit) *running_hit = e->running_hit;
    if (step) *step = e->sched_step;
}

void po_engine_store_stats(const po_engine* e, uint64_t* live, uint64_t* memory_bytes,
                           uint64_t* inserts, uint64_t* overwrites) {
    uint64_t n = 0;
    for (int r = 0; r < e->nrings; ++r) n += (uint64_t)e->live[r];
    if (live) *live = n;
    /* KVStore::memory_bytes, kvstore.cpp:193-196 */
    if (memory_bytes) *memory_bytes = 2ull * (uint64_t)e->dp * (uint64_t)e->c.elem_bytes * n;
    if (inserts) *inserts = e->st_inserts;
    if (overwrites) *overwrites = e->st_overwrites;
}

int po_engine_dump_slots(const po_engine* e, uint64_t* id, uint64_t* shard_seq, int64_t* token,
                         int32_t* expert, uint64_t* insert_step, uint64_t* last_access,
                         uint64_t* freq, double* attn_mass, double* per_layer) {
    int64_t n = po_engine_slot_count(e);
    for (int64_t i = 0; i < n; ++i) {
        const po_slot* s = &e->slots[i];
        if (id) id[i] = s->id;
        if (shard_seq) shard_seq[i] = s->shard_seq;
        if (token) token[i] = s->token;
        if (expert) expert[i] = s->expert;
        if (insert_step) insert_step[i] = s->insert_step;
        if (last_access) last_access[i] = s->last_access;
        if (freq) freq[i] = s->freq;
        if (attn_mass) attn_mass[i] = s->attn_mass;
    }
    if (per_layer && e->c.n_layers > 0)
        memcpy(per_layer, e->layers, (size_t)n * (size_t)e->c.n_layers * sizeof(double));
    return PIKV_OK;
}

/* KVStore::snapshot, kvstore.cpp:206-221: every live entry as (device, shard,
 * token, expert, age = EntryMeta::age(now) (types.hpp:19-21), freq), visited
 * device-major in for_each_live (slot) order, then sorted by (device, shard,
 * token, expert). */
static int snap_cmp(const void* a, const void* b) {
    const pikv_snapshot_record* x = (const pikv_snapshot_record*)a;
    const pikv_snapshot_record* y = (const pikv_snapshot_record*)b;
    if (x->device != y->device) return x->device < y->device ? -1 : 1;
    if (x->shard != y->shard) return x->shard < y->shard ? -1 : 1;
    if (x->token_id != y->token_id) return x->token_id < y->token_id ? -1 : 1;
    if (x->expert_id != y->expert_id) return x->expert_id < y->expert_id ? -1 : 1;
    return 0;
}

int po_engine_snapshot(const po_engine* e, uint64_t now, pikv_snapshot_record* out, int64_t cap,
                       int64_t* n_out) {
    const int64_t n_slots = po_engine_slot_count(e);
    const int spd = e->spd, S = e->c.S;
    int64_t n = 0;
    for (int64_t i = 0; i < n_slots; ++i) n += e->slots[i].id != 0;
    pikv_snapshot_record* all = (pikv_snapshot_record*)calloc((size_t)(n ? n : 1), sizeof(*all));
    if (!all) return PIKV_ERR_OUT_OF_MEMORY;
    int64_t m = 0;
    for (int64_t i = 0; i < n_slots; ++i) {
        const po_slot* sl = &e->slots[i];
        if (!sl->id) continue;
        const int64_t ring = i / S;
        pikv_snapshot_record* r = &all[m++];
        r->device = (int32_t)(ring / spd);
        r->shard = (int32_t)(ring % spd);
        r->token_id = sl->token;
        r->expert_id = sl->expert;
        r->age = now >= sl->insert_step ? now - sl->insert_step : 0;
        r->freq = sl->freq;
    }
    qsort(all, (size_t)n, sizeof(*all), snap_cmp);
    if (out) memcpy(out, all, (size_t)(n < cap ? n : cap) * sizeof(*all));
    free(all);
    if (n_out) *n_out = n;
    return PIKV_OK;
}

/* Stored K/V of slot gi as attended (zeros for an empty slot). */
int po_engine_read_payload(po_engine* e, int64_t gi, float* key, float* value) {
    if (gi < 0 || gi >= po_engine_slot_count(e)) return PIKV_ERR_INVALID_ARGUMENT;
    if (!e->slots[gi].id || !e->payload[(size_t)gi / PO_CHUNK]) {
        memset(key, 0, sizeof(float) * (size_t)e->dp), memset(value, 0, sizeof(float) * (size_t)e->dp);
        return PIKV_OK;
    }
    const float* p = slot_payload(e, (size_t)gi, 0);
    memcpy(key, p, sizeof(float) * (size_t)e->dp);
    memcpy(value, p + e->dp, sizeof(float) * (size_t)e->dp);
    return PIKV_OK;
}

/* Overwrite the stored K/V of live slot gi (test infrastructure: attend over
 * exactly the values another store holds, e.g. the GPU's rounded projections). */
int po_engine_write_payload(po_engine* e, int64_t gi, const float* key, const float* value) {
    if (gi < 0 || gi >= po_engine_slot_count(e) || !e->slots[gi].id) return PIKV_ERR_INVALID_ARGUMENT;
    float* p = slot_payload(e, (size_t)gi, 1);
    memcpy(p, key, sizeof(float) * (size_t)e->dp);
    memcpy(p + e->dp, value, sizeof(float) * (size_t)e->dp);
    return PIKV_OK;
}

int po_engine_set_attn_mass(po_engine* e, const double* attn_mass, const double* per_layer) {
    int64_t n = po_engine_slot_count(e);
    for (int64_t i = 0; i < n; ++i)
        if (attn_mass) e->slots[i].attn_mass = attn_mass[i];
    if (per_layer && e->c.n_layers > 0)
        memcpy(e->layers, per_layer, (size_t)n * (size_t)e->c.n_layers * sizeof(double));
    return PIKV_OK;
}

/* Codec::encode_vector for one K or V row (compressor.cpp:364-411), one
 * basis per head; the stored payload is rounded to the storage dtype.
 * INT8/INT4 store the dequantized values the attention kernel reads. */
static void encode_row(const po_engine* e, const double* x, double* out, int for_query) {
    const pikv_config* c = &e->c;
    const int H = e->H, hd = e->hd, r = c->rank;
    switch (c->codec) {
        case PIKV_CODEC_IDENTITY:
            for (int i = 0; i < c->d; ++i) out[i] = x[i];
            return;
        case PIKV_CODEC_LOWRANK:
        case PIKV_CODEC_LORAPLUS: /* project_encode, compressor.cpp:318-329 (+374-378) */
            for (int h = 0; h < H; ++h) {
                for (int j = 0; j < r; ++j) {
                    const double* col = e->basis + ((size_t)h * r + j) * hd;
                    double s = 0.0;
                    for (int i = 0; i < hd; ++i) {
                        double xi = x[h * hd + i];
                        if (c->codec == PIKV_CODEC_LORAPLUS) xi = xi - e->bias[h * hd + i];
                        s += col[i] * xi;
                    }
                    out[h * r + j] = for_query ? s : round_to_dtype(s, c->kv_dtype);
                }
            }
            return;
        case PIKV_CODEC_FASTV: /* compressor.cpp:396-397 */
            for (int h = 0; h < H; ++h)
                for (int j = 0; j < r; ++j) out[h * r + j] = x[h * hd + j];
            return;
        case PIKV_CODEC_PRUNE: /* compressor.cpp:398-402 */
            for (int h = 0; h < H; ++h)
                for (int j = 0; j < r; ++j) out[h * r + j] = x[h * hd + e->kept[h * r + j]];
            return;
        case PIKV_CODEC_INT8:
        case PIKV_CODEC_INT4: {
            if (for_query) {
                for (int i = 0; i < c->d; ++i) out[i] = x[i];
                return;
            }
            int bits = c->codec == PIKV_CODEC_INT8 ? 8 : 4;
            float* row = (float*)malloc(sizeof(float) * (size_t)hd);
            uint8_t* codes = (uint8_t*)malloc((size_t)hd);
            float* deq = (float*)malloc(sizeof(float) * (size_t)hd);
            for (int h = 0; h < H; ++h) {
                float scale;
                for (int i = 0; i < hd; ++i) row[i] = (float)x[h * hd + i];
                po_quantize_row(row, hd, bits, codes, &scale);
                po_dequantize_row(codes, scale, hd, bits, deq);
                for (int i = 0; i < hd; ++i) out[h * hd + i] = (double)deq[i];
            }
            free(row), free(codes), free(deq);
            return;
        }
    }
}

/* ShardBuffer::insert + KVStore::insert, kvstore.cpp:36-53, 107-120.
 * Returns 1 and fills *displaced when a live slot was overwritten. */
static int store_insert(po_engine* e, int64_t token, int expert, const double* k,
                        const double* v, const double* saliency, po_slot* displaced,
                        int* displaced_device) {
    const pikv_config* c = &e->c;
    int dev, sh;
    po_shard_assign(token, expert, c->n_tok, c->n_exp, c->G, c->additive, &dev, &sh, NULL);
    int ring = dev * e->spd + sh;
    int slot = e->head[ring];
    size_t gi = (size_t)ring * c->S + (size_t)slot;
    po_slot* s = &e->slots[gi];
    int disp = 0;
    if (s->id != 0) {
        *displaced = *s;
        *displaced_device = dev;
        disp = 1;
    } else {
        e->live[ring] += 1;
    }
    s->id = e->next_id++;
    s->shard_seq = e->seq[ring]++;
    s->token = token;
    s->expert = expert;
    s->insert_step = e->now; /* pipeline.cpp:191-193 */
    s->last_access = e->now;
    s->freq = 0;
    s->attn_mass = 0.0;
    float* pp = slot_payload(e, gi, 1);
    for (int i = 0; i < e->dp; ++i) pp[i] = (float)k[i], pp[e->dp + i] = (float)v[i];
    s->has_layers = c->n_layers > 0 && saliency != NULL;
    if (c->n_layers > 0) {
        double* pl = e->layers + gi * (size_t)c->n_layers;
        for (int l = 0; l < c->n_layers; ++l) pl[l] = saliency ? saliency[l] : 0.0;
    }
    e->head[ring] = (slot + 1) % c->S;
    e->st_inserts += 1;
    if (disp) e->st_overwrites += 1;
    return disp;
}

/* score_entry, scheduler.cpp:181-229 */
static double score_entry(const po_engine* e, const po_slot* s, size_t gi) {
    const pikv_config* c = &e->c;
    uint64_t now = e->now;
    uint64_t age = now >= s->insert_step ? now - s->insert_step : 0;
    uint64_t rec = now >= s->last_access ? now - s->last_access : 0;
    switch (c->sched_strategy) {
        case PIKV_SCHED_H2O:
            return s->attn_mass;
        case PIKV_SCHED_SL: {
            double u = (double)age <= c->tau ? 1.0 : 0.0;
            if (s->token < c->sink) u += 2.0;
            return u;
        }
        case PIKV_SCHED_FLEX: {
            uint64_t bucket = age / (uint64_t)c->flex_bucket;
            if (bucket >= (uint64_t)c->n_flex_plan) bucket = (uint64_t)c->n_flex_plan - 1;
            return c->flex_plan[bucket];
        }
        case PIKV_SCHED_LRU:
            return -(double)rec;
        case PIKV_SCHED_LRU_PLUS:
            return -(double)rec + c->lambda_freq * (double)s->freq;
        case PIKV_SCHED_ADAKV: {
            double phi[3] = {s->attn_mass, (double)s->freq, 1.0 / (1.0 + (double)age)};
            double u = 0.0;
            for (int j = 0; j < c->n_adakv_weights && j < 3; ++j) u += c->adakv_weights[j] * phi[j];
            return u;
        }
        case PIKV_SCHED_DUO: {
            double u = 0.0;
            if (!s->has_layers) return u; /* empty per_layer_scores */
            const double* pl = e->layers + gi * (size_t)c->n_layers;
            for (int l = 0; l < c->n_layers; ++l) u += pl[l];
            return u;
        }
    }
    return 0.0;
}

/* evict, scheduler.cpp:262-330 */
static int sched_evict(po_engine* e, po_step_out* out) {
    const pikv_config* c = &e->c;
    const int S = c->S, ps = c->page_size;
    for (int dev = 0; dev < c->G; ++dev) {
        /* pages keyed (shard, shard_seq / page_size); aggregates summed in
         * slot order (for_each_live, kvstore.hpp:43-48). */
        int maxp = 0;
        for (int sh = 0; sh < e->spd; ++sh) maxp += S / ps + 2;
        double* agg = (double*)calloc((size_t)maxp, sizeof(double));
        uint64_t* oldest = (uint64_t*)calloc((size_t)maxp, sizeof(uint64_t));
        int* cnt = (int*)calloc((size_t)maxp, sizeof(int));
        int* pring = (int*)calloc((size_t)maxp, sizeof(int));
        uint64_t* pno = (uint64_t*)calloc((size_t)maxp, sizeof(uint64_t));
        int np = 0;
        for (int sh = 0; sh < e->spd; ++sh) {
            int ring = dev * e->spd + sh;
            uint64_t lo_seq = e->seq[ring] > (uint64_t)S ? e->seq[ring] - (uint64_t)S : 0;
            uint64_t p0 = lo_seq / (uint64_t)ps;
            int base = np;
            int nring_pages = 0;
            for (int slot = 0; slot < S; ++slot) {
                po_slot* s = &e->slots[(size_t)ring * S + slot];
                if (!s->id) continue;
                int pi = (int)(s->shard_seq / (uint64_t)ps - p0);
                if (pi + 1 > nring_pages) nring_pages = pi + 1;
                int k = base + pi;
                if (cnt[k] == 0) oldest[k] = s->id;
                oldest[k] = oldest[k] < s->id ? oldest[k] : s->id;
                agg[k] += score_entry(e, s, (size_t)ring * S + slot);
                cnt[k] += 1;
                pring[k] = ring;
                pno[k] = p0 + (uint64_t)pi;
            }
            np = base + nring_pages;
        }
        /* compact to existing pages (map order: shard, page_no) */
        int P = 0;
        for (int i = 0; i < np; ++i) {
            if (!cnt[i]) continue;
            agg[P] = agg[i], oldest[P] = oldest[i], cnt[P] = cnt[i];
            pring[P] = pring[i], pno[P] = pno[i];
            ++P;
        }
        out->pages_before += P;
        int* idx = (int*)malloc(sizeof(int) * (size_t)(P + 1));
        int* why = (int*)malloc(sizeof(int) * (size_t)(P + 1));
        int nv = po_select_evictions(agg, oldest, P, c->budget_pages,
                                     c->sched_strategy == PIKV_SCHED_ADAKV, e->theta, idx, why);
        out->pages_after += P - nv;
        for (int v = 0; v < nv; ++v) {
            int p = idx[v], ring = pring[p];
            /* members in id order == shard_seq order within a ring */
            for (uint64_t sq = pno[p] * (uint64_t)ps; sq < (pno[p] + 1) * (uint64_t)ps; ++sq) {
                int slot = (int)(sq % (uint64_t)S);
                size_t gi = (size_t)ring * S + slot;
                po_slot* s = &e->slots[gi];
                if (!s->id || s->shard_seq != sq) continue;
                if (out->n_evictions < out->evict_cap && out->evictions) {
                    po_evict* r = &out->evictions[out->n_evictions];
                    r->step = e->sched_step;
                    r->id = s->id;
                    r->token = s->token;
                    r->expert = s->expert;
                    r->device = dev;
                    r->score = score_entry(e, s, gi);
                    r->reason = why[v];
                    r->stream = 0;
                }
                out->n_evictions += 1;
                s->id = 0; /* KVStore::erase, kvstore.cpp:180-185 */
                e->live[ring] -= 1;
            }
        }
        free(idx), free(why), free(agg), free(oldest), free(cnt), free(pring), free(pno);
    }
    e->sched_step += 1;
    return PIKV_OK;
}

typedef struct att_ref {
    int64_t token;
    int32_t expert;
    size_t gi;
} att_ref;

static int att_cmp(const void* pa, const void* pb) {
    const att_ref* a = (const att_ref*)pa;
    const att_ref* b = (const att_ref*)pb;
    if (a->token != b->token) return a->token < b->token ? -1 : 1;
    if (a->expert != b->expert) return a->expert < b->expert ? -1 : 1;
    return 0;
}

static int engine_step_impl(po_engine* e, const double* q, const double* k, const double* v,
                            const double* saliency, po_step_out* out, int attend) {
    const pikv_config* c = &e->c;
    out->inserts = out->hits = out->lookups = out->n_attended = 0;
    out->fetch_elements = 0;
    out->pages_before = out->pages_after = 0;
    out->n_evictions = 0;
    int64_t token_id = (int64_t)e->now;
    const int kk = c->k, E = c->E;

    /* 1. route (pipeline.cpp:223) */
    double* logits = (double*)malloc(sizeof(double) * (size_t)E);
    int rc = po_route(e->router, c, q, logits, out->experts, out->gates);
    if (out->logits) memcpy(out->logits, logits, sizeof(double) * (size_t)E);
    free(logits);
    if (rc) return rc;

    /* 2-4. stage one entry per expert, compress, insert (pipeline.cpp:228-246, 148-211) */
    encode_row(e, k, e->stage_k, 0);
    encode_row(e, v, e->stage_v, 0);
    for (int j = 0; j < kk; ++j) {
        po_slot disp;
        int ddev = 0;
        if (store_insert(e, token_id, out->experts[j], e->stage_k, e->stage_v, saliency, &disp,
                         &ddev)) {
            if (out->n_evictions < out->evict_cap && out->evictions) {
                po_evict* r = &out->evictions[out->n_evictions];
                r->step = e->now;
                r->id = disp.id;
                r->token = disp.token;
                r->expert = disp.expert;
                r->device = ddev;
                r->score = 0.0;
                r->reason = PIKV_EVICT_OVERWRITE;
                r->stream = 0;
            }
            out->n_evictions += 1;
        }
        out->inserts += 1;
    }

    /* 5. scheduling pass (pipeline.cpp:249-254) */
    if (!c->unbounded_budget) sched_evict(e, out);

    /* 6. retrieve (kvstore.cpp:122-178) */
    size_t ns = (size_t)e->nrings * c->S;
    att_ref* hits = (att_ref*)malloc(sizeof(att_ref) * (ns + 1));
    int nh = 0;
    int found[64] = {0};
    for (size_t gi = 0; gi < ns; ++gi) {
        po_slot* s = &e->slots[gi];
        if (!s->id || s->token >= token_id) continue;
        for (int j = 0; j < kk; ++j) {
            if (out->experts[j] == s->expert) {
                hits[nh].token = s->token;
                hits[nh].expert = s->expert;
                hits[nh].gi = gi;
                ++nh;
                found[j] += 1;
                break;
            }
        }
    }
    qsort(hits, (size_t)nh, sizeof(att_ref), att_cmp);
    for (int i = 0; i < nh; ++i) {
        po_slot* s = &e->slots[hits[i].gi];
        s->freq += 1;
        s->last_access = e->now;
    }
    int missed = 0;
    for (int j = 0; j < kk; ++j) {
        if (found[j] == 0) {
            po_record_miss(e->router, out->experts[j]);
            ++missed;
        }
    }
    out->lookups = kk;
    out->hits = kk - missed;
    /* 7. fetch_elements (pipeline.cpp:262-264, 22-26) */
    int hw = c->head_width < e->dp ? c->head_width : e->dp;
    out->fetch_elements = (int64_t)nh * (int64_t)(2 * hw + e->dp);
    out->n_attended = nh;

    if (attend) {
        /* 8-9. attention in compressed space, per head (pipeline.cpp:295-299) */
        double* qa = (double*)malloc(sizeof(double) * (size_t)e->dp);
        encode_row(e, q, qa, 1);
        const int H = e->H, w = e->dph;
        double* kbuf = (double*)malloc(sizeof(double) * (size_t)(nh > 0 ? nh : 1) * (size_t)w);
        double* vbuf = (double*)malloc(sizeof(double) * (size_t)(nh > 0 ? nh : 1) * (size_t)w);
        double* wts = (double*)malloc(sizeof(double) * (size_t)(nh > 0 ? nh : 1));
        double* alpha = (double*)calloc((size_t)(nh > 0 ? nh : 1), sizeof(double));
        for (int h = 0; h < H; ++h) {
            for (int i = 0; i < nh; ++i) {
                const float* p = slot_payload(e, hits[i].gi, 0);
                for (int o = 0; o < w; ++o) {
                    kbuf[(size_t)i * w + o] = (double)p[(size_t)h * w + o];
                    vbuf[(size_t)i * w + o] = (double)p[e->dp + (size_t)h * w + o];
                }
            }
            po_attention(qa + (size_t)h * w, kbuf, vbuf, nh, w, out->y + (size_t)h * w, wts);
            for (int i = 0; i < nh; ++i) alpha[i] += wts[i];
        }
        /* 10. fold-back (pipeline.cpp:302-312); alpha = mean over heads */
        for (int i = 0; i < nh; ++i) {
            double a = alpha[i] / H;
            po_slot* s = &e->slots[hits[i].gi];
            s->attn_mass += a;
            if (s->has_layers) e->layers[hits[i].gi * (size_t)c->n_layers + e->now % (uint64_t)c->n_layers] += a;
            if (i < out->att_cap) {
                if (out->att_token) out->att_token[i] = s->token;
                if (out->att_expert) out->att_expert[i] = s->expert;
                if (out->att_weight) out->att_weight[i] = a;
            }
        }
        free(qa), free(kbuf), free(vbuf), free(wts), free(alpha);
    }
    free(hits);

    /* 11. feedback (pipeline.cpp:337-347) */
    if (c->router_strategy == PIKV_ROUTER_ADAPTIVE) {
        double reward = out->lookups == 0 ? 0.0 : (double)out->hits / out->lookups;
        po_adapt(e->router, c, out->experts, kk, reward);
    }
    if (out->lookups > 0) { /* observe_hits, scheduler.cpp:332-338 */
        double rate = (double)out->hits / (double)out->lookups;
        e->running_hit = c->hit_decay * e->running_hit + (1.0 - c->hit_decay) * rate;
    }
    if (c->sched_strategy == PIKV_SCHED_ADAKV && !c->unbounded_budget)
        e->theta += c->adakv_step * (c->target_hit - e->running_hit); /* :340-342 */
    e->now += 1;
    return PIKV_OK;
}

/* QueryEncoder(width, seed), pipeline.cpp:29-36: w_query, w_key, w_value
 * drawn in that order from one Rng, each normal_vector(width^2, 1/sqrt(width)). */
void po_encoder_weights(int width, uint64_t seed, double* w3) {
    po_rng r;
    po_rng_init(&r, seed);
    const double scale = 1.0 / sqrt((double)width);
    const int64_t n = (int64_t)width * width;
    for (int64_t i = 0; i < 3 * n; ++i) w3[i] = scale * po_rng_normal(&r);
}

/* QueryEncoder::apply / encode, pipeline.cpp:38-57: out[i] = sum_j W[i][j] x[j]
 * in j order, for W = w_query, w_key, w_value. */
void po_encode(const double* w3, int width, const double* x, double* q, double* k, double* v) {
    double* outs[3] = {q, k, v};
    for (int m = 0; m < 3; ++m) {
        const double* W = w3 + (size_t)m * width * width;
        for (int i = 0; i < width; ++i) {
            const double* row = W + (size_t)i * width;
            double s = 0.0;
            for (int j = 0; j < width; ++j) s += row[j] * x[j];
            outs[m][i] = s;
        }
    }
}

#define PO_ENCODER_SALT 0x71c9de52ae0aefULL /* pipeline.cpp:15 kEncoderSalt */

/* Engine::step from the token's embedding (pipeline.cpp:213-351 incl. the
 * encode at :222).  q stays fp64 (routing is bit-exact); k and v are rounded
 * to the storage dtype, as the engine stores them. */
int po_engine_step_embed(po_engine* e, const double* emb, const double* saliency, po_step_out* out,
                         int attend) {
    const int d = e->c.d;
    if (!e->enc_w) {
        e->enc_w = (double*)malloc(sizeof(double) * 3 * (size_t)d * d);
        if (!e->enc_w) return PIKV_ERR_OUT_OF_MEMORY;
        po_encoder_weights(d, e->c.seed ^ PO_ENCODER_SALT, e->enc_w);
    }
    double* q = (double*)malloc(sizeof(double) * 3 * (size_t)d);
    double* k = q + d;
    double* v = k + d;
    po_encode(e->enc_w, d, emb, q, k, v);
    for (int i = 0; i < d; ++i) {
        k[i] = round_to_dtype(k[i], e->c.kv_dtype);
        v[i] = round_to_dtype(v[i], e->c.kv_dtype);
    }
    const int rc = engine_step_impl(e, q, k, v, saliency, out, attend);
    free(q);
    return rc;
}

/* The store build of a prefill: for t = 0..T-1 (steps now+t)
 * the token's k entries (experts[t][0..k-1], selection order) are encoded
 * and inserted as Engine::step inserts them (pipeline.cpp:148-211,
 * kvstore.cpp:107-120) -- no routing, eviction or retrieval -- then now
 * advances by T.  k/v rows are [T][d]; saliency [T][n_layers] or NULL. */
int po_engine_insert_bulk(po_engine* e, int64_t T, const double* k, const double* v,
                          const int32_t* experts, const double* saliency, int64_t* n_displaced) {
    const pikv_config* c = &e->c;
    int64_t nd = 0;
    for (int64_t t = 0; t < T; ++t) {
        encode_row(e, k + (size_t)t * c->d, e->stage_k, 0);
        encode_row(e, v + (size_t)t * c->d, e->stage_v, 0);
        for (int j = 0; j < c->k; ++j) {
            po_slot disp;
            int ddev = 0;
            nd += store_insert(e, (int64_t)e->now, experts[t * c->k + j], e->stage_k, e->stage_v,
                               saliency ? saliency + (size_t)t * c->n_layers : NULL, &disp, &ddev);
        }
        e->now += 1;
    }
    if (n_displaced) *n_displaced = nd;
    return PIKV_OK;
}

int po_engine_step(po_engine* e, const double* q, const double* k, const double* v,
                   const double* saliency, po_step_out* out) {
    return engine_step_impl(e, q, k, v, saliency, out, 1);
}

int po_engine_step_noattend(po_engine* e, const double* q, const double* k, const double* v,
                            const double* saliency, po_step_out* out) {
    return engine_step_impl(e, q, k, v, saliency, out, 0);
}
