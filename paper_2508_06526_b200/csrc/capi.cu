// SPDX-License-Identifier: Apache-2.0
//
// C-ABI of the B200 PiKV engine (include/pikv_b200.h): engine lifetime,
// HBM allocation, the per-step launch sequence (captured once into a CUDA
// graph and replayed), result readback and the pure-function entry points.
#include <cuda.h>  // green-context types only: the entry points come from cudaGetDriverEntryPoint
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "pikv_dev.cuh"

using namespace pikv_dev;

namespace pikv_dev {
bool pdl_enabled() {
    static const bool on = [] {
        // measured neutral on c2 with graph replay (profiles/README.md); opt in
        const char* v = std::getenv("PIKV_PDL");
        return v && v[0] == '1';
    }();
    return on;
}
__global__ void k_shard_assign(const int64_t*, const int32_t*, int32_t, int32_t, int32_t, int32_t,
                               int32_t, int32_t*, int32_t*, int32_t*);
__global__ void k_select(const double*, const uint64_t*, int32_t, int32_t, int32_t, double,
                         int32_t*, int32_t*, int32_t*);
__global__ void k_attention(const float*, const float*, const float*, int32_t, int32_t, float*,
                            float*);
__global__ void k_quantize(const void*, int32_t, int32_t, int32_t, int32_t, uint8_t*, float*);
__global__ void k_dequantize(const uint8_t*, const float*, int32_t, int32_t, int32_t, float*);
__global__ void k_lr_encode(const float*, const float*, const float*, int32_t, int32_t, int32_t,
                            int32_t, float*);
__global__ void k_lr_decode(const float*, const float*, const float*, int32_t, int32_t, int32_t,
                            int32_t, float*);
const char* attend_check(const Dims& D);
int attend_entries_per_stage(const Dims& D);
int attend_ctas_per_sm(const Dims& D);
int attend_reserve_sms(const Dims& D);
}  // namespace pikv_dev

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(x)                                                                   \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess)                                                        \
            return fail(PIKV_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

bool is_pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }

constexpr uint64_t kRouterSalt = 0x2545f4914f6cdd1dULL;  // pipeline.cpp:16

// W_r [E][d] (row-major, router.cpp:54-67) -> the device layout: chunks of
// route_ch columns, each [E][route_ch + 2] with zero padding (State::W).
static size_t router_w_elems(const Dims& D) {
    const size_t nch = (size_t)(D.d + D.route_ch - 1) / D.route_ch;
    return nch * D.E * (D.route_ch + 2);
}
static std::vector<double> pack_router_w(const Dims& D, const double* w) {
    std::vector<double> out(router_w_elems(D), 0.0);
    const int ch = D.route_ch, rs = ch + 2;
    for (int e = 0; e < D.E; ++e)
        for (int i = 0; i < D.d; ++i)
            out[((size_t)(i / ch) * D.E + e) * rs + i % ch] = w[(size_t)e * D.d + i];
    return out;
}

// n draws of Rng(seed).normal() * 1/sqrt(width): pikv::Rng's transforms
// over std::mt19937_64 (rng.hpp).  RouterState::init (router.cpp:54-67):
// W_r = normal_vector(E*d, 1/sqrt(d)); QueryEncoder (pipeline.cpp:29-36):
// w_query, w_key, w_value = three consecutive normal_vector(d*d, 1/sqrt(d)).
struct RefRng {  // pikv::Rng (rng.hpp:15-70): std::mt19937_64 + its double transforms
    explicit RefRng(uint64_t seed) : gen(seed) {}
    double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        double u1 = uniform();
        double u2 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        double radius = std::sqrt(-2.0 * std::log(u1));
        double angle = 2.0 * M_PI * u2;
        spare = radius * std::sin(angle);
        has_spare = true;
        return radius * std::cos(angle);
    }
    std::mt19937_64 gen;
    bool has_spare = false;
    double spare = 0.0;
};

std::vector<double> reference_normals(size_t n, int width, uint64_t seed) {
    RefRng rng(seed);
    const double scale = 1.0 / std::sqrt(static_cast<double>(width));
    std::vector<double> w(n);
    for (auto& x : w) x = scale * rng.normal();
    return w;
}

std::vector<double> router_matrix(int E, int d, uint64_t seed) {
    return reference_normals(static_cast<size_t>(E) * d, d, seed);
}

constexpr uint64_t kEncoderSalt = 0x71c9de52ae0aefULL;  // pipeline.cpp:15

}  // namespace

struct pikv_engine {
    pikv_config cfg{};
    Dims D{};
    Cfg C{};
    State S{};
    ExchangeLayout X{};
    cudaStream_t stream = nullptr;
    int device = 0;
    std::vector<void*> allocs;
    // staging for host-buffer steps and synthetic prefill
    void* in_q = nullptr;
    void* in_k = nullptr;
    void* in_v = nullptr;
    double* in_sal = nullptr;
    // QueryEncoder (pipeline.cpp:29-57) for the embedding step, allocated on
    // first use: W^T [3][d][d] fp64, the step's fp64 q, host-path staging
    // pikv_step_host as one graph: H2D of the packed q/k/v -> the step -> D2H
    // of y, captured once; the memcpy nodes are re-pointed at the caller's
    // (pinned) buffers on every call
    cudaGraph_t host_g = nullptr;
    cudaGraphExec_t host_ge = nullptr;
    cudaGraphNode_t host_h2d = nullptr, host_h2d_kv = nullptr, host_d2h = nullptr;
    void* host_ph = nullptr;  // pinned placeholders used at capture
    cudaStream_t side = nullptr;  // the graph's copy branch at capture
    cudaEvent_t ev_fork = nullptr, ev_kv = nullptr, ev_y = nullptr, ev_join = nullptr;
    // grow-only scratch of the bulk store build (device) and its host-path
    // staging; freed at destroy (not through the async pool: no per-call
    // map/unmap)
    void* bulk_buf = nullptr;
    size_t bulk_cap = 0;
    void* bulk_stage = nullptr;
    size_t stage_cap = 0;
    // multi-GPU exchange (pikv_engine_attach_nccl / pikv_engine_set_nccl_comm):
    // the step all-gathers every rank's exchange records into `gathered` on
    // the engine stream (inside the captured step graph) and finishes the
    // LSE merge on every rank
    ncclComm_t comm = nullptr;
    bool own_comm = false;
    uint8_t* gathered = nullptr;
    // grow-only readback scratch (pikv_read_attended_host)
    void* rb_buf = nullptr;
    size_t rb_cap = 0;
    bool exchange_path() const { return D.world > 1 || comm != nullptr; }
    std::string attend_err;  // non-empty: the decode step cannot run this layout
    cudaEvent_t y_final_event = nullptr;  // group host path, sharded: recorded after the merge
    double* enc_wt = nullptr;
    double* q64 = nullptr;
    double* in_emb = nullptr;
    float* out_y = nullptr;
    // graph cache keyed by (q, k, v, saliency, y, attend | emb | parts):
    // the executable and the number of kernels it launches
    struct Captured {
        cudaGraphExec_t ge;
        int kernels;
    };
    std::map<std::tuple<const void*, const void*, const void*, const void*, void*, int>, Captured>
        graphs;
    void drop_graphs() {
        for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.ge);
        graphs.clear();
    }
    // every captured graph: the keyed cache and the pikv_step_host graph
    // (kernels captured State by value, so new codec buffers need new graphs)
    void invalidate() {
        drop_graphs();
        if (host_ge) cudaGraphExecDestroy(host_ge);
        if (host_g) cudaGraphDestroy(host_g);
        host_ge = nullptr, host_g = nullptr;
        host_h2d = host_h2d_kv = host_d2h = nullptr;
    }
    unsigned warmed_parts = 0;  // step parts run eagerly once (kernel attributes set)
    bool warmed = false;
    int64_t launches = 0;
    int kernels_per_step = 0;
    bool fused_retrieval = false;  // PIKV_RETR_FUSED=1: single-pass k_retr_fused (measured: not faster
                                   // in graph replay, profiles/README.md)
    bool fused_control = false;  // k_control replaces route..retr_write (B <= 8; PIKV_CONTROL=0/1 forces)
    // profiling: per step kPhases+1 events on the engine stream
    bool profiling = false;
    std::vector<cudaEvent_t> ev;
    int prof_steps = 0;
    int cur = -1;  // event slot base of the step being enqueued

    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        if (n == 0) n = 1;
        if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return nullptr;
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
};

extern "C" {

const char* pikv_version(void) { return "pikv-b200 0.1 (sm_100a)"; }
const char* pikv_last_error(void) { return g_err.c_str(); }
int pikv_config_size(void) { return (int)sizeof(pikv_config); }

void pikv_config_default(pikv_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->d = 64, c->head_width = 16, c->E = 8, c->k = 2, c->L = 1024, c->G = 2, c->S = 16;
    c->K = 4, c->elem_bytes = 2, c->rho = 1.0, c->n_heads = 1;
    c->n_tok = 64, c->n_exp = 64, c->additive = 0, c->shards_per_device = 0;
    c->router_strategy = PIKV_ROUTER_TOPK, c->groups = 1, c->stride = 1;
    c->alpha = 1.0, c->lambda_miss = 1.0, c->beta_ent = 1.0, c->bandit_step = 0.05;
    c->bias_cap = 5.0, c->load_decay = 0.99;
    c->sched_strategy = PIKV_SCHED_LRU, c->budget_pages = 4, c->page_size = 16, c->sink = 4;
    c->flex_bucket = 16, c->n_adakv_weights = 3, c->n_flex_plan = 1;
    c->tau = 64.0, c->lambda_freq = 0.5, c->adakv_step = 0.05, c->target_hit = 0.9;
    c->gamma_sim = 0.5, c->theta0 = -1e18, c->hit_decay = 0.9;
    c->adakv_weights[0] = 1.0, c->adakv_weights[1] = 0.5, c->adakv_weights[2] = 0.25;
    c->flex_plan[0] = 1.0;
    c->codec = PIKV_CODEC_IDENTITY, c->rank = 8;
    c->batch = 1, c->kv_dtype = PIKV_DTYPE_F32, c->world_size = 1, c->rank_id = 0;
    c->seed = 1;
}

// ---------------------------------------------------------------------------
// pure functions
// ---------------------------------------------------------------------------
int pikv_shard_assign(const int64_t* t, const int32_t* e, int32_t n, int32_t n_tok, int32_t n_exp,
                      int32_t devices, int32_t additive, int32_t* device_out, int32_t* shard_out,
                      int32_t* raw_out) {
    if (!is_pow2(n_tok) || !is_pow2(n_exp))  // kvstore.cpp:17-19
        return fail(PIKV_ERR_INVALID_CONFIG, "shard_assign: moduli must be powers of two");
    if (devices < 1) return fail(PIKV_ERR_INVALID_CONFIG, "shard_assign: devices must be >= 1");
    if (n <= 0) return PIKV_OK;
    // negative inputs (kvstore.cpp:20-22) are checked on the device copy
    std::vector<int64_t> ht(n);
    std::vector<int32_t> he(n);
    CUDA_TRY(cudaMemcpy(ht.data(), t, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(he.data(), e, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i)
        if (ht[i] < 0 || he[i] < 0)
            return fail(PIKV_ERR_INVALID_ARGUMENT, "shard_assign: negative token or expert index");
    k_shard_assign<<<(n + 255) / 256, 256>>>(t, e, n, n_tok, n_exp, devices, additive, device_out,
                                             shard_out, raw_out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    return PIKV_OK;
}

int pikv_select_evictions(const double* aggregate, const uint64_t* oldest_id, int32_t n,
                          int32_t budget_pages, int32_t use_theta, double theta, int32_t* idx_out,
                          int32_t* reason_out, int32_t* n_out) {
    if (budget_pages < 1) return fail(PIKV_ERR_INVALID_CONFIG, "budget_pages must be >= 1");
    k_select<<<1, 1024>>>(aggregate, oldest_id, n, budget_pages, use_theta, theta, idx_out,
                          reason_out, n_out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    return PIKV_OK;
}

int pikv_attention(const float* q, const float* keys, const float* values, int32_t n_queries,
                   int32_t n, int32_t w, float* y_out, float* weights_out) {
    if (w < 1) return fail(PIKV_ERR_INVALID_ARGUMENT, "attention: width must be >= 1");
    if (n == 0) {  // pipeline.cpp:63-66: zero vector, no weights
        CUDA_TRY(cudaMemset(y_out, 0, sizeof(float) * (size_t)n_queries * w));
        return PIKV_OK;
    }
    size_t smem = sizeof(float) * (size_t)n;
    if (smem > 200 * 1024) return fail(PIKV_ERR_INVALID_ARGUMENT, "attention: n too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_attention<<<n_queries, 256, smem>>>(q, keys, values, n, w, y_out, weights_out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    return PIKV_OK;
}

int pikv_quantize(const void* x, int32_t dtype, int32_t rows, int32_t width, int32_t bits,
                  uint8_t* codes_out, float* scales_out) {
    if (bits != 8 && bits != 4) return fail(PIKV_ERR_INVALID_ARGUMENT, "bits must be 8 or 4");
    if (bits == 4 && width % 2) return fail(PIKV_ERR_INVALID_ARGUMENT, "int4 width must be even");
    k_quantize<<<(rows + 7) / 8, 256>>>(x, dtype, rows, width, bits, codes_out, scales_out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    return PIKV_OK;
}

int pikv_dequantize(const uint8_t* codes, const float* scales, int32_t rows, int32_t width,
                    int32_t bits, float* x_out) {
    if (bits != 8 && bits != 4) return fail(PIKV_ERR_INVALID_ARGUMENT, "bits must be 8 or 4");
    const int64_t n = (int64_t)rows * width;
    k_dequantize<<<(unsigned)((n + 255) / 256), 256>>>(codes, scales, rows, width, bits, x_out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    return PIKV_OK;
}

int pikv_lowrank_encode(const float* x, const float* basis, const float* bias, int32_t rows,
                        int32_t heads, int32_t hd, int32_t r, float* y_out) {
    const int64_t n = (int64_t)rows * heads * r;
    k_lr_encode<<<(unsigned)((n + 255) / 256), 256>>>(x, basis, bias, rows, heads, hd, r, y_out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    return PIKV_OK;
}

int pikv_lowrank_decode(const float* y, const float* basis, const float* bias, int32_t rows,
                        int32_t heads, int32_t hd, int32_t r, float* x_out) {
    const int64_t n = (int64_t)rows * heads * hd;
    k_lr_decode<<<(unsigned)((n + 255) / 256), 256>>>(y, basis, bias, rows, heads, hd, r, x_out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    return PIKV_OK;
}

// host-buffer wrappers ---------------------------------------------------------
namespace {
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t n) { cudaMalloc(&p, n ? n : 1); }
    ~DevBuf() { cudaFree(p); }
};
}  // namespace

int pikv_shard_assign_host(const int64_t* t, const int32_t* e, int32_t n, int32_t n_tok,
                           int32_t n_exp, int32_t devices, int32_t additive, int32_t* device_out,
                           int32_t* shard_out, int32_t* raw_out) {
    // same checks as shard_assign (kvstore.cpp:17-22), before touching the device
    if (!is_pow2(n_tok) || !is_pow2(n_exp))
        return fail(PIKV_ERR_INVALID_CONFIG, "shard_assign: moduli must be powers of two");
    if (devices < 1) return fail(PIKV_ERR_INVALID_CONFIG, "shard_assign: devices must be >= 1");
    for (int i = 0; i < n; ++i)
        if (t[i] < 0 || e[i] < 0)
            return fail(PIKV_ERR_INVALID_ARGUMENT, "shard_assign: negative token or expert index");
    if (n <= 0) return PIKV_OK;
    DevBuf dt(8 * (size_t)n), de(4 * (size_t)n), dd(4 * (size_t)n), ds(4 * (size_t)n), dr(4 * (size_t)n);
    CUDA_TRY(cudaMemcpy(dt.p, t, 8 * (size_t)n, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(de.p, e, 4 * (size_t)n, cudaMemcpyHostToDevice));
    int rc = pikv_shard_assign((int64_t*)dt.p, (int32_t*)de.p, n, n_tok, n_exp, devices, additive,
                               (int32_t*)dd.p, (int32_t*)ds.p, (int32_t*)dr.p);
    if (rc) return rc;
    if (device_out) CUDA_TRY(cudaMemcpy(device_out, dd.p, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    if (shard_out) CUDA_TRY(cudaMemcpy(shard_out, ds.p, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    if (raw_out) CUDA_TRY(cudaMemcpy(raw_out, dr.p, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_select_evictions_host(const double* aggregate, const uint64_t* oldest_id, int32_t n,
                               int32_t budget_pages, int32_t use_theta, double theta,
                               int32_t* idx_out, int32_t* reason_out, int32_t* n_out) {
    const size_t m = n > 0 ? (size_t)n : 1;
    DevBuf da(8 * m), dol(8 * m), di(4 * m), dr(4 * m), dn(4);
    if (n > 0) {
        CUDA_TRY(cudaMemcpy(da.p, aggregate, 8 * (size_t)n, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(dol.p, oldest_id, 8 * (size_t)n, cudaMemcpyHostToDevice));
    }
    int rc = pikv_select_evictions((double*)da.p, (uint64_t*)dol.p, n, budget_pages, use_theta, theta,
                                   (int32_t*)di.p, (int32_t*)dr.p, (int32_t*)dn.p);
    if (rc) return rc;
    int32_t v = 0;
    CUDA_TRY(cudaMemcpy(&v, dn.p, 4, cudaMemcpyDeviceToHost));
    *n_out = v;
    if (v > 0) {
        CUDA_TRY(cudaMemcpy(idx_out, di.p, 4 * (size_t)v, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(reason_out, dr.p, 4 * (size_t)v, cudaMemcpyDeviceToHost));
    }
    return PIKV_OK;
}

int pikv_attention_host(const float* q, const float* keys, const float* values, int32_t n_queries,
                        int32_t n, int32_t w, float* y_out, float* weights_out) {
    const size_t nq = (size_t)n_queries, nn = (size_t)(n > 0 ? n : 1);
    DevBuf dq(4 * nq * w), dk(4 * nq * nn * w), dv(4 * nq * nn * w), dy(4 * nq * w), dw(4 * nq * nn);
    CUDA_TRY(cudaMemcpy(dq.p, q, 4 * nq * w, cudaMemcpyHostToDevice));
    if (n > 0) {
        CUDA_TRY(cudaMemcpy(dk.p, keys, 4 * nq * n * w, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(dv.p, values, 4 * nq * n * w, cudaMemcpyHostToDevice));
    }
    int rc = pikv_attention((float*)dq.p, (float*)dk.p, (float*)dv.p, n_queries, n, w, (float*)dy.p,
                            (float*)dw.p);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpy(y_out, dy.p, 4 * nq * w, cudaMemcpyDeviceToHost));
    if (weights_out && n > 0) CUDA_TRY(cudaMemcpy(weights_out, dw.p, 4 * nq * n, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

// ---------------------------------------------------------------------------
// engine
// ---------------------------------------------------------------------------
static int validate(const pikv_config& c) {
    // ModelConfig::validate, config.hpp:42-54
    if (c.d < 1) return fail(PIKV_ERR_INVALID_CONFIG, "ModelConfig: d must be >= 1");
    if (c.head_width < 1 || c.head_width > c.d)
        return fail(PIKV_ERR_INVALID_CONFIG, "ModelConfig: head_width must be in [1, d]");
    if (c.E < 1) return fail(PIKV_ERR_INVALID_CONFIG, "ModelConfig: E must be >= 1");
    if (c.k < 1 || c.k > c.E) return fail(PIKV_ERR_INVALID_CONFIG, "ModelConfig: need 1 <= k <= E");
    if (c.L < 1 || c.G < 1 || c.S < 1 || c.K < 1)
        return fail(PIKV_ERR_INVALID_CONFIG, "ModelConfig: L, G, S, K must be >= 1");
    if (!(c.rho >= 1.0)) return fail(PIKV_ERR_INVALID_CONFIG, "ModelConfig: rho must be >= 1");
    if (c.elem_bytes < 1) return fail(PIKV_ERR_INVALID_CONFIG, "ModelConfig: elem_bytes must be >= 1");
    // StoreConfig::validate, kvstore.cpp:56-64
    if (!is_pow2(c.n_tok) || !is_pow2(c.n_exp))
        return fail(PIKV_ERR_INVALID_CONFIG, "StoreConfig: n_tok and n_exp must be powers of two");
    if (c.shards_per_device < 0)
        return fail(PIKV_ERR_INVALID_CONFIG, "StoreConfig: shards_per_device must be >= 0");
    // RouterConfig::validate, router.cpp:40-53
    if (c.alpha < 0 || c.lambda_miss < 0 || c.beta_ent < 0 || c.bandit_step < 0)
        return fail(PIKV_ERR_INVALID_CONFIG, "RouterConfig: coefficients must be >= 0");
    if (c.groups < 1 || c.groups > c.E)
        return fail(PIKV_ERR_INVALID_CONFIG, "RouterConfig: need 1 <= groups <= E");
    if (c.load_decay < 0 || c.load_decay >= 1.0)
        return fail(PIKV_ERR_INVALID_CONFIG, "RouterConfig: load_decay must be in [0, 1)");
    // SchedulerConfig::validate, scheduler.cpp:49-71
    if (c.budget_pages < 1) return fail(PIKV_ERR_INVALID_CONFIG, "SchedulerConfig: budget_pages must be >= 1");
    if (c.page_size < 1) return fail(PIKV_ERR_INVALID_CONFIG, "SchedulerConfig: page_size must be >= 1");
    if (c.lambda_freq < 0 || c.adakv_step < 0 || c.gamma_sim < 0)
        return fail(PIKV_ERR_INVALID_CONFIG, "SchedulerConfig: coefficients must be >= 0");
    if (c.target_hit < 0.0 || c.target_hit > 1.0)
        return fail(PIKV_ERR_INVALID_CONFIG, "SchedulerConfig: target_hit must be in [0, 1]");
    if (c.hit_decay < 0.0 || c.hit_decay >= 1.0)
        return fail(PIKV_ERR_INVALID_CONFIG, "SchedulerConfig: hit_decay must be in [0, 1)");
    if (c.n_flex_plan < 1 || c.n_flex_plan > 32 || c.flex_bucket < 1)
        return fail(PIKV_ERR_INVALID_CONFIG, "SchedulerConfig: flex plan needs >= 1 bucket");
    if (c.sink < 0 || c.tau < 0) return fail(PIKV_ERR_INVALID_CONFIG, "SchedulerConfig: sink and tau must be >= 0");
    if (c.n_adakv_weights < 0 || c.n_adakv_weights > 8)
        return fail(PIKV_ERR_INVALID_CONFIG, "SchedulerConfig: <= 8 adakv weights");
    if (c.sched_strategy == PIKV_SCHED_QUEST)  // scheduler.cpp:199-203 (fit needs Eigen; out of scope)
        return fail(PIKV_ERR_NOT_FITTED, "score: QUEST scorer not fitted");
    if (c.sched_strategy < 0 || c.sched_strategy > PIKV_SCHED_DUO || c.router_strategy < 0 ||
        c.router_strategy > PIKV_ROUTER_HIERARCHICAL)
        return fail(PIKV_ERR_INVALID_CONFIG, "unknown strategy");
    // engine limits
    if (c.E > kMaxE) return fail(PIKV_ERR_INVALID_CONFIG, "E must be <= 256");
    if (c.k > kMaxK) return fail(PIKV_ERR_INVALID_CONFIG, "k must be <= 64");
    if (c.n_heads < 1 || c.d % c.n_heads)
        return fail(PIKV_ERR_INVALID_CONFIG, "n_heads must divide d");
    if (c.batch < 1 || c.batch > 1024) return fail(PIKV_ERR_INVALID_CONFIG, "batch must be in [1, 1024]");
    if (c.world_size < 1 || c.rank_id < 0 || c.rank_id >= c.world_size)
        return fail(PIKV_ERR_INVALID_CONFIG, "bad world_size / rank_id");
    if (c.codec < PIKV_CODEC_IDENTITY || c.codec > PIKV_CODEC_INT4)
        return fail(PIKV_ERR_INVALID_CONFIG, "unknown codec");
    if (c.route_mode != PIKV_ROUTE_EXACT && c.route_mode != PIKV_ROUTE_FAST)
        return fail(PIKV_ERR_INVALID_CONFIG, "route_mode must be PIKV_ROUTE_EXACT or PIKV_ROUTE_FAST");
    if (c.kv_dtype != PIKV_DTYPE_F32 && c.kv_dtype != PIKV_DTYPE_BF16)
        return fail(PIKV_ERR_INVALID_CONFIG, "kv_dtype must be f32 or bf16");
    const int hd = c.d / c.n_heads;
    if ((c.codec >= PIKV_CODEC_LOWRANK && c.codec <= PIKV_CODEC_PRUNE) && (c.rank < 1 || c.rank > hd))
        return fail(PIKV_ERR_INVALID_CONFIG, "codec rank must be in [1, head_dim]");
    if (c.n_layers < 0) return fail(PIKV_ERR_INVALID_CONFIG, "n_layers must be >= 0");
    if (c.d > 16384) return fail(PIKV_ERR_INVALID_CONFIG, "d must be <= 16384 (router stages q in smem)");
    // k_foldback stages one stream's global (m, 1/l) per head in shared memory
    if (8.0 * c.n_heads > 227.0 * 1024)
        return fail(PIKV_ERR_INVALID_CONFIG, "n_heads too large (fold-back: 8 H <= 227 KB)");
    if (128 + 8.0 * c.d + 5.0 * c.E * (32 * 8 + 16) > 200 * 1024)
        return fail(PIKV_ERR_INVALID_CONFIG, "router: E x d too large for the shared-memory W ring");
    return PIKV_OK;
}

// The device-side scalar config (Cfg) of a pikv_config: router and
// scheduler coefficients, and whether page aggregates are exact in any order.
static void fill_cfg(const pikv_config& c, Cfg& C) {
    C.router_strategy = c.router_strategy, C.groups = c.groups, C.stride = c.stride;
    C.alpha = c.alpha, C.lambda_miss = c.lambda_miss, C.beta_ent = c.beta_ent;
    C.bandit_step = c.bandit_step, C.bias_cap = c.bias_cap, C.load_decay = c.load_decay;
    C.sched_strategy = c.sched_strategy, C.budget_pages = c.budget_pages;
    C.page_size = c.page_size, C.sink = c.sink, C.flex_bucket = c.flex_bucket;
    C.n_adakv_weights = c.n_adakv_weights, C.n_flex_plan = c.n_flex_plan;
    C.tau = c.tau, C.lambda_freq = c.lambda_freq, C.adakv_step = c.adakv_step;
    C.target_hit = c.target_hit, C.theta0 = c.theta0, C.hit_decay = c.hit_decay;
    std::memcpy(C.adakv_weights, c.adakv_weights, sizeof(C.adakv_weights));
    std::memcpy(C.flex_plan, c.flex_plan, sizeof(C.flex_plan));
    C.unbounded_budget = c.unbounded_budget, C.head_width = c.head_width;
    C.route_mode = c.route_mode;
    // Page aggregates (scheduler.cpp:276-289) are summed in slot order.  When
    // every score is an integer multiple of 2^-10 and the page sum stays below
    // 2^42 in magnitude, each partial sum is exact, so any summation order is
    // bit-identical and the kernel may use a tree reduction.  True for LRU
    // (-recency) and SL ({0,1,2,3}) always, for LRUPlus when lambda*1024 is an
    // integer, and for Flex when every plan value is such a multiple.  With
    // step counters < 2^31: LRU |sum| <= ps 2^31 < 2^53; LRUPlus needs
    // ps (1 + |lambda|) 2^31 2^10 <= 2^53; Flex |plan| < 2^20 -> ps 2^30 <= 2^53.
    {
        auto dyadic = [](double x) { return std::isfinite(x) && std::fabs(x) < 1048576.0 &&
                                            std::nearbyint(x * 1024.0) == x * 1024.0; };
        bool ex = false;
        if (c.sched_strategy == PIKV_SCHED_LRU || c.sched_strategy == PIKV_SCHED_SL) ex = true;
        if (c.sched_strategy == PIKV_SCHED_LRU_PLUS)
            ex = dyadic(c.lambda_freq) && (double)c.page_size * (1.0 + std::fabs(c.lambda_freq)) <= 4096.0;
        if (c.sched_strategy == PIKV_SCHED_FLEX) {
            ex = true;
            for (int i = 0; i < c.n_flex_plan; ++i) ex = ex && dyadic(c.flex_plan[i]);
        }
        C.exact_sum = ex && c.page_size <= 1024 ? 1 : 0;
        C.record_agg = C.exact_sum && (c.sched_strategy == PIKV_SCHED_LRU ||
                                       c.sched_strategy == PIKV_SCHED_LRU_PLUS) ? 1 : 0;
    }
}

// attend_sms > 0: the persistent attention grid spans that many SMs (the rest
// stay free for the other micro-batch's control kernels, pikv_group)
static int engine_create(const pikv_config* cfg, int32_t cuda_device, int attend_sms, pikv_engine** out,
                         int items_per_cta = 4) {
    *out = nullptr;
    int rc = validate(*cfg);
    if (rc) return rc;
    CUDA_TRY(cudaSetDevice(cuda_device));
    auto* eng = new pikv_engine();
    eng->cfg = *cfg;
    eng->device = cuda_device;
    const pikv_config& c = *cfg;
    Dims& D = eng->D;
    D.B = c.batch;
    D.G = c.G;
    D.world = c.world_size;
    D.rank = c.rank_id;
    D.Gl = 0;
    for (int g = 0; g < c.G; ++g) D.Gl += (g % c.world_size) == c.rank_id;
    // KVStore ctor, kvstore.cpp:82-100
    int spd = c.shards_per_device > 0 ? c.shards_per_device : std::max(c.n_tok, c.n_exp) / c.G;
    if (spd < 1) spd = 1;
    const int raw_span = c.additive ? c.n_tok + c.n_exp - 1 : std::max(c.n_tok, c.n_exp);
    const int needed = (raw_span + c.G - 1) / c.G;
    D.SPD = std::max(spd, needed);
    D.R = std::max(D.Gl, 1) * D.SPD;
    D.S = c.S;
    D.H = c.n_heads;
    D.d = c.d;
    D.E = c.E;
    D.k = c.k;
    D.n_layers = c.n_layers;
    D.codec = c.codec;
    D.kv_dtype = c.kv_dtype;
    const int hd = c.d / c.n_heads;
    const bool proj = c.codec >= PIKV_CODEC_LOWRANK && c.codec <= PIKV_CODEC_PRUNE;
    D.dph = proj ? c.rank : hd;
    D.dp = D.dph * D.H;
    const bool quant = c.codec == PIKV_CODEC_INT8 || c.codec == PIKV_CODEC_INT4;
    if (c.codec == PIKV_CODEC_INT8) D.payload_bytes = D.dp, D.elem_bits = 8;
    else if (c.codec == PIKV_CODEC_INT4) D.payload_bytes = D.dp / 2, D.elem_bits = 4;
    else D.payload_bytes = D.dp * (c.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4),
         D.elem_bits = c.kv_dtype == PIKV_DTYPE_BF16 ? 16 : 32;
    D.entry_bytes = 2 * D.payload_bytes + (quant ? 8 * D.H : 0);
    D.entry_bytes = (D.entry_bytes + 15) & ~15;
    D.n_tok = c.n_tok;
    D.n_exp = c.n_exp;
    D.additive = c.additive;
    D.page_size = c.page_size;
    D.ppr_sched = (c.S - 1) / c.page_size + 2;
    if (c.S % c.page_size == 0 && c.page_size <= 256) {
        D.spg = c.page_size;
    } else {
        D.spg = 1;
        while (D.spg < 16 && c.S % (D.spg * 2) == 0) D.spg *= 2;
    }
    D.ppr = c.S / D.spg;
    int sel = 1;
    while (sel < D.SPD * D.ppr_sched) sel <<= 1;
    D.sel_stride = sel;
    D.max_cand = std::min<int64_t>(D.R, (int64_t)c.k * c.n_tok);
    D.chunk_slots = std::min(1024, ((c.S + 31) / 32) * 32);
    D.nch = (c.S + D.chunk_slots - 1) / D.chunk_slots;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
    if (const char* v = std::getenv("PIKV_ATTEND_SMS")) attend_sms = std::atoi(v);
    // attend_sms > 0: that many SMs; 0: all; < 0: all but the pipeline's
    // control-plane reserve for this layout (attend_reserve_sms)
    const int use_sms = attend_sms > 0 ? std::min(attend_sms, sms)
                        : attend_sms < 0 ? std::max(1, sms - attend_reserve_sms(D)) : sms;
    D.attend_ctas = attend_ctas_per_sm(D) * use_sms;
    {
        const char* v = std::getenv("PIKV_ITEMS");
        D.items_per_cta = v ? std::max(1, std::atoi(v)) : items_per_cta;
        const char* dc = std::getenv("PIKV_DEBUG_CTL");
        D.dbg_ctl = dc && dc[0] == '1';
        const char* da = std::getenv("PIKV_DEBUG_ATT");
        D.dbg_att = da && da[0] == '1';
        // attention work as equal static shares per CTA or ticketed items
        // (PIKV_ATT_SHARE=1 / 0 overrides).  Shares win where the attention
        // CTAs start together (c2 44.1-44.4 vs 43.1-43.5 K tokens/s, c3, c4);
        // with more than 16 streams per engine the other micro-batch's control
        // kernels delay some CTAs' start and tickets let those run less (c5,
        // 32 streams per micro-batch: 152-156 vs 151-153 K); a single stream's
        // latency-bound step builds ticketed items faster (c1: 70.2 vs 72.4 us);
        // profiles/README.md
        const char* sh = std::getenv("PIKV_ATT_SHARE");
        D.att_share = sh ? sh[0] != '0' : D.B >= 2 && D.B <= 16;
    }
    D.only_s = -1;  // scheduler kernels: all streams
    D.holes = 0;    // no arbitrary erase yet: page members are contiguous
    D.item_cap = (int64_t)D.items_per_cta * D.attend_ctas + D.B + 16;
    const int64_t total_slots = (int64_t)D.B * D.R * D.S;
    if (total_slots >= (1LL << 31)) {
        delete eng;
        return fail(PIKV_ERR_INVALID_CONFIG, "B * rings * S must be < 2^31 slots");
    }
    int64_t pool_entries = c.pool_entries > 0 ? c.pool_entries : total_slots;
    {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        const int64_t cap = (int64_t)((double)fr * 0.6 / D.entry_bytes);
        if (c.pool_entries <= 0 && pool_entries > cap) pool_entries = cap;
    }
    D.pool_pages = (pool_entries + D.spg - 1) / D.spg;
    D.pool_entries = D.pool_pages * D.spg;
    D.att_stride = std::min<int64_t>((int64_t)D.max_cand * c.S, D.pool_entries);
    D.att_cap = (int64_t)D.B * D.att_stride + 1;
    D.att_eps = std::max(1, attend_entries_per_stage(D));
    // a layout the decode-attention kernel cannot run is an error of the step
    // (run_step), not of the engine: the component API (store, router,
    // scheduler, attention over stored entries) works at any width
    if (const char* msg = attend_check(D)) eng->attend_err = std::string("attention layout: ") + msg;
    fill_cfg(*cfg, eng->C);
    {
        // measured (profiles/README.md): the per-stream control kernel wins
        // when the step is launch-bound (B = 1: +5%); from B = 16 the wide
        // multi-kernel path is as fast or faster (c2 tie, c3-c5 +2-7%)
        bool want = D.B <= 8;
        if (const char* v = std::getenv("PIKV_CONTROL")) want = v[0] == '1';
        eng->fused_control = control_supported(D, eng->C) && want;
        if (const char* v = std::getenv("PIKV_RETR_FUSED")) eng->fused_retrieval = v[0] == '1';
    }

    // exchange record layout
    ExchangeLayout& X = eng->X;
    X.o_off = 0;
    X.m_off = X.o_off + 4LL * D.H * D.dph;
    X.l_off = X.m_off + 4LL * D.H;
    X.found_off = X.l_off + 4LL * D.H;
    X.stats_off = X.found_off + 4LL * D.k;
    X.bytes_per_stream = ((X.stats_off + 16 + 15) / 16) * 16;

    cudaStreamCreateWithFlags(&eng->stream, cudaStreamNonBlocking);
    State& S = eng->S;
    const int B = D.B, E = D.E, k = D.k;
    const int64_t rings = (int64_t)B * D.R;
    bool ok = true;
    auto chk = [&](void* p) { ok = ok && p != nullptr; };
    D.route_ch = pick_route_chunk(D);
    if (eng->fused_control) control_geometry(D);  // needs route_ch
    double* W = eng->alloc<double>(router_w_elems(D));
    chk(W);
    S.W = W;
    chk(S.load = eng->alloc<double>((size_t)B * E));
    chk(S.usage = eng->alloc<uint64_t>((size_t)B * E));
    chk(S.total_usage = eng->alloc<uint64_t>(B));
    chk(S.miss = eng->alloc<uint64_t>((size_t)B * E));
    chk(S.bias = eng->alloc<double>((size_t)B * E));
    chk(S.rstep = eng->alloc<uint64_t>(B));
    chk(S.theta = eng->alloc<double>(B));
    chk(S.running_hit = eng->alloc<double>(B));
    chk(S.sstep = eng->alloc<uint64_t>(B));
    chk(S.now = eng->alloc<uint64_t>(B));
    chk(S.next_id = eng->alloc<uint64_t>(B));
    chk(S.err = eng->alloc<int32_t>(B));
    chk(S.st_inserts = eng->alloc<uint64_t>(B));
    chk(S.st_overwrites = eng->alloc<uint64_t>(B));
    chk(S.st_retrievals = eng->alloc<uint64_t>(B));
    chk(S.st_misses = eng->alloc<uint64_t>(B));
    chk(S.head = eng->alloc<int32_t>(rings));
    chk(S.live = eng->alloc<int32_t>(rings));
    chk(S.seq = eng->alloc<uint64_t>(rings));
    chk(S.page_table = eng->alloc<int32_t>(rings * D.ppr));
    chk(S.id = eng->alloc<uint64_t>(total_slots));
    chk(S.shard_seq = eng->alloc<uint64_t>(total_slots));
    chk(S.token = eng->alloc<int64_t>(total_slots));
    chk(S.expert = eng->alloc<int32_t>(total_slots));
    chk(S.insert_step = eng->alloc<uint64_t>(total_slots));
    chk(S.last_access = eng->alloc<uint64_t>(total_slots));
    chk(S.freq = eng->alloc<uint64_t>(total_slots));
    chk(S.attn_mass = eng->alloc<double>(total_slots));
    chk(S.per_layer = eng->alloc<double>((size_t)total_slots * std::max(D.n_layers, 1)));
    chk(S.has_pl = eng->alloc<uint8_t>(total_slots));
    chk(S.pool = eng->alloc<uint8_t>((size_t)D.pool_entries * D.entry_bytes));
    chk(S.page_live = eng->alloc<int32_t>(D.pool_pages));
    chk(S.free_stack = eng->alloc<int32_t>(D.pool_pages));
    chk(S.free_top = eng->alloc<int32_t>(1));
    chk(S.experts = eng->alloc<int32_t>((size_t)B * k));
    chk(S.gates = eng->alloc<double>((size_t)B * k));
    chk(S.logits = eng->alloc<double>((size_t)B * E));
    chk(S.q_attn = eng->alloc<float>((size_t)B * D.dp));
    chk(S.proj = eng->alloc<float>((size_t)2 * B * D.dp));
    chk(S.cand = eng->alloc<int32_t>((size_t)B * D.max_cand));
    chk(S.ncand = eng->alloc<int32_t>(B));
    chk(S.rec_ow = eng->alloc<EvictRec>((size_t)B * k));
    chk(S.n_ow = eng->alloc<int32_t>(B));
    chk(S.rec_ev = eng->alloc<EvictRec>((size_t)B * std::max(D.Gl, 1) * D.SPD * D.S));
    chk(S.n_ev = eng->alloc<int32_t>((size_t)B * std::max(D.Gl, 1)));
    chk(S.pages_before = eng->alloc<int32_t>((size_t)B * std::max(D.Gl, 1)));
    chk(S.pages_after = eng->alloc<int32_t>((size_t)B * std::max(D.Gl, 1)));
    chk(S.pr_cnt = eng->alloc<int32_t>(rings * D.ppr_sched));
    chk(S.pr_first = eng->alloc<int32_t>(rings * D.ppr_sched));
    chk(S.pr_sla = eng->alloc<uint64_t>(rings * D.ppr_sched));
    chk(S.pr_sf = eng->alloc<uint64_t>(rings * D.ppr_sched));
    chk(S.pages_live = eng->alloc<int32_t>((size_t)B * std::max(D.Gl, 1)));
    chk(S.pg_agg = eng->alloc<double>(rings * D.ppr_sched));
    chk(S.pg_oldest = eng->alloc<uint64_t>(rings * D.ppr_sched));
    chk(S.pg_cnt = eng->alloc<int32_t>(rings * D.ppr_sched));
    chk(S.sel_idx = eng->alloc<int32_t>((size_t)B * std::max(D.Gl, 1) * D.sel_stride));
    const size_t nchunk = (size_t)B * D.max_cand * D.nch;
    chk(S.chunk_cnt = eng->alloc<int32_t>(nchunk));
    chk(S.chunk_off = eng->alloc<int32_t>(2 * nchunk));  // int32 offsets / 64-bit look-back words
    chk(S.found = eng->alloc<int32_t>((size_t)B * k));
    chk(S.att_cnt = eng->alloc<int32_t>(B));
    chk(S.att_slot = eng->alloc<int32_t>(D.att_cap));
    chk(S.att_entry = eng->alloc<int32_t>(D.att_cap));
    chk(S.scores = eng->alloc<float>((size_t)D.att_cap * D.H));
    chk(S.item_stream = eng->alloc<int32_t>(D.item_cap));
    chk(S.item_begin = eng->alloc<int32_t>(D.item_cap));
    chk(S.item_end = eng->alloc<int32_t>(D.item_cap));
    chk(S.n_items = eng->alloc<int32_t>(2));  // [count, attention's dynamic item ticket]
    chk(S.item_first = eng->alloc<int32_t>(B + 1));
    chk(S.cta_first = eng->alloc<int32_t>((size_t)D.attend_ctas + 1 + B + 1));  // + per-stream unit scratch
    chk(S.part_m = eng->alloc<float>((size_t)D.item_cap * D.H));
    chk(S.part_l = eng->alloc<float>((size_t)D.item_cap * D.H));
    chk(S.part_o = eng->alloc<float>((size_t)D.item_cap * D.H * D.dph));
    chk(S.exchange = eng->alloc<uint8_t>((size_t)B * X.bytes_per_stream));
    chk(S.gM = eng->alloc<float>((size_t)B * D.H));
    chk(S.gL = eng->alloc<float>((size_t)B * D.H));
    chk(S.summary = eng->alloc<pikv_step_summary>(B));
    chk(S.dbg = eng->alloc<long long>(64 + 8 * (size_t)B + 8 * (size_t)D.attend_ctas));
    chk(S.done_ctr = eng->alloc<unsigned>(1));
    chk(S.ctl_ctr = eng->alloc<unsigned>(4));
    const size_t in_elem = c.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4;
    // q, k, v staging: one allocation, packed back to back
    chk(eng->in_q = eng->alloc<uint8_t>((size_t)3 * B * D.d * in_elem));
    eng->in_k = (uint8_t*)eng->in_q + (size_t)B * D.d * in_elem;
    eng->in_v = (uint8_t*)eng->in_k + (size_t)B * D.d * in_elem;
    chk(eng->in_sal = eng->alloc<double>((size_t)B * std::max(D.n_layers, 1)));
    chk(eng->out_y = eng->alloc<float>((size_t)B * D.dp));
    if (!ok) {
        pikv_engine_destroy(eng);
        return fail(PIKV_ERR_OUT_OF_MEMORY, "cudaMalloc failed (reduce pool_entries / batch / S)");
    }
    // initial state
    cudaStream_t st = eng->stream;
    {
        const auto w = pack_router_w(D, router_matrix(E, D.d, c.seed ^ kRouterSalt).data());
        CUDA_TRY(cudaMemcpy(W, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
    }
    std::vector<double> theta(B, c.theta0);  // SchedulerState::init, scheduler.cpp:73-80
    CUDA_TRY(cudaMemcpyAsync(S.theta, theta.data(), sizeof(double) * B, cudaMemcpyHostToDevice, st));
    std::vector<uint64_t> ones(B, 1);  // kvstore.hpp:157 next_id_ = 1
    CUDA_TRY(cudaMemcpyAsync(S.next_id, ones.data(), sizeof(uint64_t) * B, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(S.load, 0, sizeof(double) * B * E, st));
    CUDA_TRY(cudaMemsetAsync(S.usage, 0, sizeof(uint64_t) * B * E, st));
    CUDA_TRY(cudaMemsetAsync(S.total_usage, 0, sizeof(uint64_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.miss, 0, sizeof(uint64_t) * B * E, st));
    CUDA_TRY(cudaMemsetAsync(S.bias, 0, sizeof(double) * B * E, st));
    CUDA_TRY(cudaMemsetAsync(S.rstep, 0, sizeof(uint64_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.running_hit, 0, sizeof(double) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.sstep, 0, sizeof(uint64_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.now, 0, sizeof(uint64_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.err, 0, sizeof(int32_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.st_inserts, 0, sizeof(uint64_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.st_overwrites, 0, sizeof(uint64_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.st_retrievals, 0, sizeof(uint64_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.st_misses, 0, sizeof(uint64_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.head, 0, sizeof(int32_t) * rings, st));
    CUDA_TRY(cudaMemsetAsync(S.live, 0, sizeof(int32_t) * rings, st));
    CUDA_TRY(cudaMemsetAsync(S.seq, 0, sizeof(uint64_t) * rings, st));
    CUDA_TRY(cudaMemsetAsync(S.page_table, 0xff, sizeof(int32_t) * rings * D.ppr, st));
    CUDA_TRY(cudaMemsetAsync(S.id, 0, sizeof(uint64_t) * total_slots, st));
    CUDA_TRY(cudaMemsetAsync(S.attn_mass, 0, sizeof(double) * total_slots, st));
    CUDA_TRY(cudaMemsetAsync(S.has_pl, 0, total_slots, st));
    // never-written slots read back as zeros (readback of whole slot arrays)
    CUDA_TRY(cudaMemsetAsync(S.shard_seq, 0, sizeof(uint64_t) * total_slots, st));
    CUDA_TRY(cudaMemsetAsync(S.token, 0, sizeof(int64_t) * total_slots, st));
    CUDA_TRY(cudaMemsetAsync(S.expert, 0, sizeof(int32_t) * total_slots, st));
    CUDA_TRY(cudaMemsetAsync(S.insert_step, 0, sizeof(uint64_t) * total_slots, st));
    CUDA_TRY(cudaMemsetAsync(S.last_access, 0, sizeof(uint64_t) * total_slots, st));
    CUDA_TRY(cudaMemsetAsync(S.freq, 0, sizeof(uint64_t) * total_slots, st));
    CUDA_TRY(cudaMemsetAsync(S.per_layer, 0, sizeof(double) * total_slots * std::max(D.n_layers, 1), st));
    CUDA_TRY(cudaMemsetAsync(S.pr_cnt, 0, sizeof(int32_t) * rings * D.ppr_sched, st));
    CUDA_TRY(cudaMemsetAsync(S.pages_live, 0, sizeof(int32_t) * B * std::max(D.Gl, 1), st));
    CUDA_TRY(cudaMemsetAsync(S.pr_first, 0, sizeof(int32_t) * rings * D.ppr_sched, st));
    CUDA_TRY(cudaMemsetAsync(S.pr_sla, 0, sizeof(uint64_t) * rings * D.ppr_sched, st));
    CUDA_TRY(cudaMemsetAsync(S.pr_sf, 0, sizeof(uint64_t) * rings * D.ppr_sched, st));
    CUDA_TRY(cudaMemsetAsync(S.n_ow, 0, sizeof(int32_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.n_ev, 0, sizeof(int32_t) * B * std::max(D.Gl, 1), st));
    CUDA_TRY(cudaMemsetAsync(S.pages_before, 0, sizeof(int32_t) * B * std::max(D.Gl, 1), st));
    CUDA_TRY(cudaMemsetAsync(S.pages_after, 0, sizeof(int32_t) * B * std::max(D.Gl, 1), st));
    CUDA_TRY(cudaMemsetAsync(S.summary, 0, sizeof(pikv_step_summary) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.n_items, 0, 2 * sizeof(int32_t), st));
    CUDA_TRY(cudaMemsetAsync(S.item_first, 0, sizeof(int32_t) * (B + 1), st));
    CUDA_TRY(cudaMemsetAsync(S.att_cnt, 0, sizeof(int32_t) * B, st));
    CUDA_TRY(cudaMemsetAsync(S.done_ctr, 0, sizeof(unsigned), st));
    CUDA_TRY(cudaMemsetAsync(S.ctl_ctr, 0, 4 * sizeof(unsigned), st));
    CUDA_TRY(cudaMemsetAsync(S.chunk_off, 0, 2 * sizeof(int32_t) * nchunk, st));
    std::vector<int32_t> stack(D.pool_pages);
    for (int64_t i = 0; i < D.pool_pages; ++i) stack[i] = (int32_t)(D.pool_pages - 1 - i);
    CUDA_TRY(cudaMemcpyAsync(S.free_stack, stack.data(), sizeof(int32_t) * D.pool_pages,
                             cudaMemcpyHostToDevice, st));
    const int32_t top = (int32_t)D.pool_pages;
    CUDA_TRY(cudaMemcpyAsync(S.free_top, &top, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(eng->in_sal, 0, sizeof(double) * B * std::max(D.n_layers, 1), st));
    CUDA_TRY(cudaStreamSynchronize(st));
    S.basis = nullptr, S.cbias = nullptr, S.kept = nullptr;
    *out = eng;
    return PIKV_OK;
}

int pikv_engine_create(const pikv_config* cfg, int32_t cuda_device, pikv_engine** out) {
    return engine_create(cfg, cuda_device, 0, out);
}

int pikv_engine_destroy(pikv_engine* eng) {
    if (!eng) return PIKV_OK;
    cudaSetDevice(eng->device);
    if (eng->stream) cudaStreamSynchronize(eng->stream);
    eng->drop_graphs();
    for (auto e : eng->ev) cudaEventDestroy(e);
    for (void* p : eng->allocs) cudaFree(p);
    for (auto e : {eng->ev_fork, eng->ev_kv, eng->ev_y, eng->ev_join})
        if (e) cudaEventDestroy(e);
    if (eng->side) cudaStreamDestroy(eng->side);
    if (eng->host_ge) cudaGraphExecDestroy(eng->host_ge);
    if (eng->host_g) cudaGraphDestroy(eng->host_g);
    if (eng->host_ph) cudaFreeHost(eng->host_ph);
    if (eng->bulk_buf) cudaFree(eng->bulk_buf);
    if (eng->rb_buf) cudaFree(eng->rb_buf);
    if (eng->gathered) cudaFree(eng->gathered);
    if (eng->comm && eng->own_comm) ncclCommDestroy(eng->comm);
    if (eng->bulk_stage) cudaFree(eng->bulk_stage);
    if (eng->stream) cudaStreamDestroy(eng->stream);
    delete eng;
    return PIKV_OK;
}

void* pikv_engine_stream(pikv_engine* eng) { return (void*)eng->stream; }

int pikv_set_router_matrix_host(pikv_engine* eng, const double* w_r) {
    const auto w = pack_router_w(eng->D, w_r);
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    CUDA_TRY(cudaMemcpy((void*)eng->S.W, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
    return PIKV_OK;
}

int pikv_set_codec_host(pikv_engine* eng, const float* basis, const float* bias,
                        const int32_t* kept) {
    const Dims& D = eng->D;
    const int hd = D.d / D.H, r = D.dph;
    auto up = [&](const void* src, size_t bytes) -> void* {
        void* p = eng->alloc<uint8_t>(bytes);
        if (p) cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice);
        return p;
    };
    if (basis) eng->S.basis = (const float*)up(basis, sizeof(float) * (size_t)D.H * r * hd);
    if (bias) eng->S.cbias = (const float*)up(bias, sizeof(float) * (size_t)D.d);
    if (kept) {
        for (int i = 0; i < D.H * r; ++i)
            if (kept[i] < 0 || kept[i] >= hd) return fail(PIKV_ERR_INVALID_ARGUMENT, "kept index out of range");
        eng->S.kept = (const int32_t*)up(kept, sizeof(int32_t) * (size_t)D.H * r);
    }
    cudaStreamSynchronize(eng->stream);
    eng->invalidate();  // captured kernels hold the old pointers
    return PIKV_OK;
}

static int codec_ready(pikv_engine* eng) {
    if (!eng->attend_err.empty()) return fail(PIKV_ERR_INVALID_CONFIG, eng->attend_err);
    const int c = eng->D.codec;
    if ((c == PIKV_CODEC_LOWRANK || c == PIKV_CODEC_LORAPLUS) && !eng->S.basis)
        return fail(PIKV_ERR_NOT_FITTED, "codec basis not set (pikv_set_codec_host)");
    if (c == PIKV_CODEC_LORAPLUS && !eng->S.cbias)
        return fail(PIKV_ERR_NOT_FITTED, "LoRAPlus bias not set");
    if (c == PIKV_CODEC_PRUNE && !eng->S.kept) return fail(PIKV_ERR_NOT_FITTED, "Prune kept set not set");
    return PIKV_OK;
}

// Kernels timed in profiling mode (one event after each).
constexpr int kPhases = 12;  // route insert sched_pages sched_select retr_count retr_scan
                             // retr_write attend combine finish_merge foldback feedback
constexpr int kProfSteps = 512;

static void mark(pikv_engine* eng, int phase) {
    if (eng->cur < 0) return;
    cudaEventRecord(eng->ev[eng->cur + phase], eng->stream);
}

// Parts of one step, enqueued together or separately (the micro-batch
// pipeline of pikv_group interleaves them across engines):
//   CTL    route -> insert -> evict -> retrieve (latency-bound control plane)
//   ATTEND decode attention (HBM-bound)
//   MERGE  combine (y)
//   FOLD   [finish merge] -> fold-back + feedback
enum : unsigned { kPartCtl = 1u, kPartAttend = 2u, kPartMerge = 4u, kPartFold = 8u, kPartTail = 12u,
                  kPartAll = 15u };

// The step's launch sequence (pipeline.cpp:213-351 ordering).
// kv_ready: if set, waited on (stream-ordered) right before the first
// kernel that reads k/v; y_ready: if set, recorded as soon as y is written.
static int enqueue_local(pikv_engine* eng, const void* q, const void* k, const void* v,
                         const double* sal, bool attend, float* y, bool q_f64 = false,
                         cudaEvent_t kv_ready = nullptr, cudaEvent_t y_ready = nullptr,
                         unsigned parts = kPartAll) {
    Dims D = eng->D;
    D.q_f64 = q_f64 ? 1 : 0;
    const State& S = eng->S;
    cudaStream_t st = eng->stream;
    int n = 0;
    if (parts & kPartCtl) {
        eng->cur = -1;
        if (eng->profiling && eng->prof_steps < kProfSteps) eng->cur = eng->prof_steps++ * (kPhases + 1);
    }
    mark(eng, 0);
    const bool proj = D.codec == PIKV_CODEC_LOWRANK || D.codec == PIKV_CODEC_LORAPLUS;
    if (!(parts & kPartCtl)) {
    } else if (eng->fused_control) {
        // one CTA per stream runs route -> insert -> evict -> retrieve
        if (kv_ready) cudaStreamWaitEvent(st, kv_ready, 0);
        if (proj) launch_project(D, S, q, k, v, st), ++n;
        launch_control(D, eng->C, S, q, k, v, sal, st), ++n;
        for (int p = 1; p <= 7; ++p) mark(eng, p);
    } else {
    launch_route(D, eng->C, S, q, st), ++n;
    mark(eng, 1);
    // a rank that owns no device still issues entry ids (k_insert) and joins
    // the merge with an empty record
    if (kv_ready) cudaStreamWaitEvent(st, kv_ready, 0);  // k/v arrive while routing
    if (proj) launch_project(D, S, q, k, v, st), ++n;  // q, k, v of all streams in one pass
    launch_insert(D, eng->C, S, q, k, v, sal, st), ++n;
    mark(eng, 2);
    const bool sched = D.Gl > 0 && !eng->C.unbounded_budget;
    // LRU/LRU+: both kernels exit at once for devices whose live-page counter
    // is within budget (single-CTA key computation measured slower: 32 vs 27 us)
    if (sched) launch_sched_pages(D, eng->C, S, st), ++n;
    mark(eng, 3);
    if (sched) launch_sched_select(D, eng->C, S, st), ++n;
    mark(eng, 4);
    if (eng->fused_retrieval) {
        launch_retr_fused(D, eng->C, S, st), ++n;
        mark(eng, 5), mark(eng, 6);
    } else {
        launch_retr_count(D, S, st), ++n;
        mark(eng, 5);
        launch_retr_scan(D, eng->C, S, st), ++n;
        mark(eng, 6);
        launch_retr_write(D, S, st), ++n;
    }
    mark(eng, 7);
    }
    if ((parts & kPartAttend) && attend && D.Gl > 0) launch_attend(D, S, st), ++n;
    mark(eng, 8);
    if (parts & kPartMerge) {
        const int direct = !eng->exchange_path();  // single rank: combine writes y
        if (attend || !direct) launch_combine(D, eng->C, S, eng->X, y, direct, attend, st), ++n;
        if (y_ready) cudaEventRecord(y_ready, st);
    }
    mark(eng, 9);
    CUDA_TRY(cudaGetLastError());
    eng->kernels_per_step = n;
    return PIKV_OK;
}

static int enqueue_finish(pikv_engine* eng, const uint8_t* gathered, float* y, bool attend,
                          int granks) {
    const bool xp = eng->exchange_path();
    if (xp) launch_finish_merge(eng->D, eng->C, eng->S, eng->X, gathered, y, granks, eng->stream);
    // y is final here (the cross-rank merge wrote it): a host-path group step
    // starts its D2H while the fold-back runs
    // (an external event node when captured: waited on outside the graph)
    if (xp && eng->y_final_event) cudaEventRecordWithFlags(eng->y_final_event, eng->stream, cudaEventRecordExternal);
    mark(eng, 10);
    // fold-back + feedback in one launch (last CTA runs the feedback); the
    // prefill (no attention) launches the feedback alone
    if (attend) launch_foldback(eng->D, eng->C, eng->S, eng->stream);
    mark(eng, 11);
    if (!attend) launch_feedback(eng->D, eng->C, eng->S, eng->stream);
    mark(eng, 12);
    eng->cur = -1;
    eng->kernels_per_step += 1 + (xp ? 1 : 0);
    CUDA_TRY(cudaGetLastError());
    return PIKV_OK;
}

// emb != nullptr: the step starts from the tokens' embeddings (Engine::step,
// pipeline.cpp:222): the QueryEncoder kernel writes q (fp64) and the stored
// K/V, then the step proceeds on them.
static int enqueue_step(pikv_engine* eng, const double* emb, const void* q, const void* k, const void* v,
                        const double* sal, float* y, bool attend, unsigned parts = kPartAll) {
    if (emb && (parts & kPartCtl)) {
        launch_encode(eng->D, eng->enc_wt, emb, eng->q64, eng->in_k, eng->in_v, eng->stream);
    }
    if (emb) q = eng->q64, k = eng->in_k, v = eng->in_v;
    int rc = enqueue_local(eng, q, k, v, sal, attend, y, emb != nullptr, nullptr, nullptr, parts);
    if (!rc && (parts & kPartFold)) {
        if (eng->comm) {  // the one exchange of the path: all-gather of the LSE records
            const size_t nb = (size_t)eng->D.B * eng->X.bytes_per_stream;
            const ncclResult_t r = ncclAllGather(eng->S.exchange, eng->gathered, nb, ncclUint8, eng->comm, eng->stream);
            if (r != ncclSuccess) return fail(PIKV_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
            rc = enqueue_finish(eng, eng->gathered, y, attend, eng->D.world);
        } else {
            rc = enqueue_finish(eng, eng->S.exchange, y, attend, 1);
        }
    }
    if (emb && (parts & kPartCtl)) eng->kernels_per_step += (eng->D.B + 63) / 64;
    return rc;
}

static int run_step(pikv_engine* eng, const void* q, const void* k, const void* v,
                    const double* sal, float* y, bool attend, const double* emb = nullptr,
                    unsigned parts = kPartAll) {
    int rc = codec_ready(eng);
    if (rc) return rc;
    if (eng->D.world != 1 && !eng->comm)
        return fail(PIKV_ERR_INVALID_ARGUMENT,
                    "world_size > 1: attach NCCL (pikv_engine_attach_nccl) or use pikv_step_local / pikv_step_finish");
    cudaSetDevice(eng->device);
    static const bool att_eager = [] {  // A/B experiments only: attention part launched without a graph
        const char* v = std::getenv("PIKV_ATT_EAGER");
        return v && v[0] == '1';
    }();
    const bool use_graph = (eng->warmed_parts & parts) == parts && !eng->profiling &&
                           !(att_eager && parts == kPartAttend);
    if (!use_graph) {
        rc = enqueue_step(eng, emb, q, k, v, sal, y, attend, parts);
        if (rc) return rc;
        eng->warmed_parts |= parts;  // first eager pass sets kernel attributes
        eng->warmed = eng->warmed_parts == kPartAll;
        eng->launches += eng->kernels_per_step;
        return PIKV_OK;
    }
    auto key = std::make_tuple(emb ? (const void*)emb : q, k, v, (const void*)sal, (void*)y,
                               (attend ? 1 : 0) + (emb ? 2 : 0) + (int)(parts << 2));
    auto it = eng->graphs.find(key);
    if (it == eng->graphs.end()) {
        cudaGraph_t g;
        CUDA_TRY(cudaStreamBeginCapture(eng->stream, cudaStreamCaptureModeThreadLocal));
        rc = enqueue_step(eng, emb, q, k, v, sal, y, attend, parts);
        cudaError_t ce = cudaStreamEndCapture(eng->stream, &g);
        if (rc) return rc;
        if (ce != cudaSuccess) return fail(PIKV_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ce));
        cudaGraphExec_t ge;
        CUDA_TRY(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
        if (eng->graphs.size() > 16) eng->drop_graphs();
        it = eng->graphs.emplace(key, pikv_engine::Captured{ge, eng->kernels_per_step}).first;
    }
    CUDA_TRY(cudaGraphLaunch(it->second.ge, eng->stream));
    eng->launches += it->second.kernels;
    return PIKV_OK;
}

int pikv_step(pikv_engine* eng, const void* q, const void* k, const void* v, const double* saliency,
              float* y_out) {
    return run_step(eng, q, k, v, saliency, y_out, true);
}

// QueryEncoder weights on the device as W^T [3][d][d] (k_encode layout).
static int upload_encoder(pikv_engine* eng, const double* wq, const double* wk, const double* wv) {
    const int d = eng->D.d;
    const size_t dd = (size_t)d * d;
    if (!eng->enc_wt) {
        eng->enc_wt = eng->alloc<double>(3 * dd);
        eng->q64 = eng->alloc<double>((size_t)eng->D.B * d);
        eng->in_emb = eng->alloc<double>((size_t)eng->D.B * d);
        if (!eng->enc_wt || !eng->q64 || !eng->in_emb)
            return fail(PIKV_ERR_OUT_OF_MEMORY, "cudaMalloc failed (QueryEncoder weights)");
    }
    std::vector<double> t(dd);
    const double* w3[3] = {wq, wk, wv};
    for (int m = 0; m < 3; ++m) {
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j) t[(size_t)j * d + i] = w3[m][(size_t)i * d + j];
        CUDA_TRY(cudaMemcpy(eng->enc_wt + (size_t)m * dd, t.data(), sizeof(double) * dd, cudaMemcpyHostToDevice));
    }
    return PIKV_OK;
}

static int encoder_ready(pikv_engine* eng) {
    if (eng->enc_wt) return PIKV_OK;
    const int d = eng->D.d;
    const size_t dd = (size_t)d * d;
    // QueryEncoder(d, seed ^ kEncoderSalt), pipeline.cpp:29-36, 89
    const auto w = reference_normals(3 * dd, d, eng->cfg.seed ^ kEncoderSalt);
    return upload_encoder(eng, w.data(), w.data() + dd, w.data() + 2 * dd);
}

int pikv_set_encoder_host(pikv_engine* eng, const double* w_query, const double* w_key,
                          const double* w_value) {
    if (!w_query || !w_key || !w_value) return fail(PIKV_ERR_INVALID_ARGUMENT, "encoder matrix is NULL");
    cudaSetDevice(eng->device);
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    return upload_encoder(eng, w_query, w_key, w_value);
}

int pikv_step_embed(pikv_engine* eng, const double* emb, const double* saliency, float* y_out) {
    if (!emb) return fail(PIKV_ERR_INVALID_ARGUMENT, "embedding is NULL");
    cudaSetDevice(eng->device);
    int rc = encoder_ready(eng);
    if (rc) return rc;
    return run_step(eng, nullptr, nullptr, nullptr, saliency, y_out, true, emb);
}

int pikv_step_embed_host(pikv_engine* eng, const double* emb, const double* saliency, float* y_out) {
    if (!emb) return fail(PIKV_ERR_INVALID_ARGUMENT, "embedding is NULL");
    const Dims& D = eng->D;
    cudaSetDevice(eng->device);
    int rc = encoder_ready(eng);
    if (rc) return rc;
    cudaStream_t st = eng->stream;
    CUDA_TRY(cudaMemcpyAsync(eng->in_emb, emb, sizeof(double) * D.B * D.d, cudaMemcpyHostToDevice, st));
    const double* sal = nullptr;
    if (saliency && D.n_layers > 0) {
        CUDA_TRY(cudaMemcpyAsync(eng->in_sal, saliency, sizeof(double) * D.B * D.n_layers,
                                 cudaMemcpyHostToDevice, st));
        sal = eng->in_sal;
    }
    rc = run_step(eng, nullptr, nullptr, nullptr, sal, eng->out_y, true, eng->in_emb);
    if (rc) return rc;
    if (y_out)
        CUDA_TRY(cudaMemcpyAsync(y_out, eng->out_y, sizeof(float) * D.B * D.dp, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return PIKV_OK;
}

static bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// The whole host-buffer step as one graph launch (see pikv_engine::host_g).
static int step_host_graph(pikv_engine* eng, const void* q, float* y_out, size_t n, size_t ny) {
    cudaStream_t st = eng->stream;
    if (!eng->host_ge) {
        if (!eng->host_ph) CUDA_TRY(cudaHostAlloc(&eng->host_ph, 3 * n + ny, cudaHostAllocDefault));
        uint8_t* ph = (uint8_t*)eng->host_ph;
        if (!eng->side) {
            CUDA_TRY(cudaStreamCreateWithFlags(&eng->side, cudaStreamNonBlocking));
            for (auto* e : {&eng->ev_fork, &eng->ev_kv, &eng->ev_y, &eng->ev_join})
                CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        cudaGraph_t g = nullptr;
        // main: H2D q -> route -> (wait k/v) insert ... combine -> (y ready) fold-back
        // side: H2D k, v during routing; D2H y during the fold-back
        CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        cudaEventRecord(eng->ev_fork, st);
        cudaStreamWaitEvent(eng->side, eng->ev_fork, 0);
        cudaMemcpyAsync(eng->in_k, ph + n, 2 * n, cudaMemcpyHostToDevice, eng->side);
        cudaEventRecord(eng->ev_kv, eng->side);
        cudaMemcpyAsync(eng->in_q, ph, n, cudaMemcpyHostToDevice, st);
        int rc = enqueue_local(eng, eng->in_q, eng->in_k, eng->in_v, nullptr, true, eng->out_y, false,
                               eng->ev_kv, eng->ev_y);
        cudaStreamWaitEvent(eng->side, eng->ev_y, 0);
        cudaMemcpyAsync(ph + 3 * n, eng->out_y, ny, cudaMemcpyDeviceToHost, eng->side);
        cudaEventRecord(eng->ev_join, eng->side);
        if (!rc) rc = enqueue_finish(eng, eng->S.exchange, eng->out_y, true, 1);
        cudaStreamWaitEvent(st, eng->ev_join, 0);
        const cudaError_t ce = cudaStreamEndCapture(st, &g);
        if (rc) return rc;
        if (ce != cudaSuccess) return fail(PIKV_ERR_CUDA, std::string("host capture: ") + cudaGetErrorString(ce));
        size_t nn = 0;
        CUDA_TRY(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &nn));
        for (auto nd : nodes) {
            cudaGraphNodeType t;
            CUDA_TRY(cudaGraphNodeGetType(nd, &t));
            if (t != cudaGraphNodeTypeMemcpy) continue;
            cudaMemcpy3DParms p{};
            CUDA_TRY(cudaGraphMemcpyNodeGetParams(nd, &p));
            if (p.kind == cudaMemcpyDeviceToHost) eng->host_d2h = nd;
            else if (p.dstPtr.ptr == eng->in_q) eng->host_h2d = nd;
            else if (p.dstPtr.ptr == eng->in_k) eng->host_h2d_kv = nd;
        }
        if (!eng->host_h2d || !eng->host_h2d_kv || !eng->host_d2h) {
            cudaGraphDestroy(g);
            return fail(PIKV_ERR_CUDA, "host capture: memcpy nodes not found");
        }
        CUDA_TRY(cudaGraphInstantiate(&eng->host_ge, g, 0));
        eng->host_g = g;
    }
    CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(eng->host_ge, eng->host_h2d, eng->in_q, q, n,
                                                cudaMemcpyHostToDevice));
    CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(eng->host_ge, eng->host_h2d_kv, eng->in_k,
                                                (const uint8_t*)q + n, 2 * n, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(eng->host_ge, eng->host_d2h, y_out, eng->out_y, ny,
                                                cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaGraphLaunch(eng->host_ge, st));
    eng->launches += eng->kernels_per_step;
    CUDA_TRY(cudaStreamSynchronize(st));
    return PIKV_OK;
}

int pikv_step_host(pikv_engine* eng, const void* q, const void* k, const void* v,
                   const double* saliency, float* y_out) {
    const Dims& D = eng->D;
    const size_t n = (size_t)D.B * D.d * (D.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4);
    cudaStream_t st = eng->stream;
    const uint8_t* hq = (const uint8_t*)q;
    const bool packed = (const uint8_t*)k == hq + n && (const uint8_t*)v == hq + 2 * n;
    if (packed && y_out && !(saliency && D.n_layers > 0) && !eng->exchange_path() && eng->warmed && !eng->profiling &&
        codec_ready(eng) == PIKV_OK && is_pinned(q) && is_pinned(y_out)) {
        cudaSetDevice(eng->device);
        return step_host_graph(eng, q, y_out, n, sizeof(float) * D.B * D.dp);
    }
    if ((const uint8_t*)k == hq + n && (const uint8_t*)v == hq + 2 * n) {
        // q, k, v packed back to back on the host: one transfer into the
        // (equally packed) staging buffers
        CUDA_TRY(cudaMemcpyAsync(eng->in_q, q, 3 * n, cudaMemcpyHostToDevice, st));
    } else {
        CUDA_TRY(cudaMemcpyAsync(eng->in_q, q, n, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(eng->in_k, k, n, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(eng->in_v, v, n, cudaMemcpyHostToDevice, st));
    }
    const double* sal = nullptr;
    if (saliency && D.n_layers > 0) {
        CUDA_TRY(cudaMemcpyAsync(eng->in_sal, saliency, sizeof(double) * D.B * D.n_layers,
                                 cudaMemcpyHostToDevice, st));
        sal = eng->in_sal;
    }
    int rc = run_step(eng, eng->in_q, eng->in_k, eng->in_v, sal, eng->out_y, true);
    if (rc) return rc;
    if (y_out)
        CUDA_TRY(cudaMemcpyAsync(y_out, eng->out_y, sizeof(float) * D.B * D.dp, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return PIKV_OK;
}

// ---- multi-GPU: NCCL inside the library ------------------------------------
int pikv_nccl_unique_id(uint8_t* id_out) {
    if (!id_out) return fail(PIKV_ERR_INVALID_ARGUMENT, "id_out is NULL");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(PIKV_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == PIKV_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
    return PIKV_OK;
}

static int use_comm(pikv_engine* eng, ncclComm_t comm, bool own) {
    int n = 0, r = 0;
    if (comm) {
        ncclResult_t e = ncclCommCount(comm, &n);
        if (e == ncclSuccess) e = ncclCommUserRank(comm, &r);
        if (e != ncclSuccess) return fail(PIKV_ERR_NCCL, std::string("nccl comm: ") + ncclGetErrorString(e));
        if (n != eng->D.world || r != eng->D.rank)
            return fail(PIKV_ERR_INVALID_CONFIG, "NCCL communicator size / rank != world_size / rank_id");
    }
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    if (eng->comm && eng->own_comm) ncclCommDestroy(eng->comm);
    eng->comm = comm, eng->own_comm = own && comm;
    if (comm && !eng->gathered) {
        CUDA_TRY(cudaMalloc(&eng->gathered, (size_t)eng->D.world * eng->D.B * eng->X.bytes_per_stream));
    }
    eng->invalidate();  // the captured steps change shape (exchange, all-gather, finish)
    eng->warmed_parts = 0, eng->warmed = false;
    return PIKV_OK;
}

int pikv_engine_attach_nccl(pikv_engine* eng, const uint8_t* id) {
    if (!eng || !id) return fail(PIKV_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaSetDevice(eng->device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    const ncclResult_t r = ncclCommInitRank(&comm, eng->D.world, uid, eng->D.rank);
    if (r != ncclSuccess) return fail(PIKV_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    return use_comm(eng, comm, true);
}

int pikv_engine_set_nccl_comm(pikv_engine* eng, void* nccl_comm) {
    if (!eng) return fail(PIKV_ERR_INVALID_ARGUMENT, "engine is NULL");
    cudaSetDevice(eng->device);
    return use_comm(eng, (ncclComm_t)nccl_comm, false);
}

int64_t pikv_local_attended(pikv_engine* eng) {
    cudaStreamSynchronize(eng->stream);
    std::vector<int32_t> cnt(eng->D.B), err(eng->D.B);
    cudaMemcpy(cnt.data(), eng->S.att_cnt, 4 * (size_t)eng->D.B, cudaMemcpyDeviceToHost);
    cudaMemcpy(err.data(), eng->S.err, 4 * (size_t)eng->D.B, cudaMemcpyDeviceToHost);
    int64_t n = 0;
    for (int s = 0; s < eng->D.B; ++s) n += err[s] ? 0 : cnt[s];
    return n;
}

int64_t pikv_exchange_bytes(pikv_engine* eng) { return (int64_t)eng->D.B * eng->X.bytes_per_stream; }

int pikv_step_local(pikv_engine* eng, const void* q, const void* k, const void* v,
                    const double* saliency, void** exchange_out) {
    int rc = codec_ready(eng);
    if (rc) return rc;
    cudaSetDevice(eng->device);
    rc = enqueue_local(eng, q, k, v, saliency, true, nullptr);
    if (rc) return rc;
    eng->launches += eng->kernels_per_step;
    if (exchange_out) *exchange_out = eng->S.exchange;
    return PIKV_OK;
}

int pikv_step_finish(pikv_engine* eng, const void* gathered, float* y_out) {
    cudaSetDevice(eng->device);
    int rc = enqueue_finish(eng, (const uint8_t*)gathered, y_out, true, eng->D.world);
    if (rc) return rc;
    eng->launches += 2;  // finish_merge, foldback(+feedback)
    return PIKV_OK;
}

int pikv_fill_synthetic(pikv_engine* eng, void* q, void* k, void* v, uint64_t seed) {
    launch_synth(eng->D, q, k, v, seed, 0, eng->stream);
    CUDA_TRY(cudaGetLastError());
    return PIKV_OK;
}

int pikv_prefill_synthetic(pikv_engine* eng, int64_t tokens, uint64_t seed) {
    int rc = codec_ready(eng);
    if (rc) return rc;
    cudaSetDevice(eng->device);
    const bool was_prof = eng->profiling;
    eng->profiling = false;
    for (int64_t t = 0; t < tokens; ++t) {
        launch_synth(eng->D, eng->in_q, eng->in_k, eng->in_v, seed, (uint64_t)t, eng->stream);
        if (eng->D.world == 1 || eng->comm) {  // the full step (with the collective when sharded)
            rc = run_step(eng, eng->in_q, eng->in_k, eng->in_v, nullptr, nullptr, false);
        } else {
            rc = enqueue_local(eng, eng->in_q, eng->in_k, eng->in_v, nullptr, false, nullptr);
            // synthetic prefill without a collective: each rank finishes on its own
            // record (hit/miss counts then see only local shards)
            if (!rc) rc = enqueue_finish(eng, eng->S.exchange, nullptr, false, 1);
        }
        if (rc) {
            eng->profiling = was_prof;
            return rc;
        }
        if ((t & 1023) == 1023) CUDA_TRY(cudaStreamSynchronize(eng->stream));
    }
    eng->profiling = was_prof;
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    return PIKV_OK;
}

int pikv_sync(pikv_engine* eng) {
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    std::vector<int32_t> err(eng->D.B);
    CUDA_TRY(cudaMemcpy(err.data(), eng->S.err, sizeof(int32_t) * eng->D.B, cudaMemcpyDeviceToHost));
    for (int s = 0; s < eng->D.B; ++s)
        if (err[s]) return fail(err[s], "stream " + std::to_string(s) + " failed on device (code " +
                                            std::to_string(err[s]) + ")");
    return PIKV_OK;
}

// ---------------------------------------------------------------------------
// readback
// ---------------------------------------------------------------------------
int pikv_read_step_host(pikv_engine* eng, int32_t* experts, double* gates, double* logits,
                        pikv_step_summary* summary) {
    const Dims& D = eng->D;
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    if (experts) CUDA_TRY(cudaMemcpy(experts, eng->S.experts, sizeof(int32_t) * D.B * D.k, cudaMemcpyDeviceToHost));
    if (gates) CUDA_TRY(cudaMemcpy(gates, eng->S.gates, sizeof(double) * D.B * D.k, cudaMemcpyDeviceToHost));
    if (logits) CUDA_TRY(cudaMemcpy(logits, eng->S.logits, sizeof(double) * D.B * D.E, cudaMemcpyDeviceToHost));
    if (summary)
        CUDA_TRY(cudaMemcpy(summary, eng->S.summary, sizeof(pikv_step_summary) * D.B, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_read_evictions_host(pikv_engine* eng, pikv_evict_record* out, int32_t cap, int32_t* n_out) {
    const Dims& D = eng->D;
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    const int Gl = std::max(D.Gl, 1);
    std::vector<int32_t> now(D.B), nev((size_t)D.B * Gl);
    CUDA_TRY(cudaMemcpy(now.data(), eng->S.n_ow, sizeof(int32_t) * D.B, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(nev.data(), eng->S.n_ev, sizeof(int32_t) * D.B * Gl, cudaMemcpyDeviceToHost));
    int32_t n = 0, tot = 0;  // records written (<= cap), records of the step
    for (int s = 0; s < D.B; ++s) {
        const int no = std::min(now[s], std::max(0, cap - n));
        if (no > 0)
            CUDA_TRY(cudaMemcpy(out + n, eng->S.rec_ow + (size_t)s * D.k, sizeof(pikv_evict_record) * no,
                                cudaMemcpyDeviceToHost));
        n += no, tot += now[s];
        for (int gl = 0; gl < D.Gl; ++gl) {
            const int ne = std::min(nev[(size_t)s * Gl + gl], std::max(0, cap - n));
            if (ne > 0)
                CUDA_TRY(cudaMemcpy(out + n, eng->S.rec_ev + ((size_t)s * Gl + gl) * D.SPD * D.S,
                                    sizeof(pikv_evict_record) * ne, cudaMemcpyDeviceToHost));
            n += ne, tot += nev[(size_t)s * Gl + gl];
        }
    }
    *n_out = tot;
    return PIKV_OK;
}

// The store build of a prefill, see pikv_b200.h.
int pikv_insert_bulk(pikv_engine* eng, int32_t stream, int64_t T, const void* k, const void* v,
                     const int32_t* experts, const double* saliency, int64_t* n_displaced) {
    const Dims& D = eng->D;
    if (stream < 0 || stream >= D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    if (T < 0 || (T > 0 && (!k || !v || !experts)))
        return fail(PIKV_ERR_INVALID_ARGUMENT, "insert_bulk: null input");
    int rc = codec_ready(eng);
    if (rc) return rc;
    cudaSetDevice(eng->device);
    cudaStream_t st = eng->stream;
    const bool proj = D.codec == PIKV_CODEC_LOWRANK || D.codec == PIKV_CODEC_LORAPLUS;
    const size_t n_dst = sizeof(int64_t) * (size_t)std::max<int64_t>(1, T * D.k);
    // counters [2 + Gl], then the ring scratch of the two-phase placement [R][3]
    const size_t n_ctr = sizeof(unsigned long long) * (2 + D.Gl + 3 * (size_t)std::max(D.R, 1));
    // projections [2][T][dp], then the tcgen05 path's bias B^T [H][r] and
    // pre-split basis [H][2][64][hd] bf16
    const size_t n_pr = proj ? sizeof(float) * (2 * (size_t)std::max<int64_t>(1, T) * D.dp +
                                                (((size_t)D.dp + 63) & ~(size_t)63) +
                                                (size_t)D.H * 64 * (D.d / D.H) + 64)
                             : 0;
    const size_t n_sort = sizeof(int32_t) * bulk_sort_ints(D, T);
    const size_t need = ((n_dst + 255) & ~(size_t)255) + ((n_ctr + 255) & ~(size_t)255) + ((n_pr + 255) & ~(size_t)255) +
                        n_sort;
    if (need > eng->bulk_cap) {
        CUDA_TRY(cudaStreamSynchronize(st));
        if (eng->bulk_buf) cudaFree(eng->bulk_buf);
    if (eng->rb_buf) cudaFree(eng->rb_buf);
    if (eng->gathered) cudaFree(eng->gathered);
    if (eng->comm && eng->own_comm) ncclCommDestroy(eng->comm);
        eng->bulk_buf = nullptr, eng->bulk_cap = 0;
        CUDA_TRY(cudaMalloc(&eng->bulk_buf, need));
        eng->bulk_cap = need;
    }
    int64_t* dst = (int64_t*)eng->bulk_buf;
    unsigned long long* ctr = (unsigned long long*)((uint8_t*)eng->bulk_buf + ((n_dst + 255) & ~(size_t)255));
    float* pr = proj ? (float*)((uint8_t*)ctr + ((n_ctr + 255) & ~(size_t)255)) : nullptr;
    int32_t* sort_buf = (int32_t*)((uint8_t*)ctr + ((n_ctr + 255) & ~(size_t)255) + ((n_pr + 255) & ~(size_t)255));
    cudaError_t e = cudaSuccess;
    {
        const char* tc = std::getenv("PIKV_BULK_TC");
        const char* so = std::getenv("PIKV_BULK_SORT");  // A/B: 0 = per-ring scans
        e = (cudaError_t)bulk_insert(D, eng->S, stream, T, k, v, experts, saliency, dst, pr, ctr,
                                     tc ? std::atoi(tc) : 1, st, (so && so[0] == '0') ? nullptr : sort_buf);
    }
    unsigned long long host_ctr[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(host_ctr, ctr, sizeof(host_ctr), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(PIKV_ERR_CUDA, std::string("insert_bulk: ") + cudaGetErrorString(e));
    int32_t err = 0;
    CUDA_TRY(cudaMemcpy(&err, eng->S.err + stream, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (err) return fail(err, "insert_bulk: KV page pool exhausted");
    if (n_displaced) *n_displaced = (int64_t)host_ctr[1];
    return PIKV_OK;
}

int pikv_insert_bulk_host(pikv_engine* eng, int32_t stream, int64_t T, const void* k, const void* v,
                          const int32_t* experts, const double* saliency, int64_t* n_displaced) {
    const Dims& D = eng->D;
    if (T <= 0) return pikv_insert_bulk(eng, stream, T, k, v, experts, saliency, n_displaced);
    const size_t row = (size_t)D.d * (D.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4);
    cudaSetDevice(eng->device);
    cudaStream_t st = eng->stream;
    const size_t nk = row * T, ne = sizeof(int32_t) * (size_t)T * D.k;
    const size_t ns = saliency && D.n_layers > 0 ? sizeof(double) * (size_t)T * D.n_layers : 0;
    if (2 * nk + ne + ns + 64 > eng->stage_cap) {
        CUDA_TRY(cudaStreamSynchronize(st));
        if (eng->bulk_stage) cudaFree(eng->bulk_stage);
        eng->bulk_stage = nullptr, eng->stage_cap = 0;
        CUDA_TRY(cudaMalloc(&eng->bulk_stage, 2 * nk + ne + ns + 64));
        eng->stage_cap = 2 * nk + ne + ns + 64;
    }
    uint8_t* buf = (uint8_t*)eng->bulk_stage;
    uint8_t* dk = buf;
    uint8_t* dv = buf + nk;
    int32_t* de = (int32_t*)(buf + 2 * nk);
    double* ds = ns ? (double*)(((uintptr_t)(buf + 2 * nk + ne) + 15) & ~(uintptr_t)15) : nullptr;
    cudaError_t e = cudaMemcpyAsync(dk, k, nk, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dv, v, nk, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(de, experts, ne, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && ns) e = cudaMemcpyAsync(ds, saliency, ns, cudaMemcpyHostToDevice, st);
    int rc = e == cudaSuccess ? pikv_insert_bulk(eng, stream, T, dk, dv, de, ds, n_displaced)
                              : fail(PIKV_ERR_CUDA, std::string("insert_bulk_host: ") + cudaGetErrorString(e));
    cudaStreamSynchronize(st);
    return rc;
}

// generate_trace (trace.cpp:54-82): vocabulary = Rng(seed).normal_vector(width)
// per word; embed ids by inverse-CDF sampling of p_i ~ (i+1)^-skew with
// Rng(seed ^ 0x7ace5eed); per-layer saliency float(|normal| * 0.1).
int pikv_generate_trace(uint64_t steps, int32_t width, int32_t vocab, double zipf_skew, uint64_t seed,
                        int32_t layers, double* vocab_out, uint32_t* embed_ids, float* saliency) {
    // TraceSpec::validate, trace.cpp:39-44
    if (width < 1) return fail(PIKV_ERR_INVALID_CONFIG, "TraceSpec: width must be >= 1");
    if (vocab < 1) return fail(PIKV_ERR_INVALID_CONFIG, "TraceSpec: vocab must be >= 1");
    if (zipf_skew < 0) return fail(PIKV_ERR_INVALID_CONFIG, "TraceSpec: skew must be >= 0");
    if (layers < 1) return fail(PIKV_ERR_INVALID_CONFIG, "TraceSpec: layers must be >= 1");
    if (vocab_out) {
        RefRng rng(seed);
        for (size_t i = 0; i < (size_t)vocab * width; ++i) vocab_out[i] = rng.normal();
    }
    std::vector<double> cdf(vocab);
    double total = 0.0;
    for (int i = 0; i < vocab; ++i) {
        total += std::pow(static_cast<double>(i + 1), -zipf_skew);
        cdf[i] = total;
    }
    for (auto& c : cdf) c /= total;
    RefRng rng(seed ^ 0x7ace5eedULL);
    for (uint64_t t = 0; t < steps; ++t) {
        const double u = rng.uniform();
        const auto it = std::lower_bound(cdf.begin(), cdf.end(), u);
        const uint32_t id = static_cast<uint32_t>(std::min<std::ptrdiff_t>(it - cdf.begin(), vocab - 1));
        if (embed_ids) embed_ids[t] = id;
        for (int l = 0; l < layers; ++l) {
            const float sv = static_cast<float>(std::abs(rng.normal()) * 0.1);
            if (saliency) saliency[t * layers + l] = sv;
        }
    }
    return PIKV_OK;
}

int pikv_snapshot_host(pikv_engine* eng, int32_t stream, int64_t now, pikv_snapshot_record* out,
                       int64_t cap, int64_t* n_out) {
    const Dims& D = eng->D;
    if (stream < 0 || stream >= D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    if (!n_out) return fail(PIKV_ERR_INVALID_ARGUMENT, "n_out is NULL");
    cudaSetDevice(eng->device);
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    std::vector<int32_t> live(D.R > 0 ? D.R : 1);
    if (D.R > 0)
        CUDA_TRY(cudaMemcpy(live.data(), eng->S.live + (int64_t)stream * D.R, sizeof(int32_t) * D.R,
                            cudaMemcpyDeviceToHost));
    std::vector<int64_t> off(D.R + 1, 0);
    for (int r = 0; r < D.R; ++r) off[r + 1] = off[r] + live[r];
    const int64_t n = off[D.R];
    *n_out = n;
    if (!out || cap <= 0 || n == 0) return PIKV_OK;
    uint64_t t = 0;
    if (now < 0) {
        CUDA_TRY(cudaMemcpy(&t, eng->S.now + stream, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    } else {
        t = (uint64_t)now;
    }
    int64_t* d_off = nullptr;
    pikv_snapshot_record* d_rec = nullptr;
    CUDA_TRY(cudaMalloc(&d_off, sizeof(int64_t) * (D.R + 1)));
    cudaError_t e = cudaMalloc(&d_rec, sizeof(pikv_snapshot_record) * n);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_off, off.data(), sizeof(int64_t) * (D.R + 1), cudaMemcpyHostToDevice,
                            eng->stream);
    if (e == cudaSuccess) {
        launch_snapshot(D, eng->S, stream, t, d_off, d_rec, n, eng->stream);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out, d_rec, sizeof(pikv_snapshot_record) * std::min(n, cap),
                            cudaMemcpyDeviceToHost, eng->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(eng->stream);
    cudaFree(d_off);
    cudaFree(d_rec);
    if (e != cudaSuccess) return fail(PIKV_ERR_CUDA, std::string("snapshot: ") + cudaGetErrorString(e));
    return PIKV_OK;
}

int pikv_read_attended_host(pikv_engine* eng, int32_t stream, int64_t* token, int32_t* expert,
                            double* alpha, int32_t cap, int32_t* n_out) {
    const Dims& D = eng->D;
    if (stream < 0 || stream >= D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    int32_t cnt = 0;
    CUDA_TRY(cudaMemcpy(&cnt, eng->S.att_cnt + stream, sizeof(int32_t), cudaMemcpyDeviceToHost));
    const int64_t base[1] = {(int64_t)stream * D.att_stride};
    const int n = cnt;
    *n_out = n;
    const int m = std::min(n, cap);
    if (m <= 0) return PIKV_OK;
    std::vector<int32_t> slot(m);
    std::vector<float> sc((size_t)m * D.H), gM(D.H), gL(D.H);
    CUDA_TRY(cudaMemcpy(slot.data(), eng->S.att_slot + base[0], sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(sc.data(), eng->S.scores + base[0] * D.H, sizeof(float) * m * D.H, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(gM.data(), eng->S.gM + stream * D.H, sizeof(float) * D.H, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(gL.data(), eng->S.gL + stream * D.H, sizeof(float) * D.H, cudaMemcpyDeviceToHost));
    std::vector<int64_t> ht(m);
    std::vector<int32_t> he(m);
    {
        if (eng->rb_cap < 12 * (size_t)m) {
            if (eng->rb_buf) cudaFree(eng->rb_buf);
            eng->rb_buf = nullptr, eng->rb_cap = 0;
            CUDA_TRY(cudaMalloc(&eng->rb_buf, 12 * (size_t)m));
            eng->rb_cap = 12 * (size_t)m;
        }
        uint8_t* buf = (uint8_t*)eng->rb_buf;
        launch_gather_slots(eng->S, eng->S.att_slot + base[0], m, (int64_t*)buf, (int32_t*)(buf + 8 * (size_t)m),
                            eng->stream);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpyAsync(ht.data(), buf, 8 * (size_t)m, cudaMemcpyDeviceToHost, eng->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(he.data(), buf + 8 * (size_t)m, 4 * (size_t)m, cudaMemcpyDeviceToHost, eng->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(eng->stream);
        if (e != cudaSuccess) return fail(PIKV_ERR_CUDA, std::string("read_attended: ") + cudaGetErrorString(e));
    }
    for (int i = 0; i < m; ++i) {
        if (token) token[i] = ht[i];
        if (expert) expert[i] = he[i];
        if (alpha) {  // same expression as k_foldback
            double a = 0.0;
            for (int h = 0; h < D.H; ++h)
                if (gL[h] > 0.f) a += (double)(std::exp2((double)sc[(size_t)i * D.H + h] - gM[h]) / gL[h]);
            alpha[i] = a / D.H;
        }
    }
    return PIKV_OK;
}

int pikv_read_entries_host(pikv_engine* eng, int32_t stream, const int64_t* slots, int32_t n, float* key_out,
                           float* value_out) {
    const Dims& D = eng->D;
    if (stream < 0 || stream >= D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    if (n <= 0) return PIKV_OK;
    if (!slots || !key_out || !value_out) return fail(PIKV_ERR_INVALID_ARGUMENT, "read_entries: null buffer");
    const int64_t ns = (int64_t)D.R * D.S;
    for (int i = 0; i < n; ++i)
        if (slots[i] < 0 || slots[i] >= ns) return fail(PIKV_ERR_INVALID_ARGUMENT, "read_entries: slot out of range");
    cudaSetDevice(eng->device);
    const size_t nb = 8 * (size_t)n, kb = sizeof(float) * (size_t)n * D.dp;
    uint8_t* buf = nullptr;
    CUDA_TRY(cudaMalloc(&buf, nb + 2 * kb));
    cudaStream_t st = eng->stream;
    cudaError_t e = cudaMemcpyAsync(buf, slots, nb, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        launch_read_entries(D, eng->S, stream, (const int64_t*)buf, n, (float*)(buf + nb), (float*)(buf + nb + kb), st);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(key_out, buf + nb, kb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(value_out, buf + nb + kb, kb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(buf);
    if (e != cudaSuccess) return fail(PIKV_ERR_CUDA, std::string("read_entries: ") + cudaGetErrorString(e));
    return PIKV_OK;
}

int64_t pikv_slot_count(pikv_engine* eng) { return (int64_t)eng->D.R * eng->D.S; }

int pikv_read_slots_host(pikv_engine* eng, int32_t stream, uint64_t* id, uint64_t* shard_seq,
                         int64_t* token, int32_t* expert, uint64_t* insert_step,
                         uint64_t* last_access, uint64_t* freq, double* attn_mass,
                         double* per_layer) {
    const Dims& D = eng->D;
    if (stream < 0 || stream >= D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    const size_t n = (size_t)D.R * D.S, off = (size_t)stream * n;
    auto cp = [&](void* dst, const void* src, size_t es) -> cudaError_t {
        if (!dst) return cudaSuccess;
        return cudaMemcpy(dst, (const uint8_t*)src + off * es, n * es, cudaMemcpyDeviceToHost);
    };
    CUDA_TRY(cp(id, eng->S.id, 8));
    CUDA_TRY(cp(shard_seq, eng->S.shard_seq, 8));
    CUDA_TRY(cp(token, eng->S.token, 8));
    CUDA_TRY(cp(expert, eng->S.expert, 4));
    CUDA_TRY(cp(insert_step, eng->S.insert_step, 8));
    CUDA_TRY(cp(last_access, eng->S.last_access, 8));
    CUDA_TRY(cp(freq, eng->S.freq, 8));
    CUDA_TRY(cp(attn_mass, eng->S.attn_mass, 8));
    if (per_layer && D.n_layers > 0)
        CUDA_TRY(cudaMemcpy(per_layer, eng->S.per_layer + off * D.n_layers, n * D.n_layers * 8,
                            cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_write_attn_mass_host(pikv_engine* eng, int32_t stream, const double* attn_mass,
                              const double* per_layer) {
    const Dims& D = eng->D;
    if (stream < 0 || stream >= D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    const size_t n = (size_t)D.R * D.S, off = (size_t)stream * n;
    if (attn_mass) CUDA_TRY(cudaMemcpy(eng->S.attn_mass + off, attn_mass, n * 8, cudaMemcpyHostToDevice));
    if (per_layer && D.n_layers > 0)
        CUDA_TRY(cudaMemcpy(eng->S.per_layer + off * D.n_layers, per_layer, n * D.n_layers * 8,
                            cudaMemcpyHostToDevice));
    return PIKV_OK;
}

int pikv_read_router_state_host(pikv_engine* eng, int32_t stream, double* load, uint64_t* usage,
                                uint64_t* miss, double* bias, uint64_t* step, uint64_t* total_usage) {
    const Dims& D = eng->D;
    if (stream < 0 || stream >= D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    const size_t E = D.E, o = (size_t)stream * E;
    if (load) CUDA_TRY(cudaMemcpy(load, eng->S.load + o, E * 8, cudaMemcpyDeviceToHost));
    if (usage) CUDA_TRY(cudaMemcpy(usage, eng->S.usage + o, E * 8, cudaMemcpyDeviceToHost));
    if (miss) CUDA_TRY(cudaMemcpy(miss, eng->S.miss + o, E * 8, cudaMemcpyDeviceToHost));
    if (bias) CUDA_TRY(cudaMemcpy(bias, eng->S.bias + o, E * 8, cudaMemcpyDeviceToHost));
    if (step) CUDA_TRY(cudaMemcpy(step, eng->S.rstep + stream, 8, cudaMemcpyDeviceToHost));
    if (total_usage) CUDA_TRY(cudaMemcpy(total_usage, eng->S.total_usage + stream, 8, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_read_sched_state_host(pikv_engine* eng, int32_t stream, double* theta, double* running_hit,
                               uint64_t* step) {
    if (stream < 0 || stream >= eng->D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    if (theta) CUDA_TRY(cudaMemcpy(theta, eng->S.theta + stream, 8, cudaMemcpyDeviceToHost));
    if (running_hit) CUDA_TRY(cudaMemcpy(running_hit, eng->S.running_hit + stream, 8, cudaMemcpyDeviceToHost));
    if (step) CUDA_TRY(cudaMemcpy(step, eng->S.sstep + stream, 8, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_store_stats_host(pikv_engine* eng, int32_t stream, uint64_t* live, uint64_t* memory_bytes,
                          uint64_t* inserts, uint64_t* overwrites) {
    const Dims& D = eng->D;
    if (stream < 0 || stream >= D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    std::vector<int32_t> lv(D.R);
    CUDA_TRY(cudaMemcpy(lv.data(), eng->S.live + (size_t)stream * D.R, sizeof(int32_t) * D.R, cudaMemcpyDeviceToHost));
    uint64_t n = 0;
    for (int r = 0; r < D.R; ++r) n += (uint64_t)lv[r];
    if (live) *live = n;
    // KVStore::memory_bytes, kvstore.cpp:193-196: 2 * d' * elem_bytes * live
    if (memory_bytes) *memory_bytes = 2ull * (uint64_t)D.dp * (uint64_t)eng->cfg.elem_bytes * n;
    if (inserts) CUDA_TRY(cudaMemcpy(inserts, eng->S.st_inserts + stream, 8, cudaMemcpyDeviceToHost));
    if (overwrites) CUDA_TRY(cudaMemcpy(overwrites, eng->S.st_overwrites + stream, 8, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int64_t pikv_pool_pages_in_use(pikv_engine* eng) {
    cudaStreamSynchronize(eng->stream);
    int32_t top = 0;
    cudaMemcpy(&top, eng->S.free_top, sizeof(int32_t), cudaMemcpyDeviceToHost);
    return eng->D.pool_pages - top;
}

int64_t pikv_entry_bytes(pikv_engine* eng) { return eng->D.entry_bytes; }

// Not part of the public header: debug timestamps written by kernels.
int pikv_debug_read(pikv_engine* eng, long long* out, int n) {
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    CUDA_TRY(cudaMemcpy(out, eng->S.dbg, sizeof(long long) * std::min(n, 64 + 8 * eng->D.B + 8 * eng->D.attend_ctas),
                        cudaMemcpyDeviceToHost));
    return PIKV_OK;
}
int64_t pikv_kernel_launches(pikv_engine* eng) { return eng->launches; }

int pikv_set_profiling(pikv_engine* eng, int32_t on) {
    eng->profiling = on != 0;
    if (eng->profiling && eng->ev.empty()) {
        eng->ev.resize((size_t)kProfSteps * (kPhases + 1));
        for (auto& e : eng->ev) CUDA_TRY(cudaEventCreate(&e));
    }
    eng->prof_steps = 0;
    return PIKV_OK;
}

int pikv_read_profile_host(pikv_engine* eng, float* phase_ms, int32_t n_phases, int32_t* n_steps) {
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    std::vector<float> acc(kPhases, 0.f);
    for (int st = 0; st < eng->prof_steps; ++st) {
        const int b = st * (kPhases + 1);
        for (int p = 0; p < kPhases; ++p) {
            float ms = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&ms, eng->ev[b + p], eng->ev[b + p + 1]));
            acc[p] += ms;
        }
    }
    for (int p = 0; p < n_phases && p < kPhases; ++p) phase_ms[p] = acc[p];
    if (n_steps) *n_steps = eng->prof_steps;
    eng->prof_steps = 0;
    return PIKV_OK;
}

// ---------------------------------------------------------------------------
// component API: the reference's free functions and classes on one stream
// (include/pikv_b200.h "component API"); kernels in components.cu
// ---------------------------------------------------------------------------
namespace {
// device scratch of one component call, freed on scope exit
struct Scratch {
    void* p = nullptr;
    cudaError_t e = cudaSuccess;
    explicit Scratch(size_t n) { e = cudaMalloc(&p, n ? n : 1); }
    ~Scratch() { if (p) cudaFree(p); }
    uint8_t* at(size_t off) const { return (uint8_t*)p + off; }
};
size_t al256(size_t n) { return (n + 255) & ~(size_t)255; }

int component_check(pikv_engine* eng, int32_t stream) {
    if (!eng) return fail(PIKV_ERR_INVALID_ARGUMENT, "engine is NULL");
    if (stream < 0 || stream >= eng->D.B) return fail(PIKV_ERR_INVALID_ARGUMENT, "stream out of range");
    if (eng->D.world != 1) return fail(PIKV_ERR_INVALID_ARGUMENT, "component API: world_size must be 1");
    cudaSetDevice(eng->device);
    return PIKV_OK;
}
}  // namespace

int pikv_update_config(pikv_engine* eng, const pikv_config* cfg) {
    if (!eng || !cfg) return fail(PIKV_ERR_INVALID_ARGUMENT, "NULL argument");
    const pikv_config& o = eng->cfg;
    // structural fields fix the HBM layout: they must not change
    if (cfg->d != o.d || cfg->E != o.E || cfg->k != o.k || cfg->G != o.G || cfg->S != o.S ||
        cfg->n_heads != o.n_heads || cfg->n_tok != o.n_tok || cfg->n_exp != o.n_exp ||
        cfg->additive != o.additive || cfg->page_size != o.page_size || cfg->codec != o.codec ||
        cfg->rank != o.rank || cfg->n_layers != o.n_layers || cfg->batch != o.batch ||
        cfg->kv_dtype != o.kv_dtype || cfg->world_size != o.world_size)
        return fail(PIKV_ERR_INVALID_CONFIG, "update_config: only router / scheduler coefficients may change");
    int rc = validate(*cfg);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    eng->cfg = *cfg;
    fill_cfg(*cfg, eng->C);
    eng->invalidate();  // captured kernels hold the old Cfg
    return PIKV_OK;
}

static int route_common(pikv_engine* eng, int32_t stream, const double* query, const double* logits_in,
                        int32_t* experts, double* gates, double* logits) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    const Dims& D = eng->D;
    cudaStream_t st = eng->stream;
    const size_t nq = query ? sizeof(double) * (size_t)D.B * D.d : 0;
    Scratch buf(al256(nq) + sizeof(double) * (size_t)D.E);
    if (buf.e != cudaSuccess) return fail(PIKV_ERR_CUDA, "route: cudaMalloc");
    double* dq = (double*)buf.at(0);
    double* dl = (double*)buf.at(al256(nq));
    if (query) CUDA_TRY(cudaMemcpyAsync(dq + (size_t)stream * D.d, query, sizeof(double) * D.d,
                                        cudaMemcpyHostToDevice, st));
    if (logits_in) CUDA_TRY(cudaMemcpyAsync(dl, logits_in, sizeof(double) * D.E, cudaMemcpyHostToDevice, st));
    launch_route_one(D, eng->C, eng->S, stream, query ? dq : nullptr, logits_in ? dl : nullptr, st);
    CUDA_TRY(cudaGetLastError());
    int32_t err = 0;
    CUDA_TRY(cudaMemcpyAsync(&err, eng->S.err + stream, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (err == PIKV_ERR_NUMERICAL) {  // router.cpp:131-133: throws before any state change
        CUDA_TRY(cudaMemset(eng->S.err + stream, 0, sizeof(int32_t)));
        return fail(PIKV_ERR_NUMERICAL, "route_logits: NaN logit");
    }
    if (err) return fail(err, "route: stream is in an error state");
    const size_t k = (size_t)D.k, E = (size_t)D.E;
    if (experts) CUDA_TRY(cudaMemcpy(experts, eng->S.experts + stream * k, 4 * k, cudaMemcpyDeviceToHost));
    if (gates) CUDA_TRY(cudaMemcpy(gates, eng->S.gates + stream * k, 8 * k, cudaMemcpyDeviceToHost));
    if (logits) CUDA_TRY(cudaMemcpy(logits, eng->S.logits + stream * E, 8 * E, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_route_host(pikv_engine* eng, int32_t stream, const double* query, int32_t* experts, double* gates,
                    double* logits) {
    if (!query && eng && eng->C.router_strategy != PIKV_ROUTER_BASE)
        return fail(PIKV_ERR_INVALID_ARGUMENT, "route: query is NULL");
    if (!query) {  // Base ignores the query (router.cpp:219-221)
        static const double zero = 0.0;
        return route_common(eng, stream, nullptr, &zero, experts, gates, logits);
    }
    return route_common(eng, stream, query, nullptr, experts, gates, logits);
}

int pikv_route_logits_host(pikv_engine* eng, int32_t stream, const double* logits_in, int32_t* experts,
                           double* gates, double* logits) {
    if (!logits_in) return fail(PIKV_ERR_INVALID_ARGUMENT, "route_logits: logits are NULL");
    return route_common(eng, stream, nullptr, logits_in, experts, gates, logits);
}

static int state_op(pikv_engine* eng, int32_t stream, int op, uint64_t a, uint64_t b, const int32_t* experts,
                    int n, double reward) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    Scratch buf(4 * (size_t)(n > 0 ? n : 1));
    if (buf.e != cudaSuccess) return fail(PIKV_ERR_CUDA, "cudaMalloc");
    if (n > 0) CUDA_TRY(cudaMemcpyAsync(buf.p, experts, 4 * (size_t)n, cudaMemcpyHostToDevice, eng->stream));
    launch_state_op(eng->D, eng->C, eng->S, stream, op, a, b, (const int32_t*)buf.p, n, reward, eng->stream);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    return PIKV_OK;
}

int pikv_record_miss(pikv_engine* eng, int32_t stream, int32_t expert) {
    if (eng && (expert < 0 || expert >= eng->D.E))  // router.cpp:237-239
        return fail(PIKV_ERR_INVALID_ARGUMENT, "record_miss: expert out of range");
    return state_op(eng, stream, 3, (uint64_t)expert, 0, nullptr, 0, 0.0);
}

int pikv_router_adapt(pikv_engine* eng, int32_t stream, const int32_t* experts, int32_t n, double reward) {
    if (!(reward >= 0.0 && reward <= 1.0))  // router.cpp:245-247
        return fail(PIKV_ERR_INVALID_ARGUMENT, "adapt: reward must be in [0, 1]");
    for (int j = 0; j < n; ++j)
        if (eng && (experts[j] < 0 || experts[j] >= eng->D.E))
            return fail(PIKV_ERR_INVALID_ARGUMENT, "adapt: expert out of range");
    return state_op(eng, stream, 4, 0, 0, experts, n, reward);
}

int pikv_observe_hits(pikv_engine* eng, int32_t stream, uint64_t hits, uint64_t lookups) {
    return state_op(eng, stream, 0, hits, lookups, nullptr, 0, 0.0);
}

int pikv_adakv_update(pikv_engine* eng, int32_t stream) { return state_op(eng, stream, 1, 0, 0, nullptr, 0, 0.0); }

int pikv_write_router_state_host(pikv_engine* eng, int32_t stream, const double* load, const uint64_t* usage,
                                 const uint64_t* miss, const double* bias, const uint64_t* step,
                                 const uint64_t* total_usage) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    const size_t E = eng->D.E, o = (size_t)stream * E;
    if (load) CUDA_TRY(cudaMemcpy(eng->S.load + o, load, 8 * E, cudaMemcpyHostToDevice));
    if (usage) CUDA_TRY(cudaMemcpy(eng->S.usage + o, usage, 8 * E, cudaMemcpyHostToDevice));
    if (miss) CUDA_TRY(cudaMemcpy(eng->S.miss + o, miss, 8 * E, cudaMemcpyHostToDevice));
    if (bias) CUDA_TRY(cudaMemcpy(eng->S.bias + o, bias, 8 * E, cudaMemcpyHostToDevice));
    if (step) CUDA_TRY(cudaMemcpy(eng->S.rstep + stream, step, 8, cudaMemcpyHostToDevice));
    if (total_usage) CUDA_TRY(cudaMemcpy(eng->S.total_usage + stream, total_usage, 8, cudaMemcpyHostToDevice));
    return PIKV_OK;
}

int pikv_write_sched_state_host(pikv_engine* eng, int32_t stream, const double* theta, const double* running_hit,
                                const uint64_t* step) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    if (theta) CUDA_TRY(cudaMemcpy(eng->S.theta + stream, theta, 8, cudaMemcpyHostToDevice));
    if (running_hit) CUDA_TRY(cudaMemcpy(eng->S.running_hit + stream, running_hit, 8, cudaMemcpyHostToDevice));
    if (step) CUDA_TRY(cudaMemcpy(eng->S.sstep + stream, step, 8, cudaMemcpyHostToDevice));
    return PIKV_OK;
}

int pikv_store_insert_host(pikv_engine* eng, int32_t stream, int32_t n, const pikv_entry* entries,
                           const float* key, const float* value, const double* per_layer, pikv_entry* displaced,
                           float* displaced_key, float* displaced_value, double* displaced_layers,
                           int32_t* displaced_flag) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    if (n <= 0) return PIKV_OK;
    if (!entries || !key || !value) return fail(PIKV_ERR_INVALID_ARGUMENT, "store_insert: NULL input");
    const Dims& D = eng->D;
    for (int j = 0; j < n; ++j)  // kvstore.cpp:17-22 (shard_assign of the entry)
        if (entries[j].token_id < 0 || entries[j].expert_id < 0)
            return fail(PIKV_ERR_INVALID_ARGUMENT, "shard_assign: negative token or expert index");
    const size_t dp = (size_t)D.dp, nl = (size_t)std::max(D.n_layers, 0);
    std::vector<float> kv(2 * dp * n);
    for (int j = 0; j < n; ++j) {
        std::memcpy(&kv[(2 * (size_t)j) * dp], key + (size_t)j * dp, 4 * dp);
        std::memcpy(&kv[(2 * (size_t)j + 1) * dp], value + (size_t)j * dp, 4 * dp);
    }
    const size_t o_in = 0, o_kv = al256(sizeof(pikv_entry) * n), o_ly = o_kv + al256(4 * kv.size());
    const size_t o_dsp = o_ly + al256(8 * nl * n), o_dkv = o_dsp + al256(sizeof(pikv_entry) * n);
    const size_t o_dly = o_dkv + al256(4 * kv.size()), o_flag = o_dly + al256(8 * nl * n);
    const size_t o_st = o_flag + al256(4 * (size_t)n);
    Scratch buf(o_st + 16);
    if (buf.e != cudaSuccess) return fail(PIKV_ERR_CUDA, "store_insert: cudaMalloc");
    cudaStream_t st = eng->stream;
    CUDA_TRY(cudaMemcpyAsync(buf.at(o_in), entries, sizeof(pikv_entry) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(buf.at(o_kv), kv.data(), 4 * kv.size(), cudaMemcpyHostToDevice, st));
    if (per_layer && nl) CUDA_TRY(cudaMemcpyAsync(buf.at(o_ly), per_layer, 8 * nl * n, cudaMemcpyHostToDevice, st));
    launch_store_insert(D, eng->S, stream, n, (const pikv_entry*)buf.at(o_in), (const float*)buf.at(o_kv),
                        per_layer && nl ? (const double*)buf.at(o_ly) : nullptr, (pikv_entry*)buf.at(o_dsp),
                        (float*)buf.at(o_dkv), nl ? (double*)buf.at(o_dly) : nullptr, (int32_t*)buf.at(o_flag),
                        (int32_t*)buf.at(o_st), st);
    CUDA_TRY(cudaGetLastError());
    int32_t status = 0;
    std::vector<int32_t> flag(n);
    std::vector<float> dkv(kv.size());
    CUDA_TRY(cudaMemcpyAsync(&status, buf.at(o_st), 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(flag.data(), buf.at(o_flag), 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
    if (displaced) CUDA_TRY(cudaMemcpyAsync(displaced, buf.at(o_dsp), sizeof(pikv_entry) * n, cudaMemcpyDeviceToHost, st));
    if (displaced_key || displaced_value)
        CUDA_TRY(cudaMemcpyAsync(dkv.data(), buf.at(o_dkv), 4 * dkv.size(), cudaMemcpyDeviceToHost, st));
    if (displaced_layers && nl)
        CUDA_TRY(cudaMemcpyAsync(displaced_layers, buf.at(o_dly), 8 * nl * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int j = 0; j < n; ++j) {
        if (displaced_flag) displaced_flag[j] = flag[j];
        if (!flag[j]) continue;
        if (displaced_key) std::memcpy(displaced_key + (size_t)j * dp, &dkv[2 * (size_t)j * dp], 4 * dp);
        if (displaced_value) std::memcpy(displaced_value + (size_t)j * dp, &dkv[(2 * (size_t)j + 1) * dp], 4 * dp);
    }
    if (status) return fail(status, "store_insert: KV page pool exhausted");
    return PIKV_OK;
}

int pikv_store_retrieve_host(pikv_engine* eng, int32_t stream, const int32_t* experts, int32_t n_experts,
                             int64_t since, uint64_t now, int64_t* slots_out, int32_t cap, int32_t* n_out,
                             int32_t* missed_out, int32_t* n_missed) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    if (n_experts <= 0 || !experts)  // kvstore.cpp:124-126
        return fail(PIKV_ERR_INVALID_ARGUMENT, "KVStore::retrieve: empty expert set");
    for (int j = 0; j < n_experts; ++j)
        if (experts[j] < 0) return fail(PIKV_ERR_INVALID_ARGUMENT, "KVStore::retrieve: negative expert");
    const Dims& D = eng->D;
    uint32_t want[8] = {0};
    for (int j = 0; j < n_experts; ++j)
        if (experts[j] < 256) want[experts[j] >> 5] |= 1u << (experts[j] & 31);
    cudaStream_t st = eng->stream;
    Scratch buf(retrieve_scratch_bytes(D) + 256);
    if (buf.e != cudaSuccess) return fail(PIKV_ERR_CUDA, "retrieve: cudaMalloc");
    uint32_t* dwant = (uint32_t*)buf.at(0);
    CUDA_TRY(cudaMemcpyAsync(dwant, want, sizeof(want), cudaMemcpyHostToDevice, st));
    int32_t *sorted = nullptr, *cnt = nullptr;
    uint32_t* found = nullptr;
    const int e = launch_retrieve(D, eng->S, stream, since, now, dwant, buf.at(256), &sorted, &cnt, &found, st);
    if (e) return fail(PIKV_ERR_CUDA, std::string("retrieve: ") + cudaGetErrorString((cudaError_t)e));
    int32_t n = 0;
    uint32_t hfound[256];
    CUDA_TRY(cudaMemcpyAsync(&n, cnt, 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(hfound, found, sizeof(hfound), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (n_out) *n_out = n;
    const int m = std::min(n, cap);
    if (slots_out && m > 0) {
        std::vector<int32_t> sl(m);
        CUDA_TRY(cudaMemcpy(sl.data(), sorted, 4 * (size_t)m, cudaMemcpyDeviceToHost));
        for (int i = 0; i < m; ++i) slots_out[i] = sl[i];
    }
    int nm = 0;  // missed experts in the order given (kvstore.cpp:169-174)
    for (int j = 0; j < n_experts; ++j)
        if (experts[j] >= 256 || hfound[experts[j]] == 0) {
            if (missed_out) missed_out[nm] = experts[j];
            ++nm;
        }
    if (n_missed) *n_missed = nm;
    // StoreStats: retrievals += 1, misses += |missed| (kvstore.cpp:169-176)
    std::vector<uint64_t> cs(2);
    CUDA_TRY(cudaMemcpy(&cs[0], eng->S.st_retrievals + stream, 8, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(&cs[1], eng->S.st_misses + stream, 8, cudaMemcpyDeviceToHost));
    cs[0] += 1, cs[1] += (uint64_t)nm;
    CUDA_TRY(cudaMemcpy(eng->S.st_retrievals + stream, &cs[0], 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(eng->S.st_misses + stream, &cs[1], 8, cudaMemcpyHostToDevice));
    return PIKV_OK;
}

int pikv_store_erase_host(pikv_engine* eng, int32_t stream, uint64_t entry_id, int32_t* erased) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    if (erased) *erased = 0;
    if (entry_id == 0) return PIKV_OK;  // ids start at 1 (kvstore.hpp:157)
    if (!eng->D.holes) {  // page members may have holes from now on
        CUDA_TRY(cudaStreamSynchronize(eng->stream));
        eng->D.holes = 1;
        eng->invalidate();
    }
    Scratch buf(16);
    if (buf.e != cudaSuccess) return fail(PIKV_ERR_CUDA, "erase: cudaMalloc");
    launch_store_erase(eng->D, eng->S, stream, entry_id, (int32_t*)buf.p, eng->stream);
    CUDA_TRY(cudaGetLastError());
    int32_t st = 0;
    CUDA_TRY(cudaMemcpyAsync(&st, buf.p, 4, cudaMemcpyDeviceToHost, eng->stream));
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    if (erased) *erased = st;
    return PIKV_OK;
}

int pikv_store_counters_host(pikv_engine* eng, int32_t stream, uint64_t* retrievals, uint64_t* misses) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    if (retrievals) CUDA_TRY(cudaMemcpy(retrievals, eng->S.st_retrievals + stream, 8, cudaMemcpyDeviceToHost));
    if (misses) CUDA_TRY(cudaMemcpy(misses, eng->S.st_misses + stream, 8, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_ring_live_host(pikv_engine* eng, int32_t stream, int32_t* live) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(eng->stream));
    CUDA_TRY(cudaMemcpy(live, eng->S.live + (size_t)stream * eng->D.R, 4 * (size_t)eng->D.R, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_score_entries_host(const pikv_config* cfg, const pikv_entry* entries, const double* per_layer, int32_t n,
                            uint64_t now, double* out) {
    if (!cfg || (n > 0 && (!entries || !out))) return fail(PIKV_ERR_INVALID_ARGUMENT, "NULL argument");
    if (cfg->sched_strategy == PIKV_SCHED_QUEST)  // scheduler.cpp:199-203
        return fail(PIKV_ERR_NOT_FITTED, "score: QUEST scorer not fitted");
    if (n <= 0) return PIKV_OK;
    Cfg C{};
    fill_cfg(*cfg, C);
    const size_t nl = (size_t)std::max(cfg->n_layers, 0);
    Scratch buf(al256(sizeof(pikv_entry) * n) + al256(8 * nl * n) + 8 * (size_t)n);
    if (buf.e != cudaSuccess) return fail(PIKV_ERR_CUDA, "score: cudaMalloc");
    const size_t o_ly = al256(sizeof(pikv_entry) * n), o_out = o_ly + al256(8 * nl * n);
    CUDA_TRY(cudaMemcpy(buf.at(0), entries, sizeof(pikv_entry) * n, cudaMemcpyHostToDevice));
    if (per_layer && nl) CUDA_TRY(cudaMemcpy(buf.at(o_ly), per_layer, 8 * nl * n, cudaMemcpyHostToDevice));
    launch_score_meta(C, (const pikv_entry*)buf.at(0), per_layer && nl ? (const double*)buf.at(o_ly) : nullptr,
                      (int)nl, n, now, (double*)buf.at(o_out), 0);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(out, buf.at(o_out), 8 * (size_t)n, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_evict_host(pikv_engine* eng, int32_t stream, uint64_t now, pikv_evict_record* out, int32_t cap,
                    int32_t* n_out, int32_t* pages_before, int32_t* pages_after) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    const Dims& D = eng->D;
    cudaStream_t st = eng->stream;
    const int Gl = std::max(D.Gl, 1);
    const size_t o = (size_t)stream * Gl;
    CUDA_TRY(cudaMemcpyAsync(eng->S.now + stream, &now, 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(eng->S.n_ev + o, 0, 4 * (size_t)Gl, st));
    CUDA_TRY(cudaMemsetAsync(eng->S.pages_before + o, 0, 4 * (size_t)Gl, st));
    CUDA_TRY(cudaMemsetAsync(eng->S.pages_after + o, 0, 4 * (size_t)Gl, st));
    Dims d1 = D;
    d1.only_s = stream;  // scheduler kernels for this stream only
    if (D.Gl > 0) {
        launch_sched_pages(d1, eng->C, eng->S, st);
        launch_sched_select(d1, eng->C, eng->S, st);
    }
    launch_state_op(D, eng->C, eng->S, stream, 2, 0, 0, nullptr, 0, 0.0, st);  // state.step++ (scheduler.cpp:328)
    CUDA_TRY(cudaGetLastError());
    std::vector<int32_t> nev(Gl), pb(Gl), pa(Gl);
    CUDA_TRY(cudaMemcpyAsync(nev.data(), eng->S.n_ev + o, 4 * (size_t)Gl, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(pb.data(), eng->S.pages_before + o, 4 * (size_t)Gl, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(pa.data(), eng->S.pages_after + o, 4 * (size_t)Gl, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    int32_t n = 0, sb = 0, sa = 0;
    for (int gl = 0; gl < D.Gl; ++gl) {
        sb += pb[gl], sa += pa[gl];
        const int ne = std::min(nev[gl], std::max(0, cap - n));
        if (out && ne > 0)
            CUDA_TRY(cudaMemcpy(out + n, eng->S.rec_ev + (o + gl) * D.SPD * D.S, sizeof(pikv_evict_record) * ne,
                                cudaMemcpyDeviceToHost));
        n += nev[gl];
    }
    if (n_out) *n_out = n;
    if (pages_before) *pages_before = sb;
    if (pages_after) *pages_after = sa;
    return PIKV_OK;
}

int pikv_attend_host(pikv_engine* eng, int32_t stream, const float* query, const int64_t* slots, int32_t n,
                     float* y_out, float* alpha_out) {
    int rc = component_check(eng, stream);
    if (rc) return rc;
    const Dims& D = eng->D;
    if (!query || !y_out || (n > 0 && !slots)) return fail(PIKV_ERR_INVALID_ARGUMENT, "attend: NULL argument");
    if (n == 0) {  // pipeline.cpp:63-66: zero vector, no weights
        std::memset(y_out, 0, sizeof(float) * D.dp);
        return PIKV_OK;
    }
    const int64_t ns = (int64_t)D.R * D.S;
    for (int i = 0; i < n; ++i)
        if (slots[i] < 0 || slots[i] >= ns) return fail(PIKV_ERR_INVALID_ARGUMENT, "attend: slot out of range");
    if ((size_t)n * 4 > 200 * 1024) return fail(PIKV_ERR_INVALID_ARGUMENT, "attend: too many entries for one call");
    const size_t kvb = 4 * (size_t)D.H * n * D.dph;
    const size_t o_sl = 0, o_q = al256(8 * (size_t)n), o_k = o_q + al256(4 * (size_t)D.dp), o_v = o_k + al256(kvb);
    const size_t o_y = o_v + al256(kvb), o_w = o_y + al256(4 * (size_t)D.dp), o_a = o_w + al256(4 * (size_t)D.H * n);
    Scratch buf(o_a + 4 * (size_t)n);
    if (buf.e != cudaSuccess) return fail(PIKV_ERR_CUDA, "attend: cudaMalloc");
    cudaStream_t st = eng->stream;
    CUDA_TRY(cudaMemcpyAsync(buf.at(o_sl), slots, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(buf.at(o_q), query, 4 * (size_t)D.dp, cudaMemcpyHostToDevice, st));
    launch_read_heads(D, eng->S, stream, (const int64_t*)buf.at(o_sl), n, (float*)buf.at(o_k), (float*)buf.at(o_v), st);
    const size_t smem = sizeof(float) * (size_t)n;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_attention<<<D.H, 256, smem, st>>>((const float*)buf.at(o_q), (const float*)buf.at(o_k), (const float*)buf.at(o_v),
                                        n, D.dph, (float*)buf.at(o_y), (float*)buf.at(o_w));
    launch_head_mean((const float*)buf.at(o_w), D.H, n, (float*)buf.at(o_a), st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(y_out, buf.at(o_y), 4 * (size_t)D.dp, cudaMemcpyDeviceToHost, st));
    if (alpha_out) CUDA_TRY(cudaMemcpyAsync(alpha_out, buf.at(o_a), 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return PIKV_OK;
}

int pikv_codec_encode(int32_t codec, int32_t rows, int32_t heads, int32_t hd, int32_t r, const float* basis,
                      const float* bias, const int32_t* kept, const float* x, float* y) {
    if (rows < 0 || heads < 1 || hd < 1) return fail(PIKV_ERR_INVALID_ARGUMENT, "codec: bad shape");
    switch (codec) {
        case PIKV_CODEC_IDENTITY:
            CUDA_TRY(cudaMemcpy(y, x, 4 * (size_t)rows * heads * hd, cudaMemcpyDeviceToDevice));
            return PIKV_OK;
        case PIKV_CODEC_LOWRANK:
        case PIKV_CODEC_LORAPLUS:
            if (!basis || (codec == PIKV_CODEC_LORAPLUS && !bias)) return fail(PIKV_ERR_NOT_FITTED, "codec: basis/bias");
            return pikv_lowrank_encode(x, basis, codec == PIKV_CODEC_LORAPLUS ? bias : nullptr, rows, heads, hd, r, y);
        case PIKV_CODEC_FASTV:
        case PIKV_CODEC_PRUNE:
            if (r < 1 || r > hd || (codec == PIKV_CODEC_PRUNE && !kept))
                return fail(PIKV_ERR_NOT_FITTED, "codec: rank / kept set");
            launch_codec_select(0, codec, rows, heads, hd, r, kept, x, y, 0);
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaDeviceSynchronize());
            return PIKV_OK;
    }
    return fail(PIKV_ERR_CODEC_MISMATCH, "codec_encode: int8/int4 use pikv_quantize");
}

int pikv_codec_decode(int32_t codec, int32_t rows, int32_t heads, int32_t hd, int32_t r, const float* basis,
                      const float* bias, const int32_t* kept, const float* y, float* x) {
    if (rows < 0 || heads < 1 || hd < 1) return fail(PIKV_ERR_INVALID_ARGUMENT, "codec: bad shape");
    switch (codec) {
        case PIKV_CODEC_IDENTITY:
            CUDA_TRY(cudaMemcpy(x, y, 4 * (size_t)rows * heads * hd, cudaMemcpyDeviceToDevice));
            return PIKV_OK;
        case PIKV_CODEC_LOWRANK:
        case PIKV_CODEC_LORAPLUS:
            if (!basis || (codec == PIKV_CODEC_LORAPLUS && !bias)) return fail(PIKV_ERR_NOT_FITTED, "codec: basis/bias");
            return pikv_lowrank_decode(y, basis, codec == PIKV_CODEC_LORAPLUS ? bias : nullptr, rows, heads, hd, r, x);
        case PIKV_CODEC_FASTV:
        case PIKV_CODEC_PRUNE:
            if (r < 1 || r > hd || (codec == PIKV_CODEC_PRUNE && !kept))
                return fail(PIKV_ERR_NOT_FITTED, "codec: rank / kept set");
            launch_codec_select(1, codec, rows, heads, hd, r, kept, y, x, 0);
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaDeviceSynchronize());
            return PIKV_OK;
    }
    return fail(PIKV_ERR_CODEC_MISMATCH, "codec_decode: int8/int4 use pikv_dequantize");
}

static int codec_host(bool decode, int32_t codec, int32_t rows, int32_t heads, int32_t hd, int32_t r,
                      const float* basis, const float* bias, const int32_t* kept, const float* in, float* out) {
    const int wi = decode ? (codec == PIKV_CODEC_IDENTITY ? hd : r) : hd;
    const int wo = decode ? hd : (codec == PIKV_CODEC_IDENTITY ? hd : r);
    const size_t nin = 4 * (size_t)rows * heads * wi, nout = 4 * (size_t)rows * heads * wo;
    const size_t nb = basis ? 4 * (size_t)heads * r * hd : 0, nbias = bias ? 4 * (size_t)heads * hd : 0;
    const size_t nk = kept ? 4 * (size_t)heads * r : 0;
    const size_t o_in = 0, o_out = al256(nin), o_b = o_out + al256(nout), o_bias = o_b + al256(nb);
    const size_t o_k = o_bias + al256(nbias);
    Scratch buf(o_k + nk + 16);
    if (buf.e != cudaSuccess) return fail(PIKV_ERR_CUDA, "codec: cudaMalloc");
    CUDA_TRY(cudaMemcpy(buf.at(o_in), in, nin, cudaMemcpyHostToDevice));
    if (nb) CUDA_TRY(cudaMemcpy(buf.at(o_b), basis, nb, cudaMemcpyHostToDevice));
    if (nbias) CUDA_TRY(cudaMemcpy(buf.at(o_bias), bias, nbias, cudaMemcpyHostToDevice));
    if (nk) CUDA_TRY(cudaMemcpy(buf.at(o_k), kept, nk, cudaMemcpyHostToDevice));
    auto* fb = nb ? (const float*)buf.at(o_b) : nullptr;
    auto* fbias = nbias ? (const float*)buf.at(o_bias) : nullptr;
    auto* fk = nk ? (const int32_t*)buf.at(o_k) : nullptr;
    int rc = decode ? pikv_codec_decode(codec, rows, heads, hd, r, fb, fbias, fk, (const float*)buf.at(o_in),
                                        (float*)buf.at(o_out))
                    : pikv_codec_encode(codec, rows, heads, hd, r, fb, fbias, fk, (const float*)buf.at(o_in),
                                        (float*)buf.at(o_out));
    if (rc) return rc;
    CUDA_TRY(cudaMemcpy(out, buf.at(o_out), nout, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

int pikv_codec_encode_host(int32_t codec, int32_t rows, int32_t heads, int32_t hd, int32_t r, const float* basis,
                           const float* bias, const int32_t* kept, const float* x, float* y) {
    return codec_host(false, codec, rows, heads, hd, r, basis, bias, kept, x, y);
}

int pikv_codec_decode_host(int32_t codec, int32_t rows, int32_t heads, int32_t hd, int32_t r, const float* basis,
                           const float* bias, const int32_t* kept, const float* y, float* x) {
    return codec_host(true, codec, rows, heads, hd, r, basis, bias, kept, y, x);
}

int pikv_column_variance_host(const double* rows, int32_t n, int32_t d, double* var) {
    if (n < 1 || d < 1 || !rows || !var) return fail(PIKV_ERR_INSUFFICIENT_CALIBRATION, "column variance: no rows");
    const size_t nx = 8 * (size_t)n * d;
    Scratch buf(al256(nx) + 8 * (size_t)d);
    if (buf.e != cudaSuccess) return fail(PIKV_ERR_CUDA, "variance: cudaMalloc");
    CUDA_TRY(cudaMemcpy(buf.at(0), rows, nx, cudaMemcpyHostToDevice));
    launch_col_var((const double*)buf.at(0), n, d, (double*)buf.at(al256(nx)), 0);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(var, buf.at(al256(nx)), 8 * (size_t)d, cudaMemcpyDeviceToHost));
    return PIKV_OK;
}

// ---------------------------------------------------------------------------
// micro-batch pipeline
// ---------------------------------------------------------------------------
struct pikv_group {
    int n = 0;
    int device = 0;
    std::vector<pikv_engine*> eng;
    std::vector<cudaEvent_t> att_done;  // per micro-batch: its last attention
    std::vector<cudaEvent_t> y_done;    // per micro-batch: its last y written
    std::vector<cudaEvent_t> y_ready;   // host path: y merged on the device
    std::vector<cudaStream_t> side;     // host path: D2H of y beside the fold-back
    cudaEvent_t join = nullptr;
    bool timing = false;
    // timing: per micro-batch, event pairs of submitted steps not yet read
    std::vector<std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> tev;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tfree;
    size_t in_bytes = 0, y_bytes = 0, sal_elems = 0;  // per micro-batch
    // Attention SM partition (PIKV_GREEN=1): a green context owning the
    // attention SMs; each micro-batch's attention graph is captured and run on
    // its own stream in it, so the two micro-batches' attention launches need
    // no ordering (the next one's CTAs take the partition's SMs as the
    // previous one's finish) and can never take the control plane's SMs.
    CUgreenCtx gctx = nullptr;
    std::vector<cudaStream_t> att_st;
    std::vector<cudaEvent_t> ctl_done;
    // timeline probe (PIKV_GROUP_TIMELINE=1 at create; pikv_group_read_timeline):
    // per submit, events before / after the control graph, after the cross-
    // micro-batch wait, after the attention graph, after the tail
    bool timeline = false;
    struct TL {
        int m;
        cudaEvent_t ev[5];
    };
    std::vector<TL> tl;
};

// Driver entry points for green contexts (no link against libcuda: the
// library must load on hosts without a driver, e.g. for the CPU tests).
static void* drv(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return fn;
}

// A green context of `sms` SMs (a multiple of 8) and one stream in it per
// micro-batch; false (nothing created) when the driver cannot provide it.
static bool make_attention_partition(pikv_group* g, int sms) {
    using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
    using Split = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                               unsigned int);
    using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
    using Create = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
    using StreamCreate = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);
    using DevGet = CUresult (*)(CUdevice*, int);
    auto dev_get = reinterpret_cast<DevGet>(drv("cuDeviceGet"));
    auto get_res = reinterpret_cast<GetRes>(drv("cuDeviceGetDevResource"));
    auto split = reinterpret_cast<Split>(drv("cuDevSmResourceSplitByCount"));
    auto gen = reinterpret_cast<GenDesc>(drv("cuDevResourceGenerateDesc"));
    auto create = reinterpret_cast<Create>(drv("cuGreenCtxCreate"));
    auto screate = reinterpret_cast<StreamCreate>(drv("cuGreenCtxStreamCreate"));
    if (!dev_get || !get_res || !split || !gen || !create || !screate) return false;
    CUdevice dev;
    CUdevResource all{}, part[1]{}, rest{};
    unsigned int ng = 1;
    CUdevResourceDesc desc;
    if (dev_get(&dev, g->device) != CUDA_SUCCESS || get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
        return false;
    if (split(part, &ng, &all, &rest, 0, (unsigned)sms) != CUDA_SUCCESS || ng != 1 ||
        (int)part[0].sm.smCount != sms)
        return false;
    if (gen(&desc, part, 1) != CUDA_SUCCESS || create(&g->gctx, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
        return false;
    for (int m = 0; m < g->n; ++m) {
        CUstream st = nullptr;
        if (screate(&st, g->gctx, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return false;
        g->att_st.push_back((cudaStream_t)st);
        cudaEvent_t ev;
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        g->ctl_done.push_back(ev);
    }
    return true;
}

int pikv_group_create(const pikv_config* cfg, int32_t n_micro, int32_t attend_sms, int32_t cuda_device,
                      pikv_group** out) {
    *out = nullptr;
    if (n_micro < 1 || cfg->batch % n_micro != 0)
        return fail(PIKV_ERR_INVALID_CONFIG, "batch must be a multiple of n_micro");

    int rc = validate(*cfg);
    if (rc) return rc;
    CUDA_TRY(cudaSetDevice(cuda_device));
    auto* g = new pikv_group();
    g->n = n_micro;
    g->device = cuda_device;
    pikv_config c = *cfg;
    c.batch = cfg->batch / n_micro;
    if (cfg->pool_entries > 0) c.pool_entries = cfg->pool_entries / n_micro;
    // leave SMs to the control plane of the other micro-batch: all but
    // attend_reserve_sms(layout) (sweeps in profiles/README.md: c2 flat at
    // 44 K from 100 to 116 SMs, c4-int8 39.7 K at 136 vs 36.6 K at 148,
    // c4-low-rank on the HMMA kernel 77.6-78.0 K at 108 vs 76.2-76.9 K at 116)
    if (attend_sms <= 0 && n_micro > 1) attend_sms = -1;
    for (int m = 0; m < n_micro; ++m) {
        pikv_engine* e = nullptr;
        // 2 work items per attention CTA in the pipeline (c2: 1 -> 37.6 K,
        // 2 -> 43.3 K, 4 -> 42.2 K, 8 -> 39.5 K tokens/s): half the split-K
        // partials of 4 and the item ticket absorbs the imbalance
        rc = engine_create(&c, cuda_device, attend_sms, &e, 2);
        if (rc) {
            pikv_group_destroy(g);
            return rc;
        }
        // the cluster control kernel (one CTA per SM per cluster rank) cannot
        // share SMs with the other micro-batch's attention: use the multi-kernel
        // control plane unless PIKV_CONTROL=1 forces it
        const char* cv = std::getenv("PIKV_CONTROL");
        if (!(cv && cv[0] == '1')) e->fused_control = false;
        g->eng.push_back(e);
        cudaEvent_t a, y;
        // att_done keeps timing enabled: the other micro-batch's attention waits
        // on it, and a DisableTiming event recorded right behind the attention
        // graph launch released that wait later (e2e step 0.398 -> 0.357 ms at
        // c2, profiles/microbench/e2e_timing_ab.py)
        cudaEventCreate(&a);
        cudaEventCreateWithFlags(&y, cudaEventDisableTiming);
        g->att_done.push_back(a);
        g->y_done.push_back(y);
        cudaEvent_t yr;
        cudaStream_t sd;
        cudaEventCreate(&yr);  // timing enabled: waited on by the side stream (see att_done)
        cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking);
        g->y_ready.push_back(yr);
        g->side.push_back(sd);

    }
    cudaEventCreateWithFlags(&g->join, cudaEventDisableTiming);
    g->tev.resize(n_micro);
    // default for the CUDA-core attention kernel (two CTAs per SM): c2 45.3 ->
    // 49.4 K tokens/s, c3 44.7 -> 46.2 K, c5 157 -> 163 K; the one-CTA-per-SM
    // tensor-core kernels lose 2-3 % (their control-bound steps lose the SMs
    // the attention gaps used to free): profiles/README.md.  PIKV_GREEN=0 / 1
    // overrides.  Sharded groups too: the attention part has no collective
    // (the all-gather follows in the merge part, on the engine stream).
    // The one-CTA-per-SM tensor-core kernels gain from it from four
    // micro-batches on (c4-lowrank 77.8 -> 81.9 K, c4-int4 72.1 -> 74.8 K
    // tokens/s), not with two.
    // Not by default under a CUDA tool that injects itself (the environment
    // variables ncu / nsys / compute-sanitizer set): ncu cannot prepare every
    // kernel of a green context for profiling (an all-kernel launch list
    // failed with an unknown error), and the tools' kernel lists must not
    // depend on it.
    const char* gv = std::getenv("PIKV_GREEN");
    bool tool = false;  // injected by ncu / nsys / compute-sanitizer / CUPTI injection
    for (const char* var : {"CUDA_INJECTION64_PATH", "NV_TPS_LAUNCH_TOKEN", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE",
                            "NVIDIA_PROCESS_INJECTION_CRASH_REPORTING"}) {
        const char* v = std::getenv(var);
        tool = tool || (v && v[0]);
    }
    const bool want_green =
        gv ? gv[0] == '1' : !tool && (attend_ctas_per_sm(g->eng[0]->D) == 2 || n_micro >= 4);
    if (want_green && n_micro > 1) {
        // the partition holds the attention grid's SMs, rounded down to the
        // green-context granularity (8 SMs on sm_90+)
        const int cps = std::max(1, attend_ctas_per_sm(g->eng[0]->D));
        const int sms = (g->eng[0]->D.attend_ctas / cps) & ~7;
        if (sms >= 8 && make_attention_partition(g, sms)) {
            // with the partition the static shares win at every batch (c5, 32
            // streams per engine: 165.5 vs 162.9 K tokens/s with tickets; c4-int8
            // 39.6 vs 38.5-39.1 K): no other micro-batch's control kernels hold
            // attention SMs, so the CTAs start together
            const bool share_env = std::getenv("PIKV_ATT_SHARE") != nullptr;
            for (auto* e : g->eng) {
                e->D.attend_ctas = cps * sms;
                if (!share_env && e->D.B >= 2) e->D.att_share = 1;
            }
        } else {
            for (auto st : g->att_st) cudaStreamDestroy(st);
            for (auto ev : g->ctl_done) cudaEventDestroy(ev);
            g->att_st.clear(), g->ctl_done.clear();
            g->gctx = nullptr;  // (a partly created context is left to process exit)
        }
    }
    if (const char* tv = std::getenv("PIKV_GROUP_TIMELINE")) g->timeline = tv[0] == '1';
    const Dims& D = g->eng[0]->D;
    g->in_bytes = (size_t)D.B * D.d * (D.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4);
    g->y_bytes = sizeof(float) * (size_t)D.B * D.dp;
    g->sal_elems = (size_t)D.B * D.n_layers;
    *out = g;
    return PIKV_OK;
}

int pikv_group_destroy(pikv_group* g) {
    if (!g) return PIKV_OK;
    cudaSetDevice(g->device);
    for (auto* e : g->eng) pikv_engine_destroy(e);
    for (auto e : g->att_done) cudaEventDestroy(e);
    for (auto e : g->y_done) cudaEventDestroy(e);
    for (auto e : g->y_ready) cudaEventDestroy(e);
    for (auto st : g->side) cudaStreamSynchronize(st), cudaStreamDestroy(st);
    for (auto& v : g->tev)
        for (auto& p : v) cudaEventDestroy(p.first), cudaEventDestroy(p.second);
    for (auto& p : g->tfree) cudaEventDestroy(p.first), cudaEventDestroy(p.second);
    if (g->join) cudaEventDestroy(g->join);
    for (auto& r : g->tl)
        for (auto ev : r.ev) cudaEventDestroy(ev);
    for (auto st : g->att_st) cudaStreamSynchronize(st), cudaStreamDestroy(st);
    for (auto ev : g->ctl_done) cudaEventDestroy(ev);
    if (g->gctx) {
        using Destroy = CUresult (*)(CUgreenCtx);
        if (auto d = reinterpret_cast<Destroy>(drv("cuGreenCtxDestroy"))) d(g->gctx);
    }
    delete g;
    return PIKV_OK;
}

int pikv_group_size(pikv_group* g) { return g->n; }

pikv_engine* pikv_group_engine(pikv_group* g, int32_t m) {
    return m >= 0 && m < g->n ? g->eng[m] : nullptr;
}

static thread_local cudaEvent_t* g_tl_rec = nullptr;
static void Group_TL_begin(pikv_group* g, int m) {
    pikv_group::TL r;
    r.m = m;
    for (auto& ev : r.ev) cudaEventCreate(&ev);
    g->tl.push_back(r);
}

int pikv_group_submit(pikv_group* g, int32_t m, const void* q, const void* k, const void* v,
                      const double* sal, float* y, int32_t host) {
    if (m < 0 || m >= g->n) return fail(PIKV_ERR_INVALID_ARGUMENT, "micro-batch index out of range");
    pikv_engine* e = g->eng[m];
    cudaSetDevice(g->device);
    int rc = codec_ready(e);
    if (rc) return rc;
    cudaStream_t st = e->stream;
    const void *dq = q, *dk = k, *dv = v;
    const double* ds = sal;
    float* dy = y;
    if (host) {
        const uint8_t* hq = (const uint8_t*)q;
        if ((const uint8_t*)k == hq + g->in_bytes && (const uint8_t*)v == hq + 2 * g->in_bytes) {
            // q, k, v packed back to back: one transfer into the packed staging
            CUDA_TRY(cudaMemcpyAsync(e->in_q, q, 3 * g->in_bytes, cudaMemcpyHostToDevice, st));
        } else {
            CUDA_TRY(cudaMemcpyAsync(e->in_q, q, g->in_bytes, cudaMemcpyHostToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(e->in_k, k, g->in_bytes, cudaMemcpyHostToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(e->in_v, v, g->in_bytes, cudaMemcpyHostToDevice, st));
        }
        if (sal && g->sal_elems)
            CUDA_TRY(cudaMemcpyAsync(e->in_sal, sal, sizeof(double) * g->sal_elems, cudaMemcpyHostToDevice, st));
        dq = e->in_q, dk = e->in_k, dv = e->in_v, ds = sal ? e->in_sal : nullptr, dy = e->out_y;
    }
    if (e->profiling) {
        rc = run_step(e, dq, dk, dv, ds, dy, true);
    } else {
        // control graph -> [wait for the previous micro-batch's attention] ->
        // attention graph -> [record] -> tail graph; the ordering is stream
        // API calls between the graph launches.  (Attention on a separate
        // highest-priority stream measured slower: 37.5 vs 42.1 K tokens/s at c2.)
        g_tl_rec = nullptr;
        if (g->timeline && !host && g->tl.size() < 4096) {
            Group_TL_begin(g, m);
            g_tl_rec = g->tl.back().ev;
            CUDA_TRY(cudaEventRecord(g_tl_rec[0], st));
        }
        rc = run_step(e, dq, dk, dv, ds, dy, true, nullptr, kPartCtl);
        if (g_tl_rec) CUDA_TRY(cudaEventRecord(g_tl_rec[1], st));
        if (!rc) {
            // (unordered attention launches measured: c2 43.8 vs 43.7 K, c5 145 vs 154 K)
            // attention stream: the engine stream (ordered after the previous
            // micro-batch's attention), or this micro-batch's stream in the
            // attention partition (no ordering needed)
            const bool green = !g->att_st.empty();
            cudaStream_t ast = green ? g->att_st[m] : st;
            if (green) {
                CUDA_TRY(cudaEventRecord(g->ctl_done[m], st));
                CUDA_TRY(cudaStreamWaitEvent(ast, g->ctl_done[m], 0));
            } else if (g->n > 1) {
                CUDA_TRY(cudaStreamWaitEvent(st, g->att_done[(m + g->n - 1) % g->n], 0));
            }
            if (g_tl_rec) CUDA_TRY(cudaEventRecord(g_tl_rec[2], ast));
            std::pair<cudaEvent_t, cudaEvent_t> p{nullptr, nullptr};
            if (g->timing && g->tev[m].size() < 8192) {  // bounded until pikv_group_read_timing
                if (g->tfree.empty()) {
                    CUDA_TRY(cudaEventCreate(&p.first));
                    CUDA_TRY(cudaEventCreate(&p.second));
                } else {
                    p = g->tfree.back();
                    g->tfree.pop_back();
                }
                g->tev[m].push_back(p);
                CUDA_TRY(cudaEventRecord(p.first, ast));
            }
            // the attention graph is captured and replayed on ast (a graph
            // captured on another stream would run on every SM)
            e->stream = ast;
            rc = run_step(e, dq, dk, dv, ds, dy, true, nullptr, kPartAttend);
            e->stream = st;
            if (p.second) CUDA_TRY(cudaEventRecord(p.second, ast));
            CUDA_TRY(cudaEventRecord(g->att_done[m], ast));
            if (green) CUDA_TRY(cudaStreamWaitEvent(st, g->att_done[m], 0));
            if (g_tl_rec) CUDA_TRY(cudaEventRecord(g_tl_rec[3], ast));
        }
        if (!host) {
            if (!rc) rc = run_step(e, dq, dk, dv, ds, dy, true, nullptr, kPartTail);
            if (!rc && g_tl_rec) CUDA_TRY(cudaEventRecord(g_tl_rec[4], st));
        } else if (e->exchange_path()) {
            // sharded over ranks: y is final after the all-gather and the
            // cross-rank merge, inside the fold part; the fold graph records
            // y_ready right after the merge (y_final_event) and the D2H on
            // the side stream overlaps the fold-back
            if (!rc) CUDA_TRY(cudaStreamWaitEvent(st, g->y_done[m], 0));
            if (!rc) rc = run_step(e, dq, dk, dv, ds, dy, true, nullptr, kPartMerge);
            e->y_final_event = g->y_ready[m];
            if (!rc) rc = run_step(e, dq, dk, dv, ds, dy, true, nullptr, kPartFold);
            e->y_final_event = nullptr;
            if (!rc) {
                CUDA_TRY(cudaStreamWaitEvent(g->side[m], g->y_ready[m], 0));
                CUDA_TRY(cudaMemcpyAsync(y, e->out_y, g->y_bytes, cudaMemcpyDeviceToHost, g->side[m]));
                CUDA_TRY(cudaEventRecord(g->y_done[m], g->side[m]));
            }
        } else {
            // y leaves for the host on a side stream as soon as the merge wrote
            // it, while the fold-back runs: the caller's wait returns earlier
            // the merge rewrites out_y: order it after the previous step's D2H
            // of out_y on the side stream (a no-op in the steady state)
            if (!rc) CUDA_TRY(cudaStreamWaitEvent(st, g->y_done[m], 0));
            if (!rc) rc = run_step(e, dq, dk, dv, ds, dy, true, nullptr, kPartMerge);
            if (!rc) {
                CUDA_TRY(cudaEventRecord(g->y_ready[m], st));
                CUDA_TRY(cudaStreamWaitEvent(g->side[m], g->y_ready[m], 0));
                CUDA_TRY(cudaMemcpyAsync(y, e->out_y, g->y_bytes, cudaMemcpyDeviceToHost, g->side[m]));
                CUDA_TRY(cudaEventRecord(g->y_done[m], g->side[m]));
                rc = run_step(e, dq, dk, dv, ds, dy, true, nullptr, kPartFold);
            }
        }
    }
    if (rc) return rc;
    if (e->profiling && host) CUDA_TRY(cudaMemcpyAsync(y, e->out_y, g->y_bytes, cudaMemcpyDeviceToHost, st));
    if (!host || e->profiling) CUDA_TRY(cudaEventRecord(g->y_done[m], st));
    return PIKV_OK;
}

int pikv_group_attach_nccl(pikv_group* g, const uint8_t* ids) {
    if (!g || !ids) return fail(PIKV_ERR_INVALID_ARGUMENT, "NULL argument");
    for (int m = 0; m < g->n; ++m) {  // one communicator per micro-batch stream
        const int rc = pikv_engine_attach_nccl(g->eng[m], ids + (size_t)m * PIKV_NCCL_ID_BYTES);
        if (rc) return rc;
    }
    return PIKV_OK;
}

int pikv_group_wait(pikv_group* g, int32_t m) {
    if (m < 0 || m >= g->n) return fail(PIKV_ERR_INVALID_ARGUMENT, "micro-batch index out of range");
    CUDA_TRY(cudaEventSynchronize(g->y_done[m]));
    return PIKV_OK;
}

int pikv_group_step(pikv_group* g, const void* q, const void* k, const void* v, const double* sal,
                    float* y) {
    for (int m = 0; m < g->n; ++m) {
        const size_t o = (size_t)m * g->in_bytes;
        int rc = pikv_group_submit(g, m, (const uint8_t*)q + o, (const uint8_t*)k + o, (const uint8_t*)v + o,
                                   sal ? sal + (size_t)m * g->sal_elems : nullptr,
                                   y ? (float*)((uint8_t*)y + (size_t)m * g->y_bytes) : nullptr, 0);
        if (rc) return rc;
    }
    return PIKV_OK;
}

int pikv_group_join(pikv_group* g) {
    cudaSetDevice(g->device);
    cudaStream_t s0 = g->eng[0]->stream;
    for (int m = 0; m < g->n; ++m) {
        if (m) {
            CUDA_TRY(cudaEventRecord(g->join, g->eng[m]->stream));
            CUDA_TRY(cudaStreamWaitEvent(s0, g->join, 0));
        }
        CUDA_TRY(cudaEventRecord(g->join, g->side[m]));
        CUDA_TRY(cudaStreamWaitEvent(s0, g->join, 0));
    }
    return PIKV_OK;
}

int pikv_group_sync(pikv_group* g) {
    for (auto st : g->side) CUDA_TRY(cudaStreamSynchronize(st));
    for (auto* e : g->eng) {
        int rc = pikv_sync(e);
        if (rc) return rc;
    }
    return PIKV_OK;
}

int pikv_group_set_timing(pikv_group* g, int32_t on) {
    g->timing = on != 0;
    return PIKV_OK;
}

int pikv_group_attention_partition(pikv_group* g) { return g && g->gctx ? 1 : 0; }

int pikv_group_read_timing_union(pikv_group* g, double* sum_ms, double* union_ms, int32_t* n) {
    // attention launches of all micro-batches as [start, end] on one time
    // axis; with overlapping launches (attention partition) the union is the
    // time the attention kernels had the GPU
    std::vector<std::pair<double, double>> iv;
    cudaEvent_t ref = nullptr;
    for (auto& v : g->tev)
        for (auto& p : v) {
            CUDA_TRY(cudaEventSynchronize(p.second));
            if (!ref) ref = p.first;
        }
    double tot = 0;
    for (auto& v : g->tev) {
        for (auto& p : v) {
            float a = 0, b = 0;
            CUDA_TRY(cudaEventElapsedTime(&a, ref, p.first));
            CUDA_TRY(cudaEventElapsedTime(&b, ref, p.second));
            iv.emplace_back(a, b);
            tot += b - a;
            g->tfree.push_back(p);
        }
        v.clear();
    }
    std::sort(iv.begin(), iv.end());
    double uni = 0, cs = 0, ce = -1e300;
    for (auto& x : iv) {
        if (x.first > ce) {
            if (ce > cs) uni += ce - cs;
            cs = x.first, ce = x.second;
        } else {
            ce = std::max(ce, x.second);
        }
    }
    if (!iv.empty() && ce > cs) uni += ce - cs;
    if (sum_ms) *sum_ms = tot;
    if (union_ms) *union_ms = uni;
    if (n) *n = (int32_t)iv.size();
    return PIKV_OK;
}

int pikv_group_read_timing(pikv_group* g, double* ms, int32_t* n) {
    double tot = 0;
    int cnt = 0;
    for (auto& v : g->tev) {
        for (auto& p : v) {
            CUDA_TRY(cudaEventSynchronize(p.second));
            float t = 0;
            CUDA_TRY(cudaEventElapsedTime(&t, p.first, p.second));
            tot += t, ++cnt;
            g->tfree.push_back(p);
        }
        v.clear();
    }
    if (ms) *ms = tot;
    if (n) *n = cnt;
    return PIKV_OK;
}

/* Debug probe: rows of (m, ctl_start, ctl_end, wait_done, attend_end, tail_end)
 * in ms relative to the first recorded submit; clears the record. */
int pikv_group_read_timeline(pikv_group* g, double* out, int32_t cap, int32_t* n) {
    int cnt = 0;
    if (!g->tl.empty()) {
        CUDA_TRY(cudaEventSynchronize(g->tl.back().ev[4]));
        for (auto& r : g->tl) {
            if (cnt < cap) {
                out[6 * cnt] = r.m;
                for (int i = 0; i < 5; ++i) {
                    float t = 0;
                    CUDA_TRY(cudaEventElapsedTime(&t, g->tl[0].ev[0], r.ev[i]));
                    out[6 * cnt + 1 + i] = t;
                }
                ++cnt;
            }
        }
        for (auto& r : g->tl)
            for (auto ev : r.ev) cudaEventDestroy(ev);
        g->tl.clear();
    }
    if (n) *n = cnt;
    return PIKV_OK;
}

}  // extern "C"
