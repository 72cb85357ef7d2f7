// SPDX-License-Identifier: Apache-2.0
//
// Per-step kernels of the B200 PiKV engine except decode attention
// (attend.cu).  One launch each, all on the engine stream, graph-capturable:
//
//   route      router.cpp:216-234 + 122-214 (+ codec query projection,
//              pipeline.cpp:295-297) and the retrieval candidate rings
//   insert     kvstore.cpp:107-120 + 36-53, pipeline.cpp:148-211
//   sched      scheduler.cpp:262-330 (score + page aggregate, select, erase)
//   retrieve   kvstore.cpp:122-178 (filter, compact, freq/recency bump)
//   combine    per-stream LSE merge of the attention work items
//   finish     cross-rank LSE merge -> y, global (m, l); hits/misses
//   foldback   pipeline.cpp:302-312 (attn_mass += alpha)
//   feedback   pipeline.cpp:337-347 (adapt, observe_hits, adakv_update), now++
//
// Bit-exactness: all fp64 arithmetic that the reference performs with plain
// * and + is written with __dmul_rn/__dadd_rn so nvcc cannot contract it into
// FMAs, and every reduction keeps the reference's sequential order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "pikv_dev.cuh"

namespace cg = cooperative_groups;

namespace pikv_dev {

constexpr int kMaxCluster = 8;  // k_control CTAs per stream

// ===========================================================================
// route
// ===========================================================================
// One CTA per stream.  The logits are the reference's sequential fp64 dot
// (router.cpp:229-231): s = ((0 + w0 q0) + w1 q1) + ...; thread e < E runs
// that dependent DMUL/DADD chain for expert e in column order (the rounding
// semantics make it sequential; __dmul_rn/__dadd_rn forbid FMA contraction).
// W_r rows stream through an NST-stage shared-memory ring filled by TMA bulk
// copies (one per expert row segment, issued by the producer lane of the
// last warp), so the chain never waits on L2.  Thread 0 then runs the
// strategy penalty, selection, gate softmax and note_selection.
__device__ __forceinline__ void route_select(const Dims& D, const Cfg& C, const State& S, int s,
                                             double* sm_logit, bool* sm_flag, int* sm_pool,
                                             double* load, uint64_t* usage, const uint64_t* miss,
                                             const double* bias, int* sel, const uint64_t* pre, int* errf);

constexpr int kRouteCHMax = 256;  // columns per stage (reduced so E rows x stages fit)
constexpr int kRouteStages = 5;

// Route stream s with the calling CTA (k_route, k_control); sm_raw = the
// dynamic shared memory (route_smem_bytes(CH)).
__device__ __forceinline__ const int* route_body(const Dims& D, const Cfg& C, const State& S, const int s,
                                           const void* __restrict__ qin, const int kRouteCH,
                                           uint8_t* sm_raw, const double* logits_in = nullptr) {
    uint64_t* full = (uint64_t*)sm_raw;
    uint64_t* empty = full + kRouteStages;
    double* sm_q = (double*)(sm_raw + 128);
    const int rowb = kRouteCH * 8 + 16;  // padded row: 2-way bank conflicts at worst (CH % 32 == 0)
    uint8_t* ring = (uint8_t*)(sm_q + D.d);
    __shared__ double sm_logit[kMaxE];
    __shared__ bool sm_flag[kMaxE];
    __shared__ int sm_pool[kMaxE];
    __shared__ double sm_load[kMaxE], sm_bias[kMaxE];
    __shared__ uint64_t sm_usage[kMaxE], sm_miss[kMaxE];
    __shared__ int sm_sel[kMaxK];
    const int tid = threadIdx.x;
    const int nsum_warps = (D.E + 31) / 32;
    const int prod_warp = nsum_warps;  // last warp
    // per-step scratch counters of this stream (replaces memset nodes)
    if (tid == 0) S.n_ow[s] = 0;
    for (int g = tid; g < D.Gl; g += blockDim.x) {
        S.n_ev[s * D.Gl + g] = 0;
        S.pages_before[s * D.Gl + g] = 0;
        S.pages_after[s * D.Gl + g] = 0;
    }
    for (int j = tid; j < D.k; j += blockDim.x) S.found[(int64_t)s * D.k + j] = 0;
    if (S.err[s]) return nullptr;
    // router state of this stream -> smem (thread 0's serial part reads it
    // without dependent global round trips)
    for (int e = tid; e < D.E; e += blockDim.x) {
        sm_load[e] = S.load[(int64_t)s * D.E + e];
        sm_usage[e] = S.usage[(int64_t)s * D.E + e];
        sm_miss[e] = S.miss[(int64_t)s * D.E + e];
        sm_bias[e] = S.bias[(int64_t)s * D.E + e];
    }
    // the selection's scalar state, fetched while the logit chains run
    __shared__ uint64_t sm_pre[2];  // total_usage, rstep
    __shared__ int sm_errf;         // set by route_select (NaN logits)
    if (tid == 0) sm_pre[0] = S.total_usage[s], sm_pre[1] = S.rstep[s], sm_errf = 0;
    const bool dbg = D.dbg_ctl && s == 0 && tid == 0 && S.dbg;  // PIKV_DEBUG_CTL timestamps
    if (dbg) S.dbg[0] = clock64();
    if (tid == 0) {
        for (int i = 0; i < kRouteStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], nsum_warps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // query in fp64 (exact upcast of bf16/f32, or the encoder's fp64 q);
    // 16-byte loads, all in flight.  route_logits (logits_in): no query
    if (logits_in) {
    } else if (D.q_f64) {
        const double2* qd = (const double2*)((const double*)qin + (int64_t)s * D.d);
        if (D.d % 2 == 0)
            for (int v = tid; v < D.d / 2; v += blockDim.x) ((double2*)sm_q)[v] = qd[v];
        else
            for (int i = tid; i < D.d; i += blockDim.x) sm_q[i] = ((const double*)qin)[(int64_t)s * D.d + i];
    } else {
        const int esz = D.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4;
        const int nvec = (D.d * esz) / 16;
        const uint8_t* qb = (const uint8_t*)qin + (int64_t)s * D.d * esz;
        if ((D.d * esz) % 16 == 0) {
            for (int v0 = tid; v0 < nvec; v0 += 8 * blockDim.x) {
                uint4 w[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int v = v0 + u * blockDim.x;
                    if (v < nvec) w[u] = ((const uint4*)qb)[v];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int v = v0 + u * blockDim.x;
                    if (v >= nvec) continue;
                    const uint32_t ww[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
                    if (esz == 2) {
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            sm_q[v * 8 + 2 * t] = (double)bf16_lo(ww[t]);
                            sm_q[v * 8 + 2 * t + 1] = (double)bf16_hi(ww[t]);
                        }
                    } else {
#pragma unroll
                        for (int t = 0; t < 4; ++t) sm_q[v * 4 + t] = (double)__uint_as_float(ww[t]);
                    }
                }
            }
        } else {
            for (int i = tid; i < D.d; i += blockDim.x) {
                double x;
                if (esz == 2)
                    x = (double)__uint_as_float(((uint32_t)((const uint16_t*)qin)[(int64_t)s * D.d + i]) << 16);
                else
                    x = (double)((const float*)qin)[(int64_t)s * D.d + i];
                sm_q[i] = x;
            }
        }
    }
    __syncthreads();
    if (dbg) S.dbg[1] = clock64();
    const bool base = C.router_strategy == PIKV_ROUTER_BASE;
    if (logits_in && !base) {  // route_logits, router.cpp:122-214: the given logits
        for (int e = tid; e < D.E; e += blockDim.x) sm_logit[e] = logits_in[e];
        __syncthreads();
    }
    if (!base && !logits_in && C.route_mode == PIKV_ROUTE_FAST) {
        // fast routing: the same fp64 products reduced as a tree (FMA, warp
        // shuffles) instead of the reference's sequential sum -- logits differ
        // in rounding order only; one warp per expert, W read from L2
        // (k_route launches one warp per expert in this mode; four independent
        // accumulators keep the L2 loads in flight)
        const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
        const int CH = kRouteCH, rs = CH + 2;
        for (int e = warp; e < D.E; e += nw) {
            double a[4] = {0.0, 0.0, 0.0, 0.0};
            for (int c0 = 0; c0 < D.d; c0 += CH) {
                const double* row = S.W + ((size_t)(c0 / CH) * D.E + e) * rs;
                const double* qq = sm_q + c0;
                const int w = min(CH, D.d - c0);
                if (w == CH) {
#pragma unroll
                    for (int u = 0; u < kRouteCHMax / 32; ++u)
                        if (u * 32 < CH) a[u & 3] = fma(row[lane + u * 32], qq[lane + u * 32], a[u & 3]);
                } else {
                    for (int i = lane; i < w; i += 32) a[0] = fma(row[i], qq[i], a[0]);
                }
            }
            double acc = (a[0] + a[1]) + (a[2] + a[3]);
            for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) sm_logit[e] = acc;
        }
        __syncthreads();
    } else if (!base && !logits_in) {
        const int E = D.E, CH = kRouteCH;
        const int nchunk = (D.d + CH - 1) / CH;
        const int warp = tid >> 5, lane = tid & 31;
        if (warp == prod_warp) {
            if (lane == 0) {
                int stage = 0;
                uint32_t phase = 0;
                // W is stored chunk-major with padded rows (State::W), so a
                // stage is one contiguous bulk copy of E padded rows
                const uint32_t bytes = (uint32_t)(E * rowb);
                for (int c = 0; c < nchunk; ++c) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], bytes);
                    bulk_g2s_plain(ring + (size_t)stage * E * rowb, (const uint8_t*)S.W + (size_t)c * bytes, bytes,
                                   &full[stage]);
                    if (++stage == kRouteStages) stage = 0, phase ^= 1;
                }
            }
        } else if (warp < nsum_warps) {
            double acc = 0.0;
            int stage = 0;
            uint32_t phase = 0;
            const int e = tid;
            long long t_wait = 0;
            const bool timing = D.dbg_ctl != 0;
            for (int c = 0; c < nchunk; ++c) {
                const int c0 = c * CH, w = min(CH, D.d - c0);
                const long long tw0 = timing ? clock64() : 0;
                mbar_wait(&full[stage], phase);
                if (timing) t_wait += clock64() - tw0;
                if (e < E) {
                    // 32 products into registers (LDS.128 pairs, independent
                    // DMULs), then the 32-long DADD chain: measured 10.5
                    // cycles/column on B200 vs 17.6 for a fused load-mul-add
                    // loop (profiles/microbench/chain_variants.cu)
                    const double* row = (const double*)(ring + (size_t)stage * E * rowb + (size_t)e * rowb);
                    const double* qq = sm_q + c0;
                    if (w == CH) {
                        for (int i0 = 0; i0 < CH; i0 += 32) {
                            double r[32];
#pragma unroll
                            for (int u = 0; u < 32; u += 2) {
                                const double2 a2 = *(const double2*)(row + i0 + u);
                                const double2 b2 = *(const double2*)(qq + i0 + u);
                                r[u] = __dmul_rn(a2.x, b2.x);
                                r[u + 1] = __dmul_rn(a2.y, b2.y);
                            }
#pragma unroll
                            for (int u = 0; u < 32; ++u) acc = __dadd_rn(acc, r[u]);
                        }
                    } else {
                        for (int i = 0; i < w; ++i) acc = __dadd_rn(acc, __dmul_rn(row[i], qq[i]));
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);
                if (++stage == kRouteStages) stage = 0, phase ^= 1;
            }
            if (e < E) sm_logit[e] = acc;
            if (dbg) S.dbg[5] = t_wait;
        }
        __syncthreads();
    }
    if (dbg) S.dbg[2] = clock64();
    if (dbg) S.dbg[3] = clock64();
    if (tid < 32) route_select(D, C, S, s, sm_logit, sm_flag, sm_pool, sm_load, sm_usage, sm_miss,
                               sm_bias, sm_sel, sm_pre, &sm_errf);
    __syncthreads();
    if (sm_errf) return nullptr;
    for (int e = tid; e < D.E; e += blockDim.x) S.load[(int64_t)s * D.E + e] = sm_load[e];
    for (int j = tid; j < D.k; j += blockDim.x) {
        S.usage[(int64_t)s * D.E + sm_sel[j]] = sm_usage[sm_sel[j]];
        S.experts[(int64_t)s * D.k + j] = sm_sel[j];
    }
    if (dbg) S.dbg[4] = clock64();
    return sm_sel;  // the selected experts, in this CTA's shared memory
}

__global__ void k_route(Dims D, Cfg C, State S, const void* __restrict__ qin) {
    griddep_enter();
    extern __shared__ __align__(128) uint8_t sm_raw[];
    route_body(D, C, S, blockIdx.x, qin, D.route_ch, sm_raw);
}

// route / route_logits of one stream (component API, pikv_route_host):
// q [B][d] fp64 staging with the query in row s, or logits [E].
__global__ void k_route_one(Dims D, Cfg C, State S, int s, const double* __restrict__ q,
                            const double* __restrict__ logits) {
    extern __shared__ __align__(128) uint8_t sm_raw[];
    route_body(D, C, S, s, q, D.route_ch, sm_raw, logits);
}
static size_t route_smem_bytes(const Dims& D, int ch);
void launch_route_one(const Dims& D, const Cfg& C, const State& S, int s, const double* q, const double* logits,
                      cudaStream_t st) {
    Dims d1 = D;
    d1.q_f64 = 1;
    const size_t smem = route_smem_bytes(d1, d1.route_ch);
    // static shared memory counts against the 48 KB default too: always opt in
    cudaFuncSetAttribute(k_route_one, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int threads = ((D.E + 31) / 32) * 32 + 32;
    k_route_one<<<1, threads, smem, st>>>(d1, C, S, s, q, logits);
}

// Warp 0 of k_route: penalties, selection, gates, note_selection and the
// retrieval candidate rings, on the smem copy of RouterState.  Lanes work
// over experts / rings; the reductions whose order the reference fixes
// (mean load, gate softmax) run on lane 0 in index order.
__device__ __forceinline__ void route_select(const Dims& D, const Cfg& C, const State& S, int s,
                                             double* sm_logit, bool* sm_flag, int* sm_pool,
                                             double* load, uint64_t* usage, const uint64_t* miss,
                                             const double* bias, int* sel, const uint64_t* pre, int* errf) {
    const int lane = threadIdx.x & 31;
    const int E = D.E, k = D.k;
    double* gates = S.gates + (int64_t)s * k;
    double* lg = S.logits + (int64_t)s * E;
    const bool base = C.router_strategy == PIKV_ROUTER_BASE;
    __shared__ double sm_mean;
    const uint64_t sm_tot = pre[0];  // S.total_usage[s], prefetched
    if (base) {  // base_round_robin, router.cpp:107-118
        const int64_t t = (int64_t)pre[1];  // S.rstep[s]
        for (int j = lane; j < k; j += 32) {
            sel[j] = (int)((t * C.stride + j) % E);
            gates[j] = __ddiv_rn(1.0, (double)k);
        }
        for (int e = lane; e < E; e += 32) lg[e] = 0.0;
    } else {
        bool nan_seen = false;
        for (int e = lane; e < E; e += 32) nan_seen |= isnan(sm_logit[e]);
        if (__any_sync(0xffffffffu, nan_seen)) {  // router.cpp:131-133
            if (lane == 0) S.err[s] = PIKV_ERR_NUMERICAL, *errf = 1;
            return;
        }
        if (C.router_strategy == PIKV_ROUTER_LOAD_BALANCED && lane == 0) {
            double acc = 0.0;
            for (int e = 0; e < E; ++e) acc = __dadd_rn(acc, load[e]);
            sm_mean = __ddiv_rn(acc, (double)E);
        }
        __syncwarp();
        const uint64_t tot = sm_tot;
        for (int e = lane; e < E; e += 32) {
            double x = sm_logit[e];
            switch (C.router_strategy) {
                case PIKV_ROUTER_LOAD_BALANCED:
                    x = __dsub_rn(x, __dmul_rn(C.alpha, __dsub_rn(load[e], sm_mean)));
                    break;
                case PIKV_ROUTER_CACHE_AWARE:
                    x = __dsub_rn(x, __dmul_rn(C.lambda_miss, log1p((double)miss[e])));
                    break;
                case PIKV_ROUTER_ENTROPY_LB: {
                    const double p = tot == 0 ? 0.0 : __ddiv_rn((double)usage[e], (double)tot);
                    const double h = p > 0.0 ? __dmul_rn(-p, log(p)) : 0.0;
                    x = __dsub_rn(x, __dmul_rn(C.beta_ent, h));
                    break;
                }
                case PIKV_ROUTER_ADAPTIVE:
                    x = __dadd_rn(x, bias[e]);
                    break;
                default:
                    break;
            }
            sm_logit[e] = x;
            lg[e] = x;
        }
        __syncwarp();
        // selection: (score desc, index asc), router.cpp:82-90, 174-198
        if (C.router_strategy == PIKV_ROUTER_HIERARCHICAL) {
            if (lane == 0) {
                auto better = [&](int a2, int b2) {
                    const double sa = sm_logit[a2], sb = sm_logit[b2];
                    return sa != sb ? sa > sb : a2 < b2;
                };
                const int groups = C.groups;
                const int cs = (E + groups - 1) / groups;
                int chosen = 0, npool = 0;
                bool* used = sm_flag;
                int* pool = sm_pool;
                for (int g = 0; g < groups; ++g) used[g] = false;
                while (npool < k && chosen < groups) {
                    int best = -1;
                    double bsc = 0.0;
                    for (int g = 0; g < groups; ++g) {
                        if (used[g]) continue;
                        double sc = -INFINITY;
                        for (int e = g * cs; e < min(E, g * cs + cs); ++e)
                            sc = (sc < sm_logit[e]) ? sm_logit[e] : sc;
                        if (best < 0 || sc > bsc) best = g, bsc = sc;  // ties keep lower g
                    }
                    used[best] = true;
                    ++chosen;
                    for (int e = best * cs; e < min(E, best * cs + cs); ++e) pool[npool++] = e;
                }
                for (int j = 0; j < k; ++j) {
                    int bi = j;
                    for (int i = j + 1; i < npool; ++i)
                        if (better(pool[i], pool[bi])) bi = i;
                    const int t = pool[j];
                    pool[j] = pool[bi];
                    pool[bi] = t;
                    sel[j] = pool[j];
                }
            }
        } else {
            // k rounds of warp argmax, excluding earlier picks == sorted prefix
            for (int e = lane; e < E; e += 32) sm_flag[e] = false;
            __syncwarp();
            for (int j = 0; j < k; ++j) {
                double bv = 0.0;
                int bi = -1;
                for (int e = lane; e < E; e += 32) {
                    if (sm_flag[e]) continue;
                    const double x = sm_logit[e];
                    if (bi < 0 || x > bv || (x == bv && e < bi)) bv = x, bi = e;
                }
                for (int off = 16; off; off >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                    if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) bv = ov, bi = oi;
                }
                if (lane == 0) {
                    sel[j] = bi;
                    sm_flag[bi] = true;
                }
                __syncwarp();
            }
        }
        __syncwarp();
        {  // gates = softmax(selected logits), mathops.cpp:11-30: the exps and
           // divisions on lanes j < k, the sum sequential in j order on lane 0
            __shared__ double sm_g[kMaxK];
            __shared__ double sm_gtot;
            double mx = sm_logit[sel[0]];
            for (int j = 0; j < k; ++j) mx = (mx < sm_logit[sel[j]]) ? sm_logit[sel[j]] : mx;
            for (int j = lane; j < k; j += 32) sm_g[j] = exp(__dsub_rn(sm_logit[sel[j]], mx));
            __syncwarp();
            if (lane == 0) {
                double tot2 = 0.0;
                for (int j = 0; j < k; ++j) tot2 = __dadd_rn(tot2, sm_g[j]);
                sm_gtot = tot2;
            }
            __syncwarp();
            for (int j = lane; j < k; j += 32) gates[j] = __ddiv_rn(sm_g[j], sm_gtot);
        }
    }
    __syncwarp();
    // note_selection, router.cpp:92-105
    const double one_m = __dsub_rn(1.0, C.load_decay);
    for (int e = lane; e < E; e += 32) {
        bool picked = false;
        for (int j = 0; j < k; ++j) picked |= sel[j] == e;
        load[e] = __dadd_rn(__dmul_rn(C.load_decay, load[e]), __dmul_rn(one_m, picked ? 1.0 : 0.0));
    }
    for (int j = lane; j < k; j += 32) usage[sel[j]] += 1;
    if (lane == 0) {
        S.total_usage[s] = sm_tot + (uint64_t)k;
        S.rstep[s] = pre[1] + 1;
    }
    // candidate local rings for retrieval (ascending ring id)
    int nc = 0;
    int32_t* cand = S.cand + (int64_t)s * D.max_cand;
    const int nr = D.Gl * D.SPD;
    for (int r0 = 0; r0 < nr; r0 += 32) {
        const int r = r0 + lane;
        bool ok = false;
        if (r < nr) {
            const int gl = r / D.SPD, sh = r % D.SPD;
            const int raw = sh * D.G + gl * D.world + D.rank;
            for (int j = 0; j < k && !ok; ++j) ok = ring_can_hold(raw, sel[j], D.n_tok, D.n_exp, D.additive);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        const int pos = nc + __popc(bal & ((1u << lane) - 1u));
        if (ok && pos < D.max_cand) cand[pos] = r;
        nc += __popc(bal);
    }
    if (lane == 0) S.ncand[s] = min(nc, D.max_cand);
}

static size_t route_smem_bytes(const Dims& D, int ch) {
    return 128 + sizeof(double) * (size_t)D.d + (size_t)kRouteStages * D.E * ((size_t)ch * 8 + 16);
}
// Router columns per W ring stage, fixed per engine (the W layout depends on
// it): the largest multiple of 32 <= 256 whose ring fits 200 KB.  Long
// stages matter: each stage boundary costs the chain a refill bubble
// (measured: CH 64 -> 38 us, CH 256 -> 31 us at d 4096, E 16).
int pick_route_chunk(const Dims& D) {
    int ch = kRouteCHMax;
    while (ch > 32 && route_smem_bytes(D, ch) > 200 * 1024) ch -= 32;
    return ch;
}

void launch_route(const Dims& D, const Cfg& C, const State& S, const void* q, cudaStream_t st) {
    const size_t smem = route_smem_bytes(D, D.route_ch);
    // static shared memory counts against the 48 KB default too: always opt in
    cudaFuncSetAttribute(k_route, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int threads = ((D.E + 31) / 32) * 32 + 32;
    if (C.route_mode == PIKV_ROUTE_FAST) threads = std::max(threads, std::min(1024, 32 * D.E));
    launch_pdl(k_route, dim3(D.B), dim3(threads), smem, st, D, C, S, q);
}

// ===========================================================================
// project: Codec::encode_vector for LowRank / LoRAPlus (compressor.cpp:318-329,
// 364-378, pipeline.cpp:295-297) of the step's q, k and v of every stream,
// one CTA per (head, row): the head's basis and the B input slices are staged
// in shared memory once, then y[b][j] = sum_i B[j][i] x[b][i] (i ascending,
// fp32) for all streams.  Output: S.proj[row][B][dp] (row 0 = q -> q_attn).
__global__ void k_project(Dims D, State S, const void* __restrict__ qin, const void* __restrict__ kin,
                          const void* __restrict__ vin) {
    griddep_enter();
    extern __shared__ float sm_p[];  // basis [r][hd + 1] then x [B][hd]
    const int h = blockIdx.x, row = blockIdx.y;
    const int hd = D.d / D.H, r = D.dph, tid = threadIdx.x, nt = blockDim.x;
    const int hdp = hd + 1;  // padded basis rows: lanes j = 0..31 read column i of 32 rows
                             // from 32 different banks (unpadded: one bank, 32-way conflict)
    const void* x = row == 0 ? qin : (row == 1 ? kin : vin);
    float* bs = sm_p;
    float* xs = sm_p + (size_t)r * hdp;
    for (int t = tid; t < r * hd; t += nt) bs[(t / hd) * hdp + t % hd] = S.basis[(int64_t)h * r * hd + t];
    for (int t = tid; t < D.B * hd; t += nt) {
        const int b = t / hd, i = t % hd;
        float xi = (row == 0 && D.q_f64) ? (float)((const double*)x)[(int64_t)b * D.d + h * hd + i]
                                          : load_in(x, D.kv_dtype, (int64_t)b * D.d + h * hd + i);
        if (D.codec == PIKV_CODEC_LORAPLUS) xi -= S.cbias[h * hd + i];
        xs[t] = xi;
    }
    __syncthreads();
    for (int t = tid; t < D.B * r; t += nt) {
        const int b = t / r, j = t % r;
        const float* col = bs + (size_t)j * hdp;
        const float* xb = xs + (size_t)b * hd;
        float acc = 0.f;
#pragma unroll 8
        for (int i = 0; i < hd; ++i) acc = fmaf(col[i], xb[i], acc);
        if (row == 0) S.q_attn[(int64_t)b * D.dp + h * r + j] = acc;
        else S.proj[((int64_t)(row - 1) * D.B + b) * D.dp + h * r + j] = acc;
    }
}

void launch_project(const Dims& D, const State& S, const void* q, const void* k, const void* v,
                    cudaStream_t st) {
    const int hd = D.d / D.H;
    const size_t smem = sizeof(float) * ((size_t)D.dph * (hd + 1) + (size_t)D.B * hd);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_project, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(k_project, dim3(D.H, 3), dim3(256), smem, st, D, S, q, k, v);
}

// ===========================================================================
// insert: KVStore::insert for the k staged entries of each stream
// ===========================================================================

// Encode one K or V row of stream s into smem `dst` in the stored layout.
__device__ __forceinline__ void encode_row(const Dims& D, const State& S, const void* x, int s, uint8_t* dst,
                                           float* scales_out, float* tmp, int kv_row) {
    const int H = D.H, hd = D.d / H, r = D.dph, tid = threadIdx.x, nt = blockDim.x;
    const int64_t base = (int64_t)s * D.d;
    switch (D.codec) {
        case PIKV_CODEC_IDENTITY:
            if ((D.d * (D.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4)) % 16 == 0) {
                const int nv = D.d * (D.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4) / 16;
                const uint4* src = (const uint4*)((const uint8_t*)x +
                                                  base * (D.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4));
                for (int i = tid; i < nv; i += nt) ((uint4*)dst)[i] = src[i];
            } else if (D.kv_dtype == PIKV_DTYPE_BF16) {
                for (int i = tid; i < D.d; i += nt) ((uint16_t*)dst)[i] = ((const uint16_t*)x)[base + i];
            } else {
                for (int i = tid; i < D.d; i += nt) ((float*)dst)[i] = ((const float*)x)[base + i];
            }
            return;
        case PIKV_CODEC_LOWRANK:
        case PIKV_CODEC_LORAPLUS: {  // project_encode: computed for all streams by k_project
            const float* pr = S.proj + ((int64_t)kv_row * D.B + s) * D.dp;
            for (int o = tid; o < D.dp; o += nt) {
                const float val = pr[o];
                if (D.kv_dtype == PIKV_DTYPE_BF16) ((uint16_t*)dst)[o] = f32_to_bf16_rne(val);
                else ((float*)dst)[o] = val;
            }
            return;
        }
        case PIKV_CODEC_FASTV:   // compressor.cpp:396-397
        case PIKV_CODEC_PRUNE:   // compressor.cpp:398-402
            for (int o = tid; o < D.dp; o += nt) {
                const int h = o / r, j = o % r;
                const int i = D.codec == PIKV_CODEC_FASTV ? j : S.kept[h * r + j];
                if (D.kv_dtype == PIKV_DTYPE_BF16)
                    ((uint16_t*)dst)[o] = ((const uint16_t*)x)[base + h * hd + i];
                else
                    ((float*)dst)[o] = ((const float*)x)[base + h * hd + i];
            }
            return;
        case PIKV_CODEC_INT8:
        case PIKV_CODEC_INT4: {
            // symmetric absmax per head (oracle: po_quantize_row)
            const int bits = D.codec == PIKV_CODEC_INT8 ? 8 : 4;
            const float qmax = bits == 8 ? 127.0f : 7.0f;
            for (int i = tid; i < D.d; i += nt) tmp[i] = load_in(x, D.kv_dtype, base + i);
            __syncthreads();
            const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
            for (int h = warp; h < H; h += nw) {
                float amax = 0.f;
                for (int i = lane; i < hd; i += 32) amax = fmaxf(amax, fabsf(tmp[h * hd + i]));
                for (int off = 16; off; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
                float inv = 0.f, scale = 0.f;
                if (amax > 0.f) {
                    scale = __fdiv_rn(amax, qmax);
                    inv = __fdiv_rn(qmax, amax);
                }
                if (lane == 0) scales_out[h] = scale;
                if (bits == 8) {
                    for (int i = lane; i < hd; i += 32) {
                        float c = rintf(__fmul_rn(tmp[h * hd + i], inv));
                        c = fminf(fmaxf(c, -qmax), qmax);
                        ((int8_t*)dst)[h * hd + i] = (int8_t)(int)c;
                    }
                } else {
                    for (int i2 = lane; i2 < hd / 2; i2 += 32) {
                        float c0 = rintf(__fmul_rn(tmp[h * hd + 2 * i2], inv));
                        float c1 = rintf(__fmul_rn(tmp[h * hd + 2 * i2 + 1], inv));
                        c0 = fminf(fmaxf(c0, -qmax), qmax);
                        c1 = fminf(fmaxf(c1, -qmax), qmax);
                        dst[(h * hd) / 2 + i2] = (uint8_t)(((int)c0 & 0xF) | (((int)c1 & 0xF) << 4));
                    }
                }
            }
            __syncthreads();
            return;
        }
    }
}

// KVStore::insert of stream s's k entries by the calling CTA (k_insert,
// k_control); sm_entry = dynamic smem of insert_smem_bytes().  `sel` = the
// step's experts in shared memory when the caller has them (k_control),
// else they are read from S.experts.
//
// Bookkeeping runs on warp 0 only (lane j = selected expert j) while the
// other warps stage the K/V row (identity codec) and the fp32 query.  When
// the k entries hit k distinct rings (the common case) the lanes do their
// KVStore::insert concurrently, loading everything first (ring head/seq,
// then the head slot and both page records), so the chain is a few
// independent load rounds; otherwise lane 0 runs them in order.
// Entry ids are issued in selection order on every rank (kvstore.cpp:114).
__device__ __forceinline__ void insert_book_seq(const Dims& D, const State& S, const int s, const int* sel,
                                                const double* __restrict__ saliency, int64_t* sm_dst, int* sm_n) {
    const uint64_t now = S.now[s];
    const int64_t token = (int64_t)now;
    // pass 1: the pool pages the k inserts will need (the i-th insert of the
    // step into a ring lands at head + i), reserved with one atomic before
    // any store: an exhausted pool fails the insert with no partial state
    // (pipeline.cpp:153-154)
    int64_t rng[kMaxK], newp[kMaxK];
    int nnew = 0;
    for (int j = 0; j < D.k; ++j) {
        const int e = sel ? sel[j] : S.experts[(int64_t)s * D.k + j];
        const int raw = shard_raw(token, e, D.n_tok, D.n_exp, D.additive);
        const int dev = raw % D.G;
        rng[j] = -1;
        if (dev % D.world != D.rank) continue;
        const int64_t ring = ((int64_t)s * D.Gl + dev / D.world) * D.SPD + raw / D.G;
        rng[j] = ring;
        int off = 0;
        for (int i = 0; i < j; ++i) off += rng[i] == ring;
        const int slot = (S.head[ring] + off) % D.S;
        if (off >= D.S || S.id[ring * D.S + slot] != 0) continue;  // displaces: no new page
        const int64_t pidx = ring * D.ppr + slot / D.spg;
        if (S.page_table[pidx] >= 0) continue;
        bool seen = false;
        for (int i = 0; i < nnew; ++i) seen |= newp[i] == pidx;
        if (!seen) newp[nnew++] = pidx;
    }
    int pbase = 0;
    if (nnew > 0) {
        pbase = atomicSub(S.free_top, nnew) - nnew;
        if (pbase < 0) {
            atomicAdd(S.free_top, nnew);
            S.err[s] = PIKV_ERR_OUT_OF_MEMORY;
            *sm_n = 0;
            return;
        }
    }
    int n = 0;
    for (int j = 0; j < D.k; ++j) {
        const int e = sel ? sel[j] : S.experts[(int64_t)s * D.k + j];
        const int raw = shard_raw(token, e, D.n_tok, D.n_exp, D.additive);
        const int dev = raw % D.G, sh = raw / D.G;
        const uint64_t id = S.next_id[s]++;  // every rank issues every id
        if (dev % D.world != D.rank) continue;
        const int gl = dev / D.world;
        const int64_t ring = ((int64_t)s * D.Gl + gl) * D.SPD + sh;
        const int slot = S.head[ring];
        const int64_t gi = ring * D.S + slot;
        const int64_t pidx = ring * D.ppr + slot / D.spg;
        int32_t page = S.page_table[pidx];
        if (S.id[gi] != 0) {  // displaced (kvstore.cpp:41-43; pipeline.cpp:200-208)
            rec_drop_front(D, S, ring, S.shard_seq[gi], S.last_access[gi], S.freq[gi]);
            const int no = S.n_ow[s]++;
            EvictRec& r = S.rec_ow[(int64_t)s * D.k + no];
            r.step = now;
            r.entry_id = S.id[gi];
            r.token_id = S.token[gi];
            r.expert_id = S.expert[gi];
            r.device = dev;
            r.score = 0.0;
            r.reason = PIKV_EVICT_OVERWRITE;
            r.stream = s;
            S.st_overwrites[s] += 1;
        } else {
            S.live[ring] += 1;
            if (page < 0) {  // reserved in pass 1
                page = S.free_stack[pbase++];
                S.page_table[pidx] = page;
                S.page_live[page] = 0;
            }
            S.page_live[page] += 1;
        }
        S.id[gi] = id;
        rec_append(D, S, ring, S.seq[ring], now);
        S.shard_seq[gi] = S.seq[ring]++;
        S.token[gi] = token;
        S.expert[gi] = e;
        S.insert_step[gi] = now;
        S.last_access[gi] = now;
        S.freq[gi] = 0;
        S.attn_mass[gi] = 0.0;
        for (int l = 0; l < D.n_layers; ++l)
            S.per_layer[gi * D.n_layers + l] = saliency ? saliency[(int64_t)s * D.n_layers + l] : 0.0;
        S.has_pl[gi] = D.n_layers > 0 && saliency != nullptr;
        S.head[ring] = (slot + 1) % D.S;
        S.st_inserts[s] += 1;
        sm_dst[n] = (int64_t)page * D.spg + slot % D.spg;
        ++n;
    }
    *sm_n = n;
}

// Warp 0: the k inserts of stream s (see above).  Writes the pool entry
// index of each stored entry (in id order) to sm_dst and their number to
// *sm_n.
__device__ __forceinline__ void insert_book(const Dims& D, const State& S, const int s, const int* sel,
                                            const double* __restrict__ saliency, int64_t* sm_dst, int* sm_n) {
    const int j = threadIdx.x & 31;
    const uint64_t now = S.now[s];
    const int64_t token = (int64_t)now;
    // round A: expert -> ring (local rings only)
    bool act = false;
    int e = 0, dev = 0;
    int64_t ring = -1 - j;
    if (j < D.k) {
        e = sel ? sel[j] : S.experts[(int64_t)s * D.k + j];
        const int raw = shard_raw(token, e, D.n_tok, D.n_exp, D.additive);
        dev = raw % D.G;
        if (dev % D.world == D.rank) {
            act = true;
            ring = (int64_t)s * D.R + (dev / D.world) * D.SPD + raw / D.G;
        }
    }
    bool distinct = D.k <= 32;
    if (distinct) {
        const unsigned m = __match_any_sync(0xffffffffu, ring);
        distinct = __all_sync(0xffffffffu, !act || m == (1u << j));
    }
    if (!distinct) {
        if (j == 0) insert_book_seq(D, S, s, sel, saliency, sm_dst, sm_n);
        __syncwarp();
        return;
    }
    // round B: ring state
    int slot = 0;
    uint64_t seq = 0, nid = 0;
    if (act) {
        slot = S.head[ring];
        seq = S.seq[ring];
    }
    nid = S.next_id[s];
    // round C: head slot (possibly displaced) and the append page record
    const int64_t gi = ring * D.S + slot;
    const int64_t pidx = ring * D.ppr + slot / D.spg;
    const int64_t arec = act ? page_rec(D, ring, seq) : 0;
    int32_t page = -1;
    uint64_t old = 0, osq = 0, ola = 0, ofr = 0;
    int64_t otok = 0;
    int oex = 0, acnt = 0, afirst = 0;
    uint64_t asla = 0, asf = 0;
    if (act) {
        page = S.page_table[pidx];
        old = S.id[gi];
        osq = S.shard_seq[gi];
        ola = S.last_access[gi];
        ofr = S.freq[gi];
        otok = S.token[gi];
        oex = S.expert[gi];
        acnt = S.pr_cnt[arec];
        afirst = S.pr_first[arec];
        asla = S.pr_sla[arec];
        asf = S.pr_sf[arec];
    }
    const bool disp = act && old != 0;
    // round D: the displaced entry's page record (rec_drop_front)
    int64_t drec = -1;
    int dcnt = 0, dfirst = 0;
    uint64_t dsla = 0, dsf = 0;
    int pl_delta = 0;  // pages_live change of the ring's device
    if (disp) {
        drec = page_rec(D, ring, osq);
        if (drec == arec) {
            dcnt = acnt, dfirst = afirst, dsla = asla, dsf = asf;
        } else {
            dcnt = S.pr_cnt[drec];
            dfirst = S.pr_first[drec];
            dsla = S.pr_sla[drec];
            dsf = S.pr_sf[drec];
        }
        if (--dcnt == 0) --pl_delta;  // last member displaced
        dfirst += 1;
        if (D.holes && dcnt > 0) dfirst = next_member(D, S, ring, osq / (uint64_t)D.page_size, dfirst);
        dsla -= ola;
        dsf -= ofr;
        if (drec == arec) acnt = dcnt, afirst = dfirst, asla = dsla, asf = dsf;
    }
    // page allocation for fresh slots: the step's new pages are reserved
    // with one atomic, and an exhausted pool fails the whole insert before
    // any store (no partial state, pipeline.cpp:153-154)
    bool fresh_page = false;
    {
        const bool need = act && !disp && page < 0;
        const unsigned nm = __ballot_sync(0xffffffffu, need);
        int base = 0;
        if (j == 0 && nm) {
            const int c = __popc(nm);
            base = atomicSub(S.free_top, c) - c;
            if (base < 0) atomicAdd(S.free_top, c);
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base < 0) {
            if (j == 0) S.err[s] = PIKV_ERR_OUT_OF_MEMORY, *sm_n = 0;
            __syncwarp();
            return;
        }
        if (need) {
            page = S.free_stack[base + __popc(nm & ((1u << j) - 1u))];
            fresh_page = true;
        }
    }
    const bool ins = act;
    // rec_append
    if (ins) {
        if (acnt == 0) {
            ++pl_delta;  // a page comes to life
            acnt = 1;
            afirst = (int)(seq % (uint64_t)D.page_size);
            asla = now;
            asf = 0;
        } else {
            acnt += 1;
            asla += now;
        }
    }
    // stores
    if (disp && drec != arec) {
        S.pr_cnt[drec] = dcnt;
        S.pr_first[drec] = dfirst;
        S.pr_sla[drec] = dsla;
        S.pr_sf[drec] = dsf;
    }
    if (ins || (disp && drec == arec)) {
        S.pr_cnt[arec] = acnt;
        S.pr_first[arec] = afirst;
        S.pr_sla[arec] = asla;
        S.pr_sf[arec] = asf;
    }
    if (pl_delta) atomicAdd(&S.pages_live[ring / D.SPD], pl_delta);
    if (ins) {
        if (!disp) {
            atomicAdd(&S.live[ring], 1);
            if (fresh_page) {
                S.page_table[pidx] = page;
                S.page_live[page] = 1;
            } else {
                atomicAdd(&S.page_live[page], 1);
            }
        }
        S.id[gi] = nid + (uint64_t)j;
        S.shard_seq[gi] = seq;
        S.seq[ring] = seq + 1;
        S.token[gi] = token;
        S.expert[gi] = e;
        S.insert_step[gi] = now;
        S.last_access[gi] = now;
        S.freq[gi] = 0;
        S.attn_mass[gi] = 0.0;
        for (int l = 0; l < D.n_layers; ++l)
            S.per_layer[gi * D.n_layers + l] = saliency ? saliency[(int64_t)s * D.n_layers + l] : 0.0;
        S.has_pl[gi] = D.n_layers > 0 && saliency != nullptr;
        S.head[ring] = (slot + 1) % D.S;
    }
    const unsigned dm = __ballot_sync(0xffffffffu, disp);
    const unsigned am = __ballot_sync(0xffffffffu, ins);
    if (disp) {  // displaced (kvstore.cpp:41-43; pipeline.cpp:200-208)
        EvictRec rec;
        rec.step = now;
        rec.entry_id = old;
        rec.token_id = otok;
        rec.expert_id = oex;
        rec.device = dev;
        rec.score = 0.0;
        rec.reason = PIKV_EVICT_OVERWRITE;
        rec.stream = s;
        S.rec_ow[(int64_t)s * D.k + __popc(dm & ((1u << j) - 1u))] = rec;
    }
    if (ins) sm_dst[__popc(am & ((1u << j) - 1u))] = (int64_t)page * D.spg + slot % D.spg;
    if (j == 0) {
        S.n_ow[s] = __popc(dm);
        S.st_overwrites[s] += (uint64_t)__popc(dm);
        S.st_inserts[s] += (uint64_t)__popc(am);
        S.next_id[s] = nid + (uint64_t)D.k;
        *sm_n = __popc(am);
    }
    __syncwarp();
}

__device__ __forceinline__ void insert_body(const Dims& D, const Cfg& C, const State& S, const int s,
                                            const void* __restrict__ qin, const void* __restrict__ kin,
                                            const void* __restrict__ vin,
                                            const double* __restrict__ saliency, uint8_t* sm_entry,
                                            const int* sel = nullptr) {
    __shared__ int64_t sm_dst[kMaxK];
    __shared__ int sm_n;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (S.err[s]) return;
    float* tmp = (float*)(sm_entry + ((D.entry_bytes + 15) & ~15));
    const int pay = D.payload_bytes;
    const int esz = D.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4;
    const bool proj = D.codec == PIKV_CODEC_LOWRANK || D.codec == PIKV_CODEC_LORAPLUS ||
                      D.codec == PIKV_CODEC_FASTV || D.codec == PIKV_CODEC_PRUNE;
    // the query in the stored (compressed) space, fp32 (pipeline.cpp:295-297)
    auto query = [&](int t0, int nt) {
        const int hd = D.d / D.H, r = D.dph;
        const int64_t base = (int64_t)s * D.d;
        float* qa = S.q_attn + (int64_t)s * D.dp;
        if (D.q_f64) {  // encoder output: fp64 -> fp32 (projections use the same input)
            const double* q64 = (const double*)qin + base;
            if (!proj) {
                for (int o = t0; o < D.d; o += nt) qa[o] = (float)q64[o];
            } else if (D.codec == PIKV_CODEC_FASTV || D.codec == PIKV_CODEC_PRUNE) {
                for (int o = t0; o < D.dp; o += nt) {
                    const int h = o / r, j = o % r;
                    const int i = D.codec == PIKV_CODEC_FASTV ? j : S.kept[h * r + j];
                    qa[o] = (float)q64[h * hd + i];
                }
            }
        } else if (!proj && D.kv_dtype == PIKV_DTYPE_BF16 && D.d % 8 == 0) {
            const uint4* src = (const uint4*)((const uint16_t*)qin + base);
            for (int v = t0; v < D.d / 8; v += nt) {
                const uint4 w = src[v];
                float4* dq = (float4*)(qa + v * 8);
                dq[0] = make_float4(bf16_lo(w.x), bf16_hi(w.x), bf16_lo(w.y), bf16_hi(w.y));
                dq[1] = make_float4(bf16_lo(w.z), bf16_hi(w.z), bf16_lo(w.w), bf16_hi(w.w));
            }
        } else if (!proj) {
            for (int o = t0; o < D.d; o += nt) qa[o] = load_in(qin, D.kv_dtype, base + o);
        } else if (D.codec == PIKV_CODEC_FASTV || D.codec == PIKV_CODEC_PRUNE) {
            for (int o = t0; o < D.dp; o += nt) {
                const int h = o / r, j = o % r;
                const int i = D.codec == PIKV_CODEC_FASTV ? j : S.kept[h * r + j];
                qa[o] = load_in(qin, D.kv_dtype, base + h * hd + i);
            }
        }  // LowRank / LoRAPlus: q_attn written by k_project
    };
    const bool overlap = D.codec == PIKV_CODEC_IDENTITY && (D.d * esz) % 16 == 0 && blockDim.x >= 64;
    if (overlap) {
        // warp 0: bookkeeping; warps 1..: K/V rows -> smem entry, query
        if (warp == 0) {
            insert_book(D, S, s, sel, saliency, sm_dst, &sm_n);
        } else {
            const int t0 = tid - 32, nt = blockDim.x - 32;
            const int nv = D.d * esz / 16;
            const uint4* ks = (const uint4*)((const uint8_t*)kin + (int64_t)s * D.d * esz);
            const uint4* vs = (const uint4*)((const uint8_t*)vin + (int64_t)s * D.d * esz);
            for (int i = t0; i < nv; i += nt) {
                ((uint4*)sm_entry)[i] = ks[i];
                ((uint4*)(sm_entry + pay))[i] = vs[i];
            }
            query(t0, nt);
        }
    } else {
        float* ksc = (float*)(sm_entry + 2 * pay);
        float* vsc = ksc + D.H;
        encode_row(D, S, kin, s, sm_entry, ksc, tmp, 0);
        encode_row(D, S, vin, s, sm_entry + pay, vsc, tmp, 1);
        query(tid, blockDim.x);
        if (warp == 0) insert_book(D, S, s, sel, saliency, sm_dst, &sm_n);
    }
    __syncthreads();
    const int n = sm_n;
    const int nvec = D.entry_bytes / 16;
    for (int j = 0; j < n; ++j) {
        uint4* dst = (uint4*)(S.pool + sm_dst[j] * (int64_t)D.entry_bytes);
        const uint4* src = (const uint4*)sm_entry;
        for (int i = tid; i < nvec; i += blockDim.x) dst[i] = src[i];
    }
}

__global__ void k_insert(Dims D, Cfg C, State S, const void* __restrict__ qin,
                         const void* __restrict__ kin, const void* __restrict__ vin,
                         const double* __restrict__ saliency) {
    griddep_enter();
    extern __shared__ __align__(16) uint8_t sm_entry[];  // [entry_bytes] + tmp floats [d]
    insert_body(D, C, S, blockIdx.x, qin, kin, vin, saliency, sm_entry);
}

static size_t insert_smem_bytes(const Dims& D) {
    return (size_t)((D.entry_bytes + 15) & ~15) + sizeof(float) * (size_t)D.d;
}

void launch_insert(const Dims& D, const Cfg& C, const State& S, const void* q, const void* k,
                   const void* v, const double* saliency, cudaStream_t st) {
    size_t smem = insert_smem_bytes(D);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_insert, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(k_insert, dim3(D.B), dim3(256), smem, st, D, C, S, q, k, v, saliency);
}

// ===========================================================================
// sched: evict, scheduler.cpp:262-330
// ===========================================================================
// (a) page keys (aggregate, oldest id, live count) for every candidate
//     scheduler page (ring, page_no).  Dead pages (record count 0) cost one
//     load.  LRU/LRU+ with exact sums take the aggregate from the page record:
//     -(cnt*now - sum last_access) [+ lambda*sum freq] is the exact value of the
//     reference's slot-order sum (every term and partial sum is an integer or
//     dyadic below 2^53).  Other strategies score the live member range: lane u
//     takes the u-th member in slot order (scheduler.cpp:276-289), lane 0 sums
//     in that order (or a tree sum when exact in any order).
// Key of candidate page pi of `ring` from its page record (record_agg
// strategies): live count, exact aggregate, oldest (= first member's) id.
__device__ __forceinline__ int page_key_rec(const Dims& D, const Cfg& C, const State& S, const int64_t ring,
                                            const int pi, const uint64_t now, double& agg, uint64_t& oldest) {
    const uint64_t seq = S.seq[ring];
    const uint64_t Su = (uint64_t)D.S, ps = (uint64_t)D.page_size;
    const uint64_t lo = seq > Su ? seq - Su : 0;
    const uint64_t q = lo / ps + (uint64_t)pi;
    const int64_t rec = ring * D.ppr_sched + (int64_t)(q % (uint64_t)D.ppr_sched);
    const int cnt = q * ps < seq ? S.pr_cnt[rec] : 0;
    agg = 0.0;
    oldest = 0;
    if (cnt > 0) {
        const int first = S.pr_first[rec];
        const uint64_t sla = S.pr_sla[rec];
        agg = -(double)((uint64_t)cnt * now - sla);
        if (C.sched_strategy == PIKV_SCHED_LRU_PLUS)
            agg = __dadd_rn(agg, __dmul_rn(C.lambda_freq, (double)S.pr_sf[rec]));
        oldest = S.id[ring * D.S + (int64_t)((q * ps + (uint64_t)first) % Su)];
    }
    return cnt;
}

__global__ void k_sched_pages(Dims D, Cfg C, State S, int lanes) {
    griddep_enter();
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int sub = lane / lanes, u0 = lane % lanes;
    const unsigned gmask = (lanes == 32 ? 0xffffffffu : ((1u << lanes) - 1u)) << (sub * lanes);
    const int64_t t = gt / lanes;  // page candidate index
    const int64_t total = (int64_t)D.B * D.R * D.ppr_sched;
    const bool in = t < total;
    const int64_t ring = in ? t / D.ppr_sched : 0;
    const int pi = in ? (int)(t % D.ppr_sched) : 0;
    const int s = (int)(ring / D.R);
    const bool skip = D.only_s >= 0 && s != D.only_s;  // pikv_evict_host: one stream
    const uint64_t seq = in && !skip ? S.seq[ring] : 0;
    const uint64_t Su = (uint64_t)D.S, ps = (uint64_t)D.page_size;
    const uint64_t lo = seq > Su ? seq - Su : 0;
    const uint64_t q = lo / ps + (uint64_t)pi;
    const int64_t rec = ring * D.ppr_sched + (int64_t)(q % (uint64_t)D.ppr_sched);
    if (C.record_agg) {  // lanes == 1
        // devices within budget evict nothing: select decides from the
        // live-page counter and never reads their keys
        if (!in || skip || S.pages_live[ring / D.SPD] <= C.budget_pages) return;
        double agg = 0.0;
        uint64_t oldest = 0;
        const int c2 = S.err[s] ? 0 : page_key_rec(D, C, S, ring, pi, S.now[s], agg, oldest);
        S.pg_cnt[t] = c2;
        S.pg_agg[t] = agg;
        S.pg_oldest[t] = oldest;
        return;
    }
    const int cnt = (in && !skip && q * ps < seq) ? S.pr_cnt[rec] : 0;
    const bool live_page = cnt > 0 && !S.err[s];
    const uint64_t now = in ? S.now[s] : 0;
    const int first = live_page ? S.pr_first[rec] : 0;
    const uint64_t s0 = (q * ps) % Su;
    const int w = (s0 + ps > Su) ? (int)(Su - s0) : 0;  // offsets wrapping to slot 0 come first
    double agg = 0.0;
    uint64_t oldest = ~0ull;
    for (int base = 0; base < (int)ps; base += lanes) {
        const int u = base + u0;
        bool mem = false;
        double sc = 0.0;
        uint64_t id = 0;
        if (live_page && u < (int)ps) {
            const int i = (w + u) % (int)ps;  // member offset in slot order
            if (D.holes ? page_member(D, S, ring, q, i) : (i >= first && i < first + cnt)) {
                const int64_t gi = ring * D.S + (int64_t)((q * ps + (uint64_t)i) % Su);
                id = S.id[gi];
                sc = score_entry(C, S, gi, now, D.n_layers);
                mem = true;
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, mem) & gmask;
        if (mem && id < oldest) oldest = id;
        if (C.exact_sum) {
            // every score and partial sum is exactly representable (integer /
            // dyadic scores, host-checked bound), so any order is bit-identical
            double x = mem ? sc : 0.0;
            for (int off = lanes >> 1; off; off >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, off));
            if (bal) agg = __dadd_rn(agg, x);
        } else {
            for (int v = 0; v < lanes; ++v) {  // sequential fp64 sum in slot order
                const double x = __shfl_sync(0xffffffffu, sc, sub * lanes + v);
                if (bal & (1u << (sub * lanes + v))) agg = __dadd_rn(agg, x);
            }
        }
    }
    for (int off = lanes >> 1; off; off >>= 1) {
        const uint64_t o2 = __shfl_xor_sync(0xffffffffu, oldest, off);
        oldest = o2 < oldest ? o2 : oldest;
    }
    if (in && !skip && u0 == 0) {
        S.pg_cnt[t] = live_page ? cnt : 0;
        S.pg_agg[t] = agg;
        S.pg_oldest[t] = live_page ? oldest : 0;
    }
}

__device__ __forceinline__ bool page_less(double a, uint64_t oa, double b, uint64_t ob) {
    return a != b ? a < b : oa < ob;
}

// (b) one CTA per (stream, local device): select_evictions + erase.
// Block-size generic (k_sched_select: 1024 threads, k_control: 512).
constexpr int kSelThreads = 1024;

// Erase scheduler page `pidx` of device sg (scheduler.cpp:305-326) with one
// warp: lanes over its members in id (= shard_seq) order, records from
// rec + o.  Returns the member count (lane 0's value is authoritative).
__device__ __forceinline__ int erase_page_warp(const Dims& D, const Cfg& C, const State& S, const int sg,
                                               const int pidx, const int reason, int o) {
    const int s = sg / D.Gl, gl = sg % D.Gl, lane = threadIdx.x & 31;
    const int64_t ring = (int64_t)sg * D.SPD + pidx / D.ppr_sched;
    const uint64_t seq = S.seq[ring];
    const uint64_t Su = (uint64_t)D.S, ps = (uint64_t)D.page_size;
    const uint64_t lo = seq > Su ? seq - Su : 0;
    const uint64_t q = lo / ps + (uint64_t)(pidx % D.ppr_sched);
    const uint64_t sstep = S.sstep[s], now = S.now[s];
    const int dev = gl * D.world + D.rank;
    EvictRec* rec = S.rec_ev + (int64_t)sg * D.SPD * D.S;
    const int o0 = o;
    for (uint64_t b0 = 0; b0 < ps; b0 += 32) {
        const uint64_t sq = q * ps + b0 + lane;
        bool mem = false;
        int64_t gi = 0;
        if (b0 + lane < ps) {
            gi = ring * D.S + (int64_t)(sq % Su);
            mem = S.id[gi] != 0 && S.shard_seq[gi] == sq;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, mem);
        if (mem) {
            EvictRec& r = rec[o + __popc(bal & ((1u << lane) - 1u))];
            r.step = sstep;
            r.entry_id = S.id[gi];
            r.token_id = S.token[gi];
            r.expert_id = S.expert[gi];
            r.device = dev;
            r.score = score_entry(C, S, gi, now, D.n_layers);
            r.reason = reason;
            r.stream = s;
            // KVStore::erase (kvstore.cpp:180-185) + page reclamation
            S.id[gi] = 0;
            atomicSub(&S.live[ring], 1);
            const int slot = (int)(sq % Su);
            const int64_t pt_i = ring * D.ppr + slot / D.spg;
            const int32_t page = S.page_table[pt_i];
            if (atomicSub(&S.page_live[page], 1) == 1) {
                S.page_table[pt_i] = -1;
                const int top = atomicAdd(S.free_top, 1);
                S.free_stack[top] = page;
            }
        }
        o += __popc(bal);
    }
    if (lane == 0) {  // the page is gone: reset its record
        const int64_t r = ring * D.ppr_sched + (int64_t)(q % (uint64_t)D.ppr_sched);
        if (S.pr_cnt[r] > 0) atomicSub(&S.pages_live[sg], 1);
        S.pr_cnt[r] = 0;
        S.pr_first[r] = 0;
        S.pr_sla[r] = 0;
        S.pr_sf[r] = 0;
    }
    return o - o0;
}

// Page count P, below-theta count T and the (aggregate, oldest) argmin over
// the pages i = first + tid + j * step (< np) of one device; the block's
// result lands in *out (shared memory), visible to all threads on return.
struct PageBest {
    int P, T, I;
    double A;
    uint64_t O;
};
__device__ __forceinline__ void merge_best(PageBest& a, const PageBest& b) {
    a.P += b.P;
    a.T += b.T;
    if (b.I >= 0 && (a.I < 0 || page_less(b.A, b.O, a.A, a.O))) a.A = b.A, a.O = b.O, a.I = b.I;
}
template <class KeyFn>
__device__ __forceinline__ void block_page_scan(const int np, const int first, const int step, KeyFn key,
                                                const double th, const bool ut, PageBest* out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
    PageBest b{0, 0, -1, 0.0, 0};
#pragma unroll 4
    for (int i = first + tid; i < np; i += step) {
        double a2;
        uint64_t o2;
        if (key(i, a2, o2) <= 0) continue;
        ++b.P;
        if (ut && a2 < th) ++b.T;
        if (b.I < 0 || page_less(a2, o2, b.A, b.O)) b.A = a2, b.O = o2, b.I = i;
    }
    __shared__ PageBest wb[32];
    for (int off = 16; off; off >>= 1) {
        PageBest o;
        o.P = __shfl_xor_sync(0xffffffffu, b.P, off);
        o.T = __shfl_xor_sync(0xffffffffu, b.T, off);
        o.A = __shfl_xor_sync(0xffffffffu, b.A, off);
        o.O = __shfl_xor_sync(0xffffffffu, b.O, off);
        o.I = __shfl_xor_sync(0xffffffffu, b.I, off);
        merge_best(b, o);
    }
    if (lane == 0) wb[warp] = b;
    __syncthreads();
    if (tid == 0) {
        PageBest r = wb[0];
        for (int w = 1; w < NW; ++w) merge_best(r, wb[w]);
        *out = r;
    }
    __syncthreads();
}

// select_evictions' count (scheduler.cpp:246-259) from the device's totals;
// records pages_before/after.  One thread.
__device__ __forceinline__ int decide_victims(const Cfg& C, const State& S, const int sg, const PageBest& b) {
    const int V0 = max(b.T, max(b.P - C.budget_pages, 0));
    S.pages_before[sg] = b.P;
    S.pages_after[sg] = b.P - V0;
    S.n_ev[sg] = 0;
    return V0;
}

// Fast path (the common steady state evicts 0 or 1 page): one pass over the
// page keys (key(i, agg, oldest) -> live count) computes P, T and the argmin;
// a single victim is erased directly.  Returns V (uniform); V > 1 is left to
// select_general.
template <class KeyFn>
__device__ __forceinline__ int select_fast(const Dims& D, const Cfg& C, const State& S, const int sg,
                                           KeyFn key) {
    const int s = sg / D.Gl;
    __shared__ PageBest sb;
    __shared__ int sV;
    block_page_scan(D.SPD * D.ppr_sched, 0, blockDim.x, key, S.theta[s],
                    C.sched_strategy == PIKV_SCHED_ADAKV, &sb);
    if (threadIdx.x == 0) sV = decide_victims(C, S, sg, sb);
    __syncthreads();
    const int V0 = sV;
    if (V0 == 1 && threadIdx.x < 32) {
        const int n = erase_page_warp(D, C, S, sg, sb.I, sb.T >= 1 ? PIKV_EVICT_THRESHOLD : PIKV_EVICT_BUDGET, 0);
        if (threadIdx.x == 0) S.n_ev[sg] = n;
    }
    return V0;
}

// General path (V > 1): recount from the materialised page keys (pg_*),
// select V victims (argmin rounds for V <= 32, bitonic sort otherwise) and
// erase them in order, a warp per victim page.
__device__ __forceinline__ void select_general(const Dims& D, const Cfg& C, const State& S, const int sg,
                                               const bool stage) {
    const int s = sg / D.Gl;
    const int tid = threadIdx.x, NT = blockDim.x, NW = NT / 32;
    __shared__ int sm_red[32];
    __shared__ int sm_P, sm_thr, sm_V;
    const int64_t first0 = (int64_t)sg * D.SPD * D.ppr_sched;  // pages of this device
    const int npg = D.SPD * D.ppr_sched;
    // page keys of this device: staged in shared memory when they fit (every
    // pass below then reads smem), else read in place from global memory
    extern __shared__ __align__(16) uint8_t sm_keys[];
    const double* KA = S.pg_agg + first0;
    const uint64_t* KO = S.pg_oldest + first0;
    int32_t* KC = S.pg_cnt + first0;
    if (stage) {
        double* a2 = (double*)sm_keys;
        uint64_t* o2 = (uint64_t*)(a2 + npg);
        int32_t* c2 = (int32_t*)(o2 + npg);
#pragma unroll 4
        for (int i = tid; i < npg; i += NT) {
            a2[i] = KA[i];
            o2[i] = KO[i];
            c2[i] = KC[i];
        }
        __syncthreads();
        KA = a2, KO = o2, KC = c2;
    }
    int32_t* list = S.sel_idx + (int64_t)sg * D.sel_stride;
    const double theta = S.theta[s];
    const bool use_theta = C.sched_strategy == PIKV_SCHED_ADAKV;
    // count pages and below-theta pages
    int P = 0, T = 0;
#pragma unroll 4
    for (int i = tid; i < npg; i += NT) {
        if (KC[i] > 0) {
            ++P;
            if (use_theta && KA[i] < theta) ++T;
        }
    }
    for (int off = 16; off; off >>= 1) {
        P += __shfl_xor_sync(0xffffffffu, P, off);
        T += __shfl_xor_sync(0xffffffffu, T, off);
    }
    if ((tid & 31) == 0) sm_red[tid >> 5] = P;
    __syncthreads();
    if (tid == 0) {
        int p = 0;
        for (int w = 0; w < NW; ++w) p += sm_red[w];
        sm_P = p;
    }
    __syncthreads();
    if ((tid & 31) == 0) sm_red[tid >> 5] = T;
    __syncthreads();
    if (tid == 0) {
        int t = 0;
        for (int w = 0; w < NW; ++w) t += sm_red[w];
        sm_thr = t;
        const int over = sm_P - C.budget_pages;
        sm_V = max(t, max(over, 0));  // select_evictions, scheduler.cpp:246-259
        S.pages_before[sg] = sm_P;
        S.pages_after[sg] = sm_P - sm_V;
        S.n_ev[sg] = 0;
    }
    __syncthreads();
    const int V = sm_V;
    if (V == 0) return;
    if (V <= 32) {
        // V rounds of block-wide argmin over (aggregate, oldest_id)
        for (int v = 0; v < V; ++v) {
            double ba = 0.0;
            uint64_t bo = 0;
            int bi = -1;
#pragma unroll 4
            for (int i = tid; i < npg; i += NT) {
                if (KC[i] <= 0) continue;
                const double a = KA[i];
                const uint64_t o = KO[i];
                if (bi < 0 || page_less(a, o, ba, bo)) ba = a, bo = o, bi = i;
            }
            for (int off = 16; off; off >>= 1) {
                double a2 = __shfl_xor_sync(0xffffffffu, ba, off);
                uint64_t o2 = __shfl_xor_sync(0xffffffffu, bo, off);
                int i2 = __shfl_xor_sync(0xffffffffu, bi, off);
                if (i2 >= 0 && (bi < 0 || page_less(a2, o2, ba, bo))) ba = a2, bo = o2, bi = i2;
            }
            __shared__ double wa[32];
            __shared__ uint64_t wo[32];
            __shared__ int wi[32];
            if ((tid & 31) == 0) wa[tid >> 5] = ba, wo[tid >> 5] = bo, wi[tid >> 5] = bi;
            __syncthreads();
            if (tid == 0) {
                int b = -1;
                double a = 0.0;
                uint64_t o = 0;
                for (int w = 0; w < NW; ++w) {
                    if (wi[w] >= 0 && (b < 0 || page_less(wa[w], wo[w], a, o))) a = wa[w], o = wo[w], b = wi[w];
                }
                list[v] = b;
                KC[b] = -KC[b];  // mark taken (negative count)
            }
            __syncthreads();
        }
    } else {
        // full bitonic sort of page indices by (aggregate, oldest_id) in the
        // scratch list (power-of-two capacity D.sel_stride; -1 sorts last),
        // then take the first V.
        const int n2 = D.sel_stride;
        for (int i = tid; i < n2; i += NT) list[i] = (i < npg && KC[i] > 0) ? i : -1;
        __syncthreads();
        auto key_less = [&](int a, int b) {
            if (a < 0) return false;
            if (b < 0) return true;
            return page_less(KA[a], KO[a], KA[b], KO[b]);
        };
        for (int kk = 2; kk <= n2; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < n2; i += NT) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const int a = list[i], b = list[ixj];
                        const bool up = (i & kk) == 0;
                        if (up ? key_less(b, a) : key_less(a, b)) {
                            list[i] = b;
                            list[ixj] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int v = tid; v < V; v += NT) KC[list[v]] = -KC[list[v]];
        __syncthreads();
    }
    // erase victims in order (scheduler.cpp:305-326): a warp per victim page;
    // record offsets are the exclusive prefix of member counts over victims
    // (block scan) plus the ballot rank inside the page.
    __shared__ int sm_off;
    __shared__ int vcnt_off[kSelThreads];
    if (tid == 0) sm_off = 0;
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5;
    for (int v0 = 0; v0 < V; v0 += NT) {
        const int v = v0 + tid;
        const int cnt = v < V ? -KC[list[v]] : 0;
        int x = cnt;
        for (int off = 1; off < 32; off <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        __shared__ int wsum[32];
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (tid < 32) {
            int w = tid < NW ? wsum[tid] : 0;
            for (int off = 1; off < 32; off <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, w, off);
                if (tid >= off) w += y;
            }
            wsum[tid] = w;
        }
        __syncthreads();
        vcnt_off[tid] = x - cnt + (warp ? wsum[warp - 1] : 0) + sm_off;
        __syncthreads();
        const int nv = min(NT, V - v0);
        for (int vv = warp; vv < nv; vv += NW) {
            const int reason = (v0 + vv) < sm_thr ? PIKV_EVICT_THRESHOLD : PIKV_EVICT_BUDGET;
            erase_page_warp(D, C, S, sg, list[v0 + vv], reason, vcnt_off[vv]);
        }
        __syncthreads();
        if (tid == NT - 1) sm_off = vcnt_off[tid] + cnt;
        __syncthreads();
    }
    if (tid == 0) S.n_ev[sg] = sm_off;
}

__device__ __forceinline__ bool within_budget(const Dims& D, const Cfg& C, const State& S, const int sg,
                                              const bool writer = true) {
    if (!(C.record_agg && S.pages_live[sg] <= C.budget_pages)) return false;
    if (writer && threadIdx.x == 0) {  // P <= K: nothing to evict
        const int P = S.pages_live[sg];
        S.pages_before[sg] = P;
        S.pages_after[sg] = P;
        S.n_ev[sg] = 0;
    }
    return true;
}

__device__ __forceinline__ void select_body(const Dims& D, const Cfg& C, const State& S, const int sg,
                                            const bool stage) {
    const int s = sg / D.Gl;
    if (D.only_s >= 0 && s != D.only_s) return;  // pikv_evict_host: one stream
    if (S.err[s]) return;
    if (within_budget(D, C, S, sg)) return;
    const int64_t f0 = (int64_t)sg * D.SPD * D.ppr_sched;
    const int V = select_fast(D, C, S, sg, [&](int i, double& a, uint64_t& o) {
        const int c = S.pg_cnt[f0 + i];
        if (c > 0) a = S.pg_agg[f0 + i], o = S.pg_oldest[f0 + i];
        return c;
    });
    if (V <= 1) return;
    __syncthreads();
    select_general(D, C, S, sg, stage);
}

// Evict for device sg inside k_control (record_agg strategies), by the
// stream's cluster: the page pass is split over the cluster's CTAs, partial
// (P, T, argmin) meet in rank 0's shared memory (DSMEM); rank 0 decides and
// erases.  V > 1 materialises the keys (split) and rank 0 runs select_general.
__device__ __forceinline__ void sched_device_cl(const Dims& D, const Cfg& C, const State& S, const int sg,
                                                cg::cluster_group& cl) {
    const int r = (int)cl.block_rank(), CL = (int)cl.num_blocks();
    if (within_budget(D, C, S, sg, r == 0)) return;  // uniform over the cluster
    const int s = sg / D.Gl, tid = threadIdx.x, NT = blockDim.x;
    const uint64_t now = S.now[s];
    const int64_t ring0 = (int64_t)sg * D.SPD;
    const int ppr = D.ppr_sched, np = D.SPD * ppr;
    auto rec_key = [&](int i, double& a, uint64_t& o) {
        return page_key_rec(D, C, S, ring0 + i / ppr, i % ppr, now, a, o);
    };
    __shared__ PageBest sb, parts[kMaxCluster];
    __shared__ int sV;
    block_page_scan(np, r * NT, CL * NT, rec_key, S.theta[s], C.sched_strategy == PIKV_SCHED_ADAKV, &sb);
    if (tid == 0) *cl.map_shared_rank(&parts[r], 0) = sb;
    cl.sync();
    if (r == 0 && tid == 0) {
        PageBest b = parts[0];
        for (int i = 1; i < CL; ++i) merge_best(b, parts[i]);
        sb = b;
        sV = decide_victims(C, S, sg, b);
    }
    cl.sync();
    const int V0 = *cl.map_shared_rank(&sV, 0);
    if (V0 == 1) {
        if (r == 0 && tid < 32) {
            const int n = erase_page_warp(D, C, S, sg, sb.I, sb.T >= 1 ? PIKV_EVICT_THRESHOLD : PIKV_EVICT_BUDGET, 0);
            if (tid == 0) S.n_ev[sg] = n;
        }
    } else if (V0 > 1) {
        const int64_t f0 = (int64_t)sg * np;
        for (int i = r * NT + tid; i < np; i += CL * NT) {
            double a = 0.0;
            uint64_t o = 0;
            S.pg_cnt[f0 + i] = rec_key(i, a, o);
            S.pg_agg[f0 + i] = a;
            S.pg_oldest[f0 + i] = o;
        }
        cl.sync();
        if (r == 0) select_general(D, C, S, sg, false);
    }
    cl.sync();
}

__global__ void __launch_bounds__(kSelThreads) k_sched_select(Dims D, Cfg C, State S, int stage) {
    griddep_enter();
    select_body(D, C, S, blockIdx.x, stage != 0);
}


void launch_sched_pages(const Dims& D, const Cfg& C, const State& S, cudaStream_t st) {
    int lanes = 1;
    while (!C.record_agg && lanes < D.page_size && lanes < 32) lanes <<= 1;
    const int64_t threads = (int64_t)D.B * D.R * D.ppr_sched * lanes;
    launch_pdl(k_sched_pages, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, st, D, C, S, lanes);
}

void launch_sched_select(const Dims& D, const Cfg& C, const State& S, cudaStream_t st) {
    const size_t keys = (size_t)D.SPD * D.ppr_sched * (8 + 8 + 4);
    const int stage = keys <= 200 * 1024 ? 1 : 0;
    const size_t smem = stage ? keys : 0;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_sched_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(k_sched_select, dim3(D.B * D.Gl), dim3(kSelThreads), smem, st, D, C, S, stage);
}

// ===========================================================================
// retrieve: KVStore::retrieve over the candidate rings
// ===========================================================================
// (a) count matches per (stream, candidate, chunk of chunk_slots slots)
__global__ void k_retr_count(Dims D, State S) {
    griddep_enter();
    const int s = blockIdx.x, c = blockIdx.y, ch = blockIdx.z;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ int red[32][kMaxK + 1];
    const int64_t ci = ((int64_t)s * D.max_cand + c) * D.nch + ch;
    const bool active = !S.err[s] && c < S.ncand[s];
    int j_hit = -1;
    if (active) {
        const int64_t ring = (int64_t)s * D.R + S.cand[(int64_t)s * D.max_cand + c];
        const uint64_t seq = S.seq[ring];
        const int fill = seq < (uint64_t)D.S ? (int)seq : D.S;
        const int slot = ch * D.chunk_slots + tid;
        if (slot < fill && tid < D.chunk_slots) {
            const int64_t gi = ring * D.S + slot;
            if (S.id[gi] != 0 && S.token[gi] < (int64_t)S.now[s]) {
                const int e = S.expert[gi];
                for (int j = 0; j < D.k; ++j)
                    if (S.experts[(int64_t)s * D.k + j] == e) {
                        j_hit = j;
                        break;
                    }
            }
        }
    }
    // per-warp counts: total and per selected expert
    const int nw = (int)(blockDim.x >> 5);
    const int tot = __popc(__ballot_sync(0xffffffffu, j_hit >= 0));
    if (lane == 0) red[warp][kMaxK] = tot;
    for (int j = 0; j < D.k; ++j) {
        const int cj = __popc(__ballot_sync(0xffffffffu, j_hit == j));
        if (lane == 0) red[warp][j] = cj;
    }
    __syncthreads();
    if (tid == 0) {
        int t = 0;
        for (int w = 0; w < nw; ++w) t += red[w][kMaxK];
        S.chunk_cnt[ci] = t;
    }
    if (active && tid < D.k) {
        int f = 0;
        for (int w = 0; w < nw; ++w) f += red[w][tid];
        if (f) atomicAdd(&S.found[(int64_t)s * D.k + tid], f);
    }
}

// (b) single CTA: in-stream chunk offsets (warp per stream), per-stream
//     bases and attention work items (block scans over streams).
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* wsum, int64_t* total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    int64_t x = v;
    for (int off = 1; off < 32; off <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < nw ? wsum[lane] : 0;
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    const int64_t excl = x - v + (warp ? wsum[warp - 1] : 0);
    *total = wsum[nw - 1];
    __syncthreads();
    return excl;
}

// The step's summary (StepResult counters) is complete before attention:
// this rank's view, made global by k_finish_merge.
__device__ __forceinline__ void write_summary(const Dims& D, const Cfg& C, const State& S, int s, int64_t n) {
    int nev = S.n_ow[s], pb = 0, pa = 0, hits = 0;
    for (int gl = 0; gl < D.Gl; ++gl) {
        nev += S.n_ev[s * D.Gl + gl];
        pb += S.pages_before[s * D.Gl + gl];
        pa += S.pages_after[s * D.Gl + gl];
    }
    for (int j = 0; j < D.k; ++j) hits += S.found[(int64_t)s * D.k + j] > 0;
    pikv_step_summary& sm = S.summary[s];
    sm.step = S.now[s];
    sm.inserts = D.k;
    sm.lookups = D.k;
    sm.hits = hits;
    sm.n_attended = (int32_t)n;
    const int hw = C.head_width < D.dp ? C.head_width : D.dp;  // pipeline.cpp:22-26, 262-264
    sm.fetch_elements = (int64_t)n * (int64_t)(2 * hw + D.dp);
    sm.n_evictions = nev;
    sm.pages_before = pb;
    sm.pages_after = pa;
    sm.error = S.err[s];
}

// Equal static shares (D.att_share): every stream's list is cut into units of
// one ring stage (att_eps entries, the last one partial), the units of all
// streams are laid end to end (stream-major) and attention CTA c takes units
// [floor(c U / Cn), floor((c + 1) U / Cn)) of the U in total.  A CTA's share
// becomes one work item per stream it touches, so items stay stream-major
// (item_first / k_combine unchanged), every CTA streams the same bytes (+-1
// stage) and has no ticket round trips; cta_first[c] is CTA c's first item
// (its items are cta_first[c] .. cta_first[c+1]-1).  Measured reason: with
// ~2 ticketed items per CTA, CTAs that got one item idled for half the launch,
// and a CTA's TMA ring streams at a fixed ~33 GB/s, so idle CTAs cost HBM
// bandwidth (profiles/microbench/attend_ctas.py).
__device__ __forceinline__ void build_items_shares(const Dims& D, const Cfg& C, const State& S, int64_t* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x, nw = nt >> 5;
    const int64_t eps = D.att_eps > 0 ? D.att_eps : 1;
    const int64_t Cg = D.attend_ctas;
    // pass 1: units per stream -> U
    int64_t U = 0;
    for (int s0 = 0; s0 < D.B; s0 += nt) {
        int64_t tot;
        const int64_t n = s0 + tid < D.B ? (int64_t)S.att_cnt[s0 + tid] : 0;
        block_excl_scan((n + eps - 1) / eps, wsum, &tot);
        U += tot;
    }
    // Cn CTAs get shares of >= mu units (>= 16 entries, as the ticketed items:
    // small steps would otherwise spread over many one-stage partials that the
    // merge then reads back); the rest none.
    // CTA of unit u: the largest c with floor(c U / Cn) <= u
    const int64_t mu = (16 + eps - 1) / eps;
    const int64_t Cn = U / mu < Cg ? (U / mu > 0 ? U / mu : 1) : Cg;
    auto cta_of = [&](int64_t u) { return ((u + 1) * Cn + U - 1) / U - 1; };
    // pass 2: items per stream (the CTAs its units span), item_first, summary
    int64_t carry = 0, ucarry = 0;
    for (int s0 = 0; s0 < D.B; s0 += nt) {
        const int s = s0 + tid;
        const int64_t n = s < D.B ? S.att_cnt[s] : 0;
        const int64_t us = (n + eps - 1) / eps;
        int64_t utot, tot;
        const int64_t a = block_excl_scan(us, wsum, &utot) + ucarry;
        const int64_t ni = us > 0 ? cta_of(a + us - 1) - cta_of(a) + 1 : 0;
        const int64_t first = block_excl_scan(ni, wsum, &tot) + carry;
        if (s < D.B) {
            S.item_first[s] = (int32_t)first;
            S.cta_first[Cg + 1 + s] = (int32_t)a;  // scratch: the stream's first unit
            write_summary(D, C, S, s, n);
        }
        carry += tot;
        ucarry += utot;
    }
    if (tid == 0) {
        S.item_first[D.B] = (int32_t)carry;
        S.n_items[0] = (int32_t)carry;
        S.n_items[1] = 0;
    }
    for (int64_t c = Cn + tid; c <= Cg; c += nt) S.cta_first[c] = (int32_t)carry;  // no share
    if (U == 0) {
        __syncthreads();
        return;
    }
    __syncthreads();
    // pass 3 (warp per stream): its items, and cta_first of the CTAs whose
    // share starts inside it (an empty share points at the next CTA's item)
    for (int s = warp; s < D.B; s += nw) {
        const int64_t n = S.att_cnt[s];
        const int64_t us = (n + eps - 1) / eps;
        const int64_t a = S.cta_first[Cg + 1 + s], b = a + us;
        const int64_t f = S.item_first[s];
        if (us == 0) continue;
        const int64_t clo = cta_of(a), chi = cta_of(b - 1);
        for (int64_t c = clo + lane; c <= chi; c += 32) {
            const int64_t ulo = max(c * U / Cn, a), uhi = min((c + 1) * U / Cn, b);
            const int64_t w = f + (c - clo);
            S.item_stream[w] = s;
            S.item_begin[w] = (int32_t)((ulo - a) * eps);
            S.item_end[w] = (int32_t)min((uhi - a) * eps, n);
        }
        // CTAs c with floor(c U / Cn) in [a, b): c in [ceil(a Cn / U), ceil(b Cn / U))
        const int64_t o0 = (a * Cn + U - 1) / U, o1 = (b * Cn + U - 1) / U;
        for (int64_t c = o0 + lane; c < o1 && c < Cn; c += 32) {
            const int64_t u = c * U / Cn;
            S.cta_first[c] = (int32_t)(f + (cta_of(u) - clo));
        }
    }
    __syncthreads();
}

// Attention work items from the per-stream attended counts (att_cnt): a
// stream's list is cut into items of C entries, C sized so the persistent
// attention grid gets ~items_per_cta items per CTA.  One CTA, any block size.
__device__ __forceinline__ void build_items(const Dims& D, const Cfg& C, const State& S) {
    __shared__ int64_t wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x, nw = nt >> 5;
    int64_t N = 0;
    for (int s0 = 0; s0 < D.B; s0 += nt) {
        int64_t tot;
        block_excl_scan(s0 + tid < D.B ? (int64_t)S.att_cnt[s0 + tid] : 0, wsum, &tot);
        N += tot;
    }
    if (D.att_share) {
        build_items_shares(D, C, S, wsum);
        return;
    }
    // entries per item: the smallest cs (>= 16) whose item count fits the
    // persistent attention grid (items_per_cta per CTA).  Each stream rounds
    // its own count up, so ceil(N / K) alone can overshoot K by up to B items
    // -- and a CTA running one item more than the others sets the kernel time
    // (measured: 304 items on 296 CTAs ran at 4.6 instead of 6.4 TB/s).
    const int64_t K = (int64_t)D.items_per_cta * D.attend_ctas;
    auto total_items = [&](int64_t c) {
        int64_t all = 0;
        for (int s0 = 0; s0 < D.B; s0 += nt) {
            int64_t tot;
            const int64_t n = s0 + tid < D.B ? (int64_t)S.att_cnt[s0 + tid] : 0;
            block_excl_scan((n + c - 1) / c, wsum, &tot);
            all += tot;
        }
        return all;
    };
    const int64_t eps = D.att_eps > 0 ? D.att_eps : 1;  // whole ring stages per item
    auto round_up = [&](int64_t c) { return (c + eps - 1) / eps * eps; };
    int64_t cs = round_up((N + K - 1) / K);
    if (cs < 16) cs = round_up(16);
    for (int it = 0; it < 3; ++it) {
        const int64_t t = total_items(cs);
        if (t <= K) break;
        const int64_t next = round_up((cs * t + K - 1) / K);
        cs = next > cs ? next : cs + eps;
    }
    if (K > D.B) {  // guarantee: sum ceil(n_s / cs) <= N / cs + B <= K
        const int64_t safe = round_up((N + (K - D.B) - 1) / (K - D.B));
        if (total_items(cs) > K && safe > cs) cs = safe;
    }
    int64_t carry = 0;
    for (int s0 = 0; s0 < D.B; s0 += nt) {
        const int s = s0 + tid;
        const int64_t n = s < D.B ? S.att_cnt[s] : 0;
        int64_t tot;
        const int64_t first = block_excl_scan((n + cs - 1) / cs, wsum, &tot) + carry;
        if (s < D.B) {
            S.item_first[s] = (int32_t)first;
            write_summary(D, C, S, s, n);
        }
        carry += tot;
    }
    if (tid == 0) {
        S.item_first[D.B] = (int32_t)carry;
        S.n_items[0] = (int32_t)carry;
        S.n_items[1] = 0;  // k_attend's item ticket
    }
    __syncthreads();
    for (int s = warp; s < D.B; s += nw) {
        const int64_t ns = S.att_cnt[s];
        const int64_t f = S.item_first[s];
        for (int64_t j = lane; j * cs < ns; j += 32) {
            S.item_stream[f + j] = s;
            S.item_begin[f + j] = (int32_t)(j * cs);
            S.item_end[f + j] = (int32_t)min(ns, (j + 1) * cs);
        }
    }
}

// (b) single CTA: in-stream chunk offsets (warp per stream), per-stream
//     counts, then the attention work items.
__global__ void __launch_bounds__(1024) k_retr_scan(Dims D, Cfg C, State S) {
    griddep_enter();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int per = D.max_cand * D.nch;
    for (int s = warp; s < D.B; s += nw) {
        int64_t run = 0;
        for (int b0 = 0; b0 < per; b0 += 32) {
            const int64_t ci = (int64_t)s * per + b0 + lane;
            const int c = b0 + lane < per ? S.chunk_cnt[ci] : 0;
            int x = c;
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off) x += y;
            }
            if (b0 + lane < per) S.chunk_off[ci] = (int32_t)(run + x - c);
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) S.att_cnt[s] = (int32_t)run;
    }
    __syncthreads();
    build_items(D, C, S);
}

// (c) write the compacted (slot, entry) lists; bump freq / last_access.
__global__ void k_retr_write(Dims D, State S) {
    griddep_enter();
    const int s = blockIdx.x, c = blockIdx.y, ch = blockIdx.z;
    const int tid = threadIdx.x;
    if (S.err[s] || c >= S.ncand[s]) return;
    const int64_t ci = ((int64_t)s * D.max_cand + c) * D.nch + ch;
    const int64_t ring = (int64_t)s * D.R + S.cand[(int64_t)s * D.max_cand + c];
    const uint64_t seq = S.seq[ring];
    const int fill = seq < (uint64_t)D.S ? (int)seq : D.S;
    const int slot = ch * D.chunk_slots + tid;
    const uint64_t now = S.now[s];
    int m = 0;
    int64_t gi = 0;
    if (slot < fill && tid < D.chunk_slots) {
        gi = ring * D.S + slot;
        if (S.id[gi] != 0 && S.token[gi] < (int64_t)now) {
            const int e = S.expert[gi];
            for (int j = 0; j < D.k; ++j)
                if (S.experts[(int64_t)s * D.k + j] == e) m = 1;
        }
    }
    // block exclusive scan of m (slot order)
    int x = m;
    for (int off = 1; off < 32; off <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, off);
        if ((tid & 31) >= off) x += y;
    }
    __shared__ int ws[32];
    if ((tid & 31) == 31) ws[tid >> 5] = x;
    __syncthreads();
    if (tid < 32) {
        int w = tid < (int)(blockDim.x >> 5) ? ws[tid] : 0;
        for (int off = 1; off < 32; off <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, off);
            if (tid >= off) w += y;
        }
        ws[tid] = w;
    }
    __syncthreads();
    if (m) {
        const int excl = x - 1 + ((tid >> 5) ? ws[(tid >> 5) - 1] : 0);
        const int64_t pos = (int64_t)s * D.att_stride + S.chunk_off[ci] + excl;
        S.att_slot[pos] = (int32_t)gi;
        const int32_t page = S.page_table[ring * D.ppr + slot / D.spg];
        S.att_entry[pos] = page * D.spg + slot % D.spg;
        const int64_t prec = page_rec(D, ring, S.shard_seq[gi]);
        atomicAdd((unsigned long long*)&S.pr_sla[prec], (unsigned long long)(now - S.last_access[gi]));
        atomicAdd((unsigned long long*)&S.pr_sf[prec], 1ull);
        S.freq[gi] += 1;  // kvstore.cpp:165-168
        S.last_access[gi] = now;
    }
}

// Retrieval for stream s by its cluster (k_control).  The stream's
// candidate rings (ascending) concatenated in slot order form one list of
// slots; rank r takes the r-th contiguous 1/CL of it.  Pass 1 counts the
// matches of each rank (and the per-expert hits); the counts meet in rank
// 0's shared memory and give each rank its output base; pass 2 writes the
// (slot, pool entry) lists in (ring, slot) order and bumps freq /
// last_access (kvstore.cpp:136-168) - the filter of k_retr_count/k_retr_write.
// Tiles of kRetrU x blockDim slots (thread t takes slots t, t + NT, ...).
constexpr int kRetrU = 4;

template <bool kWrite>
__device__ __forceinline__ int retrieve_tiles(const Dims& D, const State& S, const int s, const int64_t ring,
                                              const int a, const int b, const uint64_t now, const int* sm_ex,
                                              int* sm_found, int* sm_off, int* sm_tile, int64_t out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x, NW = NT >> 5;
    int mine = 0;
    for (int t0 = a; t0 < b; t0 += kRetrU * NT) {
        uint64_t id[kRetrU];
        int64_t tok[kRetrU] = {};
        int ex[kRetrU] = {};
#pragma unroll
        for (int u = 0; u < kRetrU; ++u) {
            const int slot = t0 + u * NT + tid;
            id[u] = 0;
            if (slot < b) {
                const int64_t gi = ring * D.S + slot;
                id[u] = S.id[gi];
                tok[u] = S.token[gi];
                ex[u] = S.expert[gi];
            }
        }
        int jh[kRetrU];
#pragma unroll
        for (int u = 0; u < kRetrU; ++u) {
            jh[u] = -1;
            if (id[u] != 0 && tok[u] < (int64_t)now)
                for (int j = 0; j < D.k; ++j)
                    if (sm_ex[j] == ex[u]) {
                        jh[u] = j;
                        break;
                    }
        }
        if constexpr (!kWrite) {
#pragma unroll
            for (int u = 0; u < kRetrU; ++u)
                if (jh[u] >= 0) ++mine, atomicAdd(&sm_found[jh[u]], 1);
        } else {
        unsigned bal[kRetrU];
#pragma unroll
        for (int u = 0; u < kRetrU; ++u) {
            bal[u] = __ballot_sync(0xffffffffu, jh[u] >= 0);
            if (lane == 0) sm_off[u * NW + warp] = __popc(bal[u]);
        }
        __syncthreads();
        if (warp == 0) {  // exclusive scan over (u, warp) = slot order
            const int n = kRetrU * NW, per = (n + 31) / 32;
            int loc[kRetrU];  // per <= kRetrU (NW <= 32)
            int sum = 0;
            for (int i = 0; i < per; ++i) {
                const int idx = lane * per + i;
                loc[i] = idx < n ? sm_off[idx] : 0;
                sum += loc[i];
            }
            int x = sum;
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off) x += y;
            }
            int e = x - sum;
            for (int i = 0; i < per; ++i) {
                const int idx = lane * per + i;
                if (idx < n) sm_off[idx] = e;
                e += loc[i];
            }
            if (lane == 31) *sm_tile = x;
        }
        __syncthreads();
        // every load of the tile first (all in flight), then the stores:
        // interleaving them would serialise the tile on may-alias ordering
        int32_t page[kRetrU];
        uint64_t sq[kRetrU], la[kRetrU], fr[kRetrU];
#pragma unroll
        for (int u = 0; u < kRetrU; ++u) {
            if (jh[u] < 0) continue;
            const int slot = t0 + u * NT + tid;
            const int64_t gi = ring * D.S + slot;
            page[u] = S.page_table[ring * D.ppr + slot / D.spg];
            sq[u] = S.shard_seq[gi];
            la[u] = S.last_access[gi];
            fr[u] = S.freq[gi];
        }
#pragma unroll
        for (int u = 0; u < kRetrU; ++u) {
            if (jh[u] < 0) continue;
            const int slot = t0 + u * NT + tid;
            const int64_t gi = ring * D.S + slot;
            const int64_t pos = out + sm_off[u * NW + warp] + __popc(bal[u] & ((1u << lane) - 1u));
            S.att_slot[pos] = (int32_t)gi;
            S.att_entry[pos] = page[u] * D.spg + slot % D.spg;
            const int64_t prec = page_rec(D, ring, sq[u]);
            atomicAdd((unsigned long long*)&S.pr_sla[prec], (unsigned long long)(now - la[u]));
            atomicAdd((unsigned long long*)&S.pr_sf[prec], 1ull);
            S.freq[gi] = fr[u] + 1;  // kvstore.cpp:165-168
            S.last_access[gi] = now;
        }
        out += *sm_tile;
        mine += *sm_tile;
        __syncthreads();  // sm_off / sm_tile reused by the next tile
        }
    }
    return mine;  // kWrite: block total; else this thread's count
}

__device__ __forceinline__ void gstamp(long long* p) {
    if (p && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        *p = (long long)t;
    }
}

__device__ __forceinline__ void retrieve_cl(const Dims& D, const State& S, const int s, cg::cluster_group& cl,
                                            long long* dbg) {
    const int r = (int)cl.block_rank(), CL = (int)cl.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x;
    __shared__ int sm_ex[kMaxK], sm_found[kMaxK];
    __shared__ int sm_off[kRetrU * 32];
    __shared__ int sm_tile, sm_red[32];
    __shared__ int sm_cnt[kMaxCluster];
    for (int j = tid; j < D.k; j += NT) {
        sm_ex[j] = S.experts[(int64_t)s * D.k + j];
        sm_found[j] = 0;
    }
    __syncthreads();
    const uint64_t now = S.now[s];
    const int nc = S.ncand[s];
    int64_t total = 0;
    for (int c = 0; c < nc; ++c) {
        const uint64_t seq = S.seq[(int64_t)s * D.R + S.cand[(int64_t)s * D.max_cand + c]];
        total += seq < (uint64_t)D.S ? (int64_t)seq : D.S;
    }
    const int64_t lo = total * r / CL, hi = total * (r + 1) / CL;
    // pass 1: count
    int mine = 0;
    {
        int64_t off = 0;
        for (int c = 0; c < nc; ++c) {
            const int64_t ring = (int64_t)s * D.R + S.cand[(int64_t)s * D.max_cand + c];
            const uint64_t seq = S.seq[ring];
            const int fill = seq < (uint64_t)D.S ? (int)seq : D.S;
            const int a = (int)(max(lo, off) - off), b = (int)(min(hi, off + fill) - off);
            if (a < b) mine += retrieve_tiles<false>(D, S, s, ring, a, b, now, sm_ex, sm_found, sm_off, &sm_tile, 0);
            off += fill;
        }
    }
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0) sm_red[warp] = mine;
    __syncthreads();
    if (tid == 0) {
        int t = 0;
        for (int w = 0; w < (NT >> 5); ++w) t += sm_red[w];
        *cl.map_shared_rank(&sm_cnt[r], 0) = t;
    }
    for (int j = tid; j < D.k; j += NT)
        if (sm_found[j]) atomicAdd(&S.found[(int64_t)s * D.k + j], sm_found[j]);
    gstamp(dbg);
    cl.sync();
    gstamp(dbg ? dbg + 1 : nullptr);
    int base = 0, all = 0;
    {
        const int* c0 = cl.map_shared_rank(sm_cnt, 0);
        for (int i = 0; i < CL; ++i) {
            const int x = c0[i];
            if (i < r) base += x;
            all += x;
        }
    }
    if (r == 0 && tid == 0) S.att_cnt[s] = all;
    // pass 2: write
    int64_t out = (int64_t)s * D.att_stride + base;
    int64_t off = 0;
    for (int c = 0; c < nc; ++c) {
        const int64_t ring = (int64_t)s * D.R + S.cand[(int64_t)s * D.max_cand + c];
        const uint64_t seq = S.seq[ring];
        const int fill = seq < (uint64_t)D.S ? (int)seq : D.S;
        const int a = (int)(max(lo, off) - off), b = (int)(min(hi, off + fill) - off);
        if (a < b) out += retrieve_tiles<true>(D, S, s, ring, a, b, now, sm_ex, sm_found, sm_off, &sm_tile, out);
        off += fill;
    }
    cl.sync();  // rank 0's sm_cnt stays readable until every rank has read it
}

// ===========================================================================
// control: the whole pre-attention part of the step, one cluster per stream
// ===========================================================================
// route -> insert (rank 0) -> evict (each local device) -> retrieve (whole
// cluster), with cluster barriers between phases: streams are independent
// until attention, so no stream waits for the slowest stream's phase (the
// multi-kernel path's grid barriers) and the memory-parallel phases still
// get CL SMs per stream.  The last CTA builds the attention work items.
// Used for record_agg strategies (LRU/LRU+) and unbounded budgets, whose
// eviction keys come from the page records; other strategies run the
// multi-kernel path (their keys need the wide member scan).
constexpr int kCtlThreads = 512;
__global__ void __launch_bounds__(kCtlThreads, 1)
    k_control(Dims D, Cfg C, State S, const void* __restrict__ qin, const void* __restrict__ kin,
              const void* __restrict__ vin, const double* __restrict__ saliency, int route_ch) {
    griddep_enter();
    extern __shared__ __align__(128) uint8_t sm_dyn[];
    cg::cluster_group cl = cg::this_cluster();
    const int r = (int)cl.block_rank();
    const int s = blockIdx.x / (int)cl.num_blocks(), tid = threadIdx.x;
    auto stamp = [&](int p) {
        if (D.dbg_ctl && tid == 0 && r == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            S.dbg[64 + 8 * s + p] = (long long)t;
        }
    };
    stamp(0);
    if (r == 0) {
        if (tid == 0) S.att_cnt[s] = 0;
        const int* sel = route_body(D, C, S, s, qin, route_ch, sm_dyn);
        __syncthreads();
        stamp(1);
        if (!S.err[s]) insert_body(D, C, S, s, qin, kin, vin, saliency, sm_dyn, sel);
    }
    cl.sync();
    stamp(2);
    const bool ok = !S.err[s];
    if (ok && !C.unbounded_budget)
        for (int gl = 0; gl < D.Gl; ++gl) sched_device_cl(D, C, S, s * D.Gl + gl, cl);
    stamp(3);
    if (ok) retrieve_cl(D, S, s, cl, D.dbg_ctl && r == 0 ? S.dbg + 64 + 8 * s + 6 : nullptr);
    stamp(4);
    // last CTA of the grid: attention work items over all streams
    __shared__ bool sm_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) sm_last = atomicAdd(S.ctl_ctr, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!sm_last) return;
    __threadfence();
    build_items(D, C, S);
    if (tid == 0) *S.ctl_ctr = 0;
    if (D.dbg_ctl && tid == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        S.dbg[64 + 8 * s + 5] = (long long)t;
    }
}

bool control_supported(const Dims& D, const Cfg& C) {
    return (C.record_agg || C.unbounded_budget) && D.E + 32 <= kCtlThreads;
}

// Launch geometry of k_control, fixed per engine: the route's W ring is
// sized so two CTAs fit per SM (only rank 0 uses it, but every CTA of a
// launch gets the same shared memory), and the cluster size is the largest
// power of two <= 8 whose B clusters are all co-resident
// (cudaOccupancyMaxActiveClusters): a cluster that waits for a second wave
// delays its whole stream.
// k_control launch geometry, fixed per engine (Dims::ctl_cl / ctl_smem, set
// at creation): shared memory for the route ring or the insert staging,
// and the largest cluster size <= 8 whose B clusters are co-resident
// (cudaOccupancyMaxActiveClusters) -- a cluster waiting for a second wave
// delays its whole stream.
void control_geometry(Dims& D) {
    size_t smem = std::max(route_smem_bytes(D, D.route_ch), insert_smem_bytes(D));
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_control, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int best = 1;
    for (int cl = kMaxCluster; cl > 1; --cl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(D.B * cl);
        cfg.blockDim = dim3(kCtlThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int active = 0;
        const cudaError_t e = cudaOccupancyMaxActiveClusters(&active, k_control, &cfg);
        if (D.dbg_ctl)
            fprintf(stderr, "[k_control] cluster %d: max active %d (B %d, smem %zu, ch %d)\n", cl, active, D.B, smem,
                    D.route_ch);
        if (e == cudaSuccess && active >= D.B) {
            best = cl;
            break;
        }
        cudaGetLastError();
    }
    if (const char* v = std::getenv("PIKV_CTL_CLUSTER")) best = std::max(1, std::min(kMaxCluster, std::atoi(v)));
    D.ctl_cl = best;
    D.ctl_smem = (int)smem;
}

void launch_control(const Dims& D, const Cfg& C, const State& S, const void* q, const void* k, const void* v,
                    const double* saliency, cudaStream_t st) {
    launch_cluster(k_control, dim3(D.B * D.ctl_cl), dim3(kCtlThreads), (size_t)D.ctl_smem, st, D.ctl_cl, D, C, S,
                   q, k, v, saliency, D.route_ch);
}

// Single-pass retrieval (replaces count / scan / write): chunk tiles are
// taken in (stream, candidate ring, chunk) order through a ticket (so every
// tile's predecessors are already running: no deadlock however few CTAs are
// resident); a tile counts its matches, publishes its aggregate, looks back
// for its predecessors' inclusive prefix (decoupled look-back) and writes
// its entries in (ring, slot) order.  The last tile builds the work items.
// S.chunk_off holds the look-back words: bit 63 = inclusive, bit 62 =
// aggregate only, low 32 bits the value.
__global__ void __launch_bounds__(1024) k_retr_fused(Dims D, Cfg C, State S) {
    griddep_enter();
    __shared__ int sm_tile, sm_off, ws[32];
    __shared__ int red[32][kMaxK + 1];
    __shared__ bool sm_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = (int)(blockDim.x >> 5);
    unsigned long long* look = (unsigned long long*)S.chunk_off;  // [B * max_cand * nch]
    const int per = D.max_cand * D.nch;
    if (tid == 0) sm_tile = (int)atomicAdd(S.ctl_ctr + 1, 1u);
    __syncthreads();
    const int tile = sm_tile;
    const int s = tile / per, L = tile % per, c = L / D.nch, ch = L % D.nch;
    const bool active = !S.err[s] && c < S.ncand[s];
    int j_hit = -1;
    int64_t ring = 0, gi = 0;
    const int slot = ch * D.chunk_slots + tid;
    const uint64_t now = S.now[s];
    if (active) {
        ring = (int64_t)s * D.R + S.cand[(int64_t)s * D.max_cand + c];
        const uint64_t seq = S.seq[ring];
        const int fill = seq < (uint64_t)D.S ? (int)seq : D.S;
        if (slot < fill && tid < D.chunk_slots) {
            gi = ring * D.S + slot;
            if (S.id[gi] != 0 && S.token[gi] < (int64_t)now) {
                const int e = S.expert[gi];
                for (int j = 0; j < D.k; ++j)
                    if (S.experts[(int64_t)s * D.k + j] == e) {
                        j_hit = j;
                        break;
                    }
            }
        }
    }
    // block scan of the match flags (slot order) + per-expert hit counts
    const int m = j_hit >= 0;
    int x = m;
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) ws[warp] = x;
    for (int j = 0; j < D.k; ++j) {
        const int cj = __popc(__ballot_sync(0xffffffffu, j_hit == j));
        if (lane == 0) red[warp][j] = cj;
    }
    __syncthreads();
    if (tid < 32) {
        int w = tid < nw ? ws[tid] : 0;
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, off);
            if (tid >= off) w += y;
        }
        ws[tid] = w;
    }
    if (active && tid < D.k) {
        int f = 0;
        for (int w2 = 0; w2 < nw; ++w2) f += red[w2][tid];
        if (f) atomicAdd(&S.found[(int64_t)s * D.k + tid], f);
    }
    __syncthreads();
    const int agg = ws[nw - 1];
    // publish, then look back over this stream's earlier tiles with warp 0:
    // 32 predecessors per pass, summing aggregates back to the nearest
    // inclusive prefix (every tile publishes its aggregate right after
    // counting, so this rarely waits)
    if (warp == 0) {
        unsigned long long* base = look + (int64_t)s * per;
        if (lane == 0) atomicExch(base + L, (L == 0 ? (1ull << 63) : (1ull << 62)) | (unsigned)agg);
        int acc = 0;
        for (int p0 = L - 1; p0 >= 0; p0 -= 32) {
            const int p = p0 - lane;
            unsigned long long v = 0;
            if (p >= 0) do {
                    v = atomicAdd(base + p, 0ull);
                } while ((v >> 62) == 0);
            const unsigned incl = __ballot_sync(0xffffffffu, p >= 0 && (v >> 63));
            const int stop = incl ? __ffs(incl) - 1 : 32;  // nearest inclusive predecessor
            int part = (p >= 0 && lane <= stop) ? (int)(v & 0xffffffffu) : 0;
            for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            acc += part;
            if (incl) break;
        }
        if (lane == 0) {
            if (L > 0) atomicExch(base + L, (1ull << 63) | (unsigned)(acc + agg));
            sm_off = acc;
            __threadfence();
        }
    }
    __syncthreads();
    if (m) {
        const int excl = x - 1 + (warp ? ws[warp - 1] : 0);
        const int64_t pos = (int64_t)s * D.att_stride + sm_off + excl;
        S.att_slot[pos] = (int32_t)gi;
        const int32_t page = S.page_table[ring * D.ppr + slot / D.spg];
        S.att_entry[pos] = page * D.spg + slot % D.spg;
        const int64_t prec = page_rec(D, ring, S.shard_seq[gi]);
        atomicAdd((unsigned long long*)&S.pr_sla[prec], (unsigned long long)(now - S.last_access[gi]));
        atomicAdd((unsigned long long*)&S.pr_sf[prec], 1ull);
        S.freq[gi] += 1;  // kvstore.cpp:165-168
        S.last_access[gi] = now;
    }
    if (tid == 0 && L == per - 1) S.att_cnt[s] = sm_off + agg;  // the stream's total
    // last tile: work items over all streams, then reset the look-back words
    __threadfence();
    __syncthreads();
    if (tid == 0) sm_last = atomicAdd(S.ctl_ctr + 2, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!sm_last) return;
    __threadfence();
    build_items(D, C, S);
    for (int i = tid; i < D.B * per; i += blockDim.x) look[i] = 0;
    if (tid == 0) S.ctl_ctr[1] = 0, S.ctl_ctr[2] = 0;
}

void launch_retr_fused(const Dims& D, const Cfg& C, const State& S, cudaStream_t st) {
    launch_pdl(k_retr_fused, dim3(D.B * D.max_cand * D.nch), dim3(D.chunk_slots), 0, st, D, C, S);
}

void launch_retr_count(const Dims& D, const State& S, cudaStream_t st) {
    launch_pdl(k_retr_count, dim3(D.B, D.max_cand, D.nch), dim3(D.chunk_slots), 0, st, D, S);
}
void launch_retr_scan(const Dims& D, const Cfg& C, const State& S, cudaStream_t st) {
    launch_pdl(k_retr_scan, dim3(1), dim3(1024), 0, st, D, C, S);
}
void launch_retr_write(const Dims& D, const State& S, cudaStream_t st) {
    launch_pdl(k_retr_write, dim3(D.B, D.max_cand, D.nch), dim3(D.chunk_slots), 0, st, D, S);
}

// ===========================================================================
// combine: per-stream merge of work-item partials into the exchange record
// ===========================================================================
// LSE merge of one (stream, head) over its work items: y and the global
// (M, L) (single rank), or the exchange record's (o, m, l) plus its found /
// stats part for the cross-rank merge.
__global__ void k_combine(Dims D, Cfg C, State S, ExchangeLayout X, float* __restrict__ y, int direct,
                          int attended) {
    griddep_enter();
    const int s = blockIdx.x, h = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    extern __shared__ float sm_f[];  // [n_items of stream s] scale factors
    __shared__ float red[32];
    uint8_t* rec = S.exchange + (int64_t)s * X.bytes_per_stream;
    const int w0 = S.item_first[s];
    const int nw = attended ? S.item_first[s + 1] - w0 : 0;
    const bool ok = !S.err[s];
    float M = -INFINITY;
    for (int i = tid; i < nw; i += blockDim.x) M = fmaxf(M, S.part_m[(int64_t)(w0 + i) * D.H + h]);
    for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    if (lane == 0) red[warp] = M;
    __syncthreads();
    M = -INFINITY;
    for (int w = 0; w < nwarp; ++w) M = fmaxf(M, red[w]);
    __syncthreads();
    float L = 0.f;
    for (int i = tid; i < nw; i += blockDim.x) {
        const float f = M == -INFINITY ? 0.f : exp2f(S.part_m[(int64_t)(w0 + i) * D.H + h] - M);
        sm_f[i] = f;
        L += S.part_l[(int64_t)(w0 + i) * D.H + h] * f;
    }
    for (int off = 16; off; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
    if (lane == 0) red[warp] = L;
    __syncthreads();
    L = 0.f;
    for (int w = 0; w < nwarp; ++w) L += red[w];
    // o: G groups of dph threads split the items (group g takes i = g, g+G, ...),
    // summed in group order through shared memory -- many items per stream
    // (small batches) no longer serialise on one thread per output
    const int G = (D.dph > 0 && (int)blockDim.x % D.dph == 0) ? (int)blockDim.x / D.dph : 1;
    float* red_o = sm_f + D.item_cap;  // [G][dph]
    if (G > 1) {
        const int g = tid / D.dph, o = tid % D.dph;
        float acc = 0.f;
        const float* po = S.part_o + ((int64_t)w0 * D.H + h) * D.dph + o;
        const int64_t stride = (int64_t)D.H * D.dph;
#pragma unroll 4
        for (int i = g; i < nw; i += G) acc = fmaf(po[i * stride], sm_f[i], acc);
        red_o[g * D.dph + o] = acc;
        __syncthreads();
    }
    for (int o = tid; o < D.dph; o += blockDim.x) {
        float acc = 0.f;
        if (G > 1) {
            for (int g = 0; g < G; ++g) acc += red_o[g * D.dph + o];
        } else {
            const float* po = S.part_o + ((int64_t)w0 * D.H + h) * D.dph + o;
            const int64_t stride = (int64_t)D.H * D.dph;
#pragma unroll 8
            for (int i = 0; i < nw; ++i) acc = fmaf(po[i * stride], sm_f[i], acc);
        }
        if (direct) {
            if (y && ok) y[(int64_t)s * D.dp + h * D.dph + o] = L > 0.f ? acc / L : 0.f;
        } else {
            ((float*)(rec + X.o_off))[h * D.dph + o] = ok ? acc : 0.f;
        }
    }
    if (tid != 0) return;
    if (direct) {  // single rank: the global (M, L) for the fold-back
        S.gM[s * D.H + h] = M;
        S.gL[s * D.H + h] = L;
        return;
    }
    ((float*)(rec + X.m_off))[h] = ok ? M : -INFINITY;
    ((float*)(rec + X.l_off))[h] = ok ? L : 0.f;
    if (h == 0) {
        const pikv_step_summary& sm = S.summary[s];  // this rank's counts (build_items)
        int32_t* xf = (int32_t*)(rec + X.found_off);
        int32_t* xs = (int32_t*)(rec + X.stats_off);
        for (int j = 0; j < D.k; ++j) xf[j] = S.found[(int64_t)s * D.k + j];
        xs[0] = sm.n_attended;
        xs[1] = sm.n_evictions;
        xs[2] = sm.pages_before;
        xs[3] = sm.pages_after;
    }
}

void launch_combine(const Dims& D, const Cfg& C, const State& S, const ExchangeLayout& X, float* y,
                    int direct, int attended, cudaStream_t st) {
    // dph threads per item group, up to 4 groups (512 threads)
    int threads = D.dph >= 128 ? 128 : (D.dph >= 64 ? 64 : 32);
    if (D.dph <= 128 && 128 % D.dph == 0) threads = std::max(32, std::min(512, 4 * D.dph));
    const size_t smem = sizeof(float) * ((size_t)D.item_cap + (size_t)threads);
    launch_pdl(k_combine, dim3(D.B, D.H), dim3(threads), smem, st, D, C, S, X, y, direct, attended);
}

// ===========================================================================
// finish: cross-rank merge, fold-back, feedback
// ===========================================================================

// ===========================================================================
// finish: cross-rank merge -> y, global (m, l), summary
// ===========================================================================
__global__ void k_finish_merge(Dims D, Cfg C, State S, ExchangeLayout X,
                               const uint8_t* __restrict__ gathered, float* __restrict__ y, int granks) {
    griddep_enter();
    const int s = blockIdx.x, tid = threadIdx.x;
    D.world = granks;  // records present in `gathered`
    const int64_t stride_rank = (int64_t)D.B * X.bytes_per_stream;
    for (int o = tid; o < D.H * D.dph; o += blockDim.x) {
        const int h = o / D.dph;
        float M = -INFINITY;
        for (int r = 0; r < D.world; ++r) {
            const uint8_t* rec = gathered + r * stride_rank + (int64_t)s * X.bytes_per_stream;
            M = fmaxf(M, ((const float*)(rec + X.m_off))[h]);
        }
        float L = 0.f, acc = 0.f;
        if (M != -INFINITY) {
            for (int r = 0; r < D.world; ++r) {
                const uint8_t* rec = gathered + r * stride_rank + (int64_t)s * X.bytes_per_stream;
                const float mr = ((const float*)(rec + X.m_off))[h];
                if (mr == -INFINITY) continue;
                const float f = exp2f(mr - M);
                L += ((const float*)(rec + X.l_off))[h] * f;
                acc += ((const float*)(rec + X.o_off))[o] * f;
            }
        }
        if (y && !S.err[s]) y[(int64_t)s * D.dp + o] = L > 0.f ? acc / L : 0.f;  // empty -> 0
        if (o % D.dph == 0) {
            S.gM[s * D.H + h] = M;
            S.gL[s * D.H + h] = L;
        }
    }
    if (tid == 0) {
        int n_att = 0, nev = 0, pb = 0, pa = 0, hits = 0;
        for (int j = 0; j < D.k; ++j) {
            int f = 0;
            for (int r = 0; r < D.world; ++r) {
                const uint8_t* rec = gathered + r * stride_rank + (int64_t)s * X.bytes_per_stream;
                f += ((const int32_t*)(rec + X.found_off))[j];
            }
            S.found[(int64_t)s * D.k + j] = f;  // global per-expert hit counts
            hits += f > 0;
        }
        for (int r = 0; r < D.world; ++r) {
            const int32_t* xs = (const int32_t*)(gathered + r * stride_rank +
                                                 (int64_t)s * X.bytes_per_stream + X.stats_off);
            n_att += xs[0], nev += xs[1], pb += xs[2], pa += xs[3];
        }
        pikv_step_summary& sm = S.summary[s];
        sm.step = S.now[s];
        sm.inserts = D.k;
        sm.lookups = D.k;
        sm.hits = hits;
        sm.n_attended = n_att;
        // pipeline.cpp:262-264, 22-26
        const int hw = C.head_width < D.dp ? C.head_width : D.dp;
        sm.fetch_elements = (int64_t)n_att * (int64_t)(2 * hw + D.dp);
        sm.n_evictions = nev;
        sm.pages_before = pb;
        sm.pages_after = pa;
        sm.error = S.err[s];
    }
}

// feedback for stream s (see k_feedback)
__device__ __forceinline__ void feedback_stream(const Dims& D, const Cfg& C, const State& S, int s) {
    if (S.err[s]) return;
    const int k = D.k, E = D.E;
    int hits = 0;
    for (int j = 0; j < k; ++j) {
        if (S.found[(int64_t)s * k + j] > 0) ++hits;
        else S.miss[(int64_t)s * E + S.experts[(int64_t)s * k + j]] += 1;
    }
    S.st_retrievals[s] += 1;  // KVStore::retrieve stats (kvstore.cpp:169-176)
    S.st_misses[s] += (uint64_t)(k - hits);
    const double reward = __ddiv_rn((double)hits, (double)k);
    if (C.router_strategy == PIKV_ROUTER_ADAPTIVE) {  // adapt, router.cpp:243-255
        double* bias = S.bias + (int64_t)s * E;
        double acc = 0.0;
        for (int e = 0; e < E; ++e) acc = __dadd_rn(acc, bias[e]);
        const double mean = __ddiv_rn(acc, (double)E);
        for (int j = 0; j < k; ++j) {
            const int e = S.experts[(int64_t)s * k + j];
            double b = __dadd_rn(bias[e], __dmul_rn(C.bandit_step, __dsub_rn(reward, mean)));
            bias[e] = b < -C.bias_cap ? -C.bias_cap : (C.bias_cap < b ? C.bias_cap : b);
        }
    }
    // observe_hits, scheduler.cpp:332-338
    S.running_hit[s] = __dadd_rn(__dmul_rn(C.hit_decay, S.running_hit[s]),
                                 __dmul_rn(__dsub_rn(1.0, C.hit_decay), reward));
    if (C.sched_strategy == PIKV_SCHED_ADAKV && !C.unbounded_budget)  // :340-342
        S.theta[s] = __dadd_rn(S.theta[s], __dmul_rn(C.adakv_step, __dsub_rn(C.target_hit, S.running_hit[s])));
    if (!C.unbounded_budget) S.sstep[s] += 1;
    S.now[s] += 1;
}

// attn_mass += alpha, pipeline.cpp:302-312; alpha = mean over heads.  One
// thread per retrieved entry (its H logits are contiguous: 16-byte loads);
// the global (M, 1/L) of every (stream, head) are staged in shared memory.
__global__ void k_foldback(Dims D, Cfg C, State S) {
    griddep_enter();
    // grid (X, B): blockIdx.y = stream, the X CTAs of a stream stride over its
    // attended entries (no scan of the empty tail of the stream's region, no
    // 64-bit division per slot: 3.9 M warp-instructions and 34.8 us per c4
    // launch before, profiles/README.md)
    extern __shared__ float sm_ml[];  // [H] M, then [H] 1/L (0 when empty)
    const int s = blockIdx.y;
    for (int h = threadIdx.x; h < D.H; h += blockDim.x) {
        sm_ml[h] = S.gM[s * D.H + h];
        const float L = S.gL[s * D.H + h];
        sm_ml[D.H + h] = L > 0.f ? 1.f / L : 0.f;
    }
    __syncthreads();
    const int cnt = S.err[s] ? 0 : S.att_cnt[s];
    const float* M = sm_ml;
    const float* iL = sm_ml + D.H;
    const bool vec = (D.H % 4) == 0;
    const int64_t base = (int64_t)s * D.att_stride;
    const uint64_t now = S.now[s];
    auto alpha = [&](int64_t i) {
        const float* sc = S.scores + i * D.H;
        float a = 0.f;
        if (vec) {
            for (int h = 0; h < D.H; h += 4) {
                const float4 v = *(const float4*)(sc + h);
                a += exp2f(v.x - M[h]) * iL[h] + exp2f(v.y - M[h + 1]) * iL[h + 1] +
                     exp2f(v.z - M[h + 2]) * iL[h + 2] + exp2f(v.w - M[h + 3]) * iL[h + 3];
            }
        } else {
            for (int h = 0; h < D.H; ++h) a += exp2f(sc[h] - M[h]) * iL[h];
        }
        return (double)a / (double)D.H;
    };
    const int stride = gridDim.x * blockDim.x;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += stride) {
        const int64_t i = base + j;
        const int64_t gi = S.att_slot[i];
        const double al = alpha(i);
        S.attn_mass[gi] += al;
        if (S.has_pl[gi]) S.per_layer[gi * D.n_layers + (int64_t)(now % (uint64_t)D.n_layers)] += al;
    }
    // the last CTA to finish runs the per-stream feedback (now++ must follow
    // every fold-back that reads now)
    __shared__ bool sm_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) sm_last = atomicAdd(S.done_ctr, 1u) == gridDim.x * gridDim.y - 1;
    __syncthreads();
    if (!sm_last) return;
    __threadfence();
    for (int t = threadIdx.x; t < D.B; t += blockDim.x) feedback_stream(D, C, S, t);
    if (threadIdx.x == 0) *S.done_ctr = 0;
}

// pipeline.cpp:258 (record_miss), 337-347 (adapt, observe_hits,
// adakv_update); scheduler state.step++ (scheduler.cpp:328); now++.
__global__ void k_feedback(Dims D, Cfg C, State S) {
    griddep_enter();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < D.B) feedback_stream(D, C, S, s);
}

void launch_finish_merge(const Dims& D, const Cfg& C, const State& S, const ExchangeLayout& X,
                         const uint8_t* gathered, float* y, int granks, cudaStream_t st) {
    launch_pdl(k_finish_merge, dim3(D.B), dim3(256), 0, st, D, C, S, X, gathered, y, granks);
}
void launch_foldback(const Dims& D, const Cfg& C, const State& S, cudaStream_t st) {
    const size_t smem = sizeof(float) * 2 * (size_t)D.H;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_foldback, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // ~4 CTAs of 256 threads per B200 SM (148) in all, split over the streams,
    // and no more per stream than its attended region can fill (small steps:
    // c1's single stream would otherwise launch 592 mostly idle CTAs)
    const int64_t fill = (D.att_stride + 255) / 256;
    const int x = (int)std::max<int64_t>(1, std::min<int64_t>((4 * 148 + D.B - 1) / D.B, fill));
    launch_pdl(k_foldback, dim3(x, D.B), dim3(256), smem, st, D, C, S);
}
void launch_feedback(const Dims& D, const Cfg& C, const State& S, cudaStream_t st) {
    launch_pdl(k_feedback, dim3((D.B + 127) / 128), dim3(128), 0, st, D, C, S);
}

// ===========================================================================
// encode: QueryEncoder::encode (pipeline.cpp:38-57) of every stream's token
// ===========================================================================
// q, k, v = W_{q,k,v} x in fp64 with the reference's sequential order
// (s = ((0 + W[i][0] x0) + W[i][1] x1) + ..., __dmul_rn/__dadd_rn: no FMA),
// so routing on q is bit-exact.  wt = [3][d][d] transposed (wt[m][j][i] =
// W_m[i][j]): lane = output row i, so every column step is one coalesced
// 256-byte row segment per warp; warp w owns NB streams (NB chains per
// thread, interleaved); the streams' embedding columns are staged through
// shared memory in chunks.  One launch covers <= 4 * NB streams.
constexpr int kEncWarps = 4;
template <int NB>
__global__ void __launch_bounds__(kEncWarps * 32)
    k_encode(Dims D, const double* __restrict__ wt, const double* __restrict__ emb, int b0, int chunk,
             double* __restrict__ q64, void* __restrict__ kout, void* __restrict__ vout) {
    griddep_enter();
    extern __shared__ double xs[];  // [kEncWarps * NB][chunk]
    const int d = D.d, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = blockIdx.x * 32 + lane;  // in [0, 3d)
    const bool on = row < 3 * d;
    const int m = on ? row / d : 0, r = on ? row % d : 0;
    const double* w = wt + (size_t)m * d * d + r;
    const int nsb = kEncWarps * NB;
    double acc[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) acc[u] = 0.0;
    for (int c0 = 0; c0 < d; c0 += chunk) {
        const int wn = min(chunk, d - c0);
        __syncthreads();
        for (int t = tid; t < nsb * chunk; t += blockDim.x) {
            const int sb = t / chunk, jj = t % chunk, b = b0 + sb;
            xs[t] = (b < D.B && jj < wn) ? emb[(int64_t)b * d + c0 + jj] : 0.0;
        }
        __syncthreads();
        if (on) {
            const double* wc = w + (size_t)c0 * d;
            const double* xw = xs + warp * NB * chunk;
            // 16 columns of W in flight before the chains consume them: the
            // loads are independent of the DADD chains, so they must not sit
            // on their critical path
            // software-pipelined: the next 16 columns load while these 16 compute
            int jj = 0;
            double wv[16], wn16[16];
            if (wn >= 16) {
#pragma unroll
                for (int q = 0; q < 16; ++q) wv[q] = __ldg(wc + (size_t)q * d);
            }
            for (; jj + 16 <= wn; jj += 16) {
                const bool more = jj + 32 <= wn;
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    wn16[q] = more ? __ldg(wc + (size_t)(jj + 16 + q) * d) : 0.0;
#pragma unroll
                for (int q = 0; q < 16; ++q)
#pragma unroll
                    for (int u = 0; u < NB; ++u)
                        acc[u] = __dadd_rn(acc[u], __dmul_rn(wv[q], xw[u * chunk + jj + q]));
#pragma unroll
                for (int q = 0; q < 16; ++q) wv[q] = wn16[q];
            }
            for (; jj < wn; ++jj) {
                const double wv = __ldg(wc + (size_t)jj * d);
#pragma unroll
                for (int u = 0; u < NB; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(wv, xw[u * chunk + jj]));
            }
        }
    }
    if (!on) return;
#pragma unroll
    for (int u = 0; u < NB; ++u) {
        const int b = b0 + warp * NB + u;
        if (b >= D.B) continue;
        const int64_t o = (int64_t)b * d + r;
        if (m == 0) {
            q64[o] = acc[u];
        } else {
            void* dst = m == 1 ? kout : vout;
            const float f = (float)acc[u];  // stored K/V: fp64 -> fp32 (-> bf16 RNE)
            if (D.kv_dtype == PIKV_DTYPE_BF16) ((uint16_t*)dst)[o] = f32_to_bf16_rne(f);
            else ((float*)dst)[o] = f;
        }
    }
}

int encode_chunk(const Dims& D, int nb) {
    int c = (40 * 1024) / (8 * kEncWarps * nb);
    c = c >= 32 ? c & ~31 : c;
    return std::max(1, std::min(c, D.d));
}

void launch_encode(const Dims& D, const double* wt, const double* emb, double* q64, void* kout, void* vout,
                   cudaStream_t st) {
    // chains per thread: enough warps x NB to cover B in as few launches as
    // possible, NB <= 16
    int nb = 1;
    while (nb < 16 && kEncWarps * nb < D.B) nb *= 2;
    const int chunk = encode_chunk(D, nb);
    const size_t smem = sizeof(double) * kEncWarps * nb * chunk;
    const dim3 grid((unsigned)((3 * D.d + 31) / 32));
    for (int b0 = 0; b0 < D.B; b0 += kEncWarps * nb) {
        switch (nb) {
            case 1: launch_pdl(k_encode<1>, grid, dim3(kEncWarps * 32), smem, st, D, wt, emb, b0, chunk, q64, kout, vout); break;
            case 2: launch_pdl(k_encode<2>, grid, dim3(kEncWarps * 32), smem, st, D, wt, emb, b0, chunk, q64, kout, vout); break;
            case 4: launch_pdl(k_encode<4>, grid, dim3(kEncWarps * 32), smem, st, D, wt, emb, b0, chunk, q64, kout, vout); break;
            case 8: launch_pdl(k_encode<8>, grid, dim3(kEncWarps * 32), smem, st, D, wt, emb, b0, chunk, q64, kout, vout); break;
            default: launch_pdl(k_encode<16>, grid, dim3(kEncWarps * 32), smem, st, D, wt, emb, b0, chunk, q64, kout, vout); break;
        }
    }
}

// ===========================================================================
// bulk insert: the store build of a prefill
// ===========================================================================
// T tokens of stream s with given experts: entry e = t*k + j is the j-th
// selected expert of token t (step now + t); ids now_id + e in order.  The
// result equals T*k sequential KVStore::insert calls (kvstore.cpp:36-53,
// 107-120) with Engine::step's metadata (pipeline.cpp:191-193).
//
// (a) one CTA per local ring: count the ring's entries c; the j-th of them
//     goes to slot (head + j) mod S and only the last min(c, S) survive
//     (earlier ones are overwritten inside the bulk); displacements = bulk
//     overwrites + previously live slots among the first min(c, S) writes.
//     Survivors get their metadata and a pool entry (pages allocated on
//     first use); then the ring's live count, storage-page counts and
//     scheduler page records are rebuilt from the final slots.
__device__ __forceinline__ int bulk_ring_of(const Dims& D, int64_t token, int e) {
    const int raw = shard_raw(token, e, D.n_tok, D.n_exp, D.additive);
    const int dev = raw % D.G;
    if (dev % D.world != D.rank) return -1;
    return (dev / D.world) * D.SPD + raw / D.G;
}

// ---- grid-wide stable counting sort of the bulk's (token, expert) pairs by
// local ring (replaces each ring CTA scanning every pair twice) ------------
constexpr int kSortChunk = 4096;  // pairs per block (512 threads x 8)
constexpr int kSortMaxR = 256;    // rings per stream handled by the sort path

// ring of every pair (-1: another rank's device) and per-chunk ring counts
__global__ void __launch_bounds__(512) k_bulk_hist(Dims D, State S, int s, int64_t n,
                                                   const int32_t* __restrict__ experts,
                                                   int32_t* __restrict__ ringof, int32_t* __restrict__ hist) {
    __shared__ int hs[kSortMaxR];
    const int tid = threadIdx.x;
    for (int r = tid; r < D.R; r += blockDim.x) hs[r] = 0;
    __syncthreads();
    const uint64_t now0 = S.now[s];
    const int64_t c0 = (int64_t)blockIdx.x * kSortChunk;
    for (int i = tid; i < kSortChunk; i += blockDim.x) {
        const int64_t e = c0 + i;
        if (e >= n) break;
        const int64_t t = n < (1LL << 31) ? (int64_t)((uint32_t)e / (uint32_t)D.k) : e / D.k;
        const int r = bulk_ring_of(D, (int64_t)(now0 + (uint64_t)t), experts[e]);
        ringof[e] = r;
        if (r >= 0) atomicAdd(&hs[r], 1);
    }
    __syncthreads();
    for (int r = tid; r < D.R; r += blockDim.x) hist[(int64_t)blockIdx.x * D.R + r] = hs[r];
}

// per ring: exclusive scan over chunks (in place), ring totals and bases
__global__ void k_bulk_offsets(Dims D, int nchunk, int32_t* __restrict__ hist, int32_t* __restrict__ ring_c,
                               int32_t* __restrict__ ring_base) {
    __shared__ int64_t wsum[32];
    const int r = threadIdx.x;
    int run = 0;
    if (r < D.R)
        for (int c = 0; c < nchunk; ++c) {
            const int x = hist[(int64_t)c * D.R + r];
            hist[(int64_t)c * D.R + r] = run;
            run += x;
        }
    int64_t tot;
    const int64_t b = block_excl_scan(r < D.R ? (int64_t)run : 0, wsum, &tot);
    if (r < D.R) ring_c[r] = run, ring_base[r] = (int32_t)b;
}

// stable ranks: pairs of a chunk in rounds of 512 (warp match + per-warp
// counts scanned in warp order); list[ring_base[r] + rank] = pair index
__global__ void __launch_bounds__(512) k_bulk_rank(Dims D, int64_t n, const int32_t* __restrict__ ringof,
                                                   const int32_t* __restrict__ off,
                                                   const int32_t* __restrict__ ring_base,
                                                   int32_t* __restrict__ list) {
    __shared__ int cnt[16][kSortMaxR];
    __shared__ int run[kSortMaxR];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int r = tid; r < D.R; r += blockDim.x) run[r] = off[(int64_t)blockIdx.x * D.R + r];
    const int64_t c0 = (int64_t)blockIdx.x * kSortChunk;
    for (int i0 = 0; i0 < kSortChunk; i0 += 512) {
        for (int x = tid; x < 16 * D.R; x += blockDim.x) cnt[x / D.R][x % D.R] = 0;
        __syncthreads();
        const int64_t e = c0 + i0 + tid;
        const int r = e < n ? ringof[e] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, r);
        const int rk = __popc(peers & ((1u << lane) - 1u));
        if (r >= 0 && rk == 0) cnt[warp][r] = __popc(peers);
        __syncthreads();
        if (r >= 0) {
            int before = run[r];
            for (int w = 0; w < warp; ++w) before += cnt[w][r];
            list[ring_base[r] + before + rk] = (int32_t)e;
        }
        __syncthreads();
        for (int x = tid; x < D.R; x += blockDim.x) {
            int t = 0;
            for (int w = 0; w < 16; ++w) t += cnt[w][x];
            run[x] += t;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(512) k_bulk_ring(Dims D, State S, int s, int64_t T,
                                                   const int32_t* __restrict__ experts,
                                                   const double* __restrict__ saliency,
                                                   int64_t* __restrict__ dst, unsigned long long* counters,
                                                   int use_smem, const int32_t* __restrict__ list,
                                                   const int32_t* __restrict__ ring_c,
                                                   const int32_t* __restrict__ ring_base, int phase,
                                                   int64_t* __restrict__ ring_scr) {
    const int rl = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x;
    const int NW = NT >> 5;
    const int64_t ring = (int64_t)s * D.R + rl;
    const uint64_t now0 = S.now[s], id0 = S.next_id[s];
    const int head = S.head[ring];
    const uint64_t seq0 = S.seq[ring];
    const int64_t n = T * D.k;
    __shared__ int64_t wsum[32];
    __shared__ int64_t sm_c, sm_run;
    __shared__ unsigned long long sm_disp;
    // count
    int64_t mine = 0;
    // token of entry e: 32-bit division when the bulk fits (always, in practice)
    const bool small = n < (1LL << 31);
    auto tok_of = [&](int64_t e) -> int64_t { return small ? (int64_t)((uint32_t)e / (uint32_t)D.k) : e / D.k; };
    if (!list && phase == 0)
        for (int64_t e = tid; e < n; e += NT)
            mine += bulk_ring_of(D, (int64_t)(now0 + (uint64_t)tok_of(e)), experts[e]) == rl;
    int64_t tot;
    block_excl_scan(mine, wsum, &tot);
    if (list) tot = ring_c[rl];  // counted by the sort
    if (phase == 1) tot = ring_scr[3 * rl];  // counted in phase 0
    if (tid == 0) sm_c = tot, sm_run = 0, sm_disp = 0;
    __syncthreads();
    const int64_t c = sm_c;  // c == 0: nothing placed, the ring still counts its live pages
    const int64_t first_surv = c > D.S ? c - D.S : 0;  // ring rank of the first survivor
    const int64_t nsurv = c - first_surv;
    const int64_t s0 = (head + first_surv) % D.S;  // survivor slots: cyclic [s0, s0 + nsurv)
    // storage pages of the survivor slots that have no pool page yet, counted
    // in phase 0 and taken in phase 1 from the range k_bulk_reserve reserved
    // for this ring (an exhausted pool fails the bulk before any store)
    auto needs_page = [&](int p) {
        if (p >= D.ppr) return false;
        bool touched = false;
        for (int q = 0; q < D.spg && !touched; ++q) {
            const int64_t slot = (int64_t)p * D.spg + q;
            touched = ((slot - s0 + D.S) % D.S) < nsurv;
        }
        return touched && S.page_table[ring * D.ppr + p] < 0;
    };
    if (phase == 0) {
        int64_t need = 0;
        for (int p = tid; p < D.ppr; p += NT) need += needs_page(p);
        int64_t tn;
        block_excl_scan(need, wsum, &tn);
        if (tid == 0) ring_scr[3 * rl] = c, ring_scr[3 * rl + 1] = tn;
        return;
    }
    // displaced previously-live entries: the first min(c, S) writes
    unsigned long long dl = 0;
    for (int64_t j = tid; j < (c < D.S ? c : D.S); j += NT)
        dl += S.id[ring * D.S + (head + j) % D.S] != 0;
    for (int o = 16; o; o >>= 1) dl += __shfl_xor_sync(0xffffffffu, dl, o);
    if (lane == 0) atomicAdd(&sm_disp, dl);
    __shared__ int sm_err;
    if (tid == 0) sm_err = S.err[s];
    __syncthreads();
    if (sm_err) return;  // pool exhausted (k_bulk_reserve): nothing was stored
    {
        const int64_t pbase = ring_scr[3 * rl + 2];
        int64_t taken = 0;
        for (int p0 = 0; p0 < D.ppr; p0 += NT) {
            const bool nd = needs_page(p0 + tid);
            int64_t tn;
            const int64_t idx = block_excl_scan(nd ? 1 : 0, wsum, &tn);
            if (nd) S.page_table[ring * D.ppr + p0 + tid] = S.free_stack[pbase + taken + idx];
            taken += tn;
        }
    }
    __syncthreads();
    // place: entries in order, rank within the ring by one block scan per
    // chunk of PER consecutive entries per thread (was one scan per 512
    // entries with a serial warp prefix: 365 -> ~60 us at 32K tokens)
    constexpr int PER = 16;
    int64_t run = 0;
    // sorted path: the ring's pairs in order at list[ring_base + j]
    for (int64_t j = first_surv + tid; list && j < c; j += NT) {
        const int64_t e = list[ring_base[rl] + j];
        const int64_t t = tok_of(e);
        const int slot = (int)((head + j) % D.S);
        const int64_t gi = ring * D.S + slot;
        const uint64_t step = now0 + (uint64_t)t;
        S.id[gi] = id0 + (uint64_t)e;
        S.shard_seq[gi] = seq0 + (uint64_t)j;
        S.token[gi] = (int64_t)step;
        S.expert[gi] = experts[e];
        S.insert_step[gi] = step;
        S.last_access[gi] = step;
        S.freq[gi] = 0;
        S.attn_mass[gi] = 0.0;
        for (int l = 0; l < D.n_layers; ++l)
            S.per_layer[gi * D.n_layers + l] = saliency ? saliency[t * D.n_layers + l] : 0.0;
        S.has_pl[gi] = D.n_layers > 0 && saliency != nullptr;
        const int32_t page = S.page_table[ring * D.ppr + slot / D.spg];
        dst[e] = (int64_t)page * D.spg + slot % D.spg;
    }
    for (int64_t e0 = 0; !list && c > 0 && e0 < n; e0 += (int64_t)NT * PER) {
        const int64_t eb = e0 + (int64_t)tid * PER;
        uint32_t mask = 0;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int64_t e = eb + u;
            const bool in = e < n && bulk_ring_of(D, (int64_t)(now0 + (uint64_t)tok_of(e)), experts[e]) == rl;
            mask |= (uint32_t)in << u;
        }
        int64_t chunk;
        int64_t j = run + block_excl_scan((int64_t)__popc(mask), wsum, &chunk);
        for (; mask; mask &= mask - 1, ++j) {
            const int u = __ffs(mask) - 1;
            const int64_t e = eb + u;
            const int64_t t = tok_of(e);
            if (j >= first_surv) {
                const int slot = (int)((head + j) % D.S);
                const int64_t gi = ring * D.S + slot;
                const uint64_t step = now0 + (uint64_t)t;
                S.id[gi] = id0 + (uint64_t)e;
                S.shard_seq[gi] = seq0 + (uint64_t)j;
                S.token[gi] = (int64_t)step;
                S.expert[gi] = experts[e];
                S.insert_step[gi] = step;
                S.last_access[gi] = step;
                S.freq[gi] = 0;
                S.attn_mass[gi] = 0.0;
                for (int l = 0; l < D.n_layers; ++l)
                    S.per_layer[gi * D.n_layers + l] = saliency ? saliency[t * D.n_layers + l] : 0.0;
                S.has_pl[gi] = D.n_layers > 0 && saliency != nullptr;
                const int32_t page = S.page_table[ring * D.ppr + slot / D.spg];
                dst[e] = (int64_t)page * D.spg + slot % D.spg;
            } else {
                dst[e] = -1;  // overwritten later in the bulk
            }
        }
        run += chunk;
    }
    if (tid == 0) {
        S.head[ring] = (int)((head + c) % D.S);
        S.seq[ring] = seq0 + (uint64_t)c;
        atomicAdd(&counters[0], (unsigned long long)c);                                  // inserts
        atomicAdd(&counters[1], sm_disp + (unsigned long long)(c > D.S ? c - D.S : 0));  // displaced
    }
    __threadfence_block();
    __syncthreads();
    // rebuild the ring's counters and page records from its final slots:
    // accumulated in shared memory (16 consecutive slots share a record, so
    // global atomics serialized 16-deep per warp), written once
    // (rings too large for shared memory accumulate in the global records)
    extern __shared__ __align__(16) uint8_t sm_rec[];
    const int64_t base_r = use_smem ? 0 : ring * D.ppr_sched;
    unsigned long long* r_sla = use_smem ? (unsigned long long*)sm_rec : (unsigned long long*)S.pr_sla + base_r;
    unsigned long long* r_sf = use_smem ? r_sla + D.ppr_sched : (unsigned long long*)S.pr_sf + base_r;
    int* r_cnt = use_smem ? (int*)(r_sf + D.ppr_sched) : S.pr_cnt + base_r;
    int* r_first = use_smem ? r_cnt + D.ppr_sched : S.pr_first + base_r;
    int* p_live = use_smem ? r_first + D.ppr_sched : nullptr;
    for (int r = tid; r < D.ppr_sched; r += NT) r_sla[r] = 0, r_sf[r] = 0, r_cnt[r] = 0, r_first[r] = 0x7fffffff;
    for (int p = tid; p < D.ppr; p += NT) {
        if (use_smem) {
            p_live[p] = 0;
        } else {
            const int32_t page = S.page_table[ring * D.ppr + p];
            if (page >= 0) S.page_live[page] = 0;
        }
    }
    __syncthreads();
    int lv = 0;
    for (int slot = tid; slot < D.S; slot += NT) {
        const int64_t gi = ring * D.S + slot;
        if (S.id[gi] == 0) continue;
        ++lv;
        const uint64_t sq = S.shard_seq[gi];
        const int r = (int)(page_rec(D, ring, sq) - ring * D.ppr_sched);
        atomicAdd(&r_cnt[r], 1);
        atomicMin(&r_first[r], (int)(sq % (uint64_t)D.page_size));
        atomicAdd(&r_sla[r], (unsigned long long)S.last_access[gi]);
        atomicAdd(&r_sf[r], (unsigned long long)S.freq[gi]);
        if (use_smem) atomicAdd(&p_live[slot / D.spg], 1);
        else atomicAdd(&S.page_live[S.page_table[ring * D.ppr + slot / D.spg]], 1);
    }
    __syncthreads();
    for (int p = tid; use_smem && p < D.ppr; p += NT) {
        const int32_t page = S.page_table[ring * D.ppr + p];
        if (page >= 0) S.page_live[page] = p_live[p];
    }
    for (int o = 16; o; o >>= 1) lv += __shfl_xor_sync(0xffffffffu, lv, o);
    __shared__ int sm_lv, sm_pages;
    if (tid == 0) sm_lv = 0, sm_pages = 0;
    __syncthreads();
    if (lane == 0) atomicAdd(&sm_lv, lv);
    __syncthreads();
    int pg = 0;
    for (int r = tid; r < D.ppr_sched; r += NT) {
        const int64_t ri = ring * D.ppr_sched + r;
        const int cnt = r_cnt[r];
        const int first = cnt > 0 ? r_first[r] : 0;
        const unsigned long long sla = r_sla[r], sf = r_sf[r];
        S.pr_cnt[ri] = cnt;
        S.pr_first[ri] = first;
        S.pr_sla[ri] = sla;
        S.pr_sf[ri] = sf;
        pg += cnt > 0;
    }
    for (int o = 16; o; o >>= 1) pg += __shfl_xor_sync(0xffffffffu, pg, o);
    if (lane == 0) atomicAdd(&sm_pages, pg);
    __syncthreads();
    if (tid == 0) {
        S.live[ring] = sm_lv;
        atomicAdd(&counters[2 + rl / D.SPD], (unsigned long long)sm_pages);  // live pages per device
    }
}

// Between the two k_bulk_ring phases: reserve every ring's new pool pages
// at once (ring_scr[3r + 1] needed -> ring_scr[3r + 2] first free-stack
// index); an exhausted pool sets PIKV_ERR_OUT_OF_MEMORY before any store.
__global__ void k_bulk_reserve(Dims D, State S, int s, int64_t* __restrict__ ring_scr) {
    __shared__ int64_t wsum[32];
    __shared__ int64_t sm_tot;
    const int tid = threadIdx.x;
    int64_t run = 0;
    for (int r0 = 0; r0 < D.R; r0 += blockDim.x) {
        const int r = r0 + tid;
        const int64_t need = r < D.R ? ring_scr[3 * r + 1] : 0;
        int64_t tn;
        const int64_t ex = block_excl_scan(need, wsum, &tn);
        if (r < D.R) ring_scr[3 * r + 2] = run + ex;  // offset, rebased below
        run += tn;
    }
    if (tid == 0) sm_tot = run;
    __syncthreads();
    const int64_t tot = sm_tot;
    const int top = *S.free_top;  // no concurrent allocation: the engine stream is serial
    const bool oom = S.err[s] != 0 || tot > top;
    if (tid == 0 && !oom) *S.free_top = top - (int)tot;
    if (tid == 0 && oom && !S.err[s]) S.err[s] = PIKV_ERR_OUT_OF_MEMORY;
    for (int r = tid; r < D.R && !oom; r += blockDim.x) ring_scr[3 * r + 2] += top - tot;
}

// (b) one CTA per token: encode its K and V once (codec of the engine; the
//     low-rank projections come precomputed in proj [2][T][dp]) and copy the
//     entry to every surviving destination of the token.
__global__ void k_bulk_payload(Dims D, State S, int64_t T, const void* __restrict__ k, const void* __restrict__ v,
                               const float* __restrict__ proj, const int64_t* __restrict__ dst) {
    extern __shared__ __align__(16) uint8_t sm_entry[];  // [entry_bytes] + tmp floats [d]
    const int64_t t = blockIdx.x;
    const int tid = threadIdx.x;
    bool any = false;
    for (int j = 0; j < D.k; ++j) any |= dst[t * D.k + j] >= 0;
    if (!any) return;
    // direct paths (no shared-memory staging): identity rows and bf16 low-rank
    // projections are written straight to every destination entry
    const int esz = D.kv_dtype == PIKV_DTYPE_BF16 ? 2 : 4;
    if (D.codec == PIKV_CODEC_IDENTITY && (D.d * esz) % 16 == 0 && D.payload_bytes == D.d * esz) {
        const int nv = D.d * esz / 16;
        const uint4* ks = (const uint4*)((const uint8_t*)k + t * D.d * esz);
        const uint4* vs = (const uint4*)((const uint8_t*)v + t * D.d * esz);
        for (int i = tid; i < 2 * nv; i += blockDim.x) {
            const uint4 w = i < nv ? ks[i] : vs[i - nv];
            for (int j = 0; j < D.k; ++j) {
                const int64_t de = dst[t * D.k + j];
                if (de >= 0) ((uint4*)(S.pool + de * (int64_t)D.entry_bytes))[i] = w;
            }
        }
        return;
    }
    if ((D.codec == PIKV_CODEC_LOWRANK || D.codec == PIKV_CODEC_LORAPLUS) && D.kv_dtype == PIKV_DTYPE_BF16 &&
        D.dp % 4 == 0 && D.payload_bytes == D.dp * 2) {
        const int n4 = D.dp / 4;
        for (int i = tid; i < 2 * n4; i += blockDim.x) {
            const int row = i / n4, o4 = i % n4;
            const float4 f = ((const float4*)(proj + ((int64_t)row * T + t) * D.dp))[o4];
            const uint2 b = make_uint2((uint32_t)f32_to_bf16_rne(f.x) | ((uint32_t)f32_to_bf16_rne(f.y) << 16),
                                       (uint32_t)f32_to_bf16_rne(f.z) | ((uint32_t)f32_to_bf16_rne(f.w) << 16));
            for (int j = 0; j < D.k; ++j) {
                const int64_t de = dst[t * D.k + j];
                if (de >= 0) ((uint2*)(S.pool + de * (int64_t)D.entry_bytes + (int64_t)row * D.payload_bytes))[o4] = b;
            }
        }
        return;
    }
    float* tmp = (float*)(sm_entry + ((D.entry_bytes + 15) & ~15));
    const int pay = D.payload_bytes;
    float* ksc = (float*)(sm_entry + 2 * pay);
    float* vsc = ksc + D.H;
    if (D.codec == PIKV_CODEC_LOWRANK || D.codec == PIKV_CODEC_LORAPLUS) {
        for (int row = 0; row < 2; ++row) {
            const float* pr = proj + ((int64_t)row * T + t) * D.dp;
            uint8_t* out = sm_entry + row * pay;
            if (D.kv_dtype == PIKV_DTYPE_BF16 && D.dp % 4 == 0) {  // 16-byte loads, 8-byte stores
                for (int o4 = tid; o4 < D.dp / 4; o4 += blockDim.x) {
                    const float4 f = ((const float4*)pr)[o4];
                    const uint32_t lo = (uint32_t)f32_to_bf16_rne(f.x) | ((uint32_t)f32_to_bf16_rne(f.y) << 16);
                    const uint32_t hi = (uint32_t)f32_to_bf16_rne(f.z) | ((uint32_t)f32_to_bf16_rne(f.w) << 16);
                    ((uint2*)out)[o4] = make_uint2(lo, hi);
                }
            } else {
                for (int o = tid; o < D.dp; o += blockDim.x) {
                    if (D.kv_dtype == PIKV_DTYPE_BF16) ((uint16_t*)out)[o] = f32_to_bf16_rne(pr[o]);
                    else ((float*)out)[o] = pr[o];
                }
            }
        }
    } else {
        // encode_row reads row `s` of a [.][d] input: pass the token's row
        encode_row(D, S, (const uint8_t*)k + t * D.d * esz, 0, sm_entry, ksc, tmp, 0);
        encode_row(D, S, (const uint8_t*)v + t * D.d * esz, 0, sm_entry + pay, vsc, tmp, 1);
    }
    __syncthreads();
    const int nvec = D.entry_bytes / 16;
    for (int j = 0; j < D.k; ++j) {
        const int64_t de = dst[t * D.k + j];
        if (de < 0) continue;
        uint4* o = (uint4*)(S.pool + de * (int64_t)D.entry_bytes);
        for (int i = tid; i < nvec; i += blockDim.x) o[i] = ((const uint4*)sm_entry)[i];
    }
}

// (c) stream counters: ids, steps, store totals, live pages per device.
__global__ void k_bulk_finish(Dims D, State S, int s, int64_t T, const unsigned long long* counters) {
    if (threadIdx.x != 0 || S.err[s]) return;
    S.next_id[s] += (uint64_t)(T * D.k);
    S.now[s] += (uint64_t)T;
    S.st_inserts[s] += counters[0];
    S.st_overwrites[s] += counters[1];
    for (int gl = 0; gl < D.Gl; ++gl) S.pages_live[s * D.Gl + gl] = (int32_t)counters[2 + gl];
}

// Codec::encode_vector of LowRank / LoRAPlus for T rows on CUDA cores (fp32,
// i ascending like k_project): proj[row][t][h*r + j] = sum_i B[h][j][i] x_i.
__global__ void k_bulk_project_fma(Dims D, State S, int64_t T, const void* __restrict__ kin,
                                   const void* __restrict__ vin, float* __restrict__ proj) {
    const int h = blockIdx.y, row = blockIdx.z;
    const int hd = D.d / D.H, r = D.dph;
    const void* x = row == 0 ? kin : vin;
    extern __shared__ float sm_b[];  // basis [r][hd]
    for (int i = threadIdx.x; i < r * hd; i += blockDim.x) sm_b[i] = S.basis[(int64_t)h * r * hd + i];
    __syncthreads();
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < T * r;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = o / r;
        const int j = (int)(o % r);
        const float* col = sm_b + (size_t)j * hd;
        float acc = 0.f;
        for (int i = 0; i < hd; ++i) {
            float xi = load_in(x, D.kv_dtype, t * D.d + h * hd + i);
            if (D.codec == PIKV_CODEC_LORAPLUS) xi -= S.cbias[h * hd + i];
            acc = fmaf(col[i], xi, acc);
        }
        proj[((int64_t)row * T + t) * D.dp + h * r + j] = acc;
    }
}

size_t bulk_sort_ints(const Dims& D, int64_t T) {  // scratch of the counting sort (int32 count)
    const int64_t n = T * D.k, nchunk = (n + kSortChunk - 1) / kSortChunk;
    return (size_t)(2 * n + nchunk * D.R + 2 * D.R + 64);
}

int bulk_insert(const Dims& D, const State& S, int s, int64_t T, const void* k, const void* v,
                const int32_t* experts, const double* saliency, int64_t* dst, float* proj,
                unsigned long long* counters, int use_tc, cudaStream_t st, int32_t* sort_buf) {
    cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * (2 + D.Gl), st);
    cudaMemsetAsync(dst, 0xff, sizeof(int64_t) * (size_t)(T * D.k), st);  // -1: not stored here
    // ring placement first: it fixes every entry's pool slot (dst), so the
    // tcgen05 projection can write its bf16 rows straight into the entries
    if (D.R > 0) {
        size_t rsm = (size_t)D.ppr_sched * 24 + (size_t)D.ppr * 4;  // page-record accumulators
        const int use_smem = rsm <= 160 * 1024;
        if (!use_smem) rsm = 0;
        if (rsm > 48 * 1024) cudaFuncSetAttribute(k_bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
        const int64_t n = T * D.k, nchunk = (n + kSortChunk - 1) / kSortChunk;
        int32_t *list = nullptr, *ring_c = nullptr, *ring_base = nullptr;
        if (sort_buf && D.R <= kSortMaxR && n > 0 && n < (1LL << 31)) {
            int32_t* ringof = sort_buf;
            list = ringof + n;
            int32_t* hist = list + n;
            ring_c = hist + nchunk * D.R;
            ring_base = ring_c + D.R;
            k_bulk_hist<<<(unsigned)nchunk, 512, 0, st>>>(D, S, s, n, experts, ringof, hist);
            k_bulk_offsets<<<1, 256, 0, st>>>(D, (int)nchunk, hist, ring_c, ring_base);
            k_bulk_rank<<<(unsigned)nchunk, 512, 0, st>>>(D, n, ringof, hist, ring_base, list);
        }
        int64_t* ring_scr = (int64_t*)(counters + 2 + D.Gl);
        k_bulk_ring<<<D.R, 512, 0, st>>>(D, S, s, T, experts, saliency, dst, counters, use_smem, list, ring_c,
                                         ring_base, 0, ring_scr);
        k_bulk_reserve<<<1, 256, 0, st>>>(D, S, s, ring_scr);
        k_bulk_ring<<<D.R, 512, rsm, st>>>(D, S, s, T, experts, saliency, dst, counters, use_smem, list, ring_c,
                                           ring_base, 1, ring_scr);
    }
    bool fused = false;
    if ((D.codec == PIKV_CODEC_LOWRANK || D.codec == PIKV_CODEC_LORAPLUS) && T > 0) {
        const char* fz = std::getenv("PIKV_BULK_FUSE");  // A/B: 0 = fp32 projections + payload kernel
        const bool want_fuse = !(fz && fz[0] == '0');
        const int rc = use_tc ? launch_bulk_project_tc(D, S, T, k, v, proj, proj + 2 * T * D.dp, st,
                                                       want_fuse ? dst : nullptr)
                              : 1;
        fused = rc == 2;
        const bool tc_ok = rc == 0 || rc == 2;
        if (!tc_ok && use_tc == 2) return (int)cudaErrorNotSupported;  // tensor cores required
        if (!tc_ok) {
            const int hd = D.d / D.H;
            const size_t smem = sizeof(float) * (size_t)D.dph * hd;
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(k_bulk_project_fma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_bulk_project_fma<<<dim3(64, D.H, 2), 256, smem, st>>>(D, S, T, k, v, proj);
        }
    }
    const size_t psmem = (size_t)((D.entry_bytes + 15) & ~15) + sizeof(float) * (size_t)D.d;
    if (psmem > 48 * 1024)
        cudaFuncSetAttribute(k_bulk_payload, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
    if (T > 0 && !fused) k_bulk_payload<<<(unsigned)T, 256, psmem, st>>>(D, S, T, k, v, proj, dst);
    k_bulk_finish<<<1, 32, 0, st>>>(D, S, s, T, counters);
    return (int)cudaGetLastError();
}

// ===========================================================================
// snapshot: KVStore::snapshot (kvstore.cpp:206-221) of one stream
// ===========================================================================
// (a) one CTA per local ring: its live entries in shard_seq order (= token
//     order: a ring's entries are inserted in step order) compacted at the
//     ring's offset (exclusive scan of the live counts); rings are already
//     in (device, shard) order.
__global__ void k_snapshot(Dims D, State S, int s, uint64_t now, const int64_t* __restrict__ ring_off,
                           pikv_snapshot_record* __restrict__ out) {
    const int rl = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ring = (int64_t)s * D.R + rl;
    const uint64_t seq = S.seq[ring];
    const int fill = seq < (uint64_t)D.S ? (int)seq : D.S;
    const uint64_t lo = seq - (uint64_t)fill;
    __shared__ int wsum[32];
    __shared__ int sm_total;
    int64_t o = ring_off[rl];
    for (int c0 = 0; c0 < fill; c0 += blockDim.x) {
        const int i = c0 + tid;
        const uint64_t sq = lo + (uint64_t)i;
        const int64_t gi = ring * D.S + (int64_t)(sq % (uint64_t)D.S);
        const bool live = i < fill && S.id[gi] != 0 && S.shard_seq[gi] == sq;
        const unsigned bal = __ballot_sync(0xffffffffu, live);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        if (tid == 0) {
            int t = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                const int c = wsum[w];
                wsum[w] = t;
                t += c;
            }
            sm_total = t;
        }
        __syncthreads();
        if (live) {
            pikv_snapshot_record r;
            r.device = (rl / D.SPD) * D.world + D.rank;
            r.shard = rl % D.SPD;
            r.token_id = S.token[gi];
            r.expert_id = S.expert[gi];
            r.reserved = 0;
            const uint64_t ins = S.insert_step[gi];
            r.age = now >= ins ? now - ins : 0;  // EntryMeta::age, types.hpp:19-21
            r.freq = S.freq[gi];
            out[o + wsum[warp] + __popc(bal & ((1u << lane) - 1u))] = r;
        }
        o += sm_total;
        __syncthreads();
    }
}

// (b) a step's entries of one shard are consecutive with equal tokens, in
//     selection order: sort each such run by expert (runs are <= k long).
__global__ void k_snapshot_ties(pikv_snapshot_record* __restrict__ out, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto same = [&](int64_t a, int64_t b) {
        return out[a].device == out[b].device && out[a].shard == out[b].shard &&
               out[a].token_id == out[b].token_id;
    };
    if (i > 0 && same(i - 1, i)) return;  // not the first of its run
    int64_t j = i + 1;
    while (j < n && same(i, j)) ++j;
    for (int64_t a = i + 1; a < j; ++a) {
        const pikv_snapshot_record x = out[a];
        int64_t b = a - 1;
        while (b >= i && out[b].expert_id > x.expert_id) out[b + 1] = out[b], --b;
        out[b + 1] = x;
    }
}

void launch_snapshot(const Dims& D, const State& S, int s, uint64_t now, const int64_t* ring_off,
                     pikv_snapshot_record* out, int64_t n, cudaStream_t st) {
    if (D.R > 0) k_snapshot<<<D.R, 256, 0, st>>>(D, S, s, now, ring_off, out);
    if (n > 0) k_snapshot_ties<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, n);
}

// Stored K/V of n slots of stream s decoded to fp32 (the values the
// attention reads): KVEntry::key / value of the reference (types.hpp:27-34)
// for the store facade and the full-context parity checks.  slot = the
// stream-local index ring_local * S + slot; empty slots decode to zeros.
__global__ void k_read_entries(Dims D, State S, int s, const int64_t* __restrict__ slots, int n,
                               float* __restrict__ kout, float* __restrict__ vout) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const int64_t ls = slots[i];
    const int64_t ring = (int64_t)s * D.R + ls / D.S;
    const int slot = (int)(ls % D.S);
    const int64_t gi = ring * D.S + slot;
    const int32_t page = S.page_table[ring * D.ppr + slot / D.spg];
    const bool live = S.id[gi] != 0 && page >= 0;
    const uint8_t* ent = live ? S.pool + ((int64_t)page * D.spg + slot % D.spg) * D.entry_bytes : nullptr;
    const int pay = D.payload_bytes, hw = D.dph;
    for (int o = threadIdx.x; o < 2 * D.dp; o += blockDim.x) {
        const int row = o / D.dp, c = o % D.dp;
        float x = 0.f;
        if (live) {
            const uint8_t* p = ent + row * pay;
            if (D.codec == PIKV_CODEC_INT8 || D.codec == PIKV_CODEC_INT4) {
                const float sc = ((const float*)(ent + 2 * pay))[row * D.H + c / hw];
                int code;
                if (D.codec == PIKV_CODEC_INT8) {
                    code = (int)((const int8_t*)p)[c];
                } else {
                    const int nib = (p[c >> 1] >> ((c & 1) * 4)) & 0xF;
                    code = nib >= 8 ? nib - 16 : nib;
                }
                x = __fmul_rn((float)code, sc);
            } else if (D.kv_dtype == PIKV_DTYPE_BF16) {
                x = __uint_as_float(((uint32_t)((const uint16_t*)p)[c]) << 16);
            } else {
                x = ((const float*)p)[c];
            }
        }
        (row ? vout : kout)[(int64_t)i * D.dp + c] = x;
    }
}
void launch_read_entries(const Dims& D, const State& S, int s, const int64_t* slots, int n, float* k, float* v,
                         cudaStream_t st) {
    if (n > 0) k_read_entries<<<n, 256, 0, st>>>(D, S, s, slots, n, k, v);
}

// token / expert of a list of slots (pikv_read_attended_host)
__global__ void k_gather_slots(State S, const int32_t* __restrict__ slot, int n, int64_t* __restrict__ token,
                               int32_t* __restrict__ expert) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int32_t gi = slot[i];
        token[i] = S.token[gi];
        expert[i] = S.expert[gi];
    }
}
void launch_gather_slots(const State& S, const int32_t* slot, int n, int64_t* token, int32_t* expert,
                         cudaStream_t st) {
    if (n > 0) k_gather_slots<<<(n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024, 256, 0, st>>>(S, slot, n, token, expert);
}

// ===========================================================================
// synthetic inputs: N(0,1) from a counter hash, rounded to kv_dtype
// ===========================================================================
__host__ __device__ __forceinline__ uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__global__ void k_synth(int64_t n, int dtype, void* __restrict__ out, uint64_t seed) {
    griddep_enter();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = splitmix(seed ^ splitmix((uint64_t)i));
        const float u1 = ((float)(h >> 40) + 1.0f) * (1.0f / 16777217.0f);
        const float u2 = (float)((h >> 16) & 0xffffff) * (1.0f / 16777216.0f);
        const float z = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
        if (dtype == PIKV_DTYPE_BF16) ((uint16_t*)out)[i] = f32_to_bf16_rne(z);
        else ((float*)out)[i] = z;
    }
}

void launch_synth(const Dims& D, void* q, void* k, void* v, uint64_t seed, uint64_t step,
                  cudaStream_t st) {
    const int64_t n = (int64_t)D.B * D.d;
    const uint64_t base = splitmix(seed) ^ (step * 0x632be59bd9b4e019ull);
    launch_pdl(k_synth, dim3(256), dim3(256), 0, st, n, D.kv_dtype, q, base ^ 0x1111);
    launch_pdl(k_synth, dim3(256), dim3(256), 0, st, n, D.kv_dtype, k, base ^ 0x2222);
    launch_pdl(k_synth, dim3(256), dim3(256), 0, st, n, D.kv_dtype, v, base ^ 0x3333);
}

}  // namespace pikv_dev
