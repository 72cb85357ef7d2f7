// SPDX-License-Identifier: Apache-2.0
//
// Sharded decode attention, the HBM-bound hot kernel of the PiKV step.
//
// Reproduces attention() (pipeline.cpp:59-85) per head over the retrieved
// entries (kvstore.cpp:122-178) and returns per-work-item partial softmax
// state (m, l, o) for the log-sum-exp merge, plus every
// entry's per-head logit for the alpha fold-back (pipeline.cpp:302-312).
//
// Design (B200):
//  * persistent grid: two 288-thread CTAs per SM; work items = (stream, run of
//    consecutive retrieved entries): each CTA's equal static share of all the
//    streams' entries (build_items_shares; 2..16 streams per engine), else
//    items taken from a global ticket;
//  * warp 8 is the producer: lanes issue one cp.async.bulk (TMA bulk copy,
//    SASS UBLKCP) per KV entry -- K, V (and scales) are contiguous in the
//    paged pool, 16 KiB at 32x128 bf16 -- into an NST-stage shared-memory
//    ring; full/empty mbarriers (complete_tx) hand stages to the consumers;
//  * warps 0-7 consume: each thread owns VPT 16-byte chunks of K/V (one head
//    slice), dots them with its registers of q, reduces across the CPH lanes
//    of the head with shuffles and runs the online softmax in base 2
//    (exp2f), two entries per step for ILP;
//  * the q.K products are 1 flop/byte GEMVs (one query per KV set), far below
//    the tensor-core ridge, so CUDA cores are the right unit.
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <type_traits>

#include "pikv_dev.cuh"

#ifndef PIKV_ATTEND_NOHINT
#define PIKV_ATTEND_NOHINT 0  // experiment builds only: TMA without the L2 evict-first hint
#endif
#ifndef PIKV_ATTEND_I8DOT
#define PIKV_ATTEND_I8DOT 1  // int8 q.k as IDP4A digit planes (0: decode + FFMA2, A/B builds)
#endif
#ifndef PIKV_ATTEND_NOMATH
#define PIKV_ATTEND_NOMATH 0  // experiment builds only: consumers skip the math
#endif

namespace pikv_dev {

namespace {

constexpr int kConsumers = 256;
constexpr int kThreads = kConsumers + 32;
constexpr int kSmemBudget = 110 * 1024;   // two CTAs per SM
constexpr int kSmemBudget3 = 74 * 1024;   // three CTAs per SM (bf16 heads, PIKV_ATT_CPS=3)

__device__ __forceinline__ void consumer_bar() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// ---- packed fp32x2 math (Blackwell FFMA2 / FMUL2) ------------------------
struct f2 {
    float x, y;
};
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
          "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return *reinterpret_cast<f2*>(&d);
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(d)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return *reinterpret_cast<f2*>(&d);
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(d)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return *reinterpret_cast<f2*>(&d);
}

// ---- 16-byte chunk decoders: N values as N/2 pairs -------------------------
struct DecBF16 {
    static constexpr int N = 8;
    __device__ static void dec(const uint4& w, f2* x) {
        x[0] = {bf16_lo(w.x), bf16_hi(w.x)};
        x[1] = {bf16_lo(w.y), bf16_hi(w.y)};
        x[2] = {bf16_lo(w.z), bf16_hi(w.z)};
        x[3] = {bf16_lo(w.w), bf16_hi(w.w)};
    }
};
struct DecF32 {
    static constexpr int N = 4;
    __device__ static void dec(const uint4& w, f2* x) {
        x[0] = {__uint_as_float(w.x), __uint_as_float(w.y)};
        x[1] = {__uint_as_float(w.z), __uint_as_float(w.w)};
    }
};
// int8 / int4 codes -> exact fp32 without I2F: bias the two's-complement
// codes to unsigned (xor), place each byte under the exponent of 2^23
// (PRMT -> 0x4B0000vv == 2^23 + v exactly) and subtract 2^23 + bias with one
// packed FADD2.  ~1.5 (int8) / ~2 (int4) full-rate ops per value.
__device__ __forceinline__ float magic_byte(uint32_t u, uint32_t sel) {
    return __uint_as_float(__byte_perm(u, 0x4B000000u, sel));
}
struct DecI8 {
    static constexpr int N = 16;
    __device__ static void dec(const uint4& w, f2* x) {
        const uint32_t v[4] = {w.x ^ 0x80808080u, w.y ^ 0x80808080u, w.z ^ 0x80808080u, w.w ^ 0x80808080u};
        const f2 bias = {-8388736.0f, -8388736.0f};  // -(2^23 + 128)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            x[2 * i] = add2({magic_byte(v[i], 0x7540), magic_byte(v[i], 0x7541)}, bias);
            x[2 * i + 1] = add2({magic_byte(v[i], 0x7542), magic_byte(v[i], 0x7543)}, bias);
        }
    }
};
struct DecI4 {
    static constexpr int N = 32;
    __device__ static void dec(const uint4& w, f2* x) {
        const uint32_t v[4] = {w.x ^ 0x88888888u, w.y ^ 0x88888888u, w.z ^ 0x88888888u, w.w ^ 0x88888888u};
        const f2 bias = {-8388616.0f, -8388616.0f};  // -(2^23 + 8)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t lo = v[i] & 0x0F0F0F0Fu;         // even nibbles as bytes
            const uint32_t hi = (v[i] >> 4) & 0x0F0F0F0Fu;  // odd nibbles
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t sel = 0x7540u | (uint32_t)j;
                x[4 * i + j] = add2({magic_byte(lo, sel), magic_byte(hi, sel)}, bias);
            }
        }
    }
};

template <class Dec> struct IsQuant { static constexpr bool v = false; };
template <> struct IsQuant<DecI8> { static constexpr bool v = true; };
template <> struct IsQuant<DecI4> { static constexpr bool v = true; };

struct AttParams {
    int CPH;          // 16-byte chunks per head (K payload)
    int LPH;          // lanes per head = CPH / CPT
    int TPE;          // threads per entry = H * LPH
    int EP;           // entries processed in parallel by sub-groups (256 / TPE)
    int EPS;          // entries per stage
    int NST;          // stages
    int stage_bytes;
    float scale2;     // log2(e) / sqrt(dph)
    int dyn;          // work items from the global ticket (1) or strided by CTA (0)
    int merge;        // one bulk copy per run of pool-adjacent entries (PIKV_ATT_MERGE)
};

// Thread (sub, head, j) owns chunks j + i*LPH (i < CPT) of one head: the
// q.k partial is reduced over the head's LPH lanes (xor shuffles), so every
// lane of the group holds the head's score and its own slice of o.
__device__ __forceinline__ float ex2(float x) {  // 2^x, x <= 0 (flushes to 0 below 2^-126)
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// LPHC: lanes per head as a compile-time constant (0 = P.LPH at run time)
template <class Dec, int CPT, int NB, int LPHC, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_attend(Dims D, State S, AttParams P) {
    const long long t_entry = D.dbg_att && threadIdx.x == 0 ? (long long)globaltimer() : 0;  // PIKV_DEBUG_ATT
    griddep_enter();
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int N = Dec::N, NP = N / 2;
    uint64_t* full = (uint64_t*)smem;  // [0, 8): stage ring (NST <= 8)
    uint64_t* empty = full + 16;
    // work-item queue, producer -> consumers: item index in iq, handed over
    // with ifull / iempty (the producer fetches the next item while the
    // consumers still work on the current one)
    uint64_t* ifull = full + 8;
    uint64_t* iempty = empty + 8;
    int* iq = (int*)(full + 12);
    constexpr int NQ = 4;
    uint8_t* stages = smem + 256;
    float* red = (float*)(stages + (size_t)P.NST * P.stage_bytes);  // EP merge scratch
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < P.NST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kConsumers / 32);
        }
        for (int i = 0; i < NQ; ++i) {
            mbar_init(&ifull[i], 1);
            mbar_init(&iempty[i], kConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int n_items = S.n_items[0];
    const int H = D.H, dph = D.dph;
    const int eb = D.entry_bytes, pay = D.payload_bytes;

    if (warp == kConsumers / 32) {
        // ================= producer warp =================
        const uint64_t pol = evict_first_policy();
        int stage = 0;
        uint32_t phase = 0;
        // The pool indices of the item's entries are read a 32-entry window
        // ahead (one coalesced load per window, lane i holds entry win + i),
        // so refilling a stage never waits on a global load.
        // next item's (position, count) and first index window are loaded
        // during the current item: no metadata round trips between items
        auto item_of = [&](int w, int64_t& pos, int& cnt) {
            if (w < n_items) {
                pos = (int64_t)S.item_stream[w] * D.att_stride + S.item_begin[w];
                cnt = S.item_end[w] - S.item_begin[w];
            } else {
                pos = 0, cnt = 0;
            }
        };
        // Items are taken from a global ticket (n_items[1], reset by the
        // kernel that builds them) so CTAs that start late -- their SM still
        // busy with the previous micro-batch's tail kernels -- simply run
        // fewer items; P.dyn = 0 strides them statically (blockIdx + i*grid).
        auto next_item = [&](int prev) -> int {
            if (D.att_share) {  // equal static shares: this CTA's items, then the sentinel
                const int w = prev < 0 ? S.cta_first[blockIdx.x] : prev + 1;
                return w < S.cta_first[blockIdx.x + 1] ? w : n_items;
            }
            if (!P.dyn) return prev < 0 ? (int)blockIdx.x : prev + (int)gridDim.x;
            int w = 0;
            if (lane == 0) w = atomicAdd(&S.n_items[1], 1);
            return __shfl_sync(0xffffffffu, w, 0);
        };
        int kq = 0;
        auto publish = [&](int w) {
            if (lane == 0) {
                mbar_wait_sleep(&iempty[kq % NQ], ((kq / NQ) & 1) ^ 1);
                *(volatile int*)&iq[kq % NQ] = w;
                mbar_arrive(&ifull[kq % NQ]);
            }
            ++kq;
        };
        int64_t npos;
        int ncnt;
        int w = next_item(-1);
        item_of(w, npos, ncnt);
        int32_t nwin = lane < ncnt ? S.att_entry[npos + lane] : 0;
        for (;;) {
            publish(w);
            if (w >= n_items) break;
            const int64_t pos0 = npos;
            const int cnt = ncnt;
            auto win_load = [&](int w0) { return w0 + lane < cnt ? S.att_entry[pos0 + w0 + lane] : 0; };
            int win = 0;
            int32_t cur = nwin, nxt = win_load(32);
            const int wn = next_item(w);
            item_of(wn, npos, ncnt);
            nwin = lane < ncnt ? S.att_entry[npos + lane] : 0;
            for (int b = 0; b < cnt; b += P.EPS) {
                const int n = min(P.EPS, cnt - b);
                while (b >= win + 32) win += 32, cur = nxt, nxt = win_load(win + 32);
                // entry b + lane: from the current window, or the next one when
                // the stage straddles the boundary (EPS <= 32)
                const int o = b - win + lane;
                const int32_t e_cur = __shfl_sync(0xffffffffu, cur, o & 31);
                const int32_t e_nxt = __shfl_sync(0xffffffffu, nxt, o & 31);
                const int64_t ent = o < 32 ? e_cur : e_nxt;
                if (lane == 0) {
                    mbar_wait_sleep(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], (uint32_t)(n * eb));
                }
                __syncwarp();
                // P.merge: entries adjacent in the pool (a page's run) go as one
                // bulk copy from the run's first lane (the stage's slots are
                // contiguous too)
                int len = 1;
                bool issue = lane < n;
                if (P.merge) {
                    const int64_t prev = __shfl_up_sync(0xffffffffu, ent, 1);
                    const bool start = lane < n && (lane == 0 || ent != prev + 1);
                    const uint32_t starts = __ballot_sync(0xffffffffu, start);
                    const uint32_t later = starts & ~((2u << lane) - 1u);
                    const int end = later ? __ffs(later) - 1 : n;
                    len = (end < n ? end : n) - lane;
                    issue = start;
                }
                if (issue) {
                    if (PIKV_ATTEND_NOHINT)
                        bulk_g2s_plain(stages + (size_t)stage * P.stage_bytes + (size_t)lane * eb,
                                       S.pool + ent * (int64_t)eb, (uint32_t)(len * eb), &full[stage]);
                    else
                        bulk_g2s(stages + (size_t)stage * P.stage_bytes + (size_t)lane * eb,
                                 S.pool + ent * (int64_t)eb, (uint32_t)(len * eb), &full[stage], pol);
                }
                if (++stage == P.NST) stage = 0, phase ^= 1;
            }
            w = wn;
        }
        return;
    }

    // ================= consumer warps =================
    const int sub = tid / P.TPE;
    const int r = tid % P.TPE;
    const int LPH = LPHC ? LPHC : P.LPH;
    constexpr bool QUANT = IsQuant<Dec>::v;
    constexpr bool I8DOT = QUANT && Dec::N == 16 && PIKV_ATTEND_I8DOT;  // int8: integer q.k
    constexpr bool I4DOT = QUANT && Dec::N == 32 && PIKV_ATTEND_I8DOT;  // int4: integer q.k
    const int head = r / LPH, j = r % LPH;
    const bool active_sub = sub < P.EP;
    int coff[CPT];  // byte offset of chunk i inside the K (or V) payload
#pragma unroll
    for (int i = 0; i < CPT; ++i) coff[i] = (head * P.CPH + j + i * LPH) * 16;
    int stage = 0;
    uint32_t phase = 0;
    long long t_start = 0, n_ent = 0, t_first = 0, t_wait = 0;  // PIKV_DEBUG_ATT
    if (D.dbg_att && tid == 0) t_start = (long long)globaltimer();
    for (int kq = 0;; ++kq) {
        mbar_wait_sleep(&ifull[kq % NQ], (kq / NQ) & 1);
        const int w = *(volatile int*)&iq[kq % NQ];
        __syncwarp();
        if (lane == 0) mbar_arrive(&iempty[kq % NQ]);
        if (w >= n_items) {
            if (D.dbg_att && tid == 0) {
                long long* d = S.dbg + 64 + 8 * D.B + 8 * blockIdx.x;
                d[0] = t_start, d[1] = (long long)globaltimer(), d[2] = kq, d[3] = n_ent, d[4] = smid();
                d[5] = t_entry, d[6] = t_first, d[7] = t_wait;
            }
            break;
        }
        const int s = S.item_stream[w];
        const int64_t pos0 = (int64_t)s * D.att_stride + S.item_begin[w];
        const int cnt = S.item_end[w] - S.item_begin[w];
        n_ent += cnt;
        f2 q[CPT][NP], o[CPT][NP];
        float m = -INFINITY, l = 0.f;
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
            const float* qs = S.q_attn + (int64_t)s * D.dp + head * dph + (j + i * LPH) * N;
#pragma unroll
            for (int t = 0; t < NP; ++t) {
                q[i][t] = {qs[2 * t], qs[2 * t + 1]};
                o[i][t] = {0.f, 0.f};
            }
        }
        // int8 K: q as three signed base-256 digit planes of a 23-bit fixed-point
        // q (scale 2^(22 - e), e = exponent of the head's max |q|), so q.k is
        // three exact integer dot products (IDP4A on the raw codes, no decode):
        // q.k = (S0 + 256 S1 + 65536 S2) * 2^(e - 22) up to the rounding of q to
        // 23 bits relative to the head's max (~1e-7 relative on the logit)
        int qd[I8DOT ? CPT : 1][4][3];
        float qinv = 1.f;
        // int4 K: the same digit planes, split into even / odd elements (the
        // two nibbles of a code byte); codes are biased to 0..15 (xor 8) so a
        // byte is a non-negative int8, and 8 * sum(digits) is subtracted
        int qe[I4DOT ? CPT : 1][4][2][3];
        int corr[3] = {0, 0, 0};
        if constexpr (I4DOT) {
            float mx = 0.f;
#pragma unroll
            for (int i = 0; i < CPT; ++i)
#pragma unroll
                for (int t = 0; t < NP; ++t) mx = fmaxf(mx, fmaxf(fabsf(q[i][t].x), fabsf(q[i][t].y)));
#pragma unroll
            for (int off = 16; off; off >>= 1)
                if (off < LPH) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            int ex = 0;
            if (mx > 0.f) frexpf(mx, &ex);
            const float qs_ = ldexpf(1.f, 22 - ex);
            qinv = ldexpf(1.f, ex - 22);
#pragma unroll
            for (int i = 0; i < CPT; ++i)
#pragma unroll
                for (int wd = 0; wd < 4; ++wd)
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {
                        uint32_t pk[3] = {0u, 0u, 0u};
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const f2 qq = q[i][4 * wd + b];
                            const int v = __float2int_rn((h2 ? qq.y : qq.x) * qs_);
                            const int d0 = ((v + 128) & 255) - 128;
                            const int r1 = (v - d0) >> 8;
                            const int d1 = ((r1 + 128) & 255) - 128;
                            const int d2 = (r1 - d1) >> 8;
                            corr[0] += d0, corr[1] += d1, corr[2] += d2;
                            pk[0] |= (uint32_t)(d0 & 255) << (8 * b);
                            pk[1] |= (uint32_t)(d1 & 255) << (8 * b);
                            pk[2] |= (uint32_t)(d2 & 255) << (8 * b);
                        }
                        qe[i][wd][h2][0] = (int)pk[0], qe[i][wd][h2][1] = (int)pk[1], qe[i][wd][h2][2] = (int)pk[2];
                    }
            corr[0] *= -8, corr[1] *= -8, corr[2] *= -8;
        }
        if constexpr (I8DOT) {
            float mx = 0.f;
#pragma unroll
            for (int i = 0; i < CPT; ++i)
#pragma unroll
                for (int t = 0; t < NP; ++t) mx = fmaxf(mx, fmaxf(fabsf(q[i][t].x), fabsf(q[i][t].y)));
#pragma unroll
            for (int off = 16; off; off >>= 1)
                if (off < LPH) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            int ex = 0;
            if (mx > 0.f) frexpf(mx, &ex);
            const float qs_ = ldexpf(1.f, 22 - ex);
            qinv = ldexpf(1.f, ex - 22);
#pragma unroll
            for (int i = 0; i < CPT; ++i)
#pragma unroll
                for (int wd = 0; wd < 4; ++wd) {
                    uint32_t pk[3] = {0u, 0u, 0u};
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const f2 qq = q[i][2 * wd + (b >> 1)];
                        const int v = __float2int_rn((b & 1 ? qq.y : qq.x) * qs_);
                        const int d0 = ((v + 128) & 255) - 128;
                        const int r1 = (v - d0) >> 8;
                        const int d1 = ((r1 + 128) & 255) - 128;
                        const int d2 = (r1 - d1) >> 8;
                        pk[0] |= (uint32_t)(d0 & 255) << (8 * b);
                        pk[1] |= (uint32_t)(d1 & 255) << (8 * b);
                        pk[2] |= (uint32_t)(d2 & 255) << (8 * b);
                    }
                    qd[i][wd][0] = (int)pk[0], qd[i][wd][1] = (int)pk[1], qd[i][wd][2] = (int)pk[2];
                }
        }
        for (int b = 0; b < cnt; b += P.EPS) {
            const int n = min(P.EPS, cnt - b);
            if (D.dbg_att && tid == 0) {
                const long long t0 = (long long)globaltimer();
                mbar_wait_sleep(&full[stage], phase);
                const long long t1 = (long long)globaltimer();
                if (t_first == 0) t_first = t1;
                else t_wait += t1 - t0;
            } else {
                mbar_wait_sleep(&full[stage], phase);
            }
            const uint8_t* sb = stages + (size_t)stage * P.stage_bytes;
            float* scp = S.scores + (pos0 + b) * H + head;  // this stage's logits, entry e at scp[e * H]
            // warp-uniform trip count (sub-groups of a warp see different entries)
            for (int e0 = 0; e0 < (PIKV_ATTEND_NOMATH ? 0 : n); e0 += P.EP * NB) {
                float sc[NB];
#pragma unroll
                for (int bb = 0; bb < NB; ++bb) {
                    const int e = e0 + sub + bb * P.EP;
                    const uint8_t* ent = sb + (size_t)((active_sub && e < n) ? e : 0) * eb;
                    if constexpr (I8DOT) {
                        int d0 = 0, d1 = 0, d2 = 0;
#pragma unroll
                        for (int i = 0; i < CPT; ++i) {
                            const uint4 kw = *(const uint4*)(ent + coff[i]);
                            const int kk[4] = {(int)kw.x, (int)kw.y, (int)kw.z, (int)kw.w};
#pragma unroll
                            for (int wd = 0; wd < 4; ++wd) {
                                d0 = __dp4a(kk[wd], qd[i][wd][0], d0);
                                d1 = __dp4a(kk[wd], qd[i][wd][1], d1);
                                d2 = __dp4a(kk[wd], qd[i][wd][2], d2);
                            }
                        }
                        sc[bb] = fmaf((float)d2, 65536.f, fmaf((float)d1, 256.f, (float)d0)) * qinv;
                    } else if constexpr (I4DOT) {
                        int d0 = corr[0], d1 = corr[1], d2 = corr[2];
#pragma unroll
                        for (int i = 0; i < CPT; ++i) {
                            const uint4 kw = *(const uint4*)(ent + coff[i]);
                            const uint32_t kk[4] = {kw.x ^ 0x88888888u, kw.y ^ 0x88888888u, kw.z ^ 0x88888888u,
                                                    kw.w ^ 0x88888888u};
#pragma unroll
                            for (int wd = 0; wd < 4; ++wd) {
                                const int lo = (int)(kk[wd] & 0x0F0F0F0Fu), hi = (int)((kk[wd] >> 4) & 0x0F0F0F0Fu);
                                d0 = __dp4a(lo, qe[i][wd][0][0], d0);
                                d1 = __dp4a(lo, qe[i][wd][0][1], d1);
                                d2 = __dp4a(lo, qe[i][wd][0][2], d2);
                                d0 = __dp4a(hi, qe[i][wd][1][0], d0);
                                d1 = __dp4a(hi, qe[i][wd][1][1], d1);
                                d2 = __dp4a(hi, qe[i][wd][1][2], d2);
                            }
                        }
                        sc[bb] = fmaf((float)d2, 65536.f, fmaf((float)d1, 256.f, (float)d0)) * qinv;
                    } else {
                        // two accumulators: halves the dependent FFMA2 chain (ILP)
                        f2 acc[2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
                        for (int i = 0; i < CPT; ++i) {
                            f2 kx[NP];
                            Dec::dec(*(const uint4*)(ent + coff[i]), kx);
#pragma unroll
                            for (int t = 0; t < NP; ++t) acc[t & 1] = fma2(q[i][t], kx[t], acc[t & 1]);
                        }
                        const f2 a = add2(acc[0], acc[1]);
                        sc[bb] = a.x + a.y;
                    }
                }
#pragma unroll
                for (int off = 16; off; off >>= 1) {
                    if (off < LPH) {
#pragma unroll
                        for (int bb = 0; bb < NB; ++bb) sc[bb] += __shfl_xor_sync(0xffffffffu, sc[bb], off);
                    }
                }
                float mx = m;
#pragma unroll
                for (int bb = 0; bb < NB; ++bb) {
                    const int e = e0 + sub + bb * P.EP;
                    const bool valid = active_sub && e < n;
                    const uint8_t* ent = sb + (size_t)(valid ? e : 0) * eb;
                    float x = sc[bb] * P.scale2;
                    if (QUANT) x *= ((const float*)(ent + 2 * pay))[head];
                    sc[bb] = valid ? x : -INFINITY;
                    if (valid && j == 0) scp[e * H] = x;
                    mx = fmaxf(mx, sc[bb]);
                }
                if (mx > m) {  // lazy rescale: only when the running max moves
                    const float corr = ex2(m - mx);  // m = -inf -> 0
                    l *= corr;
                    const f2 c2 = {corr, corr};
#pragma unroll
                    for (int i = 0; i < CPT; ++i)
#pragma unroll
                        for (int t = 0; t < NP; ++t) o[i][t] = mul2(o[i][t], c2);
                    m = mx;
                }
#pragma unroll
                for (int bb = 0; bb < NB; ++bb) {
                    const int e = e0 + sub + bb * P.EP;
                    if (active_sub && e < n) {
                        const uint8_t* ent = sb + (size_t)e * eb;
                        float pp = ex2(sc[bb] - m);
                        l += pp;
                        if (QUANT) pp *= ((const float*)(ent + 2 * pay))[H + head];
                        const f2 p2 = {pp, pp};
#pragma unroll
                        for (int i = 0; i < CPT; ++i) {
                            f2 vx[NP];
                            Dec::dec(*(const uint4*)(ent + pay + coff[i]), vx);
#pragma unroll
                            for (int t = 0; t < NP; ++t) o[i][t] = fma2(p2, vx[t], o[i][t]);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == P.NST) stage = 0, phase ^= 1;
        }
        // ---- write the item's partial (m, l, o), merging sub-groups ----
        if (P.EP == 1) {
#pragma unroll
            for (int i = 0; i < CPT; ++i) {
                float* po = S.part_o + ((int64_t)w * H + head) * dph + (j + i * LPH) * N;
#pragma unroll
                for (int t = 0; t < NP; ++t) po[2 * t] = o[i][t].x, po[2 * t + 1] = o[i][t].y;
            }
            if (j == 0) {
                S.part_m[(int64_t)w * H + head] = m;
                S.part_l[(int64_t)w * H + head] = l;
            }
        } else {
            // red layout: [EP][H*dph] o, then [EP][H] m, [EP][H] l
            float* ro = red;
            float* rm = red + (size_t)P.EP * H * dph;
            float* rl = rm + (size_t)P.EP * H;
            if (active_sub) {
#pragma unroll
                for (int i = 0; i < CPT; ++i) {
                    float* dst = ro + (size_t)sub * H * dph + head * dph + (j + i * LPH) * N;
#pragma unroll
                    for (int t = 0; t < NP; ++t) dst[2 * t] = o[i][t].x, dst[2 * t + 1] = o[i][t].y;
                }
                if (j == 0) {
                    rm[sub * H + head] = m;
                    rl[sub * H + head] = l;
                }
            }
            consumer_bar();
            if (sub == 0) {
                float M = -INFINITY;
                for (int g = 0; g < P.EP; ++g) M = fmaxf(M, rm[g * H + head]);
                float L = 0.f;
                f2 acc[CPT][NP];
#pragma unroll
                for (int i = 0; i < CPT; ++i)
#pragma unroll
                    for (int t = 0; t < NP; ++t) acc[i][t] = {0.f, 0.f};
                for (int g = 0; g < P.EP; ++g) {
                    const float mg = rm[g * H + head];
                    const float f = mg == -INFINITY ? 0.f : exp2f(mg - M);
                    L += rl[g * H + head] * f;
#pragma unroll
                    for (int i = 0; i < CPT; ++i) {
                        const float* src = ro + (size_t)g * H * dph + head * dph + (j + i * LPH) * N;
#pragma unroll
                        for (int t = 0; t < NP; ++t) {
                            acc[i][t].x += src[2 * t] * f;
                            acc[i][t].y += src[2 * t + 1] * f;
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < CPT; ++i) {
                    float* po = S.part_o + ((int64_t)w * H + head) * dph + (j + i * LPH) * N;
#pragma unroll
                    for (int t = 0; t < NP; ++t) po[2 * t] = acc[i][t].x, po[2 * t + 1] = acc[i][t].y;
                }
                if (j == 0) {
                    S.part_m[(int64_t)w * H + head] = M;
                    S.part_l[(int64_t)w * H + head] = L;
                }
            }
            consumer_bar();
        }
    }
}

struct Plan {
    AttParams P;
    int cpt;
    int cps;  // CTAs per SM (2, or 3 with a two-stage ring)
    size_t smem;
};

// Three CTAs per SM (PIKV_ATT_CPS=3; 72 registers, two-stage ring of ~32 KiB
// stages): bf16 / f32 heads only (the int8 / int4 consumers spill at 72).
int cps_of(const Dims& D) {
    if (D.codec == PIKV_CODEC_INT8 || D.codec == PIKV_CODEC_INT4 || D.kv_dtype != PIKV_DTYPE_BF16) return 2;
    const char* v = std::getenv("PIKV_ATT_CPS");
    return v && v[0] == '3' ? 3 : 2;
}

Plan make_plan(const Dims& D) {
    Plan pl{};
    pl.cps = cps_of(D);
    const int budget = pl.cps == 3 ? kSmemBudget3 : kSmemBudget;
    const int min_st = pl.cps == 3 ? 2 : 3;
    int elem_bytes_x2 = 0;  // payload bytes per element * 2
    switch (D.codec) {
        case PIKV_CODEC_INT8: elem_bytes_x2 = 2; break;
        case PIKV_CODEC_INT4: elem_bytes_x2 = 1; break;
        default: elem_bytes_x2 = D.kv_dtype == PIKV_DTYPE_BF16 ? 4 : 8; break;
    }
    const int head_bytes = D.dph * elem_bytes_x2 / 2;
    pl.P.CPH = head_bytes / 16;
    // chunks per thread: aim for 8 lanes per head, and a whole entry within
    // the 256 consumer threads
    int cpt = pl.P.CPH >= 8 ? pl.P.CPH / 8 : 1;
    while (cpt < 8 && cpt < pl.P.CPH && D.H * (pl.P.CPH / cpt) > kConsumers) cpt *= 2;
    if (const char* v = std::getenv("PIKV_ATT_CPT")) {  // A/B experiments only
        const int want = std::atoi(v);
        if (want >= cpt && want <= 8 && want <= pl.P.CPH && (want & (want - 1)) == 0) cpt = want;
    }
    pl.cpt = cpt;
    pl.P.LPH = pl.P.CPH / cpt;
    pl.P.TPE = D.H * pl.P.LPH;
    pl.P.EP = pl.P.TPE > 0 ? kConsumers / pl.P.TPE : 0;
    // entries per stage: ~32 KiB, at least one per sub-group when possible,
    // and small enough that the ring keeps >= 3 stages in flight
    const size_t redb = pl.P.EP > 1 ? sizeof(float) * (size_t)pl.P.EP * D.H * (D.dph + 2) : 0;
    const int ring_max = (int)((budget - 256 - redb) / D.entry_bytes);  // entries that fit
    // a stage holds whole consumer batches (EP sub-groups x NB entries): a
    // partly filled batch still decodes and dots its K chunks
    const int nb = (D.codec == PIKV_CODEC_INT8 || D.codec == PIKV_CODEC_INT4 || cpt == 1) ? 4 : 2;  // BatchOf::NB
    const int batch = std::max(1, pl.P.EP * nb);
    int eps = (32 * 1024) / D.entry_bytes;
    eps = std::max(eps, std::min(batch, 32));
    if (eps % batch && (eps / batch + 1) * batch <= std::max(1, ring_max / min_st)) eps = (eps / batch + 1) * batch;
    eps = std::min(eps, std::max(1, ring_max / min_st));
    eps = eps < 1 ? 1 : (eps > 32 ? 32 : eps);
    pl.P.EPS = eps;
    pl.P.stage_bytes = eps * D.entry_bytes;
    int nst = (int)((budget - 256 - redb) / pl.P.stage_bytes);
    pl.P.NST = nst > 8 ? 8 : nst;
    pl.P.scale2 = 1.4426950408889634f / sqrtf((float)D.dph);
    {
        const char* st = std::getenv("PIKV_ATT_STATIC");  // A/B experiments only
        pl.P.dyn = st && st[0] == '1' ? 0 : 1;
        const char* mg = std::getenv("PIKV_ATT_MERGE");
        pl.P.merge = mg && mg[0] == '1' ? 1 : 0;
    }


    pl.smem = 256 + (size_t)pl.P.NST * pl.P.stage_bytes + redb;
    return pl;
}

// entries per consumer batch: 4 where a thread's share of an entry is small
// (int8 / int4 codes; one 16-byte chunk of a bf16/f32 head, e.g. rank-32
// projections) to amortize the per-entry softmax work, else 2 (registers)
template <class Dec, int CPT> struct BatchOf { static constexpr int NB = CPT == 1 ? 4 : 2; };
template <int CPT> struct BatchOf<DecI8, CPT> { static constexpr int NB = 4; };
template <int CPT> struct BatchOf<DecI4, CPT> { static constexpr int NB = 4; };

template <class Dec, int CPT, int LPHC>
void launch_t(const Dims& D, const State& S, const Plan& pl, cudaStream_t st) {
    auto kern = k_attend<Dec, CPT, BatchOf<Dec, CPT>::NB, LPHC, 2>;
    if constexpr (std::is_same<Dec, DecBF16>::value)
        if (pl.cps == 3) kern = k_attend<Dec, CPT, BatchOf<Dec, CPT>::NB, LPHC, 3>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
    launch_pdl(kern, dim3(D.attend_ctas), dim3(kThreads), pl.smem, st, D, S, pl.P);
}

// lanes per head fixed at compile time for the common layouts (4 or 8 lanes:
// 128-dim bf16/int8/int4 heads, rank-32 projections), run-time otherwise
template <class Dec, int CPT>
void launch_lph(const Dims& D, const State& S, const Plan& pl, cudaStream_t st) {
    if (pl.P.LPH == 8) launch_t<Dec, CPT, 8>(D, S, pl, st);
    else if (pl.P.LPH == 4) launch_t<Dec, CPT, 4>(D, S, pl, st);
    else launch_t<Dec, CPT, 0>(D, S, pl, st);
}

template <class Dec>
void launch_dec(const Dims& D, const State& S, const Plan& pl, cudaStream_t st) {
    switch (pl.cpt) {
        case 1: launch_lph<Dec, 1>(D, S, pl, st); break;
        case 2: launch_lph<Dec, 2>(D, S, pl, st); break;
        case 4: launch_t<Dec, 4, 0>(D, S, pl, st); break;
        case 8: launch_t<Dec, 8, 0>(D, S, pl, st); break;
        default: break;
    }
}

}  // namespace

// Valid iff the head slice is a whole number of 16-byte chunks, CPH is a
// power of two <= 32, and the K payload is <= 1024 chunks (VPT <= 4) with the
// thread mapping exact.  Returns a message or nullptr.
const char* attend_check(const Dims& D) {
    if (attend_i4tc_applies(D))
        return attend_i4tc_stages(D) < 2 ? "KV entry too large for the shared-memory ring" : nullptr;
    if (attend_bf16tc_applies(D))
        return attend_bf16tc_stages(D) < 2 ? "KV entry too large for the shared-memory ring" : nullptr;
    Plan pl = make_plan(D);
    int elem_x2 = D.codec == PIKV_CODEC_INT8 ? 2 : D.codec == PIKV_CODEC_INT4 ? 1
                                                 : (D.kv_dtype == PIKV_DTYPE_BF16 ? 4 : 8);
    if (D.dph * elem_x2 % 32 != 0) return "stored head width must be a multiple of 16 bytes";
    const int cph = pl.P.CPH;
    if (cph < 1 || cph > 64 || (cph & (cph - 1))) return "stored head width must be 16..1024 B, power of 2";
    if (pl.P.LPH > 32 || pl.P.TPE > kConsumers || kConsumers % pl.P.TPE)
        return "heads x lanes-per-head must divide 256 (reduce heads or head width)";
    if (pl.P.NST < 2) return "KV entry too large for the shared-memory ring";
    return nullptr;
}

int attend_max_smem() { return kSmemBudget; }

// entries per ring stage of the attention plan (work items are sized in
// multiples of it so no item ends in a partly filled stage)
int attend_entries_per_stage(const Dims& D) {
    if (attend_i4tc_applies(D)) return attend_i4tc_eps();
    if (attend_bf16tc_applies(D)) return attend_bf16tc_eps();
    return make_plan(D).P.EPS;
}

// resident attention CTAs per SM: one CTA of up to 544 threads for the
// tensor-core kernels, two 288-thread CTAs otherwise
// SMs the micro-batch pipeline leaves free of attention CTAs for the other
// micro-batch's control plane (profiles/README.md sweeps): the int8 / int4
// consumers need more issue slots per byte than the control tail, the HMMA
// low-rank kernel sustains more per SM than the CUDA-core bf16 kernel.
int attend_reserve_sms(const Dims& D) {
    // (with static shares and two ring producers, profiles/scripts/r02_tc_sms.sh:
    // c4-int4 72.3 K at 116 SMs vs 71.1 K at 124; c4-lowrank 77.6-78.0 K at 108
    // vs 76.2-76.9 K at 116)
    if (attend_i4tc_applies(D)) return 32;
    if (attend_bf16tc_applies(D)) return 40;
    if (D.codec == PIKV_CODEC_INT8 || D.codec == PIKV_CODEC_INT4) return 12;
    return 44;
}

int attend_ctas_per_sm(const Dims& D) {
    return attend_i4tc_applies(D) || attend_bf16tc_applies(D) ? 1 : make_plan(D).cps;
}

void launch_attend(const Dims& D, const State& S, cudaStream_t st) {
    if (attend_i4tc_applies(D)) {
        launch_attend_i4tc(D, S, st);
        return;
    }
    if (attend_bf16tc_applies(D)) {
        launch_attend_bf16tc(D, S, st);
        return;
    }
    Plan pl = make_plan(D);
    switch (D.codec) {
        case PIKV_CODEC_INT8: launch_dec<DecI8>(D, S, pl, st); break;
        case PIKV_CODEC_INT4: launch_dec<DecI4>(D, S, pl, st); break;
        default:
            if (D.kv_dtype == PIKV_DTYPE_BF16) launch_dec<DecBF16>(D, S, pl, st);
            else launch_dec<DecF32>(D, S, pl, st);
            break;
    }
}

}  // namespace pikv_dev
