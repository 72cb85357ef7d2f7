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
//  * persistent grid: one 288-thread CTA per SM; work items = (stream, run of
//    C consecutive retrieved entries), strided over CTAs;
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

#include "pikv_dev.cuh"

namespace pikv_dev {

namespace {

constexpr int kConsumers = 256;
constexpr int kThreads = kConsumers + 32;
constexpr int kSmemBudget = 220 * 1024;

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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void consumer_bar() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// ---- 16-byte chunk decoders ------------------------------------------------
struct DecBF16 {
    static constexpr int N = 8;
    __device__ static void dec(const uint4& w, float* x) {
        x[0] = bf16_lo(w.x), x[1] = bf16_hi(w.x), x[2] = bf16_lo(w.y), x[3] = bf16_hi(w.y);
        x[4] = bf16_lo(w.z), x[5] = bf16_hi(w.z), x[6] = bf16_lo(w.w), x[7] = bf16_hi(w.w);
    }
};
struct DecF32 {
    static constexpr int N = 4;
    __device__ static void dec(const uint4& w, float* x) {
        x[0] = __uint_as_float(w.x), x[1] = __uint_as_float(w.y);
        x[2] = __uint_as_float(w.z), x[3] = __uint_as_float(w.w);
    }
};
struct DecI8 {
    static constexpr int N = 16;
    __device__ static void dec(const uint4& w, float* x) {
        const uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) x[i * 4 + j] = (float)((int32_t)(v[i] << (24 - 8 * j)) >> 24);
    }
};
struct DecI4 {
    static constexpr int N = 32;
    __device__ static void dec(const uint4& w, float* x) {
        const uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) x[i * 8 + j] = (float)((int32_t)(v[i] << (28 - 4 * j)) >> 28);
    }
};

struct AttParams {
    int CPH;          // 16-byte chunks per head (K payload)
    int cpe;          // chunks per entry (K payload) = H * CPH
    int EP;           // entries processed in parallel by sub-groups
    int EPS;          // entries per stage
    int NST;          // stages
    int stage_bytes;
    int quant;        // INT8/INT4: per-(entry, head) scales after the payloads
    float scale2;     // log2(e) / sqrt(dph)
};

template <class Dec, int VPT, int NB>
__global__ void __launch_bounds__(kThreads, 1) k_attend(Dims D, State S, AttParams P) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int N = Dec::N;
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = full + 16;
    uint8_t* stages = smem + 256;
    float* red = (float*)(stages + (size_t)P.NST * P.stage_bytes);  // EP merge scratch
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < P.NST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kConsumers / 32);
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
        for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
            const int s = S.item_stream[w];
            const int64_t pos0 = S.att_base[s] + S.item_begin[w];
            const int cnt = S.item_end[w] - S.item_begin[w];
            for (int b = 0; b < cnt; b += P.EPS) {
                const int n = min(P.EPS, cnt - b);
                if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], (uint32_t)(n * eb));
                }
                __syncwarp();
                if (lane < n) {
                    const int64_t ent = S.att_entry[pos0 + b + lane];
                    bulk_g2s(stages + (size_t)stage * P.stage_bytes + (size_t)lane * eb,
                             S.pool + ent * (int64_t)eb, (uint32_t)eb, &full[stage], pol);
                }
                if (++stage == P.NST) stage = 0, phase ^= 1;
            }
        }
        return;
    }

    // ================= consumer warps =================
    int sub, cbase;
    if (P.EP > 1) {
        sub = tid / P.cpe;
        cbase = tid % P.cpe;
    } else {
        sub = 0;
        cbase = tid;
    }
    int head[VPT], cc[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int c = cbase + i * kConsumers;
        head[i] = c / P.CPH;
        cc[i] = c % P.CPH;
    }
    int stage = 0;
    uint32_t phase = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const int s = S.item_stream[w];
        const int64_t pos0 = S.att_base[s] + S.item_begin[w];
        const int cnt = S.item_end[w] - S.item_begin[w];
        float q[VPT][N], o[VPT][N], m[VPT], l[VPT];
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            const float* qs = S.q_attn + (int64_t)s * D.dp + head[i] * dph + cc[i] * N;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                q[i][j] = qs[j];
                o[i][j] = 0.f;
            }
            m[i] = -INFINITY;
            l[i] = 0.f;
        }
        for (int b = 0; b < cnt; b += P.EPS) {
            const int n = min(P.EPS, cnt - b);
            mbar_wait(&full[stage], phase);
            const uint8_t* sb = stages + (size_t)stage * P.stage_bytes;
            // warp-uniform trip count: sub-groups of one warp may see
            // different entries, never different loop counts (shuffles below)
            for (int e0 = 0; e0 < n; e0 += P.EP * NB) {
                float sc[NB][VPT];
#pragma unroll
                for (int bb = 0; bb < NB; ++bb) {
                    const int e = e0 + sub + bb * P.EP;
                    const bool valid = e < n;
                    const uint8_t* ent = sb + (size_t)(valid ? e : 0) * eb;
#pragma unroll
                    for (int i = 0; i < VPT; ++i) {
                        const uint4 kw = *(const uint4*)(ent + (size_t)(cbase + i * kConsumers) * 16);
                        float kx[N];
                        Dec::dec(kw, kx);
                        float acc = 0.f;
#pragma unroll
                        for (int j = 0; j < N; ++j) acc = fmaf(q[i][j], kx[j], acc);
                        sc[bb][i] = acc;
                    }
                }
#pragma unroll
                for (int off = 16; off; off >>= 1) {
                    if (off < P.CPH) {
#pragma unroll
                        for (int bb = 0; bb < NB; ++bb)
#pragma unroll
                            for (int i = 0; i < VPT; ++i)
                                sc[bb][i] += __shfl_xor_sync(0xffffffffu, sc[bb][i], off);
                    }
                }
#pragma unroll
                for (int bb = 0; bb < NB; ++bb) {
                    const int e = e0 + sub + bb * P.EP;
                    const bool valid = e < n;
                    const uint8_t* ent = sb + (size_t)(valid ? e : 0) * eb;
#pragma unroll
                    for (int i = 0; i < VPT; ++i) {
                        float x = sc[bb][i] * P.scale2;
                        if (P.quant) x *= ((const float*)(ent + 2 * pay))[head[i]];
                        sc[bb][i] = valid ? x : -INFINITY;
                        if (valid && cc[i] == 0)
                            S.scores[(pos0 + b + e) * H + head[i]] = x;
                    }
                }
#pragma unroll
                for (int i = 0; i < VPT; ++i) {
                    float mx = m[i];
#pragma unroll
                    for (int bb = 0; bb < NB; ++bb) mx = fmaxf(mx, sc[bb][i]);
                    const bool none = mx == -INFINITY;  // no entry yet for this lane
                    const float corr = none ? 1.f : exp2f(m[i] - mx);
                    float p[NB];
                    float psum = 0.f;
#pragma unroll
                    for (int bb = 0; bb < NB; ++bb) {
                        p[bb] = none ? 0.f : exp2f(sc[bb][i] - mx);
                        psum += p[bb];
                    }
                    l[i] = fmaf(l[i], corr, psum);
                    m[i] = mx;
#pragma unroll
                    for (int j = 0; j < N; ++j) o[i][j] *= corr;
#pragma unroll
                    for (int bb = 0; bb < NB; ++bb) {
                        const int e = e0 + sub + bb * P.EP;
                        if (e < n) {
                            const uint8_t* ent = sb + (size_t)e * eb;
                            const uint4 vw = *(const uint4*)(ent + pay + (size_t)(cbase + i * kConsumers) * 16);
                            float vx[N];
                            Dec::dec(vw, vx);
                            float pp = p[bb];
                            if (P.quant) pp *= ((const float*)(ent + 2 * pay))[H + head[i]];
#pragma unroll
                            for (int j = 0; j < N; ++j) o[i][j] = fmaf(pp, vx[j], o[i][j]);
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
            for (int i = 0; i < VPT; ++i) {
                float* po = S.part_o + ((int64_t)w * H + head[i]) * dph + cc[i] * N;
#pragma unroll
                for (int j = 0; j < N; ++j) po[j] = o[i][j];
                if (cc[i] == 0) {
                    S.part_m[(int64_t)w * H + head[i]] = m[i];
                    S.part_l[(int64_t)w * H + head[i]] = l[i];
                }
            }
        } else {
            // red layout: [EP][H*dph] o, then [EP][H] m, [EP][H] l
            float* ro = red;
            float* rm = red + (size_t)P.EP * H * dph;
            float* rl = rm + (size_t)P.EP * H;
            {
                float* dst = ro + (size_t)sub * H * dph + head[0] * dph + cc[0] * N;
#pragma unroll
                for (int j = 0; j < N; ++j) dst[j] = o[0][j];
                if (cc[0] == 0) {
                    rm[sub * H + head[0]] = m[0];
                    rl[sub * H + head[0]] = l[0];
                }
            }
            consumer_bar();
            if (sub == 0) {
                const int h = head[0];
                float M = -INFINITY;
                for (int g = 0; g < P.EP; ++g) M = fmaxf(M, rm[g * H + h]);
                float L = 0.f, acc[N];
#pragma unroll
                for (int j = 0; j < N; ++j) acc[j] = 0.f;
                for (int g = 0; g < P.EP; ++g) {
                    const float mg = rm[g * H + h];
                    const float f = mg == -INFINITY ? 0.f : exp2f(mg - M);
                    L += rl[g * H + h] * f;
                    const float* src = ro + (size_t)g * H * dph + h * dph + cc[0] * N;
#pragma unroll
                    for (int j = 0; j < N; ++j) acc[j] += src[j] * f;
                }
                float* po = S.part_o + ((int64_t)w * H + h) * dph + cc[0] * N;
#pragma unroll
                for (int j = 0; j < N; ++j) po[j] = acc[j];
                if (cc[0] == 0) {
                    S.part_m[(int64_t)w * H + h] = M;
                    S.part_l[(int64_t)w * H + h] = L;
                }
            }
            consumer_bar();
        }
    }
}

struct Plan {
    AttParams P;
    int vpt;
    size_t smem;
};

Plan make_plan(const Dims& D) {
    Plan pl{};
    int elem_bytes_x2 = 0;  // payload bytes per element * 2
    switch (D.codec) {
        case PIKV_CODEC_INT8: elem_bytes_x2 = 2; break;
        case PIKV_CODEC_INT4: elem_bytes_x2 = 1; break;
        default: elem_bytes_x2 = D.kv_dtype == PIKV_DTYPE_BF16 ? 4 : 8; break;
    }
    const int head_bytes = D.dph * elem_bytes_x2 / 2;
    pl.P.CPH = head_bytes / 16;
    pl.P.cpe = pl.P.CPH * D.H;
    if (pl.P.cpe >= kConsumers) {
        pl.vpt = pl.P.cpe / kConsumers;
        pl.P.EP = 1;
    } else {
        pl.vpt = 1;
        pl.P.EP = kConsumers / pl.P.cpe;
    }
    int eps = (32 * 1024) / D.entry_bytes;
    eps = eps < 1 ? 1 : (eps > 32 ? 32 : eps);
    pl.P.EPS = eps;
    pl.P.stage_bytes = eps * D.entry_bytes;
    const size_t redb = pl.P.EP > 1 ? sizeof(float) * (size_t)pl.P.EP * D.H * (D.dph + 2) : 0;
    int nst = (int)((kSmemBudget - 256 - redb) / pl.P.stage_bytes);
    pl.P.NST = nst > 8 ? 8 : nst;
    pl.P.quant = D.codec == PIKV_CODEC_INT8 || D.codec == PIKV_CODEC_INT4;
    pl.P.scale2 = 1.4426950408889634f / sqrtf((float)D.dph);
    pl.smem = 256 + (size_t)pl.P.NST * pl.P.stage_bytes + redb;
    return pl;
}

template <class Dec, int VPT>
void launch_t(const Dims& D, const State& S, const Plan& pl, cudaStream_t st) {
    auto kern = k_attend<Dec, VPT, 2>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
    kern<<<D.attend_ctas, kThreads, pl.smem, st>>>(D, S, pl.P);
}

template <class Dec>
void launch_dec(const Dims& D, const State& S, const Plan& pl, cudaStream_t st) {
    switch (pl.vpt) {
        case 1: launch_t<Dec, 1>(D, S, pl, st); break;
        case 2: launch_t<Dec, 2>(D, S, pl, st); break;
        case 4: launch_t<Dec, 4>(D, S, pl, st); break;
        default: break;
    }
}

}  // namespace

// Valid iff the head slice is a whole number of 16-byte chunks, CPH is a
// power of two <= 32, and the K payload is <= 1024 chunks (VPT <= 4) with the
// thread mapping exact.  Returns a message or nullptr.
const char* attend_check(const Dims& D) {
    Plan pl = make_plan(D);
    int elem_x2 = D.codec == PIKV_CODEC_INT8 ? 2 : D.codec == PIKV_CODEC_INT4 ? 1
                                                 : (D.kv_dtype == PIKV_DTYPE_BF16 ? 4 : 8);
    if ((D.dph * elem_x2 / 2) % 16 != 0 || D.dph * elem_x2 % 2)
        return "stored head width must be a multiple of 16 bytes";
    const int cph = pl.P.CPH;
    if (cph < 1 || cph > 32 || (cph & (cph - 1))) return "stored head width must be 16..512 B, power of 2";
    if (pl.P.cpe >= kConsumers && (pl.P.cpe % kConsumers || pl.vpt > 4 || pl.vpt == 3))
        return "H * head bytes must be <= 16 KiB and a multiple of 4 KiB above 4 KiB";
    if (pl.P.cpe < kConsumers && kConsumers % pl.P.cpe) return "H * head chunks must divide 256";
    if (pl.P.NST < 2) return "KV entry too large for the shared-memory ring";
    return nullptr;
}

int attend_max_smem() { return kSmemBudget; }

void launch_attend(const Dims& D, const State& S, cudaStream_t st) {
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
