// SPDX-License-Identifier: Apache-2.0
//
// Decode attention over 32-wide bf16 head slices on the tensor cores (HMMA:
// mma.sync m16n8k16 bf16, fp32 accumulate): the c4 rank-32 low-rank layout
// (LowRank / LoRAPlus / FastV / Prune projections stored as bf16; also plain
// bf16 heads of width 32).  Same contract as k_attend (attend.cu):
// attention() of pipeline.cpp:59-85 per head over a work item's retrieved
// entries -> the item's partial softmax state (m, l, o) and every entry's
// per-head base-2 logit.
//
// The CUDA-core kernel spends ~344 warp-instructions per 4 KiB entry on the
// per-entry softmax bookkeeping of 16-value chunks (profiles/README.md); here
// a warp owns a head pair and handles 16 entries per MMA:
//  * q.k: the K rows of 16 entries are the A operand, loaded straight from the
//    ring by ldmatrix (no conversion); q (fp32) is split exactly enough into
//    three bf16 parts hi + mid + lo (24 bits) in three B columns, so the
//    products are exact and the MMA sums them in fp32;
//  * p.v: V^T by ldmatrix.trans (entries become the k index), the weights p in
//    three bf16 parts in the B columns, fp32 accumulators in registers,
//    rescaled when the running max moves;
//  * two heads per MMA: head h in k-slots 0-7 / columns 0-2, head h+1 in
//    k-slots 8-15 / columns 4-6 (block-diagonal B).
// Ring: attend_ring.cuh, 3 stages x 16 entries (PIKV_BF16TC_EPS=8: 7 x 8),
// slot stride = entry + 16 B (ldmatrix's 8 row addresses fall in 8 different
// 16-B bank groups).  Default for these layouts (PIKV_BF16TC=0: the CUDA-core
// kernel), see attend_bf16tc_applies.
#include <cuda_runtime.h>

#include <cstdlib>

#include "attend_ring.cuh"

namespace pikv_dev {

namespace {

constexpr int kDPH = 32;  // head slice width (bf16 values)
constexpr int kPadB = 16;
constexpr unsigned kAllB = 0xffffffffu;

struct BTcParams {
    RingParams R;
    float scale2;  // log2(e) / sqrt(dph)
    int early;     // release each stage once its fragments are in registers (PIKV_BF16TC_EARLY=1; default after the math)
};

// Scoreboard wait on every loaded fragment register (an empty asm that reads
// them): the ldmatrix reads of the stage are complete before it is released.
template <int A, int J, int T>
__device__ __forceinline__ void regs_ready(const uint32_t (&ka)[A][4], const uint32_t (&va)[J][T][4]) {
#pragma unroll
    for (int i = 0; i < A; ++i) asm volatile("" ::"r"(ka[i][0]), "r"(ka[i][1]), "r"(ka[i][2]), "r"(ka[i][3]) : "memory");
#pragma unroll
    for (int j = 0; j < J; ++j)
#pragma unroll
        for (int t = 0; t < T; ++t)
            asm volatile("" ::"r"(va[j][t][0]), "r"(va[j][t][1]), "r"(va[j][t][2]), "r"(va[j][t][3]) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2b(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// x = hi + mid + lo as three bf16 (truncations: each subtraction is exact,
// 24 significant bits in all), as fp32 bit patterns (bf16 = the upper half)
struct Parts3 {
    uint32_t hi, mid, lo;
};
__device__ __forceinline__ Parts3 split3(float x) {
    const uint32_t hi = __float_as_uint(x) & 0xFFFF0000u;
    const float r1 = x - __uint_as_float(hi);
    const uint32_t mid = __float_as_uint(r1) & 0xFFFF0000u;
    const float r2 = r1 - __uint_as_float(mid);
    return Parts3{hi, mid, __float_as_uint(r2) & 0xFFFF0000u};
}
// two values' part p (0 hi, 1 mid, 2 lo, 3 zero) packed as bf16x2 (a low)
__device__ __forceinline__ uint32_t pack_part(const Parts3& a, const Parts3& b, int p) {
    const uint32_t x = p == 0 ? a.hi : p == 1 ? a.mid : a.lo;
    const uint32_t y = p == 0 ? b.hi : p == 1 ? b.mid : b.lo;
    return p == 3 ? 0u : __byte_perm(x, y, 0x7632);
}

// EPS entries per ring stage: 16 (q.k rows g / g + 8, p.v two halves) or 8
// (q.k rows g + 8 repeat rows g; one p.v MMA per d tile; twice the stages)
template <int EPS>
__global__ void __launch_bounds__(19 * 32, 1) k_attend_bf16tc(Dims D, State S, BTcParams P) {
    const long long t_entry = D.dbg_att && threadIdx.x == 0 ? (long long)globaltimer() : 0;  // PIKV_DEBUG_ATT
    long long t_wait = 0, n_stage = 0, n_ent = 0;
    griddep_enter();
    extern __shared__ __align__(128) uint8_t smem[];
    const RingSmem R = ring_smem(smem);
    const int H = D.H;
    const int ncw = H / 2;
    uint8_t* stages = smem + 256;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) ring_init(R, P.R, ncw);
    __syncthreads();
    const int n_items = S.n_items[0];
    const int pay = D.payload_bytes;
    if (warp >= ncw) {  // producers: two with static shares (ring_produce)
        const int nprod = P.R.nprod;
        if (warp - ncw < nprod) ring_produce(D, S, P.R, R, stages, n_items, lane, warp - ncw, nprod);
        return;
    }

    // MMA fragment coordinates: g = lane / 4, t = lane % 4.  q.k tile rows g /
    // g + 8 = entries g / g + 8 of the stage; lanes t = 0, 1 hold head h0,
    // t = 2, 3 head h1 in the softmax and output layout
    const int g = lane >> 2, t = lane & 3, odd = t & 1;
    const int h0 = 2 * warp, h1 = h0 + 1;
    const int hm = t < 2 ? h0 : h1;
    // ldmatrix roles: lane = 8 * matrix + row
    const int mi = lane >> 3, mr = lane & 7;
    const int mh = mi < 2 ? h0 : h1;
    // q.k (non-transposed): matrix mi = entries 8 (mi & 1) + row, 8 dims of head mh
    const int qk_off = ((EPS == 16 ? (mi & 1) << 3 : 0) + mr) * P.R.stride + mh * kDPH * 2;
    // p.v (transposed): matrix mi = entries 8j + row, d 16T + 8 (mi & 1) of head mh
    const int pv_off = mr * P.R.stride + pay + mh * kDPH * 2 + (mi & 1) * 16;
    const int part = g & 3;  // B column g: part g of head h0 (g < 3) or g - 4 of h1
    // p.v B fragment select: part 0 = low halves of (hi | mid), 1 = high
    // halves, 2 = the lo words' high halves, 3 = zero column; b0 for h0 lanes
    const uint32_t psel = part == 0 ? 0x5410u : 0x7632u;
    const bool plo = part == 2;
    const uint32_t pz = part == 3 ? 0u : 0xFFFFFFFFu;
    const uint32_t bm0 = g < 4 ? 0xFFFFFFFFu : 0u;
    int stage = 0;
    uint32_t phase = 0;
    for (int kq = 0;; ++kq) {
        const int w = ring_next_item(R, kq, lane);
        if (w >= n_items) {
            if (D.dbg_att && tid == 0) {
                long long* d = S.dbg + 64 + 8 * D.B + 8 * blockIdx.x;
                d[0] = t_entry, d[1] = (long long)globaltimer(), d[2] = kq, d[3] = n_ent, d[4] = smid();
                d[5] = t_entry, d[6] = t_wait, d[7] = n_stage;
            }
            break;
        }
        const int s = S.item_stream[w];
        const int64_t pos0 = (int64_t)s * D.att_stride + S.item_begin[w];
        const int cnt = S.item_end[w] - S.item_begin[w];
        n_ent += cnt;
        // q.k B fragments: MMA i covers dims 8i..8i+7 of both heads; b0 = head
        // h0 dims 8i + 2t, +1 (k-slots 2t, 2t+1), b1 = head h1 (k-slots 8 + 2t)
        uint32_t qB[kDPH / 8][2];
        {
            const float* qh = S.q_attn + (int64_t)s * D.dp + (g < 4 ? h0 : h1) * kDPH + 2 * t;
#pragma unroll
            for (int i = 0; i < kDPH / 8; ++i) {
                const float2 qq = *(const float2*)(qh + 8 * i);
                const uint32_t pk = pack_part(split3(qq.x), split3(qq.y), part);
                qB[i][0] = g < 4 ? pk : 0u;
                qB[i][1] = g < 4 ? 0u : pk;
            }
        }
        float* scp = S.scores + (pos0 + g + 8 * odd) * H + hm;  // this lane's logit slot, stage 0
        float m = -INFINITY, l = 0.f;
        // p.v accumulators: tile T rows g / g + 8 = d 16T + g / 16T + 8 + g,
        // columns 2t, 2t + 1 (parts of head hm)
        float acc[kDPH / 16][4];
#pragma unroll
        for (int T = 0; T < kDPH / 16; ++T) acc[T][0] = acc[T][1] = acc[T][2] = acc[T][3] = 0.f;

        for (int b = 0; b < cnt; b += EPS, scp += EPS * H) {
            const int n = min(EPS, cnt - b);
            if (D.dbg_att && tid == 0) {
                const long long t0 = (long long)globaltimer();
                mbar_wait_sleep(&R.full[stage], phase);
                t_wait += (long long)globaltimer() - t0, ++n_stage;
            } else {
                mbar_wait_sleep(&R.full[stage], phase);
            }
            const uint8_t* sb = stages + (size_t)stage * P.R.stage_bytes;
            // The stage's K and V^T fragments go to registers first and the
            // stage is released before any math: the ring slot is busy for the
            // ldmatrix round trip only, not the whole q.k -> softmax -> p.v
            // chain (consumers waited 26-33 % of the time for data with the
            // release after the math: profiles/README.md)
            uint32_t ka[kDPH / 8][4], va[EPS / 8][kDPH / 16][4];
#pragma unroll
            for (int i = 0; i < kDPH / 8; ++i) ldsm_x4(ka[i], sb + qk_off + 16 * i);
#pragma unroll
            for (int j = 0; j < EPS / 8; ++j)
#pragma unroll
                for (int T = 0; T < kDPH / 16; ++T) ldsm_x4_t(va[j][T], sb + pv_off + (8 * j) * P.R.stride + 32 * T);
            if (P.early) {
                regs_ready(ka, va);  // the loads have landed before the slot is handed back
                __syncwarp();
                if (lane == 0) mbar_arrive(&R.empty[stage]);
            }
            // ---------------- q.k ----------------
            float dq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < kDPH / 8; ++i) hmma(dq, ka[i], qB[i][0], qB[i][1]);
            // column 2t (+1): hi + mid (t even) or lo (t odd) of head hm
            float s0 = dq[0] + dq[1], s1 = dq[2] + dq[3];
            s0 += __shfl_xor_sync(kAllB, s0, 1);
            s1 += __shfl_xor_sync(kAllB, s1, 1);
            const bool v0 = g < n, v1 = EPS == 16 && g + 8 < n;
            const float x0 = v0 ? s0 * P.scale2 : -INFINITY;
            const float x1 = v1 ? s1 * P.scale2 : -INFINITY;
            if (odd ? v1 : v0) *scp = odd ? x1 : x0;
            // ---------------- online softmax of head hm ----------------
            float mx = fmaxf(x0, x1);
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(kAllB, mx, off));
            if (mx > m) {
                const float c = ex2b(m - mx);  // m = -inf -> 0
                l *= c;
#pragma unroll
                for (int T = 0; T < kDPH / 16; ++T) acc[T][0] *= c, acc[T][1] *= c, acc[T][2] *= c, acc[T][3] *= c;
                m = mx;
            }
            const float p0 = ex2b(x0 - m), p1 = ex2b(x1 - m);
            l += p0 + p1;
            // the weights' bf16 parts, split once by the lane that owns them:
            // (hi | mid) packed, lo in the upper half
            const Parts3 q0 = split3(p0), q1 = split3(p1);
            const uint32_t hm0 = __byte_perm(q0.hi, q0.mid, 0x7632), hm1 = __byte_perm(q1.hi, q1.mid, 0x7632);
            // ---------------- p.v: two halves of 8 entries ----------------
            // the stage's MMAs start from zero and are added to acc in fp32 (the
            // tensor core's accumulate aligns to the largest term and truncates:
            // carried across a whole item it would drift by ~1e-5)
            float st[kDPH / 16][4];
#pragma unroll
            for (int T = 0; T < kDPH / 16; ++T) st[T][0] = st[T][1] = st[T][2] = st[T][3] = 0.f;
            const int hs = g < 4 ? 0 : 2;
#pragma unroll
            for (int j = 0; j < EPS / 8; ++j) {
                // k-slots 2t, 2t + 1 = entries 8j + 2t, +1: their weights live in
                // lanes (2t) * 4 and (2t + 1) * 4 (+2 for head h1), register j
                const uint32_t shm = j ? hm1 : hm0, slo = j ? q1.lo : q0.lo;
                const int sa = (2 * t) * 4 + hs, sbb = (2 * t + 1) * 4 + hs;
                const uint32_t ahm = __shfl_sync(kAllB, shm, sa), bhm = __shfl_sync(kAllB, shm, sbb);
                const uint32_t alo = __shfl_sync(kAllB, slo, sa), blo = __shfl_sync(kAllB, slo, sbb);
                // branch-free part select (lane constants psel / plo / pz)
                const uint32_t pk = __byte_perm(plo ? alo : ahm, plo ? blo : bhm, psel) & pz;
                const uint32_t b0 = pk & bm0, b1 = pk & ~bm0;
#pragma unroll
                for (int T = 0; T < kDPH / 16; ++T) {
                    uint32_t* a = va[j][T];
                    if (n < EPS) {
                        // a partly filled stage: the unused slots hold stale bytes
                        // (NaN patterns included) -- zero their V so 0 * NaN cannot
                        // reach o
                        const uint32_t vm = (8 * j + 2 * t < n ? 0x0000FFFFu : 0u) |
                                            (8 * j + 2 * t + 1 < n ? 0xFFFF0000u : 0u);
                        a[0] &= vm, a[1] &= vm, a[2] &= vm, a[3] &= vm;
                    }
                    hmma(st[T], va[j][T], b0, b1);
                }
            }
#pragma unroll
            for (int T = 0; T < kDPH / 16; ++T)
                acc[T][0] += st[T][0], acc[T][1] += st[T][1], acc[T][2] += st[T][2], acc[T][3] += st[T][3];
            if (!P.early) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&R.empty[stage]);
            }
            if (++stage == P.R.NST) stage = 0, phase ^= 1;
        }
        // ---- the item's partial (m, l, o) of heads h0, h1 ----
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) l += __shfl_xor_sync(kAllB, l, off);
        float* po = S.part_o + ((int64_t)w * H + hm) * kDPH + g + 8 * odd;
#pragma unroll
        for (int T = 0; T < kDPH / 16; ++T) {
            const float r0 = acc[T][0] + acc[T][1], r1 = acc[T][2] + acc[T][3];
            // t even keeps row g, t odd row g + 8: swap halves, then add
            const float mine = odd ? r1 : r0, other = odd ? r0 : r1;
            po[16 * T] = mine + __shfl_xor_sync(kAllB, other, 1);
        }
        if (g == 0 && !odd) {
            S.part_m[(int64_t)w * H + hm] = m;
            S.part_l[(int64_t)w * H + hm] = l;
        }
    }
}

}  // namespace

// bf16 stored head slices of width 32 (rank-32 projections or 32-dim heads),
// even H <= 32; default (PIKV_BF16TC=0 selects the CUDA-core kernel).  With
// equal static work shares the HMMA kernel beats the CUDA-core one at
// c4-lowrank: 73.6-74.4 K vs 71.1-73.3 K tokens/s, e2e 72-73 K vs 64-66 K
// (three runs each), attention frac 0.87-0.89 on 116 SMs
// (profiles/scripts/r02_lowrank_rep.sh, profiles/README.md).
bool attend_bf16tc_applies(const Dims& D) {
    if (D.codec == PIKV_CODEC_INT8 || D.codec == PIKV_CODEC_INT4) return false;
    if (D.kv_dtype != PIKV_DTYPE_BF16 || D.dph != kDPH || D.H < 2 || D.H > 32 || (D.H & 1)) return false;
    const char* v = std::getenv("PIKV_BF16TC");  // read at engine creation and graph capture
    return !(v && v[0] == '0');
}

static int btc_eps() {
    const char* v = std::getenv("PIKV_BF16TC_EPS");  // A/B experiments only
    return v && std::atoi(v) == 8 ? 8 : 16;
}

static BTcParams btc_params(const Dims& D, size_t* smem) {
    BTcParams P{};
    P.R = ring_params(D, btc_eps(), kPadB, 0);
    P.scale2 = 1.4426950408889634f / sqrtf((float)D.dph);
    // release after the math (default: c4-lowrank 0.185 vs 0.190 ms per launch
    // with the release right after the fragment loads, PIKV_BF16TC_EARLY=1)
    const char* ea = std::getenv("PIKV_BF16TC_EARLY");  // A/B experiments only
    P.early = ea && ea[0] == '1';
    if (smem) *smem = 256 + (size_t)P.R.NST * P.R.stage_bytes;
    return P;
}

int attend_bf16tc_stages(const Dims& D) { return btc_params(D, nullptr).R.NST; }
int attend_bf16tc_eps() { return btc_eps(); }

void launch_attend_bf16tc(const Dims& D, const State& S, cudaStream_t st) {
    size_t smem = 0;
    const BTcParams P = btc_params(D, &smem);
    auto kern = P.R.eps == 16 ? k_attend_bf16tc<16> : k_attend_bf16tc<8>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kern, dim3(D.attend_ctas), dim3((D.H / 2 + P.R.nprod) * 32), smem, st, D, S, P);
}

}  // namespace pikv_dev
