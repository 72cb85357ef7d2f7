// SPDX-License-Identifier: Apache-2.0
//
// int4 decode attention on the tensor cores (IMMA: mma.sync m16n8k32 u8).
//
// Same contract as k_attend (attend.cu): attention() of pipeline.cpp:59-85
// per head over the retrieved entries of a work item, returning the item's
// partial softmax state (m, l, o) and every entry's per-head base-2 logit.
// Taken for int4 codes with 128-dim heads and an even head count <= 32 (the
// c4 layout); the CUDA-core kernel spends ~1000 warp-instructions per 4352-B
// entry decoding nibbles (profiles/README.md), this one ~250.
//
// Both products are exact integer GEMMs on the raw codes:
//  * q.k: q is quantized per head to a 24-bit fixed point and split into
//    three signed base-256 digit planes (the int8 path's scheme), the MMA's
//    B operand (columns = planes).  A = the K codes of 16 entries (rows),
//    nibbles biased to u8 (c + 8) by one LOP3 per 4 codes; the bias is
//    removed exactly per plane in integers.  Error: the q rounding (~1e-7).
//  * p.v: the entry weights w = p * v_scale are quantized per "epoch" to
//    24-bit integers (headroom kTau bits below 2^24) and split into three u8
//    digit planes (B columns); A = V^T, the transposed V codes of 16
//    entries (one 4x8 nibble transpose per 4 entries: 8 PRMT + LOP3), so the
//    s32 accumulators hold sum_e digit_p(w_e) * (c_e,d + 8) exactly.  The
//    epoch's integer sums are folded into fp32 o (exact fp64 combine of the
//    planes minus 8 * sum w) when a weight would overflow 2^24 (the running
//    max moved by more than the headroom) and at the end of the item.
//    Error: the weight rounding, 2^-(24 - kTau) of the epoch's largest.
//  * block-diagonal packing: one MMA carries two heads -- K (and V) of head
//    h in k-slots 0-15 and of head h+1 in 16-31, their digit planes in B
//    columns 0-2 and 4-6 -- so 6 of the tile's 8 columns are useful.
//
// Layout: one 544-thread CTA per SM (16 consumer warps, one head pair each,
// + a TMA producer warp); a ring of 3 stages x 16 entries (entry stride
// padded by 32 B so both the K row loads and the V column loads are
// bank-conflict free); the producer is the same per-entry cp.async.bulk
// ring as k_attend.
#include <cuda_runtime.h>

#include <cstdlib>

#include "attend_ring.cuh"

namespace pikv_dev {

namespace {

constexpr int kEPS = kRingEPS;     // entries per stage = MMA rows / k-slots per head
constexpr int kPad = 32;           // smem entry stride = entry_bytes + kPad
constexpr int kTau = 5;            // epoch headroom bits
constexpr float kLim = 16777215.f;  // weights must round to < 2^24 (three u8 digits)
constexpr int kEpochMax = 32768;    // entries per epoch: 255 * 240 * n < 2^31
constexpr unsigned kFull = 0xffffffffu;
// q digit planes of a head pair in smem: [head 2][plane 3][K word 16][even, odd],
// planes padded to 36 words (bank spread of the per-lane LDS.128 reads)
constexpr int kQPlane = 36;
constexpr int kQWords = 2 * 3 * kQPlane;
__host__ __device__ constexpr int q_area_bytes(int ncw) { return ((ncw * kQWords + 8) * 4 + 127) / 128 * 128; }

struct I4Params {
    RingParams R;
    float scale2;     // log2(e) / sqrt(128)
    uint32_t c88, c0f;  // nibble masks (kernel parameters, so they stay in registers)
};

__device__ __forceinline__ void imma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void imma_u8u8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2a(float x) {  // 2^x, x <= 0
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// two's-complement nibbles -> biased u8 lanes (c + 8), one LOP3 each with the
// masks in registers (c88 = 0x88888888, c0f = 0x0F0F0F0F): even nibbles as
// c + 8, odd nibbles as 16 (c + 8) (no shift; the x16 is removed in integers)
__device__ __forceinline__ uint32_t nlo(uint32_t w, uint32_t c88, uint32_t c0f) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(d) : "r"(w), "r"(c88), "r"(c0f));  // (w ^ c88) & c0f
    return d;
}
__device__ __forceinline__ uint32_t nhi(uint32_t w, uint32_t c88, uint32_t c0f) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x14;" : "=r"(d) : "r"(w), "r"(c88), "r"(c0f));  // (w ^ c88) & ~c0f
    return d;
}
__device__ __forceinline__ float rcpa(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void __launch_bounds__(19 * 32, 1) k_attend_i4tc(Dims D, State S, I4Params P) {
    griddep_enter();
    extern __shared__ __align__(128) uint8_t smem[];
    const RingSmem R = ring_smem(smem);
    const int H = D.H;
    const int ncw = H / 2;  // consumer warps
    // per consumer warp: its q digit planes in B-fragment order (kQWords),
    // then 32 zero bytes (the B fragment of inactive lanes), then the ring
    uint32_t* qsm = (uint32_t*)(smem + 256);
    const uint4* qzero = (const uint4*)(qsm + ncw * kQWords);
    uint8_t* stages = smem + 256 + q_area_bytes(ncw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid < 8) qsm[ncw * kQWords + tid] = 0u;
    if (tid == 0) ring_init(R, P.R, ncw);
    __syncthreads();
    const int n_items = S.n_items[0];
    const int pay = D.payload_bytes;
    if (warp >= ncw) {  // producers: two with static shares (ring_produce)
        const int nprod = P.R.nprod;
        if (warp - ncw < nprod) ring_produce(D, S, P.R, R, stages, n_items, lane, warp - ncw, nprod);
        return;
    }

    // ================= consumer warps: heads h0, h1 =================
    // MMA fragment coordinates: g = lane / 4 (row / column group), t = lane % 4
    const int g = lane >> 2, t = lane & 3, odd = t & 1;
    const int h0 = 2 * warp, h1 = h0 + 1;
    // softmax / output layout: lanes t = 0, 1 hold head h0, t = 2, 3 head h1;
    // rows g, g + 8 of the q.k tile are entries 2g, 2g + 1 of the stage
    const int hm = t < 2 ? h0 : h1;
    const int koff0 = h0 * 64 + 16 * t, koff1 = h1 * 64 + 16 * t;
    int stage = 0;
    uint32_t phase = 0;
    for (int kq = 0;; ++kq) {
        const int w = ring_next_item(R, kq, lane);
        if (w >= n_items) break;
        const int s = S.item_stream[w];
        const int64_t pos0 = (int64_t)s * D.att_stride + S.item_begin[w];
        const int cnt = S.item_end[w] - S.item_begin[w];

        // ---- q -> three signed base-256 digit planes per head ----
        // lanes 0-15 quantize head h0, 16-31 head h1; lane holds d 8j..8j+7
        // (K word j), stored as the even / odd d of the word per plane
        uint32_t* qw = qsm + warp * kQWords;
        int cA, cB;  // bias corrections of this lane's two q.k columns
        float xs;    // qinv * scale2 of this lane's head
        {
            const int qh = lane < 16 ? h0 : h1, j = lane & 15;
            const float4* qp = (const float4*)(S.q_attn + (int64_t)s * D.dp + qh * 128 + j * 8);
            const float4 qa = qp[0], qb = qp[1];
            const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
            float mx = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) mx = fmaxf(mx, fabsf(qv[i]));
#pragma unroll
            for (int off = 1; off < 16; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, off));
            int ex = 0;
            if (mx > 0.f) frexpf(mx, &ex);
            const float qsc = ldexpf(1.f, 22 - ex);
            const float qinv = ldexpf(1.f, ex - 22);
            uint32_t dg[3][2] = {{0u, 0u}, {0u, 0u}, {0u, 0u}};
            int cs[3] = {0, 0, 0};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int v = __float2int_rn(qv[i] * qsc);
                const int d0 = ((v + 128) & 255) - 128;
                const int r1 = (v - d0) >> 8;
                const int d1 = ((r1 + 128) & 255) - 128;
                const int d2 = (r1 - d1) >> 8;
                cs[0] += d0, cs[1] += d1, cs[2] += d2;
                dg[0][i >> 2] |= (uint32_t)(d0 & 255) << (8 * (i & 3));
                dg[1][i >> 2] |= (uint32_t)(d1 & 255) << (8 * (i & 3));
                dg[2][i >> 2] |= (uint32_t)(d2 & 255) << (8 * (i & 3));
            }
#pragma unroll
            for (int off = 1; off < 16; off <<= 1)
#pragma unroll
                for (int p = 0; p < 3; ++p) cs[p] += __shfl_xor_sync(kFull, cs[p], off);
            __syncwarp();  // the previous item's reads of qw are done
#pragma unroll
            for (int p = 0; p < 3; ++p)
                *(uint2*)(qw + ((lane >> 4) * 3 + p) * kQPlane + 2 * j) =
                    make_uint2(__byte_perm(dg[p][0], dg[p][1], 0x6420), __byte_perm(dg[p][0], dg[p][1], 0x7531));
            __syncwarp();
            const int hsrc = t < 2 ? 0 : 16;
            const int c0 = __shfl_sync(kFull, cs[0], hsrc), c1 = __shfl_sync(kFull, cs[1], hsrc),
                      c2 = __shfl_sync(kFull, cs[2], hsrc);
            cA = 8 * (odd ? c2 : c0);
            cB = odd ? 0 : 8 * c1;
            xs = __shfl_sync(kFull, qinv, hsrc) * P.scale2;
        }
        // B fragments of the q.k MMAs: column g = digit plane g of head h0
        // (g < 3) or g - 4 of head h1 (4 <= g < 7); lane t reads the even / odd
        // digits of K words 4t..4t+3; inactive lanes read zeros
        const uint4* qf0 = g < 3 ? (const uint4*)(qw + g * kQPlane + 8 * t) : qzero;
        const uint4* qf1 = (g >= 4 && g < 7) ? (const uint4*)(qw + (3 + g - 4) * kQPlane + 8 * t) : qzero;
        float* scp = S.scores + (pos0 + 2 * g + odd) * H + hm;  // this lane's logit slot, stage 0

        float m = -INFINITY, l = 0.f, E = 1.f, invE = 1.f;
        bool have = false;
        int since = 0;  // entries in the current epoch (s32 headroom of the x16 tiles)
        unsigned long long wsum = 0ull;
        // p.v tiles: tile 4 wh + T rows g / g + 8 = d 64 wh + 8g + T / + 4;
        // odd T are high nibbles (x16)
        int acc[8][4];
        // o of head hm at d = 64 wh + 8g + T (+ 4 for t odd): the values this
        // lane writes at the end of the item
        float oF[8];
#pragma unroll
        for (int T = 0; T < 8; ++T) {
            acc[T][0] = acc[T][1] = acc[T][2] = acc[T][3] = 0;
            oF[T] = 0.f;
        }
        // fold the epoch's integer sums into oF: o = sum_p 256^p D_p (/16 for
        // high-nibble tiles) - 8 sum w, exact in fp64, scaled by the epoch's E
        auto fold = [&]() {
            unsigned long long W = wsum;
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) W += __shfl_xor_sync(kFull, W, off);
            const double fa = odd ? 65536.0 : 1.0, fb = odd ? 0.0 : 256.0;
            const double cw = odd ? 8.0 * (double)W : 0.0;
            const double Ed = (double)E;
#pragma unroll
            for (int T = 0; T < 8; ++T) {
                const double sc = (T & 1) ? 0.0625 : 1.0;
                const double v0 = ((double)acc[T][0] * fa + (double)acc[T][1] * fb) * sc - cw;
                const double v1 = ((double)acc[T][2] * fa + (double)acc[T][3] * fb) * sc - cw;
                // t even keeps row g, t odd row g + 8: swap halves, then add
                const double mine = odd ? v1 : v0, other = odd ? v0 : v1;
                oF[T] += (float)((mine + __shfl_xor_sync(kFull, other, 1)) * Ed);
                acc[T][0] = acc[T][1] = acc[T][2] = acc[T][3] = 0;
            }
            wsum = 0ull;
            since = 0;
        };
        const uint32_t c88 = P.c88, c0f = P.c0f;  // LOP3 operands (both masks in one op)

        // one pass per stage, plus a final pass (b >= cnt) that only folds: the
        // fold is inlined once
        for (int b = 0;; b += kEPS, scp += kEPS * H) {
            const bool fin = b >= cnt;
            const uint8_t* sb = stages + (size_t)stage * P.R.stage_bytes;
            float z0 = 0.f, z1 = 0.f, wf0 = 0.f, wf1 = 0.f;
            bool need = false;
            if (!fin) {
                const int n = min(kEPS, cnt - b);
                mbar_wait_sleep(&R.full[stage], phase);
                const uint8_t* r0 = sb + (size_t)(2 * g) * P.R.stride;  // entry 2g
                const uint8_t* r1 = r0 + P.R.stride;                    // entry 2g + 1
                // ---------------- q.k: 8 MMAs ----------------
                // per head: K words 4t..4t+3 of entries 2g, 2g+1; low nibbles (even
                // d) and high nibbles (odd d, x16) in separate MMAs and accumulators
                int dl[4] = {0, 0, 0, 0}, dh[4] = {0, 0, 0, 0};
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint4 f0 = (hh ? qf1 : qf0)[0], f1 = (hh ? qf1 : qf0)[1];
                    const uint4 ka = *(const uint4*)(r0 + (hh ? koff1 : koff0));
                    const uint4 kb = *(const uint4*)(r1 + (hh ? koff1 : koff0));
                    imma_u8s8(dl, nlo(ka.x, c88, c0f), nlo(kb.x, c88, c0f), nlo(ka.y, c88, c0f), nlo(kb.y, c88, c0f),
                              f0.x, f0.z);
                    imma_u8s8(dh, nhi(ka.x, c88, c0f), nhi(kb.x, c88, c0f), nhi(ka.y, c88, c0f), nhi(kb.y, c88, c0f),
                              f0.y, f0.w);
                    imma_u8s8(dl, nlo(ka.z, c88, c0f), nlo(kb.z, c88, c0f), nlo(ka.w, c88, c0f), nlo(kb.w, c88, c0f),
                              f1.x, f1.z);
                    imma_u8s8(dh, nhi(ka.z, c88, c0f), nhi(kb.z, c88, c0f), nhi(ka.w, c88, c0f), nhi(kb.w, c88, c0f),
                              f1.y, f1.w);
                }
                const float sk0 = *(const float*)(r0 + 2 * pay + 4 * hm), sk1 = *(const float*)(r1 + 2 * pay + 4 * hm);
                const float sv0 = *(const float*)(r0 + 2 * pay + 4 * (H + hm));
                const float sv1 = *(const float*)(r1 + 2 * pay + 4 * (H + hm));
                // column 2t (+ 2t + 1): planes 0, 1 (t even) or plane 2 (t odd) of head hm
                const float fa = odd ? 65536.f : 1.f, fb = odd ? 0.f : 256.f;
                float s0 = (float)(dl[0] + (dh[0] >> 4) - cA) * fa + (float)(dl[1] + (dh[1] >> 4) - cB) * fb;
                float s1 = (float)(dl[2] + (dh[2] >> 4) - cA) * fa + (float)(dl[3] + (dh[3] >> 4) - cB) * fb;
                s0 += __shfl_xor_sync(kFull, s0, 1);
                s1 += __shfl_xor_sync(kFull, s1, 1);
                const bool v0 = 2 * g < n, v1 = 2 * g + 1 < n;
                const float x0 = v0 ? s0 * xs * sk0 : -INFINITY;
                const float x1 = v1 ? s1 * xs * sk1 : -INFINITY;
                if (odd ? v1 : v0) *scp = odd ? x1 : x0;
                // ---------------- online softmax of head hm ----------------
                float mx = fmaxf(x0, x1);
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, off));
                if (mx > m) {
                    const float c = ex2a(m - mx);  // m = -inf -> 0
                    l *= c;
#pragma unroll
                    for (int T = 0; T < 8; ++T) oF[T] *= c;
                    E *= c;
                    invE = rcpa(E);
                    m = mx;
                }
                const float p0 = ex2a(x0 - m), p1 = ex2a(x1 - m);
                l += p0 + p1;
                z0 = v0 ? p0 * sv0 : 0.f, z1 = v1 ? p1 * sv1 : 0.f;
                wf0 = z0 * invE, wf1 = z1 * invE;
                since += kEPS;
                need = !have || !(wf0 < kLim) || !(wf1 < kLim) || since > kEpochMax;
            }
            if (__any_sync(kFull, fin || need)) {
                // fold the epoch; then (unless the item is done) a new epoch:
                // first stage, a weight outgrew the headroom, or the x16
                // accumulators near their s32 range
                if (have) fold();
                if (fin) break;
                since = kEPS;
                float zm = fmaxf(z0, z1);
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) zm = fmaxf(zm, __shfl_xor_sync(kFull, zm, off));
                int ez = 0;
                if (zm > 0.f) frexpf(zm, &ez);
                E = zm > 0.f ? ldexpf(1.f, ez - (24 - kTau)) : 1.f;
                invE = zm > 0.f ? ldexpf(1.f, (24 - kTau) - ez) : 1.f;
                have = true;
                wf0 = z0 * invE, wf1 = z1 * invE;
            }
            const uint32_t w0 = __float2uint_rn(wf0), w1 = __float2uint_rn(wf1);
            wsum += (unsigned long long)(w0 + w1);
            // ---------------- weight digits -> B fragment ----------------
            // k-slot 4t + i (head h0: slots 0-15, h1: 16-31) = entry t + 4i; the
            // weight of entry e, head hh lives in lane (e / 2) * 4 + e % 2 (+2 for h1)
            uint32_t pb0, pb1;
            {
                const uint32_t send = odd ? w1 : w0;
                const int hs = g >= 4 ? 2 : 0;
                uint32_t pv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) pv[i] = __shfl_sync(kFull, send, (((t >> 1) + 2 * i) << 2) + odd + hs);
                const uint32_t pb = (uint32_t)(g & 3);
                const uint32_t sel = pb | ((pb + 4) << 4);
                uint32_t pk = __byte_perm(__byte_perm(pv[0], pv[1], sel), __byte_perm(pv[2], pv[3], sel), 0x5410);
                if (pb == 3) pk = 0u;
                pb0 = g < 4 ? pk : 0u;
                pb1 = g < 4 ? 0u : pk;
            }
            // ---------------- p.v: 8 MMAs (16 d rows each, both heads) ----------------
            // lane (g, t) transposes V word g (wh = 0: d 8g..) and g + 8 (wh = 1:
            // d 64 + 8g..) of entries t + 4i for both heads: x[hh][k] = byte k of
            // the 4 entries (nibbles d 2k, 2k + 1 of the word)
#pragma unroll
            for (int wh = 0; wh < 2; ++wh) {
                uint32_t xr[2][4];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint8_t* vb = sb + (size_t)t * P.R.stride + pay + (hh ? h1 : h0) * 64 + 4 * (g + 8 * wh);
                    const uint32_t w_0 = *(const uint32_t*)(vb);
                    const uint32_t w_1 = *(const uint32_t*)(vb + 4 * P.R.stride);
                    const uint32_t w_2 = *(const uint32_t*)(vb + 8 * P.R.stride);
                    const uint32_t w_3 = *(const uint32_t*)(vb + 12 * P.R.stride);
                    const uint32_t u01l = __byte_perm(w_0, w_1, 0x5140), u01h = __byte_perm(w_0, w_1, 0x7362);
                    const uint32_t u23l = __byte_perm(w_2, w_3, 0x5140), u23h = __byte_perm(w_2, w_3, 0x7362);
                    xr[hh][0] = __byte_perm(u01l, u23l, 0x5410);
                    xr[hh][1] = __byte_perm(u01l, u23l, 0x7632);
                    xr[hh][2] = __byte_perm(u01h, u23h, 0x5410);
                    xr[hh][3] = __byte_perm(u01h, u23h, 0x7632);
                }
                // tile T: rows g = d 8g + T (byte T/2), g + 8 = d 8g + T + 4 (byte T/2 + 2)
                imma_u8u8(acc[4 * wh + 0], nlo(xr[0][0], c88, c0f), nlo(xr[0][2], c88, c0f), nlo(xr[1][0], c88, c0f),
                          nlo(xr[1][2], c88, c0f), pb0, pb1);
                imma_u8u8(acc[4 * wh + 1], nhi(xr[0][0], c88, c0f), nhi(xr[0][2], c88, c0f), nhi(xr[1][0], c88, c0f),
                          nhi(xr[1][2], c88, c0f), pb0, pb1);
                imma_u8u8(acc[4 * wh + 2], nlo(xr[0][1], c88, c0f), nlo(xr[0][3], c88, c0f), nlo(xr[1][1], c88, c0f),
                          nlo(xr[1][3], c88, c0f), pb0, pb1);
                imma_u8u8(acc[4 * wh + 3], nhi(xr[0][1], c88, c0f), nhi(xr[0][3], c88, c0f), nhi(xr[1][1], c88, c0f),
                          nhi(xr[1][3], c88, c0f), pb0, pb1);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&R.empty[stage]);
            if (++stage == P.R.NST) stage = 0, phase ^= 1;
        }
        // ---- the item's partial (m, l, o) of heads h0, h1 ----
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) l += __shfl_xor_sync(kFull, l, off);
        // tile 4 wh + T, T = 0..3: d 64 wh + 8g + T (+ 4 for t odd)
        float* po = S.part_o + ((int64_t)w * H + hm) * 128 + 8 * g + (odd ? 4 : 0);
        *(float4*)po = make_float4(oF[0], oF[1], oF[2], oF[3]);
        *(float4*)(po + 64) = make_float4(oF[4], oF[5], oF[6], oF[7]);
        if (g == 0 && !odd) {
            S.part_m[(int64_t)w * H + hm] = m;
            S.part_l[(int64_t)w * H + hm] = l;
        }
    }
}

}  // namespace

// The tensor-core int4 path: int4 codes, 128-dim heads, even H <= 32.
// PIKV_I4TC=0 selects the CUDA-core kernel (A/B builds of the bench).
bool attend_i4tc_applies(const Dims& D) {
    if (D.codec != PIKV_CODEC_INT4 || D.dph != 128 || D.H < 2 || D.H > 32 || (D.H & 1)) return false;
    const char* v = std::getenv("PIKV_I4TC");  // read at engine creation and graph capture
    return !(v && v[0] == '0');
}

static I4Params i4_params(const Dims& D, size_t* smem) {
    I4Params P{};
    P.R = ring_params(D, kEPS, kPad, q_area_bytes(D.H / 2));
    if (P.R.NST > 4) P.R.NST = 4;
    P.scale2 = 1.4426950408889634f / sqrtf(128.f);
    P.c88 = 0x88888888u;
    P.c0f = 0x0F0F0F0Fu;
    if (smem) *smem = 256 + (size_t)q_area_bytes(D.H / 2) + (size_t)P.R.NST * P.R.stage_bytes;
    return P;
}

int attend_i4tc_stages(const Dims& D) { return i4_params(D, nullptr).R.NST; }
int attend_i4tc_eps() { return kEPS; }

void launch_attend_i4tc(const Dims& D, const State& S, cudaStream_t st) {
    size_t smem = 0;
    const I4Params P = i4_params(D, &smem);
    cudaFuncSetAttribute(k_attend_i4tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(k_attend_i4tc, dim3(D.attend_ctas), dim3((D.H / 2 + P.R.nprod) * 32), smem, st, D, S, P);
}

}  // namespace pikv_dev
