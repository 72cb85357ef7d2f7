// SPDX-License-Identifier: Apache-2.0
//
// The TMA ring shared by the tensor-core attention kernels (attend_i4tc.cu,
// attend_bf16tc.cu): one CTA per SM, `ncw` consumer warps + one or two
// producer warps.  The producers take work items (stream, run of retrieved
// entries) -- the CTA's static share, or from the global ticket -- hand each
// to the consumers through a small smem queue, and stream the items' entries
// into an NST-stage ring of kRingEPS entries per stage (one cp.async.bulk per
// entry, slot stride padded for the consumers' bank pattern; full/empty
// mbarriers).  Same protocol as k_attend
// (attend.cu), which keeps its own copy for its 2-CTA geometry.
#pragma once

#include <cstdlib>

#include "pikv_dev.cuh"

namespace pikv_dev {

constexpr int kRingEPS = 16;  // max entries per stage: the MMA's 16 rows / k-slots
constexpr int kRingNQ = 4;    // work-item queue depth
constexpr int kRingMaxStages = 8;

struct RingParams {
    int NST;          // ring stages (<= kRingMaxStages)
    int eps;          // entries per stage (<= kRingEPS)
    int stride;       // smem bytes per entry slot (entry_bytes + pad)
    int stage_bytes;  // eps * stride
    int dyn;          // work items from the global ticket (1) or strided by CTA (0)
    int nprod;        // producer warps (ring_produce)
};

// smem header: barriers and the item queue (256 B at the start of the
// dynamic shared memory)
struct RingSmem {
    uint64_t* full;    // [8]
    uint64_t* empty;   // [8]
    uint64_t* ifull;   // [4]
    uint64_t* iempty;  // [4]
    int* iq;           // [4]
};

__device__ __forceinline__ RingSmem ring_smem(uint8_t* smem) {
    uint64_t* b = (uint64_t*)smem;
    return RingSmem{b, b + 8, b + 16, b + 20, (int*)(b + 24)};
}

__device__ __forceinline__ void ring_init(const RingSmem& R, const RingParams& P, int ncw) {
    for (int i = 0; i < P.NST; ++i) {
        mbar_init(&R.full[i], 1);
        mbar_init(&R.empty[i], ncw);
    }
    for (int i = 0; i < kRingNQ; ++i) {
        mbar_init(&R.ifull[i], 1);
        mbar_init(&R.iempty[i], ncw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// The producer warp's whole life: items until the ticket runs out, then the
// sentinel item (w >= n_items) that ends the consumers.
// With static work shares (D.att_share) nprod producer warps split the stages
// (producer `me` fills stages k = me mod nprod) and producer 0 alone publishes
// the items: one warp's wait-expect-issue loop per stage limited a one-CTA ring
// of 16-entry stages to ~6.1-6.6 TB/s (profiles/microbench/ring_sweep.cu).
__device__ __forceinline__ void ring_produce(const Dims& D, const State& S, const RingParams& P, const RingSmem& R,
                                             uint8_t* stages, int n_items, int lane, int me = 0, int nprod = 1) {
    constexpr unsigned kAll = 0xffffffffu;
    const int eb = D.entry_bytes;
    const uint64_t pol = evict_first_policy();
    int stage = 0, ks = 0;
    uint32_t phase = 0;
    auto item_of = [&](int w, int64_t& pos, int& cnt) {
        if (w < n_items) {
            pos = (int64_t)S.item_stream[w] * D.att_stride + S.item_begin[w];
            cnt = S.item_end[w] - S.item_begin[w];
        } else {
            pos = 0, cnt = 0;
        }
    };
    auto next_item = [&](int prev) -> int {
        if (D.att_share) {  // equal static shares: this CTA's items, then the sentinel
            const int w = prev < 0 ? S.cta_first[blockIdx.x] : prev + 1;
            return w < S.cta_first[blockIdx.x + 1] ? w : n_items;
        }
        if (!P.dyn) return prev < 0 ? (int)blockIdx.x : prev + (int)gridDim.x;
        int w = 0;
        if (lane == 0) w = atomicAdd(&S.n_items[1], 1);
        return __shfl_sync(kAll, w, 0);
    };
    int kq = 0;
    auto publish = [&](int w) {
        if (lane == 0 && me == 0) {
            mbar_wait_sleep(&R.iempty[kq % kRingNQ], ((kq / kRingNQ) & 1) ^ 1);
            *(volatile int*)&R.iq[kq % kRingNQ] = w;
            mbar_arrive(&R.ifull[kq % kRingNQ]);
        }
        ++kq;
    };
    // the pool indices of an item's entries are read a 32-entry window ahead
    // (one coalesced load per window); the next item's first window during
    // the current item
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
        for (int b = 0; b < cnt; b += P.eps) {
            const int n = min(P.eps, cnt - b);
            while (b >= win + 32) win += 32, cur = nxt, nxt = win_load(win + 32);
            const int o = b - win + lane;
            const int32_t e_cur = __shfl_sync(kAll, cur, o & 31);
            const int32_t e_nxt = __shfl_sync(kAll, nxt, o & 31);
            const int64_t ent = o < 32 ? e_cur : e_nxt;
            if (ks++ % nprod == me) {
                if (lane == 0) {
                    mbar_wait_sleep(&R.empty[stage], phase ^ 1);
                    mbar_expect_tx(&R.full[stage], (uint32_t)(n * eb));
                }
                __syncwarp();
                if (lane < n)
                    bulk_g2s(stages + (size_t)stage * P.stage_bytes + (size_t)lane * P.stride,
                             S.pool + ent * (int64_t)eb, (uint32_t)eb, &R.full[stage], pol);
            }
            if (++stage == P.NST) stage = 0, phase ^= 1;
        }
        w = wn;
    }
}

// Consumer side of the item queue: the next item index (>= n_items: done).
__device__ __forceinline__ int ring_next_item(const RingSmem& R, int kq, int lane) {
    mbar_wait_sleep(&R.ifull[kq % kRingNQ], (kq / kRingNQ) & 1);
    const int w = *(volatile int*)&R.iq[kq % kRingNQ];
    __syncwarp();
    if (lane == 0) mbar_arrive(&R.iempty[kq % kRingNQ]);
    return w;
}

// Ring geometry for an entry size, entries per stage, a slot pad and the smem
// left after a kernel-specific area of `extra` bytes (after the 256-B header).
inline RingParams ring_params(const Dims& D, int eps, int pad, int extra) {
    RingParams P{};
    P.eps = eps;
    P.stride = D.entry_bytes + pad;
    P.stage_bytes = eps * P.stride;
    const int budget = 227 * 1024 - 256 - extra;
    const int nst = budget / P.stage_bytes;
    P.NST = nst > kRingMaxStages ? kRingMaxStages : nst;
    const char* st = std::getenv("PIKV_ATT_STATIC");  // A/B experiments only
    P.dyn = st && st[0] == '1' ? 0 : 1;
    // two producer warps when the work items are static shares (both walk the
    // same items), one with ticketed items; PIKV_RING_PROD=1..3 (A/B)
    const char* rp = std::getenv("PIKV_RING_PROD");
    P.nprod = D.att_share ? (rp && rp[0] >= '1' && rp[0] <= '3' ? rp[0] - '0' : 2) : 1;
    return P;
}

}  // namespace pikv_dev
