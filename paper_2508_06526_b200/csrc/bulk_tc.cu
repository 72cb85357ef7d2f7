// SPDX-License-Identifier: Apache-2.0
//
// The bulk low-rank projection of a prefill on the
// 5th-generation tensor cores:
//
//   proj[kv][t][h*r + j] = sum_i B[h][j][i] * (x[t][h*hd + i] - bias[h*hd + i])
//
// = per head a [T x hd] @ [hd x r] GEMM (compressor.cpp:318-329 for every
// row at once; LoRAPlus by linearity: x B^T - bias B^T).
//
// One CTA (4 warps) per (128-row tile, head, K|V): the A tile (token rows,
// K-major) and B (the head's basis rows, K-major) are staged in shared memory
// in the SWIZZLE_NONE canonical layout (8-row x 16-byte core matrices; LBO =
// next 16 bytes of K, SBO = next 8 rows); thread 0 issues the
// tcgen05.mma.cta_group::1.kind::f16 chain (M = 128, N = r padded to a
// multiple of 16, K = 16 per instruction) into a TMEM fp32 accumulator,
// commits to an mbarrier, and each warp reads its 32 accumulator rows back
// with tcgen05.ld.  fp32 operands are split into bf16 hi + lo, and the
// products hi*hi + hi*lo (+ lo*hi for fp32 inputs) keep ~2^-16 relative
// accuracy, i.e. fp32-level agreement with the CUDA-core projection.
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point; no -lcuda)
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>

#include "pikv_dev.cuh"

namespace pikv_dev {

namespace {

constexpr int kTcM = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, SWIZZLE_NONE K-major (CuTe SmemDescriptor:
// start [0,14), LBO [16,30), SBO [32,46), version 1 at [46,48), layout 0).
__device__ __forceinline__ uint64_t umma_desc(uint32_t start, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((start >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// Instruction descriptor: D f32, A/B bf16, both K-major, N, M = 128.
__device__ __forceinline__ uint32_t umma_idesc_bf16(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, int acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// byte offset of element (row, k) of a K-major tile with `kc` 16-byte chunks per row
__device__ __forceinline__ uint32_t core_off(int row, int k, int kc) {
    return (uint32_t)((row >> 3) * (kc * 128) + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint16_t bf16_rne(float f) { return f32_to_bf16_rne(f); }
__device__ __forceinline__ float bf16_val(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

template <int NP>
__device__ __forceinline__ void tmem_ld_rows(uint32_t taddr, float* out) {
    static_assert(NP == 16 || NP == 32 || NP == 64, "NP");
    uint32_t r[NP];
    if constexpr (NP == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else {
#pragma unroll
        for (int c = 0; c < NP; c += 16)
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                : "=r"(r[c + 0]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]),
                  "=r"(r[c + 6]), "=r"(r[c + 7]), "=r"(r[c + 8]), "=r"(r[c + 9]), "=r"(r[c + 10]), "=r"(r[c + 11]),
                  "=r"(r[c + 12]), "=r"(r[c + 13]), "=r"(r[c + 14]), "=r"(r[c + 15])
                : "r"(taddr + (uint32_t)c));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < NP; ++j) out[j] = __uint_as_float(r[j]);
}

// One accumulator row (r <= NP values) to global memory: 16-byte stores when
// the row is 16-byte aligned (r % 4 == 0), minus the LoRAPlus bias term.
template <int NP>
__device__ __forceinline__ void store_row(float* out, const float (&v)[NP], int r, const float* bias) {
    if ((r & 3) == 0 && (((uintptr_t)out) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < NP; j += 4) {
            if (j >= r) break;
            float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            if (bias) o.x -= bias[j], o.y -= bias[j + 1], o.z -= bias[j + 2], o.w -= bias[j + 3];
            *(float4*)(out + j) = o;
        }
    } else {
        for (int j = 0; j < r; ++j) out[j] = v[j] - (bias ? bias[j] : 0.f);
    }
}

template <int NP>
__global__ void __launch_bounds__(128) k_bulk_project_tc(Dims D, State S, int64_t T, const void* __restrict__ kin,
                                                         const void* __restrict__ vin, float* __restrict__ proj,
                                                         const float* __restrict__ bias_proj) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int hd = D.d / D.H, r = D.dph, kc = hd / 8;
    const int h = blockIdx.y, row = blockIdx.z, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t t0 = (int64_t)blockIdx.x * kTcM;
    const bool f32in = D.kv_dtype != PIKV_DTYPE_BF16;
    const uint32_t a_bytes = (uint32_t)kTcM * hd * 2, b_bytes = (uint32_t)NP * hd * 2;
    uint8_t* a_hi = sm;
    uint8_t* a_lo = a_hi + a_bytes;
    uint8_t* b_hi = a_lo + (f32in ? a_bytes : 0);
    uint8_t* b_lo = b_hi + b_bytes;
    uint64_t* mbar = (uint64_t*)(b_lo + b_bytes);
    uint32_t* tmem_slot = (uint32_t*)(mbar + 1);
    const void* x = row == 0 ? kin : vin;

    if (warp == 0) {  // TMEM accumulator: NP fp32 columns (power of two >= 32)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(NP < 32 ? 32 : NP));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // A: rows t0.. of head h (zero beyond T)
    for (int i = tid; i < kTcM * kc; i += blockDim.x) {
        const int rr = i / kc, c = i % kc;
        const int64_t t = t0 + rr;
        uint16_t hi[8], lo[8];
        if (t < T) {
            if (!f32in) {
                const uint4 w = *(const uint4*)((const uint16_t*)x + t * D.d + h * hd + c * 8);
                *(uint4*)hi = w;
            } else {
                const float* src = (const float*)x + t * D.d + h * hd + c * 8;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float f = src[u];
                    hi[u] = bf16_rne(f);
                    lo[u] = bf16_rne(f - bf16_val(hi[u]));
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) hi[u] = 0, lo[u] = 0;
        }
        *(uint4*)(a_hi + core_off(rr, c * 8, kc)) = *(uint4*)hi;
        if (f32in) *(uint4*)(a_lo + core_off(rr, c * 8, kc)) = *(uint4*)lo;
    }
    // B: the head's basis rows (fp32 -> bf16 hi + lo), zero rows r..NP
    for (int i = tid; i < NP * kc; i += blockDim.x) {
        const int j = i / kc, c = i % kc;
        uint16_t hi[8], lo[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float f = j < r ? S.basis[((int64_t)h * r + j) * hd + c * 8 + u] : 0.f;
            hi[u] = bf16_rne(f);
            lo[u] = bf16_rne(f - bf16_val(hi[u]));
        }
        *(uint4*)(b_hi + core_off(j, c * 8, kc)) = *(uint4*)hi;
        *(uint4*)(b_lo + core_off(j, c * 8, kc)) = *(uint4*)lo;
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (tid == 0) {
        const uint32_t idesc = umma_idesc_bf16(NP);
        const uint32_t lbo = 128, sbo_a = (uint32_t)kc * 128, sbo_b = (uint32_t)kc * 128;
        const uint32_t A[2] = {smem_u32(a_hi), smem_u32(a_lo)};
        const uint32_t B[2] = {smem_u32(b_hi), smem_u32(b_lo)};
        // products: hi*hi, hi*lo (+ lo*hi for fp32 inputs)
        const int np = f32in ? 3 : 2;
        const int pa[3] = {0, 0, 1}, pb[3] = {0, 1, 0};
        int acc = 0;
        for (int p = 0; p < np; ++p)
            for (int ks = 0; ks < hd / 16; ++ks) {
                umma_bf16(tmem, umma_desc(A[pa[p]] + ks * 256, lbo, sbo_a), umma_desc(B[pb[p]] + ks * 256, lbo, sbo_b),
                          idesc, acc);
                acc = 1;
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" ::"l"(
                         (uint64_t)__cvta_generic_to_shared(mbar))
                     : "memory");
    }
    mbar_wait(mbar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float accv[NP];
    tmem_ld_rows<NP>(tmem + ((uint32_t)(warp * 32) << 16), accv);
    const int64_t t = t0 + warp * 32 + lane;
    if (t < T) {
        float* out = proj + ((int64_t)row * T + t) * D.dp + h * r;
        store_row(out, accv, r, bias_proj ? bias_proj + h * r : nullptr);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(NP < 32 ? 32 : NP));
}

// bias B^T per head for LoRAPlus (fp32, i ascending)
__global__ void k_bias_proj(Dims D, State S, float* __restrict__ out) {
    const int hd = D.d / D.H, r = D.dph;
    for (int o = threadIdx.x + blockIdx.x * blockDim.x; o < D.H * r; o += blockDim.x * gridDim.x) {
        const int h = o / r, j = o % r;
        float acc = 0.f;
        for (int i = 0; i < hd; ++i) acc = fmaf(S.basis[((int64_t)h * r + j) * hd + i], S.cbias[h * hd + i], acc);
        out[o] = acc;
    }
}

// ---- pipelined variant -------------------------------------------------
// The basis of every head split once into bf16 hi / lo, already in the
// core-matrix layout: bhl[h][2][NP x hd].
template <int NP>
__global__ void k_basis_split(Dims D, State S, uint16_t* __restrict__ bhl) {
    const int hd = D.d / D.H, r = D.dph, kc = hd / 8;
    const int64_t per = (int64_t)NP * hd;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < (int64_t)D.H * per;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int h = (int)(o / per), rem = (int)(o % per), j = rem / hd, i = rem % hd;
        const float f = j < r ? S.basis[((int64_t)h * r + j) * hd + i] : 0.f;
        const uint16_t hi = bf16_rne(f), lo = bf16_rne(f - bf16_val(hi));
        const uint32_t off = core_off(j, i, kc) / 2;
        bhl[(int64_t)h * 2 * per + off] = hi;
        bhl[(int64_t)h * 2 * per + per + off] = lo;
    }
}

// Persistent CTA per (head, K|V) slice of the M tiles: B (hi, lo) staged
// once; A tiles double-buffered in shared memory with the next tile's
// global loads in flight (registers) while thread 0 issues this tile's MMAs
// into one of two TMEM accumulators and the warps drain the previous tile's
// accumulator (tcgen05.ld) to global memory.  bf16 inputs only (fp32 K/V
// keep the single-tile kernel).
template <int NP, int KC>
__global__ void __launch_bounds__(128) k_bulk_project_tc2(Dims D, int64_t T, const void* __restrict__ kin,
                                                          const void* __restrict__ vin,
                                                          const uint16_t* __restrict__ bhl,
                                                          float* __restrict__ proj,
                                                          const float* __restrict__ bias_proj) {
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr int HD = KC * 8;
    constexpr uint32_t A_BYTES = (uint32_t)kTcM * HD * 2, B_BYTES = (uint32_t)NP * HD * 2;
    constexpr int NACC = NP < 32 ? 32 : NP;  // TMEM columns per accumulator
    const int r = D.dph;
    const int h = blockIdx.y, row = blockIdx.z, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t* a_st[2] = {sm, sm + A_BYTES};
    uint8_t* b_hl = sm + 2 * A_BYTES;  // hi then lo
    uint64_t* mbar = (uint64_t*)(b_hl + 2 * B_BYTES);  // [2]
    uint32_t* tmem_slot = (uint32_t*)(mbar + 2);
    const uint16_t* x = (const uint16_t*)(row == 0 ? kin : vin);
    const int64_t ntiles = (T + kTcM - 1) / kTcM;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(2 * NACC));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {  // B: contiguous copy of the pre-split basis
        const uint4* src = (const uint4*)(bhl + (int64_t)h * 2 * NP * HD);
        for (int i = tid; i < (int)(2 * B_BYTES / 16); i += blockDim.x) ((uint4*)b_hl)[i] = src[i];
    }
    // A tile t -> registers: thread handles rows rr = tid / KC ... (KC chunks of 16 B per row)
    constexpr int PER = kTcM * KC / 128;  // 16-byte chunks per thread
    uint4 regs[PER];
    auto load_tile = [&](int64_t t) {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int i = tid + u * 128, rr = i / KC, c = i % KC;
            const int64_t g = t * kTcM + rr;
            regs[u] = g < T ? *(const uint4*)(x + g * D.d + h * HD + c * 8) : make_uint4(0, 0, 0, 0);
        }
    };
    auto store_tile = [&](uint8_t* dst) {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int i = tid + u * 128, rr = i / KC, c = i % KC;
            *(uint4*)(dst + core_off(rr, c * 8, KC)) = regs[u];
        }
    };
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = umma_idesc_bf16(NP);
    // epilogue: the warp's 32 accumulator rows -> smem (transpose) -> one
    // coalesced row per store instruction (lanes over the row's r values)
    float* tr = (float*)(tmem_slot + 4) + warp * 32 * (NP + 1);
    auto drain = [&](int pb, int64_t tile) {
        float accv[NP];
        tmem_ld_rows<NP>(tmem + (uint32_t)(pb * NACC) + ((uint32_t)(warp * 32) << 16), accv);
#pragma unroll
        for (int j = 0; j < NP; ++j) tr[lane * (NP + 1) + j] = accv[j];
        __syncwarp();
        const float bj = (bias_proj && lane < r) ? bias_proj[h * r + lane] : 0.f;
        for (int rr = 0; rr < 32; ++rr) {
            const int64_t g = tile * kTcM + warp * 32 + rr;
            if (g < T && lane < r)
                proj[((int64_t)row * T + g) * D.dp + h * r + lane] = tr[rr * (NP + 1) + lane] - bj;
        }
        if (NP > 32)  // r > 32: second half of the row
            for (int rr = 0; rr < 32; ++rr) {
                const int64_t g = tile * kTcM + warp * 32 + rr;
                const int c = 32 + lane;
                if (g < T && c < r)
                    proj[((int64_t)row * T + g) * D.dp + h * r + c] =
                        tr[rr * (NP + 1) + c] - (bias_proj ? bias_proj[h * r + c] : 0.f);
            }
        __syncwarp();
    };
    int64_t t = blockIdx.x;
    if (t < ntiles) load_tile(t);
    int it = 0;
    int64_t prev = -1;
    for (; t < ntiles; t += gridDim.x, ++it) {
        const int buf = it & 1;
        store_tile(a_st[buf]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (tid == 0) {
            const uint32_t A = smem_u32(a_st[buf]), Bh = smem_u32(b_hl), Bl = Bh + B_BYTES;
            const uint32_t acc = tmem + (uint32_t)(buf * NACC);
            const uint32_t sbo = KC * 128;
#pragma unroll
            for (int ks = 0; ks < KC / 2; ++ks)
                umma_bf16(acc, umma_desc(A + ks * 256, 128, sbo), umma_desc(Bh + ks * 256, 128, sbo), idesc, ks > 0);
#pragma unroll
            for (int ks = 0; ks < KC / 2; ++ks)
                umma_bf16(acc, umma_desc(A + ks * 256, 128, sbo), umma_desc(Bl + ks * 256, 128, sbo), idesc, 1);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" ::"l"(
                             (uint64_t)__cvta_generic_to_shared(&mbar[buf]))
                         : "memory");
        }
        // next tile's global loads fly while the MMAs run and the previous
        // accumulator drains
        if (t + gridDim.x < ntiles) load_tile(t + gridDim.x);
        if (prev >= 0) {
            const int pb = buf ^ 1;
            mbar_wait(&mbar[pb], (uint32_t)(((it - 1) >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            drain(pb, prev);
        }
        prev = t;
    }
    if (prev >= 0) {  // drain the last tile
        const int pb = (it - 1) & 1;
        mbar_wait(&mbar[pb], (uint32_t)(((it - 1) >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        drain(pb, prev);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(2 * NACC));
}

// ---- TMA-fed variant ----------------------------------------------------
// A tiles arrive by TMA (cp.async.bulk.tensor.2d, one elected thread) into a
// 2-stage ring in the SWIZZLE_128B K-major layout the UMMA descriptor reads
// directly (two 128-row x 64-column boxes per 128 x 128 tile, rows beyond T
// zero-filled by the TMA unit), so no thread touches the A bytes; B (basis
// hi / lo) stays in the SWIZZLE_NONE canonical layout (k_basis_split).  The
// MMA of tile i+1 and the TMA of tile i+2 run while the warps drain tile i's
// accumulator.  Persistent CTA per (head, K|V) slice of the tiles.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t start) {
    // start >> 4, LBO (unused for swizzled K-major) = 1, SBO = 1024 B (8 rows
    // x 128 B), version 1, layout SWIZZLE_128B (2) at bits [61, 64)
    return (uint64_t)((start >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n" ::"l"((uint64_t)map),
        "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// MODE 0: the epilogue stores the fp32 projections with thread stores; 1:
// through TMA (r == NP, a multiple of 32: each warp's 32 accumulator rows go
// to a SWIZZLE_128B smem box per 32 columns, one cp.async.bulk.tensor store
// each; rows beyond T are clipped by the unit); 2: fused with the bulk
// payload -- each row is rounded to bf16 and written straight into the KV
// pool entries of its token's experts (dst from the ring placement), so the
// fp32 projections never go to HBM
template <int NP, int MODE>
__global__ void __launch_bounds__(128) k_bulk_project_tc3(const __grid_constant__ CUtensorMap map_k,
                                                          const __grid_constant__ CUtensorMap map_v,
                                                          const __grid_constant__ CUtensorMap map_o, Dims D,
                                                          int64_t T, const uint16_t* __restrict__ bhl,
                                                          float* __restrict__ proj,
                                                          const float* __restrict__ bias_proj,
                                                          const int64_t* __restrict__ dst,
                                                          uint8_t* __restrict__ pool) {
    constexpr bool TST = MODE == 1;
    extern __shared__ __align__(1024) uint8_t sm3[];
    constexpr int HD = 128, KC = 16;
    constexpr uint32_t A_BYTES = (uint32_t)kTcM * HD * 2, B_BYTES = (uint32_t)NP * HD * 2;
    constexpr int NACC = NP < 32 ? 32 : NP;
    constexpr int NBOX = TST ? NP / 32 : 0;  // 32-column output boxes per warp
    const int r = D.dph;
    const int h = blockIdx.y, row = blockIdx.z, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // 1024-byte aligned stages (SWIZZLE_128B atoms)
    uint8_t* base = (uint8_t*)(((uintptr_t)sm3 + 1023) & ~(uintptr_t)1023);
    uint8_t* a_st[2] = {base, base + A_BYTES};
    uint8_t* b_hl = base + 2 * A_BYTES;
    uint8_t* obuf = b_hl + 2 * B_BYTES + (size_t)warp * NBOX * 4096;  // TST: this warp's boxes
    uint64_t* full = (uint64_t*)(b_hl + 2 * B_BYTES + 4 * NBOX * 4096);  // [2] TMA landed
    uint64_t* done = full + 2;                         // [2] MMAs of the stage finished
    uint32_t* tmem_slot = (uint32_t*)(done + 2);
    float* tr = (float*)(tmem_slot + 4) + warp * 32 * (NP + 1);
    const CUtensorMap* map = row == 0 ? &map_k : &map_v;
    const int64_t ntiles = (T + kTcM - 1) / kTcM;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(2 * NACC));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) mbar_init(&full[i], 1), mbar_init(&done[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
    }
    {
        const uint4* src = (const uint4*)(bhl + (int64_t)h * 2 * NP * HD);
        for (int i = tid; i < (int)(2 * B_BYTES / 16); i += blockDim.x) ((uint4*)b_hl)[i] = src[i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = umma_idesc_bf16(NP);
    auto issue_load = [&](int stg, int64_t tile) {  // thread 0
        mbar_expect_tx(&full[stg], A_BYTES);
        tma_load_2d(a_st[stg], map, h * HD, (int)(tile * kTcM), &full[stg]);
        tma_load_2d(a_st[stg] + A_BYTES / 2, map, h * HD + 64, (int)(tile * kTcM), &full[stg]);
    };
    auto drain = [&](int pb, int64_t tile) {
        float accv[NP];
        tmem_ld_rows<NP>(tmem + (uint32_t)(pb * NACC) + ((uint32_t)(warp * 32) << 16), accv);
        if constexpr (MODE == 2) {
            const int64_t g = tile * kTcM + warp * 32 + lane;  // this lane's token row
            if (g < T) {
                uint4 pk[NP / 8];
#pragma unroll
                for (int q = 0; q < NP / 8; ++q) {
                    uint32_t w[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int c = q * 8 + 2 * u;
                        const float a = accv[c] - (bias_proj ? bias_proj[h * NP + c] : 0.f);
                        const float b = accv[c + 1] - (bias_proj ? bias_proj[h * NP + c + 1] : 0.f);
                        w[u] = (uint32_t)f32_to_bf16_rne(a) | ((uint32_t)f32_to_bf16_rne(b) << 16);
                    }
                    pk[q] = make_uint4(w[0], w[1], w[2], w[3]);
                }
                for (int j = 0; j < D.k; ++j) {
                    const int64_t de = dst[g * D.k + j];
                    if (de < 0) continue;
                    uint4* o = (uint4*)(pool + de * (int64_t)D.entry_bytes + (int64_t)row * D.payload_bytes +
                                        (int64_t)h * NP * 2);
#pragma unroll
                    for (int q = 0; q < NP / 8; ++q) o[q] = pk[q];
                }
            }
        } else if constexpr (TST) {
            if (bias_proj) {
#pragma unroll
                for (int j = 0; j < NP; ++j) accv[j] -= bias_proj[h * NP + j];
            }
            // the previous tile's store must have read the boxes
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int bx = 0; bx < NBOX; ++bx)
#pragma unroll
                for (int c = 0; c < 8; ++c)  // row = lane: 16-byte chunk c at c ^ (row & 7)
                    *(float4*)(obuf + bx * 4096 + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                        make_float4(accv[bx * 32 + 4 * c], accv[bx * 32 + 4 * c + 1], accv[bx * 32 + 4 * c + 2],
                                    accv[bx * 32 + 4 * c + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int bx = 0; bx < NBOX; ++bx)
                    tma_store_3d(&map_o, obuf + bx * 4096, h * NP + bx * 32, (int)(tile * kTcM) + warp * 32, row);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else {
#pragma unroll
            for (int j = 0; j < NP; ++j) tr[lane * (NP + 1) + j] = accv[j];
            __syncwarp();
            for (int c = lane; c < r; c += 32) {
                const float bj = bias_proj ? bias_proj[h * r + c] : 0.f;
                for (int rr = 0; rr < 32; ++rr) {
                    const int64_t g = tile * kTcM + warp * 32 + rr;
                    if (g < T) proj[((int64_t)row * T + g) * D.dp + h * r + c] = tr[rr * (NP + 1) + c] - bj;
                }
            }
            __syncwarp();
        }
    };
    const int64_t t0 = blockIdx.x, step = gridDim.x;
    if (tid == 0) {
        if (t0 < ntiles) issue_load(0, t0);
        if (t0 + step < ntiles) issue_load(1, t0 + step);
    }
    int it = 0;
    int64_t prev = -1;
    for (int64_t t = t0; t < ntiles; t += step, ++it) {
        const int stg = it & 1;
        if (tid == 0) {
            mbar_wait(&full[stg], (uint32_t)((it >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t A = smem_u32(a_st[stg]), Bh = smem_u32(b_hl), Bl = Bh + B_BYTES;
            const uint32_t acc = tmem + (uint32_t)(stg * NACC);
            // K = 128 = two 64-column swizzle atoms (A + kb * 16 KB), 4 MMAs of
            // K = 16 (32 B) each; B canonical: 256 B per K = 16 step
#pragma unroll
            for (int hl = 0; hl < 2; ++hl)
#pragma unroll
                for (int ks = 0; ks < KC / 2; ++ks) {
                    const uint32_t a_addr = A + (uint32_t)(ks >> 2) * (A_BYTES / 2) + (uint32_t)(ks & 3) * 32;
                    umma_bf16(acc, umma_desc_sw128(a_addr), umma_desc((hl ? Bl : Bh) + ks * 256, 128, KC * 128),
                              idesc, (hl | ks) != 0);
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" ::"l"(
                             (uint64_t)__cvta_generic_to_shared(&done[stg]))
                         : "memory");
        }
        if (prev >= 0) {
            const int pb = stg ^ 1;
            mbar_wait(&done[pb], (uint32_t)(((it - 1) >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // stage pb is free (its MMAs finished): refill it with tile t + step
            if (tid == 0 && t + step < ntiles) issue_load(pb, t + step);
            drain(pb, prev);
        }
        prev = t;
    }
    if (prev >= 0) {
        const int pb = (it - 1) & 1;
        mbar_wait(&done[pb], (uint32_t)(((it - 1) >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        drain(pb, prev);
    }
    if (TST && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(2 * NACC));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}

// [T][d] bf16 rows, boxes of 128 rows x 64 columns (128 B), SWIZZLE_128B
bool make_kv_map(CUtensorMap* m, const void* x, int64_t T, int d) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn || ((uintptr_t)x & 15) || (d * 2) % 16) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)T};
    const cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)kTcM};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// proj [2][T][dp] fp32 as a 3-D map, boxes of 32 columns (128 B) x 32 rows x 1,
// SWIZZLE_128B (the epilogue's conflict-free box layout)
bool make_out_map(CUtensorMap* m, float* proj, int64_t T, int dp) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn || ((uintptr_t)proj & 15) || (dp * 4) % 16) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)dp, (cuuint64_t)T, 2};
    const cuuint64_t strides[2] = {(cuuint64_t)dp * 4, (cuuint64_t)T * dp * 4};
    const cuuint32_t box[3] = {32, 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, proj, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NP, int MODE>
int launch_tc3(const Dims& D, int64_t T, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mo,
               const uint16_t* bhl, float* proj, const float* bias_proj, cudaStream_t st,
               const int64_t* dst = nullptr, uint8_t* pool = nullptr) {
    constexpr bool TST = MODE == 1;
    const size_t smem = 1024 + 2 * (size_t)kTcM * 128 * 2 + 2 * (size_t)NP * 128 * 2 + 64 +
                        (TST ? (size_t)4 * (NP / 32) * 4096 : sizeof(float) * 4 * 32 * (NP + 1));
    cudaFuncSetAttribute(k_bulk_project_tc3<NP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t ntiles = (T + kTcM - 1) / kTcM;
    int sms = 148, smem_sm = 228 * 1024;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
    const int occ = std::max(1, std::min(4, smem_sm / (int)(smem + 1024)));  // CTAs per SM by shared memory
    // one wave: (head, K|V) pairs x slices <= resident CTAs
    int64_t per = (int64_t)occ * sms / (2LL * D.H);
    if (per > ntiles) per = ntiles;
    if (per < 1) per = 1;
    k_bulk_project_tc3<NP, MODE><<<dim3((unsigned)per, D.H, 2), 128, smem, st>>>(mk, mv, mo, D, T, bhl, proj,
                                                                                 bias_proj, dst, pool);
    return cudaGetLastError() == cudaSuccess ? (MODE == 2 ? 2 : 0) : 1;
}

template <int NP>
int launch_np(const Dims& D, const State& S, int64_t T, const void* k, const void* v, float* proj,
              const float* bias_proj, float* scratch_b, cudaStream_t st, const int64_t* fuse_dst) {
    const int hd = D.d / D.H;
    const bool f32in = D.kv_dtype != PIKV_DTYPE_BF16;
    const char* tv = std::getenv("PIKV_BULK_TMA");  // A/B: 0 = register-staged tc2
    CUtensorMap mk, mv;
    if (!f32in && hd == 128 && scratch_b && !(tv && tv[0] == '0') && make_kv_map(&mk, k, T, D.d) &&
        make_kv_map(&mv, v, T, D.d)) {
        uint16_t* bhl = (uint16_t*)scratch_b;
        k_basis_split<NP><<<64, 256, 0, st>>>(D, S, bhl);
        const char* ts = std::getenv("PIKV_BULK_TSTORE");  // A/B: 0 = thread stores
        CUtensorMap mo;
        if (fuse_dst && D.dph == NP && D.payload_bytes == D.dp * 2)  // fused payload (returns 2)
            return launch_tc3<NP, 2>(D, T, mk, mv, mk, bhl, proj, bias_proj, st, fuse_dst, S.pool);
        if constexpr (NP % 32 == 0) {
            if (D.dph == NP && !(ts && ts[0] == '0') && make_out_map(&mo, proj, T, D.dp))
                return launch_tc3<NP, 1>(D, T, mk, mv, mo, bhl, proj, bias_proj, st);
        }
        return launch_tc3<NP, 0>(D, T, mk, mv, mk, bhl, proj, bias_proj, st);
    }
    if (!f32in && hd == 128 && scratch_b) {  // pipelined persistent kernel
        uint16_t* bhl = (uint16_t*)scratch_b;
        k_basis_split<NP><<<64, 256, 0, st>>>(D, S, bhl);
        constexpr int KC = 16;
        const size_t smem = 2 * (size_t)kTcM * 128 * 2 + 2 * (size_t)NP * 128 * 2 + 64 +
                            sizeof(float) * 4 * 32 * (NP + 1);  // + epilogue transpose
        cudaFuncSetAttribute(k_bulk_project_tc2<NP, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t ntiles = (T + kTcM - 1) / kTcM;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        // ~2 CTAs per SM over all (head, K|V) pairs
        int64_t per = (2LL * sms + 2LL * D.H - 1) / (2LL * D.H);
        if (per > ntiles) per = ntiles;
        if (per < 1) per = 1;
        k_bulk_project_tc2<NP, KC><<<dim3((unsigned)per, D.H, 2), 128, smem, st>>>(D, T, k, v, bhl, proj,
                                                                                    bias_proj);
        return cudaGetLastError() == cudaSuccess ? 0 : 1;
    }
    const size_t smem = (size_t)kTcM * hd * 2 * (f32in ? 2 : 1) + (size_t)NP * hd * 2 * 2 + 16 + 16;
    if (smem > 200 * 1024) return 1;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_bulk_project_tc<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const dim3 grid((unsigned)((T + kTcM - 1) / kTcM), D.H, 2);
    k_bulk_project_tc<NP><<<grid, 128, smem, st>>>(D, S, T, k, v, proj, bias_proj);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace

int launch_bulk_project_tc(const Dims& D, const State& S, int64_t T, const void* k, const void* v, float* proj,
                           float* bias_scratch, cudaStream_t st, const int64_t* fuse_dst) {
    const int hd = D.d / D.H, r = D.dph;
    if (hd % 16 != 0 || r < 1 || r > 64 || T <= 0) return 1;
    // scratch: [H][r] bias B^T, then the pre-split basis (H x 2 x NP x hd bf16)
    float* bias_proj = nullptr;
    if (D.codec == PIKV_CODEC_LORAPLUS) {
        bias_proj = bias_scratch;
        k_bias_proj<<<1, 256, 0, st>>>(D, S, bias_proj);
    }
    float* bsplit = bias_scratch + ((D.H * r + 63) & ~63);
    int rc;
    if (r <= 16) rc = launch_np<16>(D, S, T, k, v, proj, bias_proj, bsplit, st, fuse_dst);
    else if (r <= 32) rc = launch_np<32>(D, S, T, k, v, proj, bias_proj, bsplit, st, fuse_dst);
    else rc = launch_np<64>(D, S, T, k, v, proj, bias_proj, bsplit, st, fuse_dst);
    return rc;
}

}  // namespace pikv_dev
