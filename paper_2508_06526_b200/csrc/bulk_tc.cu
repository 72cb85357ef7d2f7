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
#include <cuda_runtime.h>

#include <cstdlib>

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
        for (int j = 0; j < r; ++j) out[j] = accv[j] - (bias_proj ? bias_proj[h * r + j] : 0.f);
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

template <int NP>
int launch_np(const Dims& D, const State& S, int64_t T, const void* k, const void* v, float* proj,
              const float* bias_proj, cudaStream_t st) {
    const int hd = D.d / D.H;
    const bool f32in = D.kv_dtype != PIKV_DTYPE_BF16;
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
                           float* bias_scratch, cudaStream_t st) {
    const int hd = D.d / D.H, r = D.dph;
    if (hd % 16 != 0 || r < 1 || r > 64 || T <= 0) return 1;
    // LoRAPlus: bias B^T [H][r] in the caller's scratch
    float* bias_proj = nullptr;
    if (D.codec == PIKV_CODEC_LORAPLUS) {
        bias_proj = bias_scratch;
        k_bias_proj<<<1, 256, 0, st>>>(D, S, bias_proj);
    }
    int rc;
    if (r <= 16) rc = launch_np<16>(D, S, T, k, v, proj, bias_proj, st);
    else if (r <= 32) rc = launch_np<32>(D, S, T, k, v, proj, bias_proj, st);
    else rc = launch_np<64>(D, S, T, k, v, proj, bias_proj, st);
    return rc;
}

}  // namespace pikv_dev
