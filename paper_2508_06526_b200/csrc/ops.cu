// SPDX-License-Identifier: Apache-2.0
//
// Standalone device kernels behind the C-ABI's pure functions: the
// reference's free functions (shard_assign, select_evictions, attention,
// project_encode/decode) and this engine's int8/int4 quantizer, each run on
// the GPU over caller device arrays.
#include <cuda_runtime.h>

#include "pikv_dev.cuh"

namespace pikv_dev {

// shard_assign, kvstore.cpp:14-30
__global__ void k_shard_assign(const int64_t* t, const int32_t* e, int32_t n, int32_t n_tok,
                               int32_t n_exp, int32_t devices, int32_t additive, int32_t* dev,
                               int32_t* shard, int32_t* raw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = shard_raw(t[i], e[i], n_tok, n_exp, additive);
    if (raw) raw[i] = r;
    if (dev) dev[i] = r % devices;
    if (shard) shard[i] = r / devices;
}

// select_evictions, scheduler.cpp:231-260.  Rank sort: each page's position
// in the (aggregate asc, oldest_id asc) order is the number of pages before
// it; strict total order when oldest ids are distinct, index order otherwise
// (std::sort is then unspecified; ties on both keys do not occur in evict()).
__global__ void k_select(const double* agg, const uint64_t* oldest, int32_t n, int32_t budget,
                         int32_t use_theta, double theta, int32_t* idx_out, int32_t* reason_out,
                         int32_t* n_out) {
    __shared__ int sm_T;
    if (threadIdx.x == 0) sm_T = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (use_theta && agg[i] < theta) atomicAdd(&sm_T, 1);
    __syncthreads();
    const int T = sm_T;
    const int V = max(T, max(n - budget, 0));
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const bool less = agg[j] != agg[i] ? agg[j] < agg[i]
                              : oldest[j] != oldest[i] ? oldest[j] < oldest[i] : j < i;
            rank += less;
        }
        if (rank < V) {
            idx_out[rank] = i;
            reason_out[rank] = rank < T ? PIKV_EVICT_THRESHOLD : PIKV_EVICT_BUDGET;
        }
    }
    if (threadIdx.x == 0) *n_out = V;
}

// attention, pipeline.cpp:59-85: one CTA per query, fp32.
__global__ void k_attention(const float* q, const float* keys, const float* values, int32_t n,
                            int32_t w, float* y, float* weights) {
    extern __shared__ float sm[];  // [n] scores
    __shared__ float red[32];
    const int b = blockIdx.x, tid = threadIdx.x;
    const float* qb = q + (int64_t)b * w;
    const float* kb = keys + (int64_t)b * n * w;
    const float* vb = values + (int64_t)b * n * w;
    const float scale = 1.0f / sqrtf((float)w);
    for (int i = tid; i < n; i += blockDim.x) {
        float acc = 0.f;
        for (int j = 0; j < w; ++j) acc = fmaf(qb[j], kb[(int64_t)i * w + j], acc);
        sm[i] = acc * scale;
    }
    __syncthreads();
    float mx = -INFINITY;
    for (int i = tid; i < n; i += blockDim.x) mx = fmaxf(mx, sm[i]);
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    if (tid < 32) {
        float v = tid < (int)(blockDim.x >> 5) ? red[tid] : -INFINITY;
        for (int off = 16; off; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (tid == 0) red[0] = v;
    }
    __syncthreads();
    mx = red[0];
    __syncthreads();
    float tot = 0.f;
    for (int i = tid; i < n; i += blockDim.x) {
        const float e = expf(sm[i] - mx);
        sm[i] = e;
        tot += e;
    }
    for (int off = 16; off; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
    if ((tid & 31) == 0) red[tid >> 5] = tot;
    __syncthreads();
    if (tid < 32) {
        float v = tid < (int)(blockDim.x >> 5) ? red[tid] : 0.f;
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (tid == 0) red[0] = v;
    }
    __syncthreads();
    tot = red[0];
    for (int i = tid; i < n; i += blockDim.x) {
        sm[i] /= tot;
        if (weights) weights[(int64_t)b * n + i] = sm[i];
    }
    __syncthreads();
    for (int j = tid; j < w; j += blockDim.x) {
        float acc = 0.f;
        for (int i = 0; i < n; ++i) acc = fmaf(sm[i], vb[(int64_t)i * w + j], acc);
        y[(int64_t)b * w + j] = acc;
    }
}

// quantizer: one warp per row (oracle: po_quantize_row)
__global__ void k_quantize(const void* x, int32_t dtype, int32_t rows, int32_t width,
                           int32_t bits, uint8_t* codes, float* scales) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    auto ld = [&](int i) -> float {
        const int64_t gi = (int64_t)row * width + i;
        if (dtype == PIKV_DTYPE_BF16) return __uint_as_float(((uint32_t)((const uint16_t*)x)[gi]) << 16);
        return ((const float*)x)[gi];
    };
    const float qmax = bits == 8 ? 127.0f : 7.0f;
    float amax = 0.f;
    for (int i = lane; i < width; i += 32) amax = fmaxf(amax, fabsf(ld(i)));
    for (int off = 16; off; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    float inv = 0.f, scale = 0.f;
    if (amax > 0.f) {
        scale = __fdiv_rn(amax, qmax);
        inv = __fdiv_rn(qmax, amax);
    }
    if (lane == 0) scales[row] = scale;
    if (bits == 8) {
        for (int i = lane; i < width; i += 32) {
            float c = fminf(fmaxf(rintf(__fmul_rn(ld(i), inv)), -qmax), qmax);
            codes[(int64_t)row * width + i] = (uint8_t)(int8_t)(int)c;
        }
    } else {
        for (int i2 = lane; i2 < width / 2; i2 += 32) {
            float c0 = fminf(fmaxf(rintf(__fmul_rn(ld(2 * i2), inv)), -qmax), qmax);
            float c1 = fminf(fmaxf(rintf(__fmul_rn(ld(2 * i2 + 1), inv)), -qmax), qmax);
            codes[(int64_t)row * (width / 2) + i2] = (uint8_t)(((int)c0 & 0xF) | (((int)c1 & 0xF) << 4));
        }
    }
}

__global__ void k_dequantize(const uint8_t* codes, const float* scales, int32_t rows,
                             int32_t width, int32_t bits, float* x) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)rows * width) return;
    const int64_t row = i / width, col = i % width;
    int c;
    if (bits == 8) {
        c = (int)(int8_t)codes[i];
    } else {
        const int nib = (codes[row * (width / 2) + col / 2] >> ((col & 1) * 4)) & 0xF;
        c = nib >= 8 ? nib - 16 : nib;
    }
    x[i] = __fmul_rn((float)c, scales[row]);
}

// project_encode / project_decode per head (compressor.cpp:318-340)
__global__ void k_lr_encode(const float* x, const float* basis, const float* bias, int32_t rows,
                            int32_t H, int32_t hd, int32_t r, float* y) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)rows * H * r) return;
    const int64_t row = t / (H * r);
    const int h = (int)((t / r) % H), j = (int)(t % r);
    const float* col = basis + ((int64_t)h * r + j) * hd;
    const float* xr = x + row * (int64_t)H * hd + h * hd;
    float acc = 0.f;
    for (int i = 0; i < hd; ++i) acc = fmaf(col[i], bias ? xr[i] - bias[h * hd + i] : xr[i], acc);
    y[t] = acc;
}

__global__ void k_lr_decode(const float* y, const float* basis, const float* bias, int32_t rows,
                            int32_t H, int32_t hd, int32_t r, float* x) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)rows * H * hd) return;
    const int64_t row = t / (H * hd);
    const int h = (int)((t / hd) % H), i = (int)(t % hd);
    const float* yr = y + row * (int64_t)H * r + h * r;
    float acc = 0.f;
    for (int j = 0; j < r; ++j) acc = fmaf(basis[((int64_t)h * r + j) * hd + i], yr[j], acc);
    x[t] = bias ? acc + bias[h * hd + i] : acc;
}

}  // namespace pikv_dev
