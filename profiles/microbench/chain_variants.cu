// Formulations of the router's exact sequential fp64 dot (router.cpp:229-231)
// on one warp (16 lanes = 16 experts), operands in shared memory.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int D = 4096, DR = 512, E = 16, LD = DR + 2;  // rows reused 8x
__global__ void k(int variant, double* out, long long* cyc) {
    extern __shared__ double sm[];
    double* W = sm;              // [E][LD]
    double* P = sm + E * LD;     // [E][LD] precomputed products
    double* q = P + E * LD;      // [D]
    for (int i = threadIdx.x; i < E * LD; i += blockDim.x) { W[i] = 1e-3 * (i % 97); P[i] = 1e-4 * (i % 89); }
    for (int i = threadIdx.x; i < DR; i += blockDim.x) q[i] = 0.5 + 1e-5 * i;
    __syncthreads();
    if (threadIdx.x >= E) return;
    const int e = threadIdx.x;
    const double* w = W + e * LD;
    const double* p = P + e * LD;
    double acc = 0.0;
    long long t0 = clock64();
    if (variant == 1) {
#pragma unroll 8
        for (int i = 0; i < D; ++i) acc = __dadd_rn(acc, p[i & (DR - 1)]);
    } else if (variant == 2) {
#pragma unroll 4
        for (int i = 0; i < D; i += 2) {
            double2 v = *(const double2*)(p + (i & (DR - 1)));
            acc = __dadd_rn(acc, v.x);
            acc = __dadd_rn(acc, v.y);
        }
    } else if (variant == 3) {
#pragma unroll 8
        for (int i = 0; i < D; ++i) acc = __dadd_rn(acc, __dmul_rn(w[i & (DR - 1)], q[i & (DR - 1)]));
    } else if (variant == 4) {
        // products of 32 elements into registers via LDS.128, then the chain
        for (int i0 = 0; i0 < D; i0 += 32) {
            double r[32];
#pragma unroll
            for (int u = 0; u < 32; u += 2) {
                double2 a = *(const double2*)(w + ((i0 + u) & (DR - 1)));
                double2 b = *(const double2*)(q + ((i0 + u) & (DR - 1)));
                r[u] = __dmul_rn(a.x, b.x);
                r[u + 1] = __dmul_rn(a.y, b.y);
            }
#pragma unroll
            for (int u = 0; u < 32; ++u) acc = __dadd_rn(acc, r[u]);
        }
    } else if (variant == 5) {
        // double-buffered register batches: batch b+1's loads/muls are
        // independent of batch b's chain
        double ra[16], rb[16];
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
            double2 a = *(const double2*)(w + u), b = *(const double2*)(q + u);
            ra[u] = __dmul_rn(a.x, b.x); ra[u + 1] = __dmul_rn(a.y, b.y);
        }
        for (int i0 = 0; i0 < D; i0 += 32) {
#pragma unroll
            for (int u = 0; u < 16; u += 2) {
                double2 a = *(const double2*)(w + ((i0 + 16 + u) & (DR - 1))), b = *(const double2*)(q + ((i0 + 16 + u) & (DR - 1)));
                rb[u] = __dmul_rn(a.x, b.x); rb[u + 1] = __dmul_rn(a.y, b.y);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, ra[u]);
            if (i0 + 32 < D) {
#pragma unroll
                for (int u = 0; u < 16; u += 2) {
                    double2 a = *(const double2*)(w + ((i0 + 32 + u) & (DR - 1))), b = *(const double2*)(q + ((i0 + 32 + u) & (DR - 1)));
                    ra[u] = __dmul_rn(a.x, b.x); ra[u + 1] = __dmul_rn(a.y, b.y);
                }
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, rb[u]);
        }
    } else if (variant == 6) {
        // precomputed products (smem), batches of 32 in registers; the next
        // batch's LDS.128 interleaved between the current batch's DADDs
        double cur[32], nxt[32];
#pragma unroll
        for (int u = 0; u < 32; u += 2) {
            double2 v = *(const double2*)(p + u);
            cur[u] = v.x; cur[u + 1] = v.y;
        }
        for (int i0 = 0; i0 < D; i0 += 32) {
            const int nb = (i0 + 32) & (DR - 1);
#pragma unroll
            for (int u = 0; u < 32; u += 2) {
                acc = __dadd_rn(acc, cur[u]);
                double2 v = *(const double2*)(p + nb + u);
                acc = __dadd_rn(acc, cur[u + 1]);
                nxt[u] = v.x; nxt[u + 1] = v.y;
            }
#pragma unroll
            for (int u = 0; u < 32; ++u) cur[u] = nxt[u];
        }
    } else if (variant == 7) {
        // LDS + DMUL of the next batch interleaved between the current DADDs
        double cur[32], nxt[32];
#pragma unroll
        for (int u = 0; u < 32; u += 2) {
            double2 a = *(const double2*)(w + u), b = *(const double2*)(q + u);
            cur[u] = __dmul_rn(a.x, b.x); cur[u + 1] = __dmul_rn(a.y, b.y);
        }
        for (int i0 = 0; i0 < D; i0 += 32) {
            const int nb = (i0 + 32) & (DR - 1);
#pragma unroll
            for (int u = 0; u < 32; u += 2) {
                double2 a = *(const double2*)(w + nb + u), b = *(const double2*)(q + nb + u);
                acc = __dadd_rn(acc, cur[u]);
                nxt[u] = __dmul_rn(a.x, b.x);
                acc = __dadd_rn(acc, cur[u + 1]);
                nxt[u + 1] = __dmul_rn(a.y, b.y);
            }
#pragma unroll
            for (int u = 0; u < 32; ++u) cur[u] = nxt[u];
        }
    }
    long long t1 = clock64();
    out[e] = acc;
    if (e == 0) cyc[variant] = t1 - t0;
}
int main() {
    double* d_out; long long* d_c;
    cudaMalloc(&d_out, 8 * E); cudaMalloc(&d_c, 8 * 8);
    size_t smem = sizeof(double) * (2 * E * LD + DR);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int v = 1; v <= 7; ++v) {
        k<<<1, 32, smem>>>(v, d_out, d_c);
        k<<<1, 32, smem>>>(v, d_out, d_c);
        long long c[8];
        cudaMemcpy(c, d_c, sizeof(c), cudaMemcpyDeviceToHost);
        printf("variant %d: %.2f cycles/element (%s)\n", v, c[v] / (double)D, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
