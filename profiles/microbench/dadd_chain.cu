// Dependent fp64 add latency on the GPU (floor of the router's exact
// sequential dot, router.cpp:229-231).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, const double* in, int n, long long* cyc) {
    double a = in[0], b = in[1];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
    long long t1 = clock64();
    out[0] = a;
    cyc[0] = t1 - t0;
}
__global__ void chain_lds(double* out, int n, long long* cyc) {
    __shared__ double buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 1e-3 * i;
    __syncthreads();
    if (threadIdx.x) return;
    double a = 0.0;
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, buf[i & 4095]);
    long long t1 = clock64();
    out[0] = a;
    cyc[0] = t1 - t0;
}
int main() {
    double *d_out, *d_in;
    long long* d_c;
    cudaMalloc(&d_out, 8); cudaMalloc(&d_in, 16); cudaMalloc(&d_c, 8);
    double h_in[2] = {1.0, 1e-9};
    cudaMemcpy(d_in, h_in, 16, cudaMemcpyHostToDevice);
    long long c;
    chain<<<1, 1>>>(d_out, d_in, 4096, d_c);
    chain<<<1, 1>>>(d_out, d_in, 4096, d_c);
    cudaMemcpy(&c, d_c, 8, cudaMemcpyDeviceToHost);
    printf("register DADD chain: %.2f cycles/add\n", c / 4096.0);
    chain_lds<<<1, 256>>>(d_out, 4096, d_c);
    chain_lds<<<1, 256>>>(d_out, 4096, d_c);
    cudaMemcpy(&c, d_c, 8, cudaMemcpyDeviceToHost);
    printf("smem-operand DADD chain: %.2f cycles/add\n", c / 4096.0);
    return 0;
}
