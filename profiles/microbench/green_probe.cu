// Do green contexts partition the SMs for runtime-API kernels and graphs?
// Splits the device's SMs into a partition of `want` SMs and the rest, creates
// a stream in each, and records which SMs the CTAs of a runtime-API launch
// (direct and through a graph captured on the green stream) ran on.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a green_probe.cu -lcuda -o green_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <set>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        CUresult r_ = (x);                                                                 \
        if (r_ != CUDA_SUCCESS) {                                                          \
            const char* s_ = nullptr;                                                      \
            cuGetErrorString(r_, &s_);                                                     \
            printf("%s:%d %s -> %d %s\n", __FILE__, __LINE__, #x, (int)r_, s_ ? s_ : "?"); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)
#define RK(x)                                                                                          \
    do {                                                                                               \
        cudaError_t e_ = (x);                                                                          \
        if (e_ != cudaSuccess) {                                                                       \
            printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));                \
            return 1;                                                                                  \
        }                                                                                              \
    } while (0)

__global__ void k_smid(int* out, int spin) {
    int id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    if (threadIdx.x == 0) out[blockIdx.x] = id;
    long long t0 = clock64();
    while (clock64() - t0 < spin) {
    }
}

static int count_sms(const std::vector<int>& v, std::set<int>* out = nullptr) {
    std::set<int> s(v.begin(), v.end());
    if (out) *out = s;
    return (int)s.size();
}

int main(int argc, char** argv) {
    const int want = argc > 1 ? atoi(argv[1]) : 104;
    RK(cudaFree(0));  // primary context via the runtime
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", all.sm.smCount);
    CUdevResource part[1], rest;
    unsigned int ng = 1;
    CK(cuDevSmResourceSplitByCount(part, &ng, &all, &rest, 0, want));
    printf("partition: %u SMs, remaining %u SMs (groups %u)\n", part[0].sm.smCount, rest.sm.smCount, ng);
    CUdevResourceDesc da, db;
    CK(cuDevResourceGenerateDesc(&da, part, 1));
    CK(cuDevResourceGenerateDesc(&db, &rest, 1));
    CUgreenCtx ga, gb;
    CK(cuGreenCtxCreate(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sa, sb;
    CK(cuGreenCtxStreamCreate(&sa, ga, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&sb, gb, CU_STREAM_NON_BLOCKING, 0));
    const int n = 2048;
    int* d;
    RK(cudaMalloc(&d, n * sizeof(int)));  // primary-context allocation used by green streams
    std::vector<int> h(n);
    std::set<int> setA, setB;
    // 1) runtime launch into the green streams
    k_smid<<<n, 64, 0, (cudaStream_t)sa>>>(d, 20000);
    RK(cudaGetLastError());
    RK(cudaStreamSynchronize((cudaStream_t)sa));
    RK(cudaMemcpy(h.data(), d, n * sizeof(int), cudaMemcpyDeviceToHost));
    printf("runtime launch on partition A: %d distinct SMs\n", count_sms(h, &setA));
    k_smid<<<n, 64, 0, (cudaStream_t)sb>>>(d, 20000);
    RK(cudaGetLastError());
    RK(cudaStreamSynchronize((cudaStream_t)sb));
    RK(cudaMemcpy(h.data(), d, n * sizeof(int), cudaMemcpyDeviceToHost));
    printf("runtime launch on partition B: %d distinct SMs\n", count_sms(h, &setB));
    int overlap = 0;
    for (int x : setA) overlap += setB.count(x);
    printf("A/B overlap: %d SMs\n", overlap);
    // 2) graph captured on the green stream, launched on it
    cudaGraph_t g;
    cudaGraphExec_t ge;
    RK(cudaStreamBeginCapture((cudaStream_t)sa, cudaStreamCaptureModeThreadLocal));
    k_smid<<<n, 64, 0, (cudaStream_t)sa>>>(d, 20000);
    RK(cudaStreamEndCapture((cudaStream_t)sa, &g));
    RK(cudaGraphInstantiate(&ge, g, 0));
    RK(cudaGraphLaunch(ge, (cudaStream_t)sa));
    RK(cudaStreamSynchronize((cudaStream_t)sa));
    RK(cudaMemcpy(h.data(), d, n * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> setG;
    printf("graph captured on A, launched on A: %d distinct SMs\n", count_sms(h, &setG));
    // 3) graph captured on a plain runtime stream, launched on the green stream
    cudaStream_t plain;
    RK(cudaStreamCreateWithFlags(&plain, cudaStreamNonBlocking));
    cudaGraph_t g2;
    cudaGraphExec_t ge2;
    RK(cudaStreamBeginCapture(plain, cudaStreamCaptureModeThreadLocal));
    k_smid<<<n, 64, 0, plain>>>(d, 20000);
    RK(cudaStreamEndCapture(plain, &g2));
    RK(cudaGraphInstantiate(&ge2, g2, 0));
    RK(cudaGraphLaunch(ge2, (cudaStream_t)sa));
    RK(cudaStreamSynchronize((cudaStream_t)sa));
    RK(cudaMemcpy(h.data(), d, n * sizeof(int), cudaMemcpyDeviceToHost));
    printf("graph captured on a plain stream, launched on A: %d distinct SMs\n", count_sms(h));
    // 4) plain stream launch (primary context): all SMs?
    k_smid<<<n, 64, 0, plain>>>(d, 20000);
    RK(cudaStreamSynchronize(plain));
    RK(cudaMemcpy(h.data(), d, n * sizeof(int), cudaMemcpyDeviceToHost));
    printf("plain stream: %d distinct SMs\n", count_sms(h));
    // 5) events across partitions
    cudaEvent_t ev;
    RK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    RK(cudaEventRecord(ev, (cudaStream_t)sa));
    RK(cudaStreamWaitEvent((cudaStream_t)sb, ev, 0));
    RK(cudaStreamWaitEvent(plain, ev, 0));
    RK(cudaDeviceSynchronize());
    printf("events across partitions: ok\n");
    return 0;
}
