// Probe: CDP2 tail-launch scheduler loop, stream ordering, graph capture (tools only).
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned int g_log[4096];
__device__ unsigned int g_n;
__global__ void k_work(int level, int* data, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) data[i] += 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) { unsigned p = atomicAdd(&g_n, 1); if (p < 4096) g_log[p] = level; }
}
__global__ void k_ff(int level, int* data, int n) {
    if (threadIdx.x == 0) { unsigned p = atomicAdd(&g_n, 1); if (p < 4096) g_log[p] = 1000 + level; }
}
__global__ void k_sched(int level, int levels, int* data, int n) {
    if (level >= levels) return;
    k_ff<<<1, 32, 0, cudaStreamFireAndForget>>>(level, data, n);
    k_work<<<148, 256, 0, cudaStreamTailLaunch>>>(level, data, n);
    k_work<<<148, 256, 0, cudaStreamTailLaunch>>>(level, data, n);
    k_sched<<<1, 1, 0, cudaStreamTailLaunch>>>(level + 1, levels, data, n);
}
__global__ void k_check(int* data, int n, int expect, int* bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (data[i] != expect) atomicAdd(bad, 1);
}
int main() {
    int n = 1 << 20; int *d, *bad;
    cudaMalloc(&d, n * 4); cudaMalloc(&bad, 4);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int levels : {1, 10, 100}) {
        cudaMemsetAsync(d, 0, n * 4, s); cudaMemsetAsync(bad, 0, 4, s);
        unsigned z = 0; cudaMemcpyToSymbolAsync(g_n, &z, 4, 0, cudaMemcpyHostToDevice, s);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, s);
        k_sched<<<1, 1, 0, s>>>(0, levels, d, n);
        cudaEventRecord(b, s);
        k_check<<<148, 256, 0, s>>>(d, n, 2 * levels, bad);   // stream order: must see all levels
        int hb = -1; cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s);
        cudaError_t e = cudaStreamSynchronize(s);
        float ms = 0; cudaEventElapsedTime(&ms, a, b);
        unsigned cnt; cudaMemcpyFromSymbol(&cnt, g_n, 4);
        printf("levels=%d err=%s bad=%d launches=%u time=%.3f ms (%.2f us/level)\n", levels, cudaGetErrorString(e), hb, cnt, ms, 1000 * ms / levels);
    }
    // graph capture
    {
        cudaMemsetAsync(d, 0, n * 4, s); cudaMemsetAsync(bad, 0, 4, s); cudaStreamSynchronize(s);
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaError_t e1 = cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        k_sched<<<1, 1, 0, s>>>(0, 5, d, n);
        cudaError_t e2 = cudaStreamEndCapture(s, &g);
        cudaError_t e3 = cudaGraphInstantiate(&ge, g, 0);
        printf("capture: %s / %s / %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3));
        if (e3 == cudaSuccess) {
            for (int r = 0; r < 3; ++r) cudaGraphLaunch(ge, s);
            k_check<<<148, 256, 0, s>>>(d, n, 30, bad);
            int hb = -1; cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s);
            cudaError_t e = cudaStreamSynchronize(s);
            printf("graph replay x3: err=%s bad=%d\n", cudaGetErrorString(e), hb);
        }
    }
    return 0;
}
