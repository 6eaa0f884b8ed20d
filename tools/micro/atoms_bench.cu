// Microbenchmark (tuning aid, not product): shared-memory atomic ranking throughput.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned int u32;
template <int MODE>
__global__ void k_atoms(const u32* in, u32* out, int iters) {
    __shared__ u32 cnt[32 * 256 + 64];
    for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    u32 v = in[blockIdx.x * blockDim.x + threadIdx.x];
    u32 acc = 0;
    const u32 w = threadIdx.x >> 5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const u32 d = (v >> (u * 3)) & 255u;
            if (MODE == 0) acc += atomicAdd(&cnt[d], 1u);                 // one shared counter set
            else if (MODE == 1) acc += atomicAdd(&cnt[(w & 31) * 256 + d], 1u);  // per-warp counter sets
            else acc += atomicAdd(&cnt[(w & 31) * 256 + ((d * 33) & 255)], 1u);
        }
        v = v * 1664525u + 1013904223u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    const int blocks = 148 * 4, threads = 512, iters = 100;
    const size_t n = (size_t)blocks * threads;
    u32 *in, *out;
    cudaMalloc(&in, n * 4); cudaMalloc(&out, n * 4);
    u32* h = new u32[n]; for (size_t i = 0; i < n; ++i) h[i] = (u32)(i * 2654435761u) ^ (u32)(i >> 3) * 40503u;
    cudaMemcpy(in, h, n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
    int sm = 0; cudaDeviceGetAttribute(&sm, cudaDevAttrClockRate, 0);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); k_atoms<0><<<blocks, threads>>>(in, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("atoms shared-set : %.3f ms  %.3f elem/cycle/SM\n", ms, (double)n * iters * 8 / (ms * 1e-3 * sm * 1e3) / 148);
        cudaEventRecord(a); k_atoms<1><<<blocks, threads>>>(in, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("atoms per-warp   : %.3f ms  %.3f elem/cycle/SM\n", ms, (double)n * iters * 8 / (ms * 1e-3 * sm * 1e3) / 148);
        cudaEventRecord(a); k_atoms<2><<<blocks, threads>>>(in, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("atoms per-warp-b : %.3f ms  %.3f elem/cycle/SM\n", ms, (double)n * iters * 8 / (ms * 1e-3 * sm * 1e3) / 148);
    }
    return 0;
}
