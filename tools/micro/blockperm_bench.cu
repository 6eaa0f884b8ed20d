// Microbenchmark (tuning aid, not product): bandwidth of moving random BS-byte blocks
// (read block i, write it to block perm[i]) over a 2 GiB array, one warp per block, as the
// block permutation does; and a plain streaming copy for reference.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
typedef unsigned long long u64;

template <int BS>
__global__ void k_move(const uint4* __restrict__ src, uint4* __restrict__ dst, const unsigned* perm, unsigned nblk) {
    constexpr int V = BS / 16 / 32;  // uint4 per lane
    const unsigned lane = threadIdx.x & 31;
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (unsigned b = w; b < nblk; b += nw) {
        const unsigned d = perm[b];
        uint4 r[V];
#pragma unroll
        for (int i = 0; i < V; ++i) r[i] = src[(u64)b * (BS / 16) + i * 32 + lane];
#pragma unroll
        for (int i = 0; i < V; ++i) dst[(u64)d * (BS / 16) + i * 32 + lane] = r[i];
    }
}
__global__ void k_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) dst[i] = src[i];
}

template <int BS>
void run(const uint4* a, uint4* b, u64 bytes, int blocks) {
    const unsigned nblk = (unsigned)(bytes / BS);
    std::vector<unsigned> h(nblk);
    for (unsigned i = 0; i < nblk; ++i) h[i] = i;
    std::mt19937 g(1);
    std::shuffle(h.begin(), h.end(), g);
    unsigned* d; cudaMalloc(&d, nblk * 4ull); cudaMemcpy(d, h.data(), nblk * 4ull, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_move<BS><<<blocks, 256>>>(a, b, d, nblk);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("random %5d-B blocks, grid %5d: %.3f ms  %.0f GB/s (read+write)\n", BS, blocks, ms, 2.0 * bytes / ms / 1e6);
    }
    cudaFree(d);
}

int main() {
    const u64 bytes = 2ull << 30;
    uint4 *a, *b;
    cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
    cudaMemset(a, 1, bytes); cudaMemset(b, 0, bytes);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0); k_copy<<<148 * 8, 256>>>(a, b, bytes / 16); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("stream copy: %.3f ms  %.0f GB/s\n", ms, 2.0 * bytes / ms / 1e6);
    }
    for (int g : {148 * 8, 148 * 16}) {
        run<512>(a, b, bytes, g); run<1024>(a, b, bytes, g); run<2048>(a, b, bytes, g);
    }
    return 0;
}
