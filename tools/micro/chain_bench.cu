// Microbenchmark (tuning aid, not product): a block move preceded by a dependent L2 atomic
// (the permutation's "claim, then read" step), vs the plain random block move.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
typedef unsigned long long u64;

template <int MODE, int SLOTS>
__global__ void k_chain(const uint4* __restrict__ src, uint4* __restrict__ dst, const unsigned* perm, unsigned nblk,
                        u64* ctr, unsigned nctr) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (unsigned b0 = w * SLOTS; b0 < nblk; b0 += nw * SLOTS) {
        unsigned s[SLOTS];
        u64 old = 0;
        if (lane < SLOTS && b0 + lane < nblk) {
            const unsigned b = b0 + lane;
            if (MODE == 1) old = atomicAdd(&ctr[(perm[b] * 2654435761u) % nctr], 1ull);
            else old = 0;
        }
#pragma unroll
        for (int c = 0; c < SLOTS; ++c) s[c] = b0 + c + (unsigned)(__shfl_sync(0xffffffffu, old, c) & 0);
        uint4 r[SLOTS];
#pragma unroll
        for (int c = 0; c < SLOTS; ++c) if (s[c] < nblk) r[c] = src[(u64)perm[s[c]] * 32 + lane];
#pragma unroll
        for (int c = 0; c < SLOTS; ++c) if (s[c] < nblk) dst[(u64)s[c] * 32 + lane] = r[c];
    }
}

int main() {
    const u64 bytes = 2ull << 30;
    const unsigned nblk = (unsigned)(bytes / 512);
    uint4 *a, *b; u64* ctr;
    cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&ctr, 65536 * 8);
    cudaMemset(a, 1, bytes); cudaMemset(ctr, 0, 65536 * 8);
    std::vector<unsigned> h(nblk); for (unsigned i = 0; i < nblk; ++i) h[i] = i;
    std::mt19937 g(1); std::shuffle(h.begin(), h.end(), g);
    unsigned* d; cudaMalloc(&d, nblk * 4ull); cudaMemcpy(d, h.data(), nblk * 4ull, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    auto run = [&](const char* name, auto kern, int grid, unsigned nctr) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0); kern<<<grid, 256>>>(a, b, d, nblk, ctr, nctr); cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("%-34s grid %5d nctr %6u: %.3f ms  %.0f GB/s\n", name, grid, nctr, ms, 2.0 * bytes / ms / 1e6);
    };
    for (int grid : {592, 1184, 2368}) {
        run("move, 1 block/warp", k_chain<0, 1>, grid, 256);
        run("atomic+move, 1 block/warp", k_chain<1, 1>, grid, 256);
        run("atomic+move, 1 block/warp", k_chain<1, 1>, grid, 43520);
        run("atomic+move, 4 blocks/warp", k_chain<1, 4>, grid, 256);
        run("atomic+move, 4 blocks/warp", k_chain<1, 4>, grid, 43520);
    }
    return 0;
}
