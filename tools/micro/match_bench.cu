// Microbenchmark (tuning aid, not product): throughput of warp aggregation primitives on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned int u32;
typedef unsigned long long u64;

__global__ void k_match(const u32* in, u32* out, int iters) {
    u32 v = in[blockIdx.x * blockDim.x + threadIdx.x];
    u32 acc = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            u32 m = __match_any_sync(0xffffffffu, (v + u) & 255u);
            acc += m;
        }
        v = v * 1664525u + 1013904223u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_ballot8(const u32* in, u32* out, int iters) {
    u32 v = in[blockIdx.x * blockDim.x + threadIdx.x];
    u32 acc = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            u32 b = (v + u) & 255u;
            u32 peers = 0xffffffffu;
#pragma unroll
            for (int l = 0; l < 8; ++l) {
                bool p = (b >> l) & 1u;
                u32 x = __ballot_sync(0xffffffffu, p);
                peers &= p ? x : ~x;
            }
            acc += peers;
        }
        v = v * 1664525u + 1013904223u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
// dependent-chain descent over a 256-leaf BFS tree in shared memory, 8 keys per thread
template <bool BALLOT>
__global__ void k_descent(const u64* keys_in, const u64* tree_g, u32* out, int iters) {
    __shared__ u64 tree[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tree[i] = tree_g[i];
    __syncthreads();
    u64 key[8];
    for (int e = 0; e < 8; ++e) key[e] = keys_in[(blockIdx.x * blockDim.x + threadIdx.x) * 8 + e];
    u32 acc = 0;
    const char* tb = reinterpret_cast<const char*>(tree);
    for (int it = 0; it < iters; ++it) {
        u32 a[8], peers[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) { a[e] = 8; peers[e] = ~0u; }
#pragma unroll
        for (int l = 0; l < 8; ++l)
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const bool p = key[e] >= *reinterpret_cast<const u64*>(tb + a[e]);
                if (BALLOT) {
                    const u32 x = __ballot_sync(0xffffffffu, p);
                    peers[e] &= p ? x : ~x;
                }
                a[e] = (a[e] << 1) + (p ? 8u : 0u);
            }
#pragma unroll
        for (int e = 0; e < 8; ++e) { acc += a[e] + peers[e]; key[e] += acc; }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    const int blocks = 148 * 4, threads = 512, iters = 200;
    const size_t n = (size_t)blocks * threads;
    u32 *in, *out; u64 *keys, *tree;
    cudaMalloc(&in, n * 4); cudaMalloc(&out, n * 4); cudaMalloc(&keys, n * 8 * 8); cudaMalloc(&tree, 256 * 8);
    u32* h = new u32[n]; for (size_t i = 0; i < n; ++i) h[i] = (u32)(i * 2654435761u);
    cudaMemcpy(in, h, n * 4, cudaMemcpyHostToDevice);
    u64* hk = new u64[n * 8]; u64 s = 88172645463325252ull;
    for (size_t i = 0; i < n * 8; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hk[i] = s; }
    cudaMemcpy(keys, hk, n * 64, cudaMemcpyHostToDevice);
    u64 ht[256]; for (int j = 1; j < 256; ++j) { int l = 31 - __builtin_clz(j); int pos = j - (1 << l); int idx = (2 * pos + 1) * (256 >> (l + 1)); ht[j] = (u64)idx << 56; } ht[0] = 0;
    cudaMemcpy(tree, ht, 2048, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
    int sm = 0; cudaDeviceGetAttribute(&sm, cudaDevAttrClockRate, 0);
    auto report = [&](const char* name, double ops) {
        double cyc = ms * 1e-3 * sm * 1e3;  // SM clock kHz -> cycles
        printf("%-14s %8.3f ms  %.3f warp-ops/cycle/SM\n", name, ms, ops / cyc / 148.0);
    };
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); k_match<<<blocks, threads>>>(in, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); report("match_any", (double)n / 32 * iters * 8);
        cudaEventRecord(a); k_ballot8<<<blocks, threads>>>(in, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); report("ballot8-peers", (double)n / 32 * iters * 8);
        cudaEventRecord(a); k_descent<false><<<blocks, threads>>>(keys, tree, out, iters / 4); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); report("descent", (double)n / 32 * (iters / 4) * 8);
        cudaEventRecord(a); k_descent<true><<<blocks, threads>>>(keys, tree, out, iters / 4); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); report("descent+ballot", (double)n / 32 * (iters / 4) * 8);
    }
    printf("(ops = warp-level element classifications / aggregations; clock %d kHz)\n", sm);
    return 0;
}
