// Microbenchmark (tuning aid, not product): the data movement of K2 without classification.
// Persistent CTAs (one per SM, 640 threads, ~225 KB shared memory like K2) stream their slice of
// a 2 GiB array in 5120-element tiles through two TMA stages and write every tile back behind the
// read frontier either as 80 TMA bulk stores of 512 B (variant 0, K2's flushes) or by plain
// coalesced 16-byte stores (variant 1), or not at all (variant 2: read only).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
typedef unsigned u32;
constexpr int NT = 640, TILE = 5120, BLK = 64;

__device__ __forceinline__ void mbar_init(u64* m, u32 c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((u32)__cvta_generic_to_shared(m)), "r"(c));
}
__device__ __forceinline__ void g2s(void* dst, const void* src, u32 bytes, u64* m) {
    const u32 d = (u32)__cvta_generic_to_shared(dst), mb = (u32)__cvta_generic_to_shared(m);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d), "l"(src),
                 "r"(bytes), "r"(mb) : "memory");
}
__device__ __forceinline__ void wait(u64* m, u32 ph) {
    const u32 mb = (u32)__cvta_generic_to_shared(m);
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(mb), "r"(ph) : "memory");
}
__device__ __forceinline__ void s2g(void* dst, const void* src, u32 bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"((u32)__cvta_generic_to_shared(src)), "r"(bytes) : "memory");
}

template <int VAR>
__global__ void __launch_bounds__(NT, 1) k(u64* a, u64 n) {
    extern __shared__ __align__(128) unsigned char sm[];
    u64* st = reinterpret_cast<u64*>(sm);
    __shared__ __align__(8) u64 mb[2];
    const u32 tid = threadIdx.x;
    if (tid == 0) { mbar_init(&mb[0], 1); mbar_init(&mb[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const u64 per = n / gridDim.x / TILE * TILE, lo = blockIdx.x * per, nt = per / TILE;
    if (tid == 0) for (u64 t = 0; t < 2 && t < nt; ++t) g2s(st + t * TILE, a + lo + t * TILE, TILE * 8, &mb[t]);
    u32 ph = 0;
    for (u64 t = 0; t < nt; ++t) {
        const u32 s = t & 1;
        wait(&mb[s], (ph >> s) & 1); ph ^= 1u << s;
        __syncthreads();
        u64* src = st + s * TILE;
        u64* dst = a + lo + (t ? t - 1 : 0) * TILE;  // behind the read frontier
        if (VAR == 0) {
            if (tid < TILE / BLK) {
                s2g(dst + tid * BLK, src + tid * BLK, BLK * 8);
                asm volatile("cp.async.bulk.commit_group;");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        } else if (VAR == 1) {
            const uint4* s4 = reinterpret_cast<const uint4*>(src);
            uint4* d4 = reinterpret_cast<uint4*>(dst);
            for (u32 i = tid; i < TILE / 2; i += NT) d4[i] = s4[i];
        }
        __syncthreads();
        if (tid == 0 && t + 2 < nt) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            g2s(st + s * TILE, a + lo + (t + 2) * TILE, TILE * 8, &mb[s]);
        }
    }
    if (tid < TILE / BLK) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const u64 n = 1ull << 28;
    u64* a; cudaMalloc(&a, n * 8); cudaMemset(a, 1, n * 8);
    const int smem = 225 * 1024;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[3] = {"TMA 512-B block stores", "plain 16-B stores", "read only"};
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) k<0><<<148, NT, smem>>>(a, n);
            if (v == 1) k<1><<<148, NT, smem>>>(a, n);
            if (v == 2) k<2><<<148, NT, smem>>>(a, n);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 3) printf("%-24s %.3f ms  %.0f GB/s (algorithmic %s)\n", names[v], ms, (v == 2 ? 1.0 : 2.0) * n * 8 / ms / 1e6, v == 2 ? "read" : "read+write");
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
