// k_base.cuh -- K5: base-case sort of small subproblems in shared memory, and the T1
// classification debug kernel.
//
// The paper stops the recursion below n0 = 16 elements and uses insertion sort
// (PAPER.md:403, 416).  On the GPU the leaves are whole shared-memory tiles: a task of at
// most CAP elements is loaded into shared memory, padded to a power of two with the
// all-ones element, sorted by a bitonic network, and written back.
#pragma once
#include "common.cuh"

namespace ips4o {

constexpr int K5_THREADS = 1024;

template <class TR>
__global__ void __launch_bounds__(K5_THREADS) k_basecase(TaskDesc* tasks, u32 ntasks, void* vdata) {
    typedef typename TR::V V;
    extern __shared__ __align__(16) unsigned char smem5[];
    V* s = reinterpret_cast<V*>(smem5);
    V* data = reinterpret_cast<V*>(vdata);
    for (u32 ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
        const TaskDesc td = tasks[ti];
        const u32 n = (u32)(td.hi - td.lo);
        u32 P = 1;
        while (P < n) P <<= 1;
        for (u32 i = threadIdx.x; i < P; i += blockDim.x) s[i] = i < n ? data[td.lo + i] : TR::pad();
        __syncthreads();
        for (u32 kk = 2; kk <= P; kk <<= 1) {
            for (u32 jj = kk >> 1; jj > 0; jj >>= 1) {
                for (u32 p = threadIdx.x; p < P / 2; p += blockDim.x) {
                    const u32 i = 2 * p - (p & (jj - 1));
                    const u32 x = i + jj;
                    const bool up = (i & kk) == 0;
                    const V a = s[i], c = s[x];
                    if (TR::less(c, a) == up) {
                        s[i] = c;
                        s[x] = a;
                    }
                }
                __syncthreads();
            }
        }
        for (u32 i = threadIdx.x; i < n; i += blockDim.x) data[td.lo + i] = s[i];
        __syncthreads();
    }
}

template <class TR>
__global__ void k_debug_classify(const void* vin, u64 n, const u64* tree_g, const u64* spl_g,
                                 const TaskParam* tp, u32* out) {
    __shared__ u64 tree[MAXK], spl[MAXK];
    for (u32 i = threadIdx.x; i < (u32)MAXK; i += blockDim.x) {
        tree[i] = tree_g[i];
        spl[i] = spl_g[i];
    }
    __syncthreads();
    const typename TR::V* in = reinterpret_cast<const typename TR::V*>(vin);
    const u32 logk = tp->logk, kp = tp->kprime, eq = tp->eq;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = classify_key(TR::key(in[i]), tree, spl, logk, kp, eq);
}

}  // namespace ips4o
