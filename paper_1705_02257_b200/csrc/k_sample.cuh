// k_sample.cuh -- K1: oversampled splitter selection and the implicit search tree.
//
// One CTA per task.  PAPER.md:134-141 (§3): sort alpha*k-1 sampled elements, pick k-1
// equidistant splitters, store them as a complete binary search tree a_1 = s_{k/2},
// a_2 = s_{k/4}, a_3 = s_{3k/4}, ...  PAPER.md:399-401 (§4.7): remove duplicate
// splitters; equality buckets only if duplicates were found.  alpha = 0.2 log n
// (PAPER.md:414).  The sample lives in shared memory instead of being swapped to the
// front of the array: same splitters, no writes to the input.
#pragma once
#include "common.cuh"
#include "k_base.cuh"

namespace ips4o {

// A K1 CTA has 1024 threads: 4 (ordinary tasks) or 8 (big tasks) sample keys per thread
// (register network + merge passes).
#ifndef IPS4O_K1_THREADS
#define IPS4O_K1_THREADS 1024
#endif
constexpr int K1_THREADS = IPS4O_K1_THREADS;
constexpr int K1_SAMPLE = 4096;        // sample capacity for ordinary tasks
constexpr int K1_SAMPLE_BIG = 8192;    // for tasks of >= 2^22 elements (dynamic smem, 64 KB)
constexpr size_t K1_SMEM = (size_t)(K1_SAMPLE_BIG + K1_SAMPLE_BIG / 16) * 8 + 16;
#ifndef IPS4O_K1_BIG_LOG
#define IPS4O_K1_BIG_LOG 22
#endif
constexpr u64 K1_BIG_TASK = 1ull << IPS4O_K1_BIG_LOG;

// Builds the padded splitter array spl[1..k'-1] and the BFS tree from nd distinct sorted
// splitters held in s_dist[0..nd).  k' = next power of two >= nd+1; padding repeats the
// largest splitter.  Writes the task's classifier fields.
// Bucket-hint table (common.cuh, LUT_N): for every cell, A = #{padded splitters <= the
// cell's first key} and d = #{padded splitters inside the cell, above its first key}, for
// the padded splitters s_i = s_dist[min(i, nd) - 1], i in [1, kp-1].  Every splitter is
// counted in its cell (two 16-bit counters: equal to the cell's first key / above it), and
// A is the exclusive prefix over the cells plus the cell's "equal" count.  scr: LUT_N words
// of shared memory.  Block-wide; LUT_N must be a multiple of blockDim.x.
__device__ void build_lut_block(const u64* s_dist, u32 nd, u32 kp, unsigned short* g_lut, TaskParam* tp,
                                u32* scr) {
    __shared__ u32 s_ws[32];
    auto S = [&](u32 i) { return s_dist[(i <= nd ? i : nd) - 1]; };
    const u64 s1 = S(1), span = S(kp - 1) - s1;
    u32 sh = 0;
    if (span) {
        const u32 bl = 64u - (u32)__clzll((long long)span);
        sh = bl > LUT_LOG ? bl - LUT_LOG : 0u;  // span >> sh < LUT_N
    }
    // the cells start at lo = s_1 rounded down to a multiple of 2^sh, so that K2 can take a
    // key's cell as (key >> sh) - (lo >> sh) (one 32-bit subtraction when sh >= 32); if the
    // rounding pushes the last splitter past the table, the cells double
    u64 lo = sh ? s1 & ~((1ull << sh) - 1ull) : s1;
    if (((S(kp - 1) - lo) >> sh) >= LUT_N) {
        ++sh;
        lo = s1 & ~((1ull << sh) - 1ull);
    }
    // thread t owns cells [t*per, (t+1)*per) (any block size: the last owners may own none)
    const u32 tid = threadIdx.x, nt = blockDim.x, per = (LUT_N + nt - 1) / nt, lane = tid & 31, w = tid >> 5;
    for (u32 c = tid; c < LUT_N; c += nt) scr[c] = 0u;
    __syncthreads();
    for (u32 i = 1 + tid; i < kp; i += nt) {
        const u64 sv = S(i);
        const u64 y = (sv - lo) >> sh;
        const u32 c = y >= LUT_N ? LUT_N - 1u : (u32)y;
        atomicAdd(&scr[c], sv == lo + ((u64)c << sh) ? 0x10000u : 1u);
    }
    __syncthreads();
    u32 sum = 0;
    for (u32 k = 0; k < per && tid * per + k < LUT_N; ++k) {
        const u32 x = scr[tid * per + k];
        sum += (x & 0xFFFFu) + (x >> 16);
    }
    u32 incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (u32)o) incl += y;
    }
    if (lane == 31) s_ws[w] = incl;
    __syncthreads();
    u32 run = incl - sum;
    for (u32 ww = 0; ww < w; ++ww) run += s_ws[ww];
    for (u32 k = 0; k < per && tid * per + k < LUT_N; ++k) {
        const u32 c = tid * per + k, x = scr[c];
        const u32 eqc = x >> 16, gtc = x & 0xFFFFu;
        g_lut[c] = (unsigned short)((run + eqc) | gtc << 8);
        run += eqc + gtc;
    }
    for (u32 c = LUT_N + tid; c < LUT_STRIDE; c += nt) g_lut[c] = 0;  // keys below s_1; padding
    if (tid == 0) {
        tp->lut_lo = lo;
        tp->lut_sh = sh;
    }
}

__device__ void build_tree_block(const u64* s_dist, u32 nd, u32 eq, u64* g_tree, u64* g_spl,
                                 TaskParam* tp, u64* btot, unsigned short* g_lut, u32* scr) {
    u32 kp = 2;
    while (kp < nd + 1) kp <<= 1;
    u32 logk = 0;
    while ((1u << logk) < kp) ++logk;
    for (u32 i = threadIdx.x; i < (u32)MAXK; i += blockDim.x) {
        u64 s = 0;
        if (i >= 1 && i < kp) s = s_dist[(i <= nd ? i : nd) - 1];
        g_spl[i] = s;
    }
    for (u32 j = threadIdx.x; j < (u32)MAXK; j += blockDim.x) {
        u64 v = 0;
        if (j >= 1 && j < kp) {
            u32 l = 31 - __clz(j);
            u32 pos = j - (1u << l);
            u32 idx = (2 * pos + 1) * (kp >> (l + 1));  // 1-based splitter index
            v = s_dist[(idx <= nd ? idx : nd) - 1];
        }
        g_tree[j] = v;
    }
    for (u32 i = threadIdx.x; i < (u32)MAXK; i += blockDim.x) btot[i] = 0ull;
    if (threadIdx.x == 0) {
        tp->kprime = kp;
        tp->logk = logk;
        tp->eq = eq;
        tp->K = eq ? 2 * kp - 1 : kp;
    }
    build_lut_block(s_dist, nd, kp, g_lut, tp, scr);
}

// the sample's keys as a base-case element type (order-preserving u64 images)
struct TKey {
    typedef u64 V;
    __device__ __forceinline__ static bool less(V a, V b) { return a < b; }
    __host__ __device__ __forceinline__ static V pad() { return ~0ull; }
};

// One task t: sample, sort the sample, pick the splitters, build the classifier.
template <class TR, int SAMPLE>
__device__ __forceinline__ void k1_task(const LevelArgs& A, u32 t, u64* keys, u64* dist, u32& s_flag, u32& s_nd) {
    TaskParam* tp = const_cast<TaskParam*>(A.tp) + t;
    const u64 lo = tp->lo, hi = tp->hi, n = hi - lo;
    const Mem<TR> mem(A.data, A.vals);

    // Bucket count: the last levels use an adaptive k aimed at
    // base-case tiles of ~LEAF elements: k = min(256, max(4, pow2_ceil(n/LEAF))).
    // Oversampling: the paper's alpha = 0.2 log n is a CPU-cache choice;
    // sorting the sample costs the same ~10 us here for any alpha <= 2048/k, so the GPU
    // takes alpha = max(0.2 log2 n, 2048/k - 1 rounded down), which keeps subproblems
    // close to their expected size (fewer extra levels).  Any alpha gives the same output.
    u32 k = 4;
    while ((u64)k * TR::LEAF < n && k < (u32)MAXK) k *= 2;
    u32 alpha = (u32)llround(0.2 * log2((double)n));
    if (alpha < 1) alpha = 1;
    const u32 amax = (SAMPLE - 1) / k;
    if (alpha < amax) alpha = amax;
    // the sample must fit the task (m <= n): a task smaller than the shared-memory sample
    // (records: 1025..4095 elements) takes alpha = (n+1)/k (>= 1 since n > k here)
    const u64 acap = (n + 1) / k;
    if ((u64)alpha > acap) alpha = (u32)(acap > 0 ? acap : 1);
    const u32 m = alpha * k - 1;
    // stratified random sample without replacement: one element per stratum; sorted in
    // shared memory by the block merge sort of the base case (register networks of
    // SAMPLE/K1_THREADS keys per thread + merge-path passes), padded with the largest key
    // (all of a thread's random reads are issued before any is used: each one is a TLB and
    // DRAM miss somewhere in the array)
    constexpr int PER = SAMPLE / K1_THREADS;
    u64 sk[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const u32 j = q * K1_THREADS + threadIdx.x;
        sk[q] = ~0ull;
        if (j < m) {
            // stratum [a, b) of the task (n * (j+1) < 2^64 for n < 2^50); the offset inside
            // it is the high half of a 64x64-bit product (no division)
            const u64 a = lo + n * j / m;
            const u64 b = lo + n * (j + 1) / m;
            const u64 r = mix64(A.seed ^ mix64(lo * 0x9E3779B97F4A7C15ull + j));
            sk[q] = mem.key(a + __umul64hi(r, b - a), tp->part);
        }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) keys[padidx(q * K1_THREADS + threadIdx.x)] = sk[q];
    __syncthreads();
    block_sort_smem<TKey, K1_THREADS, PER>(keys, (u32)SAMPLE);
    // equidistant picks s_i = S[i*alpha - 1]; duplicates?
    if (threadIdx.x == 0) s_flag = 0;
    __syncthreads();
    for (u32 i = 1 + threadIdx.x; i + 1 < k; i += blockDim.x)
        if (keys[padidx(i * alpha - 1)] == keys[padidx((i + 1) * alpha - 1)]) s_flag = 1;
    __syncthreads();
    u32 eq = s_flag;
    if (!eq) {
        for (u32 i = threadIdx.x; i + 1 < k; i += blockDim.x) dist[i] = keys[padidx((i + 1) * alpha - 1)];
        if (threadIdx.x == 0) s_nd = k - 1;
    } else {
        // Equality buckets.  Take k/2-1 equidistant picks so
        // that 2k'-1 <= 255 buckets fit the shared-memory budget, then keep
        // one copy of each distinct value.
        const u32 k2 = k / 2, a2 = 2 * alpha;
        if (threadIdx.x == 0) {
            u32 nd = 0;
            for (u32 i = 1; i < k2; ++i) {
                u64 v = keys[padidx(i * a2 - 1)];
                if (nd == 0 || dist[nd - 1] != v) dist[nd++] = v;
            }
            s_nd = nd;
        }
    }
    __syncthreads();
    build_tree_block(dist, s_nd, eq, A.tree + (u64)t * MAXK, A.spl + (u64)t * MAXK, tp, A.btot + (u64)t * MAXK,
                     A.lut + (u64)t * LUT_STRIDE, reinterpret_cast<u32*>(keys));  // (the sample is done)
    if (threadIdx.x == 0 && eq) atomicAdd(&A.ctr[CTR_EQ], 1u);
}

// K1: one CTA per task of the batch (grid = the workspace's task capacity; CTAs past the
// batch exit).  Tasks of >= 2^22 elements take an 8192-key sample, the others 4096.  The
// debug partition step (dyn->from_splitters) builds task 0's classifier from given splitters.
template <class TR>
__global__ void __launch_bounds__(K1_THREADS) k_sample(LevelArgs A0) {
    const LevelArgs A = with_dyn(A0);
    extern __shared__ __align__(16) unsigned char smem1[];
    u64* keys = reinterpret_cast<u64*>(smem1);
    __shared__ u64 dist[MAXK];
    __shared__ u32 s_flag, s_nd;
    for (u32 t = blockIdx.x; t < A.ntasks; t += gridDim.x) {
        if (A0.dyn->from_splitters) {
            const u32 ns = A0.dyn->nspl;
            for (u32 i = threadIdx.x; i < ns; i += blockDim.x) dist[i] = A.dsplit[i];
            __syncthreads();
            build_tree_block(dist, ns, A0.dyn->spl_eq, A.tree, A.spl, const_cast<TaskParam*>(A.tp), A.btot, A.lut,
                             reinterpret_cast<u32*>(keys));
            return;
        }
        const u64 n = A.tp[t].hi - A.tp[t].lo;
        if (n >= K1_BIG_TASK) k1_task<TR, K1_SAMPLE_BIG>(A, t, keys, dist, s_flag, s_nd);
        else k1_task<TR, K1_SAMPLE>(A, t, keys, dist, s_flag, s_nd);
        __syncthreads();
    }
}

// Debug path: classifier from splitters given by the caller (already key-transformed).
__global__ void k_tree_from_splitters(LevelArgs A, const u64* splitters, u32 nspl, u32 eq) {
    __shared__ u64 dist[MAXK];
    __shared__ u32 scr[LUT_N];
    for (u32 i = threadIdx.x; i < nspl; i += blockDim.x) dist[i] = splitters[i];
    __syncthreads();
    build_tree_block(dist, nspl, eq, A.tree, A.spl, const_cast<TaskParam*>(A.tp), A.btot, A.lut, scr);
}

}  // namespace ips4o
