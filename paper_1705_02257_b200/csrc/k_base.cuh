// k_base.cuh -- K5: base-case sort of small subproblems, and the T1 classification debug kernel.
//
// The paper stops the recursion below n0 = 16 elements and finishes with insertion sort
// (PAPER.md:403, 416).  On the GPU a leaf is a whole shared-memory tile: one CTA loads a
// subproblem of at most THREADS*ITEMS elements, pads it with the all-ones element (which
// is >= every key and, for records, identical to any equal real element, so the first n
// outputs are exactly the sorted input), and sorts it:
//   1. every thread sorts ITEMS consecutive elements in registers with a bitonic network
//      (compile-time indices, no branches: the GPU counterpart of the paper's
//      branch-free base case);
//   2. log2(TILE/ITEMS) merge passes: each thread locates its output window in the pair
//      of runs by a merge-path binary search and merges ITEMS elements serially from
//      shared memory into registers;
//   3. coalesced write-back of the first n elements.
// Shared memory is padded by one element per 16 so that the blocked (thread-contiguous)
// accesses of 64-bit elements are free of bank conflicts beyond the 2-wavefront minimum.
// Subproblems are binned by size class (2K/4K/8K/16K elements) by the cleanup kernel so
// that each launch uses a CTA sized to its tasks.
#pragma once
#include <type_traits>
#include "common.cuh"

namespace ips4o {

__host__ __device__ constexpr u32 padidx(u32 i) { return i + (i >> 4); }

template <class TR>
__device__ __forceinline__ void ce(typename TR::V& a, typename TR::V& b, bool up) {
    const bool sw = TR::less(b, a) == up;
    const typename TR::V x = a, y = b;
    a = sw ? y : x;
    b = sw ? x : y;
}

// Sorts the n elements held in s[padidx(0..n)) in place (block-wide; all threads call it).
// Precondition: positions [n, n16) hold TR::pad(); ends with a __syncthreads().
template <class TR, int THREADS, int ITEMS>
__device__ __forceinline__ void block_sort_smem(typename TR::V* s, u32 n) {
    typedef typename TR::V V;
    constexpr u32 TILE = THREADS * ITEMS;
    const u32 tid = threadIdx.x;
    const u32 n16 = (n + ITEMS - 1) / ITEMS * ITEMS;  // only these positions are touched
    const bool active = tid * ITEMS < n;
    V v[ITEMS];
    if (active) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) v[k] = s[padidx(tid * ITEMS + k)];
        // 1. bitonic network over the thread's ITEMS registers (ascending)
#pragma unroll
        for (int kk = 2; kk <= ITEMS; kk <<= 1) {
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const int l = i ^ jj;
                    if (l > i) ce<TR>(v[i], v[l], (i & kk) == 0);
                }
            }
        }
    }
    // 2. merge passes over the n16 real positions only (runs are merged by their real
    //    lengths, so padding beyond n16 is never read).  While a run pair lies inside one
    //    warp's 32*ITEMS elements a warp barrier suffices.
#pragma unroll 1
    for (u32 w = ITEMS; w < TILE; w <<= 1) {
        const bool warp_local = 2 * w <= 32u * ITEMS;
        if (warp_local) __syncwarp(); else __syncthreads();
        if (active) {
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) s[padidx(tid * ITEMS + k)] = v[k];
        }
        if (warp_local) __syncwarp(); else __syncthreads();
        if (!active) continue;
        const u32 out0 = tid * ITEMS;
        const u32 ps = out0 & ~(2 * w - 1);  // start of the run pair
        const u32 diag = out0 - ps;
        const u32 A0 = ps, B0 = ps + w;
        const u32 ra = n16 > A0 ? (n16 - A0 < w ? n16 - A0 : w) : 0u;
        const u32 rb = n16 > B0 ? (n16 - B0 < w ? n16 - B0 : w) : 0u;
        // merge path over A[0, ra) and B[0, rb): number of A elements among the first diag
        u32 lo = diag > rb ? diag - rb : 0u, hi = diag < ra ? diag : ra;
        while (lo < hi) {
            const u32 mid = (lo + hi) >> 1;
            if (TR::less(s[padidx(B0 + diag - 1 - mid)], s[padidx(A0 + mid)])) hi = mid;
            else lo = mid + 1;
        }
        u32 ai = A0 + lo, bi = B0 + (diag - lo);
        const u32 ae = A0 + ra, be = B0 + rb;
        V av = s[padidx(ai < ae ? ai : A0)];
        V bv = s[padidx(bi < be ? bi : (rb ? B0 : A0))];
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const bool takeA = ai < ae && (bi >= be || !TR::less(bv, av));
            v[k] = takeA ? av : bv;
            if (takeA) {
                ++ai;
                av = s[padidx(ai < ae ? ai : A0)];
            } else {
                ++bi;
                bv = s[padidx(bi < be ? bi : (rb ? B0 : A0))];
            }
        }
    }
    __syncthreads();
    if (active) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) s[padidx(tid * ITEMS + k)] = v[k];
    }
    __syncthreads();
}

template <class TR, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) k_base_merge(const TaskDesc* tasks, u32 start, const u32* d_ntasks,
                                                         const LevelDyn* dyn, u32 cap) {
    const u32 ntasks = min(*d_ntasks, cap);  // tasks [start, ntasks) (the count lives on the device)
    typedef typename TR::V V;
    extern __shared__ __align__(16) unsigned char smem5[];
    V* s = reinterpret_cast<V*>(smem5);
    const Mem<TR> mem(dyn->data, dyn->vals);
    const u32 tid = threadIdx.x;
    for (u32 ti = start + blockIdx.x; ti < ntasks; ti += gridDim.x) {
        const TaskDesc td = tasks[ti];
        const u32 n = (u32)(td.hi - td.lo);
        const u32 n16 = (n + ITEMS - 1) / ITEMS * ITEMS;
        // coalesced load; the last thread's items past n are padding
        for (u32 i = tid; i < n16; i += THREADS) s[padidx(i)] = i < n ? mem.ld(td.lo + i) : TR::pad();
        __syncthreads();
        block_sort_smem<TR, THREADS, ITEMS>(s, n);
        for (u32 i = tid; i < n; i += THREADS) mem.st(td.lo + i, s[padidx(i)]);
        __syncthreads();
    }
}

// Records: sort (key part 0, key part 1 << 32 | index) items in shared memory, then gather
// the records into their sorted positions through a shared-memory copy of the leaf.
struct TRecItem {
    typedef ulonglong2 V;
    __device__ __forceinline__ static bool less(V a, V b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }
    __host__ __device__ __forceinline__ static V pad() { return make_ulonglong2(~0ull, ~0ull); }
};
// Two size classes: leaves of <= 512 records (2 items per thread, ~110 KB of shared memory:
// two CTAs per SM) and of <= 1024 (4 items, one CTA per SM).
constexpr int KREC_THREADS = 256;
template <int ITEMS>
struct RecBase {
    static constexpr size_t items_bytes = (size_t)padidx(KREC_THREADS * ITEMS) * 16 + 16;
    static constexpr u32 rec_words = KREC_THREADS * ITEMS * 25 + 8;  // + alignment slack
    static constexpr size_t smem = items_bytes + (size_t)2 * rec_words * 4;  // two leaves
};

// Records of one leaf arrive in shared memory by a TMA bulk copy of the 16-byte aligned body
// (the < 16 bytes before / after it by plain loads), one leaf ahead: the copy of leaf t+1
// overlaps the sort of leaf t.  Returns the word offset of the leaf's first record.
__device__ __forceinline__ u32 rec_fetch(const TaskDesc& td, const u32* gw, u32* buf, u64* mbar, bool edges_now) {
    const uintptr_t p0 = (uintptr_t)(gw + td.lo * 25), p1 = (uintptr_t)(gw + td.hi * 25);
    const uintptr_t a0 = (p0 + 15) & ~(uintptr_t)15, a1 = p1 & ~(uintptr_t)15, w0 = p0 & ~(uintptr_t)15;
    if (edges_now) {
        if (a1 > a0) bulk_g2s(reinterpret_cast<char*>(buf) + (a0 - w0), reinterpret_cast<const void*>(a0),
                              (u32)(a1 - a0), mbar);
        else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((u32)__cvta_generic_to_shared(mbar)) : "memory");
    }
    return (u32)((p0 - w0) / 4);
}

// Sort of a record leaf's (key part 0, key part 1 << 32 | index) items: the cell distribution
// of the 8-byte base case on key part 0 (cells of the key range, shared-memory atomic ranks,
// block scan, scatter, cells of several items ordered by insertion), or the merge sort when
// part 0 does not separate the items (all equal, e.g. a part-1 task) or a cell grows large.
// Items enter in registers (item q of thread t = index q*KREC_THREADS + t) and leave sorted
// in it[padidx(0..n)].  Block-wide.
template <int ITEMS>
__device__ void rec_items_sort(ulonglong2 (&itm)[ITEMS], u32 n, ulonglong2* it, u32* cnt, u64* s_range,
                               u32* s_flag, u32* s_wsum) {
    const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    constexpr u32 NT = KREC_THREADS, CAPI = NT * ITEMS;
    u64 kmin = ~0ull, kmax = 0;
#pragma unroll
    for (int q = 0; q < ITEMS; ++q)
        if (q * NT + tid < n) {
            kmin = min(kmin, itm[q].x);
            kmax = max(kmax, itm[q].x);
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (tid == 0) {
        s_range[0] = ~0ull;
        s_range[1] = 0;
        *s_flag = 0;
    }
    for (u32 c = tid; c < CAPI + 1; c += NT) cnt[c] = 0;
    __syncthreads();
    if (lane == 0 && w * 32 < n) {
        atomicMin(reinterpret_cast<unsigned long long*>(&s_range[0]), kmin);
        atomicMax(reinterpret_cast<unsigned long long*>(&s_range[1]), kmax);
    }
    __syncthreads();
    kmin = s_range[0];
    const u64 span = s_range[1] - kmin;
    const u32 cb = n > 1 ? 32u - (u32)__clz(n - 1) : 1u;
    const u32 ncell = 1u << cb;  // <= CAPI
    const bool cells = span != 0 && n >= 64;
    u32 cr[ITEMS];
    if (cells) {
        const u64 mul = span < ncell ? 0ull : (span == ~0ull ? (u64)ncell : (~0ull / (span + 1)) * ncell);
#pragma unroll
        for (int q = 0; q < ITEMS; ++q)
            if (q * NT + tid < n) {
                const u64 x = itm[q].x - kmin;
                const u32 c = mul ? (u32)__umul64hi(x, mul) : (u32)x;
                cr[q] = c | atomicAdd(&cnt[c], 1u) << 16;
            }
        __syncthreads();
        // exclusive scan over the ncell counters: thread t owns cells [t*ITEMS, (t+1)*ITEMS)
        u32 loc[ITEMS], sum = 0;
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            loc[q] = cnt[tid * ITEMS + q];
            sum += loc[q];
            if (loc[q] > 32u) *s_flag = 1u;  // a large cell: the merge sort is cheaper
        }
        u32 incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (u32)o) incl += y;
        }
        if (lane == 31) s_wsum[w] = incl;
        __syncthreads();
        u32 run = incl - sum;
        for (u32 ww = 0; ww < w; ++ww) run += s_wsum[ww];
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            cnt[tid * ITEMS + q] = run;
            run += loc[q];
        }
        if (tid == NT - 1) cnt[CAPI] = run;  // == n
        __syncthreads();
#pragma unroll
        for (int q = 0; q < ITEMS; ++q)
            if (q * NT + tid < n) it[padidx(cnt[cr[q] & 0xFFFFu] + (cr[q] >> 16))] = itm[q];
        __syncthreads();
        if (*s_flag == 0u) {
            // order the cells of this thread's run that hold several items (also when every
            // cell is one part-0 value: the items still differ in part 1)
#pragma unroll
            for (int q = 0; q < ITEMS; ++q) {
                const u32 b = cnt[tid * ITEMS + q], e = cnt[tid * ITEMS + q + 1];
                for (u32 i = b + 1; i < e; ++i) {
                    const ulonglong2 x = it[padidx(i)];
                    u32 j = i;
                    while (j > b && TRecItem::less(x, it[padidx(j - 1)])) {
                        it[padidx(j)] = it[padidx(j - 1)];
                        --j;
                    }
                    it[padidx(j)] = x;
                }
            }
        }
        __syncthreads();
        if (*s_flag == 0u) return;
        // large cells: fall through to the merge sort of the (permuted) items
        const u32 n16 = (n + ITEMS - 1) / ITEMS * ITEMS;
        for (u32 i = n + tid; i < n16; i += NT) it[padidx(i)] = TRecItem::pad();
        __syncthreads();
        block_sort_smem<TRecItem, NT, ITEMS>(it, n);
        return;
    }
    const u32 n16 = (n + ITEMS - 1) / ITEMS * ITEMS;
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
        const u32 i = q * NT + tid;
        if (i < n16) it[padidx(i)] = i < n ? itm[q] : TRecItem::pad();
    }
    __syncthreads();
    block_sort_smem<TRecItem, NT, ITEMS>(it, n);
}

template <int KREC_ITEMS>
__global__ void __launch_bounds__(KREC_THREADS) k_base_rec(const TaskDesc* tasks, const u32* d_ntasks, const LevelDyn* dyn, u32 cap) {
    const u32 ntasks = min(*d_ntasks, cap);
    void* vdata = dyn->data;
    typedef RecBase<KREC_ITEMS> RecBase;
    extern __shared__ __align__(16) unsigned char smem5[];
    ulonglong2* it = reinterpret_cast<ulonglong2*>(smem5);
    u32* const sbuf = reinterpret_cast<u32*>(smem5 + RecBase::items_bytes);
    u32* gw = reinterpret_cast<u32*>(vdata);
    const u32 tid = threadIdx.x;
    __shared__ __align__(8) u64 s_mbar[2];
    __shared__ u32 s_cnt[KREC_THREADS * KREC_ITEMS + 1];
    __shared__ u64 s_range[2];
    __shared__ u32 s_flag, s_wsum[KREC_THREADS / 32];
    if (tid == 0) {
        mbar_init(&s_mbar[0], 1);
        mbar_init(&s_mbar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    u32 phase = 0, cur = 0;
    if (blockIdx.x < ntasks && tid == 0) rec_fetch(tasks[blockIdx.x], gw, sbuf, &s_mbar[0], true);
    for (u32 ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
        const TaskDesc td = tasks[ti];
        const u32 n = (u32)(td.hi - td.lo);
        const u32 n16 = (n + KREC_ITEMS - 1) / KREC_ITEMS * KREC_ITEMS;
        u32* g = gw + td.lo * 25;
        u32* srec0 = sbuf + cur * RecBase::rec_words;
        if (tid == 0 && ti + gridDim.x < ntasks) {
            fence_proxy_async_smem();
            rec_fetch(tasks[ti + gridDim.x], gw, sbuf + (cur ^ 1) * RecBase::rec_words, &s_mbar[cur ^ 1], true);
        }
        const u32 dw = rec_fetch(td, gw, srec0, nullptr, false);
        u32* srec = srec0 + dw;
        {
            // this leaf's head / tail words outside the aligned body
            const uintptr_t p0 = (uintptr_t)g, p1 = (uintptr_t)(g + n * 25);
            const uintptr_t a0 = (p0 + 15) & ~(uintptr_t)15, a1 = p1 & ~(uintptr_t)15;
            const u32 nh = (u32)(((a0 < p1 ? a0 : p1) - p0) / 4);
            const uintptr_t t0 = a1 > a0 ? a1 : (a0 < p1 ? a0 : p1);
            const u32 nt = (u32)((p1 - t0) / 4);
            if (tid < nh) srec[tid] = g[tid];
            if (tid >= 32 && tid - 32 < nt) srec[(t0 - p0) / 4 + (tid - 32)] = reinterpret_cast<const u32*>(t0)[tid - 32];
        }
        mbar_wait(&s_mbar[cur], (phase >> cur) & 1u);
        phase ^= 1u << cur;
        __syncthreads();
        {
            ulonglong2 itm[KREC_ITEMS];
#pragma unroll
            for (int q = 0; q < KREC_ITEMS; ++q) {
                const u32 i = q * KREC_THREADS + tid;
                itm[q] = TRecItem::pad();
                if (i < n) {
                    const u32* r = srec + i * 25;
                    itm[q].x = TRec::hi_of(r[0], r[1]);
                    itm[q].y = (TRec::lo_of(r[2]) << 32) | i;
                }
            }
            rec_items_sort<KREC_ITEMS>(itm, n, it, s_cnt, s_range, &s_flag, s_wsum);
        }
        for (u32 i = tid; i < n * 25; i += KREC_THREADS) {
            const u32 r = i / 25, wd = i - r * 25;
            const u32 src = (u32)(it[padidx(r)].y & 0xFFFFFFFFu);
            g[i] = srec[src * 25 + wd];
        }
        __syncthreads();
        cur ^= 1u;
    }
}

// ---------------------------------------------------------------- cell base case
//
// Leaves of up to 16384 (8-byte types) / 8192 (pairs) elements are sorted by one CTA in
// shared memory.
// A leaf's keys already lie between two splitters, so one more distribution step needs no
// splitters: the key range [kmin, kmax] is cut into 2^cb >= n equal cells by the
// order-preserving map floor((key - kmin) * 2^cb / (kmax - kmin + 1)).  Then, as in the
// paper (distribution down to tiny subproblems, finished by insertion sort):
//   1. coalesced load into registers, the key range (warp shuffles + shared atomics);
//   2. cell of every element; its rank inside the cell is the value a shared-memory
//      atomic increment of the cell counter returns (order inside a cell is irrelevant);
//   3. exclusive scan of the cell counts -- thread t owns the run of cells [tE, tE+E), read
//      and written with 128-bit accesses (the counter array has 4 pad words after each
//      run, which also makes those accesses conflict-free) -- and the scatter of every
//      element to base[cell] + rank;
//   4. each thread orders the cells of its run that hold several elements (about one
//      element per cell on average): cells of 2 by one compare-exchange, of 3-4 by a
//      4-element network, larger ones by insertion sort (the cells are already in order);
//   5. write-back by one TMA bulk store of the leaf's 16-byte aligned body (the leaf is
//      staged at the same offset modulo 16 as in global memory).
// f64 leaves are sorted as their order-preserving u64 images (CellWork).
// When every cell is a single key value (span < cells) step 4 has nothing to do.  A leaf
// whose cells would need too much insertion work (keys clustered far below the resolution
// of the cells, e.g. heavy duplicates) is handed to the merge-sort kernel (fallback queue)
// untouched.
#ifndef IPS4O_BASE_WARP_WB  // each warp writes back its threads' cells as soon as it has ordered them
#define IPS4O_BASE_WARP_WB 1
#endif
#ifndef IPS4O_BASE_TMA_WB  // whole-leaf write-back by TMA bulk stores (1) or plain stores (0)
#define IPS4O_BASE_TMA_WB 1
#endif
// Phase profile of the cell base case (tuning builds only): thread 0 of each CTA adds the
// clock64 intervals between the leaf's barriers; the host prints the shares per class.
#ifdef IPS4O_BASE_PROF
__device__ unsigned long long g_base_prof[2][8];
#define BASE_PROF_INIT()                                          \
    unsigned long long bp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};      \
    unsigned long long bp_last = clock64()
#define BASE_PROF_MARK(i)                                         \
    do {                                                          \
        if (threadIdx.x == 0) {                                   \
            const unsigned long long c_ = clock64();              \
            bp_acc[i] += c_ - bp_last;                            \
            bp_last = c_;                                         \
        }                                                         \
    } while (0)
#define BASE_PROF_FLUSH(cls)                                                               \
    do {                                                                                   \
        if (threadIdx.x == 0)                                                              \
            for (int i_ = 0; i_ < 8; ++i_) atomicAdd(&g_base_prof[cls][i_], bp_acc[i_]);  \
    } while (0)
#else
#define BASE_PROF_INIT() do {} while (0)
#define BASE_PROF_MARK(i) do {} while (0)
#define BASE_PROF_FLUSH(cls) do {} while (0)
#endif
template <class TR, int NT, int E>
struct CellBase {
    static constexpr u32 TILE = NT * E;
    static constexpr size_t x_bytes = (size_t)TILE * sizeof(typename TR::V) + 16;  // + alignment shift
    static constexpr size_t cnt_bytes = (size_t)((E + 4) * NT + 8) * 4;
    static constexpr size_t smem = x_bytes + cnt_bytes;
};
template <int E>
__device__ __forceinline__ u32 cpad(u32 c) { return c + 4u * (c / E); }
#ifndef IPS4O_CELL_TILE_CELLS  // cells of a leaf with a wide key span: one per tile slot (1) or one per element (0)
#define IPS4O_CELL_TILE_CELLS 1
#endif
#ifndef IPS4O_CELL_FIX_BUDGET
#define IPS4O_CELL_FIX_BUDGET 16384
#endif
constexpr u32 CELL_FIX_BUDGET = IPS4O_CELL_FIX_BUDGET;  // estimated insertion moves per leaf before falling back

// The cell kernel works on order-preserving u64 images of f64 keys (mapped on load, mapped
// back in shared memory before the write-back): every comparison is then a plain u64 one.
template <class TR> struct CellWork {
    typedef TR T;
    __device__ __forceinline__ static typename TR::V in(typename TR::V v) { return v; }
    __device__ __forceinline__ static typename TR::V out(typename TR::V v) { return v; }
};
template <> struct CellWork<TF64> {
    typedef TU64 T;
    __device__ __forceinline__ static u64 in(u64 v) { return TF64::key(v); }
    __device__ __forceinline__ static u64 out(u64 k) { return (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k; }
};
template <> struct CellWork<TPairF64> {  // f64-key pairs: the key word as its image
    typedef TPair T;
    __device__ __forceinline__ static ulonglong2 in(ulonglong2 v) { return make_ulonglong2(TF64::key(v.x), v.y); }
    __device__ __forceinline__ static ulonglong2 out(ulonglong2 k) {
        return make_ulonglong2((k.x >> 63) ? (k.x & 0x7FFFFFFFFFFFFFFFull) : ~k.x, k.y);
    }
};
template <> struct CellWork<TKV> {  // key-value pairs: sorted as {key, value} pairs
    typedef TPair T;
    __device__ __forceinline__ static ulonglong2 in(ulonglong2 v) { return v; }
    __device__ __forceinline__ static ulonglong2 out(ulonglong2 v) { return v; }
};
template <> struct CellWork<TKVF64> : CellWork<TPairF64> {};
// quartets: cells on the image of k0, the cells' elements ordered by the full lexicographic key
template <> struct CellWork<TQuad> {
    typedef TQuad T;
    __device__ __forceinline__ static Quad in(const Quad& v) { return v; }
    __device__ __forceinline__ static Quad out(const Quad& v) { return v; }
};

#ifndef IPS4O_CELL_MINB1  // resident CTAs per SM the 256-thread class of 8-byte keys is compiled for
#define IPS4O_CELL_MINB1 3
#endif
template <class TR, int NT, int E>
struct CellMinB {
    static constexpr int v = sizeof(typename TR::V) == 8
                                 ? (E >= 16 ? (NT <= 128 ? 6 : NT <= 256 ? IPS4O_CELL_MINB1 : NT <= 512 ? 2 : 1)
                                            : (NT <= 128 ? 8 : NT <= 256 ? 4 : NT <= 512 ? 2 : 1))
                             : sizeof(typename TR::V) == 16 ? (NT <= 256 ? 3 : NT <= 512 ? 2 : 1)
                                                            : (NT <= 256 ? 2 : 1);
};
__device__ __forceinline__ u32 atoms_inc(u32 saddr) {
    u32 r;
    asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(r) : "r"(saddr));
    return r;
}
// predicated forms (the slots of a tile past the leaf's n elements): straight-line code, so that
// the tile's E atomics / loads are in flight together instead of one per basic block
__device__ __forceinline__ u32 atoms_inc_if(u32 saddr, bool p) {
    u32 r = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q atom.shared.add.u32 %0, [%1], 1;\n\t}"
                 : "+r"(r)
                 : "r"(saddr), "r"((u32)p));
    return r;
}
template <class V>
__device__ __forceinline__ void sts_v_if(u32 saddr, const V& v, bool p) {
    if constexpr (sizeof(V) == 8) {
        u64 x;
        memcpy(&x, &v, 8);
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u64 [%0], %1;\n\t}" ::"r"(saddr), "l"(x),
                     "r"((u32)p));
    } else {
        static_assert(sizeof(V) % 16 == 0, "16-byte multiples");
#pragma unroll
        for (u32 o = 0; o < sizeof(V); o += 16) {
            ulonglong2 x;
            memcpy(&x, reinterpret_cast<const char*>(&v) + o, 16);
            asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q st.shared.v2.u64 [%0], {%1, %2};\n\t}" ::"r"(saddr + o),
                         "l"(x.x), "l"(x.y), "r"((u32)p));
        }
    }
}
#ifndef IPS4O_BASE_M2X2  // cells of two elements ordered two per loop iteration
#define IPS4O_BASE_M2X2 0
#endif
#ifndef IPS4O_BASE_PRED  // rank and scatter as predicated straight-line code (1; measured no faster: H base 1.86 = 1.86 ms, C4 1.45 -> 1.50) or one branch per slot (0)
#define IPS4O_BASE_PRED 0
#endif
__device__ __forceinline__ u32 lds_u32(u32 saddr) {
    u32 r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(saddr));
    return r;
}
template <class V>
__device__ __forceinline__ void sts_v(u32 saddr, const V& v) {
    if constexpr (sizeof(V) == 8) {
        u64 x;
        memcpy(&x, &v, 8);
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(saddr), "l"(x));
    } else {
        static_assert(sizeof(V) % 16 == 0, "16-byte multiples");
#pragma unroll
        for (u32 o = 0; o < sizeof(V); o += 16) {
            ulonglong2 x;
            memcpy(&x, reinterpret_cast<const char*>(&v) + o, 16);
            asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(saddr + o), "l"(x.x), "l"(x.y));
        }
    }
}
// Leaves are taken from the class queue through an atomic ticket (the grid is the resident
// CTAs: a CTA that finishes early takes the next leaf); the next leaf's descriptor is known
// one leaf ahead and its elements are prefetched into L2 by a TMA bulk prefetch.
// Shared scalars of one cell-sort leaf.
template <int NW>
struct CellSh {
    u32 r[4];        // 32-bit key-range halves: hi min / max, lo min / max
    u64 r64[2];      // exact 64-bit range (leaves whose high halves are close)
    u32 flag, wsum[NW];
};

// The cell sort of one leaf td (<= NT*E elements) by the whole CTA (steps 1-5 above): X0 is the
// leaf's shared-memory tile (TILE elements + 16 bytes), cnt the cell counters.  after_range() is
// called by every thread between the barriers that follow the key-range reduction (the caller's
// next-leaf bookkeeping).  Returns 0 when the leaf is sorted in place, 1 when its keys are too
// clustered for the cells (it is left untouched for the merge sort).
// The leaf's elements into registers (element j*NT + tid; the slots past n load a copy of
// element n-1, which changes no range and takes no part in the steps after the range): plain
// loads with no use of the values, so that they stay in flight behind whatever the caller does
// next (k_base_cell issues the next leaf's loads while this leaf's cells are ordered).
template <class TR, int NT, int E>
__device__ __forceinline__ void cell_load(const TaskDesc& td, const Mem<TR>& mem, typename TR::V (&v)[E]) {
    const u32 n = (u32)(td.hi - td.lo);
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = mem.ld(td.lo + min((u32)(j * NT) + threadIdx.x, n - 1u));
}

// v: the leaf's elements as cell_load left them.  after_scatter() is called once v has been
// consumed (the scatter), unless the leaf returns early (all keys equal, or 1): it may refill v.
template <class TR, int NT, int E, class F, class G>
__device__ __forceinline__ int cell_leaf_pre(const TaskDesc& td, const Mem<TR>& mem, typename TR::V* data,
                                             typename TR::V* X0, u32* cnt, CellSh<NT / 32>& S,
                                             typename TR::V (&v)[E], F&& after_range, G&& after_scatter) {
    typedef typename TR::V V;
    typedef CellBase<TR, NT, E> CB;
    typedef typename CellWork<TR>::T TW;
    constexpr bool PRED = IPS4O_BASE_PRED && NT < 1024;  // (1024 threads: 64 registers, the straight-line form spills)
    const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint4* myrun = reinterpret_cast<uint4*>(cnt + cpad<E>(tid * E));  // this thread's E counters
    const u32 n = (u32)(td.hi - td.lo);
    V* g = data + td.lo;
    // the leaf in shared memory starts at the same offset modulo 16 bytes as in global
    // memory, so that its aligned body leaves by one TMA bulk store
    const u32 p = (sizeof(V) == 8 && !TR::KV) ? (u32)((reinterpret_cast<uintptr_t>(g) >> 3) & 1u) : 0u;
    V* const X = X0 + p;
    if (tid == 0) {
        S.r[0] = ~0u;
        S.r[1] = 0u;
        S.r[2] = ~0u;
        S.r[3] = 0u;
        S.r64[0] = ~0ull;
        S.r64[1] = 0ull;
        S.flag = 0;
    }
#pragma unroll
    for (int k = 0; k < E / 4; ++k) myrun[k] = make_uint4(0u, 0u, 0u, 0u);
    // 1. load (element j*NT + tid) and the range of the keys' high 32-bit halves
    //    (warp reductions in one REDUX instruction each)
    //    (branch-free over the whole tile: the slots past n load a copy of element n-1,
    //    which changes no range; they take no part in the steps below)
    u32 hmin = ~0u, hmax = 0u;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        v[j] = CellWork<TR>::in(v[j]);
        const u32 h = (u32)(TW::key(v[j]) >> 32);
        hmin = min(hmin, h);
        hmax = max(hmax, h);
    }
    hmin = __reduce_min_sync(0xffffffffu, hmin);
    hmax = __reduce_max_sync(0xffffffffu, hmax);
    __syncthreads();  // the range words and the counters are reset; the previous leaf is done
    BASE_PROF_MARK(1);
    if (lane == 0) {
        atomicMin(&S.r[0], hmin);
        atomicMax(&S.r[1], hmax);
    }
    __syncthreads();
    BASE_PROF_MARK(2);
    after_range();  // (the caller: next-leaf bookkeeping between the barriers)
    // the key range: from the high halves when they are far apart (a conservative range
    // at most (d+1)/(d-1) wider than the exact one for d = hmax - hmin >= 16); exact from
    // the low halves when all high halves are equal; exact 64-bit otherwise
    const u32 H0 = S.r[0], H1 = S.r[1];
    u64 kmin, span;
    if (H1 - H0 >= 16u) {
        kmin = (u64)H0 << 32;
        span = ((((u64)H1) << 32) | 0xFFFFFFFFull) - kmin;
    } else if (H1 == H0) {
        u32 lmin = ~0u, lmax = 0u;
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const u32 l = (u32)TW::key(v[j]);
            lmin = min(lmin, l);
            lmax = max(lmax, l);
        }
        lmin = __reduce_min_sync(0xffffffffu, lmin);
        lmax = __reduce_max_sync(0xffffffffu, lmax);
        if (lane == 0) {
            atomicMin(&S.r[2], lmin);
            atomicMax(&S.r[3], lmax);
        }
        __syncthreads();
        kmin = ((u64)H0 << 32) | S.r[2];
        span = (u64)(S.r[3] - S.r[2]);
    } else {
        u64 mn = ~0ull, mx = 0ull;
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const u64 k = TW::key(v[j]);
            mn = k < mn ? k : mn;
            mx = k > mx ? k : mx;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const u64 a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
        }
        if (lane == 0) {
            atomicMin(&S.r64[0], mn);
            atomicMax(&S.r64[1], mx);
        }
        __syncthreads();
        kmin = S.r64[0];
        span = S.r64[1] - kmin;
    }
    // all keys equal: already sorted (no write) -- for keys of several parts (quartets) only
    // the first part is equal: the merge sort orders the rest
    if (span == 0) return TR::PARTS > 1 ? 1 : 0;
    // cell(key) = floor(x * ncell / (span32 + 1)) for x = (key - kmin) >> s, the top 32
    // bits of the offset (s = 0 when the span fits 32 bits): one 32x32 multiply-high with
    // a per-leaf multiplier, monotone, onto [0, ncell).  (mul = floor(ncell * 2^32 /
    // (span32 + 1)) < 2^32 for span32 >= ncell; otherwise s = 0 and the cell is x itself,
    // a single key value.)
    const u32 bl = 64u - (u32)__clzll((long long)span);
    const u32 sh = bl > 32u ? bl - 32u : 0u;
    const u32 span32 = (u32)(span >> sh);
    // cells: one per key value when the span fits the tile (nothing to order inside a cell),
    // else one per element (at most one element per cell on average)
#if IPS4O_CELL_TILE_CELLS
    // (every counter of the tile is a cell: the counter scan covers the whole tile anyway, more
    // cells than elements mean fewer elements per cell, and every thread owns cells to order)
    const u32 ncell = span < (u64)CB::TILE ? max(n, (u32)span + 1u) : CB::TILE;
#else
    const u32 ncell = span < (u64)CB::TILE ? max(n, (u32)span + 1u) : n;
#endif
    const u32 mul = span32 >= ncell ? (u32)(((u64)ncell << 32) / ((u64)span32 + 1ull)) : 0u;
    // 2. cell and rank inside the cell
    const u32 s_cnt = (u32)__cvta_generic_to_shared(cnt);
    u32 cr[E];  // cell | rank << 16
#pragma unroll
    for (int j = 0; j < E; ++j) {
        if constexpr (PRED) {
            // (a slot past n holds a copy of element n-1: its cell is a valid one, only the count is skipped)
            const u32 x = (u32)((TW::key(v[j]) - kmin) >> sh);
            const u32 c = mul ? __umulhi(x, mul) : x;
            cr[j] = c | (atoms_inc_if(s_cnt + 4u * cpad<E>(c), (u32)(j * NT) + tid < n) << 16);
        } else if (j * NT + tid < n) {
            const u32 x = (u32)((TW::key(v[j]) - kmin) >> sh);
            const u32 c = mul ? __umulhi(x, mul) : x;
            cr[j] = c | (atoms_inc(s_cnt + 4u * cpad<E>(c)) << 16);
        }
    }
    __syncthreads();
    BASE_PROF_MARK(3);
    // 3. exclusive scan of the counts (own run of E cells, 128-bit accesses)
    u32 sum = 0;
#pragma unroll
    for (int k = 0; k < E / 4; ++k) {
        const uint4 q = myrun[k];
        sum += q.x + q.y + q.z + q.w;
    }
    u32 incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (u32)o) incl += y;
    }
    if (lane == 31) S.wsum[w] = incl;
    __syncthreads();
    BASE_PROF_MARK(4);
    u32 base = incl - sum;
    for (u32 ww = 0; ww < w; ++ww) base += S.wsum[ww];
    u32 bigwork = 0;  // insertion work of this run's cells (~m^2 / 4 for large cells)
    {
        u32 run = base;
#pragma unroll
        for (int k = 0; k < E / 4; ++k) {
            uint4 q = myrun[k];
            u32 x;
            x = q.x; q.x = run; run += x; if (x > 8) bigwork += x * x / 4;
            x = q.y; q.y = run; run += x; if (x > 8) bigwork += x * x / 4;
            x = q.z; q.z = run; run += x; if (x > 8) bigwork += x * x / 4;
            x = q.w; q.w = run; run += x; if (x > 8) bigwork += x * x / 4;
            myrun[k] = q;
        }
    }
    if (bigwork && (mul || TR::PARTS > 1)) atomicAdd(&S.flag, bigwork);
    if (IPS4O_BASE_TMA_WB && tid == 0) bulk_wait_read0();  // the previous leaf has left X
    __syncthreads();
    BASE_PROF_MARK(5);
    if (S.flag > CELL_FIX_BUDGET) return 1;  // clustered keys (heavy duplicates in few cells): the caller hands the leaf on
    // the end of this thread's run of cells (the next thread's first base), read while every
    // counter is still this leaf's: with per-warp write-back a thread may start the next leaf
    // (and reset its counters) while this one still orders its cells
    const u32 run_end = tid + 1 < (u32)NT ? cnt[cpad<E>((tid + 1) * E)] : n;
    const u32 run_beg = cnt[cpad<E>(tid * E)];
    {
        const u32 s_x = (u32)__cvta_generic_to_shared(X);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            if constexpr (PRED) {
                const u32 pos = lds_u32(s_cnt + 4u * cpad<E>(cr[j] & 0xFFFFu)) + (cr[j] >> 16);
                sts_v_if<V>(s_x + pos * (u32)sizeof(V), v[j], (u32)(j * NT) + tid < n);
            } else if (j * NT + tid < n) {
                const u32 pos = lds_u32(s_cnt + 4u * cpad<E>(cr[j] & 0xFFFFu)) + (cr[j] >> 16);
                sts_v<V>(s_x + pos * (u32)sizeof(V), v[j]);
            }
        }
    }
    after_scatter();
    __syncthreads();
    BASE_PROF_MARK(6);
    // 4. order the cells of this thread's run that hold several elements (PAPER.md:403
    //    finishes small subproblems by insertion sort): cells of 2-4 elements by a
    //    4-element sorting network over the cell padded with the largest key (pads never
    //    move: a comparator swaps only on strictly smaller keys), larger ones by insertion
    //    sort.  Singleton cells need nothing; nothing at all when every cell is a single
    //    key value.
    if (mul || TR::PARTS > 1) {  // (cells of one key part value may differ in the later parts)
        u32 bs[E + 1];
#pragma unroll
        for (int k = 0; k < E / 4; ++k) {
            const uint4 q = myrun[k];
            bs[4 * k] = q.x;
            bs[4 * k + 1] = q.y;
            bs[4 * k + 2] = q.z;
            bs[4 * k + 3] = q.w;
        }
        bs[E] = run_end;
        // cells of 2 (most multi-element cells), of 3-4 and larger ones in separate
        // loops, so that a warp's lanes run the same code in each
        u32 m2 = 0, m34 = 0, mbig = 0;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const u32 m = bs[k + 1] - bs[k];
            m2 |= (m == 2u ? 1u : 0u) << k;
            m34 |= (m - 3u <= 1u ? 1u : 0u) << k;
            mbig |= (m > 4u ? 1u : 0u) << k;
        }
        const u32 enext = bs[E];
#if IPS4O_BASE_M2X2
        // (two cells per iteration: their dependent shared-memory loads overlap)
        while (m2) {
            const u32 k = (u32)__ffs(m2) - 1u;
            m2 &= m2 - 1u;
            const u32 k2 = m2 ? (u32)__ffs(m2) - 1u : k;
            m2 &= m2 - 1u;
            const u32 b = cnt[cpad<E>(tid * E + k)], b2 = cnt[cpad<E>(tid * E + k2)];
            const V x0 = X[b], x1 = X[b + 1], y0 = X[b2], y1 = X[b2 + 1];
            if (TW::less(x1, x0)) {
                X[b] = x1;
                X[b + 1] = x0;
            }
            if (k2 != k && TW::less(y1, y0)) {
                X[b2] = y1;
                X[b2 + 1] = y0;
            }
        }
#else
        while (m2) {
            const u32 k = (u32)__ffs(m2) - 1u;
            m2 &= m2 - 1u;
            const u32 b = cnt[cpad<E>(tid * E + k)];
            const V x0 = X[b], x1 = X[b + 1];
            if (TW::less(x1, x0)) {
                X[b] = x1;
                X[b + 1] = x0;
            }
        }
#endif
        while (m34) {
            const u32 k = (u32)__ffs(m34) - 1u;
            m34 &= m34 - 1u;
            const u32 b = cnt[cpad<E>(tid * E + k)];
            const u32 e = k + 1 < (u32)E ? cnt[cpad<E>(tid * E + k + 1)] : enext;
            const V pd = TW::pad();
            V x0 = X[b], x1 = X[b + 1], x2 = X[b + 2];
            V x3 = e - b > 3u ? X[b + 3] : pd;
            auto cas = [](V& lo, V& hi) {
                const bool sw = TW::less(hi, lo);
                const V t = sw ? hi : lo;
                hi = sw ? lo : hi;
                lo = t;
            };
            cas(x0, x1);
            cas(x2, x3);
            cas(x0, x2);
            cas(x1, x3);
            cas(x1, x2);
            X[b] = x0;
            X[b + 1] = x1;
            X[b + 2] = x2;
            if (e - b > 3u) X[b + 3] = x3;
        }
        while (mbig) {
            const u32 k = (u32)__ffs(mbig) - 1u;
            mbig &= mbig - 1u;
            const u32 b = cnt[cpad<E>(tid * E + k)];
            const u32 e = k + 1 < (u32)E ? cnt[cpad<E>(tid * E + k + 1)] : enext;
            for (u32 i = b + 1; i < e; ++i) {
                const V x = X[i];
                u32 q = i;
                while (q > b && TW::less(x, X[q - 1])) {
                    X[q] = X[q - 1];
                    --q;
                }
                X[q] = x;
            }
        }
    }
#if IPS4O_BASE_WARP_WB
    // 5. write back of a leaf whose cells were ordered: warp by warp -- the cells of a warp's
    //    32 runs are the contiguous range [first base of lane 0, end of lane 31) of the tile,
    //    so each warp stores its range (coalesced) as soon as its own lanes are done, with no
    //    CTA barrier waiting for the slowest warp's cells; the next leaf's barriers order
    //    these reads of X before X is overwritten.  (Leaves with one key value per cell have
    //    nothing to order: the whole-leaf TMA store below.)
    if (mul || TR::PARTS > 1) {
        __syncwarp();
        const u32 wbeg = __shfl_sync(0xffffffffu, run_beg, 0), wend = __shfl_sync(0xffffffffu, run_end, 31);
        for (u32 i = wbeg + lane; i < wend; i += 32) mem.st(td.lo + i, CellWork<TR>::out(X[i]));
        return 0;
    }
#endif
    if constexpr (TR::KV) {
        // 5. write back: key and value arrays by coalesced stores
        __syncthreads();
        for (u32 i = tid; i < n; i += NT) mem.st(td.lo + i, CellWork<TR>::out(X[i]));
        return 0;
    }
    if constexpr (!std::is_same<TW, TR>::value) {
        __syncthreads();
        for (u32 i = tid; i < n; i += NT) X[i] = CellWork<TR>::out(X[i]);
    }
#if IPS4O_BASE_TMA_WB
    fence_proxy_async_smem();
    __syncthreads();
    BASE_PROF_MARK(7);
    // 5. write back: the 16-byte aligned body by one TMA bulk store (read before the next
    //    leaf's scatter), the element before / after it by plain stores
    {
        const u32 i0 = p < n ? p : n;
        const u32 i1 = sizeof(V) == 8 ? i0 + ((n - i0) & ~1u) : n;
        if (tid == 0 && i1 > i0) {
            bulk_s2g(g + i0, X + i0, (i1 - i0) * (u32)sizeof(V));
            bulk_commit();
        }
        if (tid == 32 && i0 > 0) g[0] = X[0];
        if (tid == 64 && i1 < n) g[n - 1] = X[n - 1];
    }
#else
    __syncthreads();
    BASE_PROF_MARK(7);
    // 5. write back
    for (u32 i = tid; i < n; i += NT) g[i] = X[i];
#endif
    return 0;
}

// One leaf, loaded here.
template <class TR, int NT, int E, class F>
__device__ __forceinline__ int cell_leaf(const TaskDesc& td, const Mem<TR>& mem, typename TR::V* data,
                                         typename TR::V* X0, u32* cnt, CellSh<NT / 32>& S, F&& after_range) {
    typename TR::V v[E];
    cell_load<TR, NT, E>(td, mem, v);
    return cell_leaf_pre<TR, NT, E>(td, mem, data, X0, cnt, S, v, after_range, []() {});
}

#ifndef IPS4O_BASE_PIPE  // the next leaf's loads issued behind this leaf's scatter (measured slower: H base 1.86 -> 1.88 ms; off)
#define IPS4O_BASE_PIPE 0
#endif
template <class TR, int NT, int E>
__global__ void __launch_bounds__(NT, (CellMinB<TR, NT, E>::v))
    k_base_cell(const TaskDesc* tasks, const u32* d_ntasks, u32 qcap, u32* ticket, const LevelDyn* dyn,
                TaskDesc* fb_queue, u32* fb_count, u32 fb_cap) {
    typedef typename TR::V V;
    typedef CellBase<TR, NT, E> CB;
    static_assert(E % 4 == 0, "cell runs are read as 128-bit vectors");
    extern __shared__ __align__(16) unsigned char smc[];
    V* const X0 = reinterpret_cast<V*>(smc);
    u32* cnt = reinterpret_cast<u32*>(smc + CB::x_bytes);
    __shared__ CellSh<NT / 32> sh;
    __shared__ u32 s_next[2];
    const u32 ntasks = min(*d_ntasks, qcap);  // (the count lives on the device: the grid is fixed)
    const Mem<TR> mem(dyn->data, dyn->vals);
    V* data = reinterpret_cast<V*>(dyn->data);  // (AoS types: the leaf's TMA write-back)
    const u32 tid = threadIdx.x;
    if (tid == 0) s_next[0] = atomicAdd(ticket, 1u);
    __syncthreads();
    constexpr bool PIPE = IPS4O_BASE_PIPE && NT < 1024;  // (1024 threads: 64 registers, no room for a second leaf)
    u32 cur = s_next[0], par = 1;
    V v[E];
    TaskDesc td = cur < ntasks ? tasks[cur] : TaskDesc{0, 1, 0u, 0u};
    if (PIPE && cur < ntasks) cell_load<TR, NT, E>(td, mem, v);
    while (cur < ntasks) {
        if (tid == 0) s_next[par] = atomicAdd(ticket, 1u);  // the next leaf (read after the barriers below)
        u32 nxt = ntasks;
        TaskDesc tn = td;
        if ((u64)(td.hi - td.lo) > (u64)CB::TILE) {
            // (a class whose tile is smaller than the base-case capacity: the rare larger leaves
            // go to the merge sort)
            __syncthreads();
            nxt = s_next[par];
            if (tid == 0) {
                const u32 q = atomicAdd(fb_count, 1u);
                if (q < fb_cap) fb_queue[q] = td;
            }
            __syncthreads();
            cur = nxt;
            par ^= 1u;
            if (cur < ntasks) {
                td = tasks[cur];
                if (PIPE) cell_load<TR, NT, E>(td, mem, v);
            }
            continue;
        }
        if (!PIPE) cell_load<TR, NT, E>(td, mem, v);
        bool pre = false;
        const int r = cell_leaf_pre<TR, NT, E>(td, mem, data, X0, cnt, sh, v, [&]() {
            nxt = s_next[par];
            if (nxt < ntasks) tn = tasks[nxt];
            if (tid == 0 && nxt < ntasks) {
                // the next leaf's elements into L2 (TMA bulk prefetch)
                if constexpr (TR::KV) {
                    for (int h = 0; h < 2; ++h) {
                        const u64* arr = h ? mem.v : mem.k;
                        const uintptr_t a0 = reinterpret_cast<uintptr_t>(arr + tn.lo) & ~(uintptr_t)15;
                        const uintptr_t a1 = (reinterpret_cast<uintptr_t>(arr + tn.hi) + 15) & ~(uintptr_t)15;
                        if (a1 > a0) bulk_prefetch_l2(reinterpret_cast<const void*>(a0), (u32)(a1 - a0));
                    }
                } else {
                    const uintptr_t a0 = reinterpret_cast<uintptr_t>(data + tn.lo) & ~(uintptr_t)15;
                    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(data + tn.hi) + 15) & ~(uintptr_t)15;
                    if (a1 > a0) bulk_prefetch_l2(reinterpret_cast<const void*>(a0), (u32)(a1 - a0));
                }
            }
        }, [&]() {
            // v has been scattered: the next leaf's loads fly while this leaf's cells are ordered
            pre = true;
            if (PIPE && nxt < ntasks) cell_load<TR, NT, E>(tn, mem, v);
        });
        if (r == 1 && tid == 0) {
            const u32 q = atomicAdd(fb_count, 1u);
            if (q < fb_cap) fb_queue[q] = td;
        }
        if (PIPE && !pre && nxt < ntasks) cell_load<TR, NT, E>(tn, mem, v);
        cur = nxt;
        td = tn;
        par ^= 1u;
    }
    if (IPS4O_BASE_TMA_WB && tid == 0) bulk_wait0();
}

template <class TR, int THREADS, int ITEMS>
struct BaseClass {
    static constexpr u32 TILE = THREADS * ITEMS;
    static constexpr size_t smem = (size_t)padidx(TILE) * sizeof(typename TR::V) + 16;
};

// The fallback queue of the 8-byte key types: leaves the cell kernels of the smaller classes
// handed back get a second chance in the largest tile (a leaf of few distinct values whose key
// span exceeds its own class's tile but not this one has one key value per cell here: nothing
// to order), and only leaves that are clustered at this resolution too are merge-sorted.
#ifndef IPS4O_FB_CELL2
#define IPS4O_FB_CELL2 1
#endif
template <class TR, int THREADS, int ITEMS>
struct FbCell2 {
    static constexpr bool on = IPS4O_FB_CELL2 && sizeof(typename TR::V) == 8 && !TR::KV && TR::PARTS == 1;
    static constexpr size_t cell_smem = CellBase<TR, THREADS, ITEMS>::smem;
    static constexpr size_t merge_smem = (size_t)padidx(THREADS * ITEMS) * sizeof(typename TR::V) + 16;
    static constexpr size_t smem = on ? (cell_smem > merge_smem ? cell_smem : merge_smem) : merge_smem;
};
template <class TR, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) k_base_fb(const TaskDesc* tasks, u32 start, const u32* d_ntasks,
                                                      const LevelDyn* dyn, u32 cap) {
    const u32 ntasks = min(*d_ntasks, cap);  // tasks [start, ntasks) (the count lives on the device)
    typedef typename TR::V V;
    typedef CellBase<TR, THREADS, ITEMS> CB;
    extern __shared__ __align__(16) unsigned char smem5[];
    V* s = reinterpret_cast<V*>(smem5);
    u32* cnt = reinterpret_cast<u32*>(smem5 + CB::x_bytes);
    __shared__ CellSh<THREADS / 32> sh;
    const Mem<TR> mem(dyn->data, dyn->vals);
    V* data = reinterpret_cast<V*>(dyn->data);
    const u32 tid = threadIdx.x;
    for (u32 ti = start + blockIdx.x; ti < ntasks; ti += gridDim.x) {
        const TaskDesc td = tasks[ti];
        const u32 n = (u32)(td.hi - td.lo);
        if (n < 2) continue;
        if (cell_leaf<TR, THREADS, ITEMS>(td, mem, data, s, cnt, sh, []() {}) == 0) continue;
        // clustered at this resolution too: merge sort (the tile is free once every warp has left
        // the previous leaf and its TMA store has read the tile)
        if (IPS4O_BASE_TMA_WB && tid == 0) bulk_wait_read0();
        __syncthreads();
        const u32 n16 = (n + ITEMS - 1) / ITEMS * ITEMS;
        for (u32 i = tid; i < n16; i += THREADS) s[padidx(i)] = i < n ? mem.ld(td.lo + i) : TR::pad();
        __syncthreads();
        block_sort_smem<TR, THREADS, ITEMS>(s, n);
        for (u32 i = tid; i < n; i += THREADS) mem.st(td.lo + i, s[padidx(i)]);
        __syncthreads();
    }
    if (IPS4O_BASE_TMA_WB && tid == 0) bulk_wait0();
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
        out[i] = classify_key(TR::key(in[i], 0), tree, spl, logk, kp, eq);
}

}  // namespace ips4o
