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
__global__ void __launch_bounds__(THREADS) k_base_merge(const TaskDesc* tasks, const u32* d_ntasks, void* vdata) {
    const u32 ntasks = *d_ntasks;
    typedef typename TR::V V;
    extern __shared__ __align__(16) unsigned char smem5[];
    V* s = reinterpret_cast<V*>(smem5);
    V* data = reinterpret_cast<V*>(vdata);
    const u32 tid = threadIdx.x;
    for (u32 ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
        const TaskDesc td = tasks[ti];
        const u32 n = (u32)(td.hi - td.lo);
        const u32 n16 = (n + ITEMS - 1) / ITEMS * ITEMS;
        V* g = data + td.lo;
        // coalesced load; the last thread's items past n are padding
        for (u32 i = tid; i < n16; i += THREADS) s[padidx(i)] = i < n ? g[i] : TR::pad();
        __syncthreads();
        block_sort_smem<TR, THREADS, ITEMS>(s, n);
        for (u32 i = tid; i < n; i += THREADS) g[i] = s[padidx(i)];
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
constexpr int KREC_THREADS = 256, KREC_ITEMS = 4;  // CAP = 1024 records
struct RecBase {
    static constexpr size_t items_bytes = (size_t)padidx(KREC_THREADS * KREC_ITEMS) * 16 + 16;
    static constexpr size_t smem = items_bytes + (size_t)KREC_THREADS * KREC_ITEMS * 100;
};

__global__ void __launch_bounds__(KREC_THREADS) k_base_rec(const TaskDesc* tasks, u32 ntasks, void* vdata) {
    extern __shared__ __align__(16) unsigned char smem5[];
    ulonglong2* it = reinterpret_cast<ulonglong2*>(smem5);
    u32* srec = reinterpret_cast<u32*>(smem5 + RecBase::items_bytes);
    u32* gw = reinterpret_cast<u32*>(vdata);
    const u32 tid = threadIdx.x;
    for (u32 ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
        const TaskDesc td = tasks[ti];
        const u32 n = (u32)(td.hi - td.lo);
        const u32 n16 = (n + KREC_ITEMS - 1) / KREC_ITEMS * KREC_ITEMS;
        u32* g = gw + td.lo * 25;
        for (u32 i = tid; i < n * 25; i += KREC_THREADS) srec[i] = g[i];
        __syncthreads();
        for (u32 i = tid; i < n16; i += KREC_THREADS) {
            ulonglong2 x = TRecItem::pad();
            if (i < n) {
                const u32* r = srec + i * 25;
                x.x = TRec::hi_of(r[0], r[1]);
                x.y = (TRec::lo_of(r[2]) << 32) | i;
            }
            it[padidx(i)] = x;
        }
        __syncthreads();
        block_sort_smem<TRecItem, KREC_THREADS, KREC_ITEMS>(it, n);
        for (u32 i = tid; i < n * 25; i += KREC_THREADS) {
            const u32 r = i / 25, wd = i - r * 25;
            const u32 src = (u32)(it[padidx(r)].y & 0xFFFFFFFFu);
            g[i] = srec[src * 25 + wd];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- radix base case
//
// Leaves of up to 8192 elements (8/16-byte types) are sorted by one CTA entirely in shared
// memory.  A merge sort spends one pass over shared memory per bit of order it establishes;
// a k-way distribution establishes log2(k) bits per pass (the point of the paper's
// samplesort), and for a leaf -- whose keys already lie between two
// splitters -- the distribution needs no splitters: the keys' most significant varying bits
// are a monotone bucket function.  So:
//   1. load the leaf (coalesced) into registers, "warp-striped" (warp w holds positions
//      [32*E*w, 32*E*(w+1)), lane l every 32nd of them), and find its key range
//      [kmin, kmax]; (key - kmin) is order-preserving with h = bitlen(kmax - kmin) bits;
//   2. two stable 8-bit counting passes (least significant digit first) over the window
//      [h-16, h) of (key - kmin): per pass, warp-aggregated ranks from 8 ballots
//      (no shared-memory atomics), per-warp digit counters turned into offsets by one
//      thread per digit, and a scatter into the shared-memory tile;
//   3. the leaf is now ordered by its 16 most significant varying bits; runs of keys equal
//      in that window (rare: a few pairs per leaf for spread keys; equal keys need nothing)
//      are finished by insertion sort -- the paper's own base-case sort --
//      in place in shared memory;
//   4. coalesced write-back.
// A leaf whose runs would need too much insertion work is handed to the merge-sort kernel
// (fallback queue) untouched.  Padding elements (positions >= n in a partly filled warp)
// get the largest digit and, the passes being stable, stay behind every real element.
template <class TR, int NT>
struct RadixBase {
    static constexpr int E = 8;
    static constexpr int NW = NT / 32;
    static constexpr u32 TILE = NT * E;
    static constexpr size_t x_bytes = (size_t)TILE * sizeof(typename TR::V);
    static constexpr size_t cnt_bytes = (size_t)NW * 256 * 2;
    static constexpr size_t smem = x_bytes + cnt_bytes;
};
constexpr u32 RADIX_FIX_BUDGET = 2048;  // insertion-sort moves per thread before falling back

template <class TR, int NT>
__global__ void __launch_bounds__(NT) k_base_radix(const TaskDesc* tasks, u32 ntasks, void* vdata,
                                                   TaskDesc* fb_queue, u32* fb_count, u32 fb_cap) {
    typedef typename TR::V V;
    typedef RadixBase<TR, NT> RB;
    constexpr int E = RB::E, NW = RB::NW;
    extern __shared__ __align__(16) unsigned char smr[];
    V* X = reinterpret_cast<V*>(smr);
    unsigned short* cnt0 = reinterpret_cast<unsigned short*>(smr + RB::x_bytes);
    __shared__ u64 s_range[2];
    __shared__ u32 s_flag, s_wsum[8], s_dbase[256], s_part[NT];
    V* data = reinterpret_cast<V*>(vdata);
    const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const u32 lt = lanemask_lt();
    // counters start at zero; each pass zeroes its set once the scatter is done
    for (u32 i = tid; i < (u32)NW * 256u; i += NT) cnt0[i] = 0;
    for (u32 ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
        const TaskDesc td = tasks[ti];
        const u32 n = (u32)(td.hi - td.lo);
        V* g = data + td.lo;
        __syncthreads();  // the previous leaf is finished (tile, flags)
        if (tid == 0) {
            s_range[0] = ~0ull;
            s_range[1] = 0ull;
            s_flag = 0;
        }
        __syncthreads();
        // 1. load (warp-striped) and the key range [kmin, kmax] of the leaf
        const u32 wbase = w * 32u * E;
        const bool wact = wbase < n;
        V v[E];
        u64 kmin = ~0ull, kmax = 0ull;
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const u32 idx = wbase + j * 32 + lane;
            if (idx < n) {
                v[j] = g[idx];
                const u64 k = TR::key(v[j]);
                kmin = k < kmin ? k : kmin;
                kmax = k > kmax ? k : kmax;
            } else {
                v[j] = TR::pad();
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const u64 a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
            kmin = a < kmin ? a : kmin;
            kmax = b > kmax ? b : kmax;
        }
        if (lane == 0 && wact) {
            atomicMin(&s_range[0], kmin);
            atomicMax(&s_range[1], kmax);
        }
        __syncthreads();
        kmin = s_range[0];
        const u64 span = s_range[1] - kmin;
        if (span == 0) continue;  // all keys equal: already sorted (no write)
        // the keys are ordered by (key - kmin); its h significant bits, the top 16 of them
        // in the counting passes
        const u32 h = 64u - (u32)__clzll((long long)span);
        const u32 lo_bit = h > 16u ? h - 16u : 0u;
        const u32 npass = (h - lo_bit + 7u) / 8u;
        // 2. stable counting passes over the window [lo_bit, h)
        for (u32 p = 0; p < npass; ++p) {
            const u32 shift = lo_bit + 8u * p;
            unsigned short* cnt = cnt0;
            u32 pos[E], dig[E];
            if (wact) {
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    // digit of (key - kmin); padding takes the largest digit
                    const bool real = wbase + j * 32 + lane < n;
                    const u32 d = real ? (u32)((TR::key(v[j]) - kmin) >> shift) & 255u : 255u;
                    dig[j] = d;
                    u32 peers = 0xffffffffu;
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const bool bit = (d >> b) & 1u;
                        const u32 x = __ballot_sync(0xffffffffu, bit);
                        peers &= bit ? x : ~x;
                    }
                    const u32 leader = __ffs(peers) - 1;
                    u32 base = 0;
                    if (lane == leader) {
                        base = cnt[w * 256 + d];
                        cnt[w * 256 + d] = (unsigned short)(base + __popc(peers));
                    }
                    base = __shfl_sync(0xffffffffu, base, leader);
                    pos[j] = base + __popc(peers & lt);
                    __syncwarp();
                }
            }
            __syncthreads();
            // offsets: thread (q, d) owns digit d of warps [8q, 8q+8); group partial sums,
            // exclusive prefixes over groups and over digits, then per-warp offsets
            const u32 d = tid & 255u, q = tid >> 8;
            u32 c[8], part = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                c[k] = cnt[(8 * q + k) * 256 + d];
                const u32 t = part;
                part += c[k];
                c[k] = t;
            }
            s_part[q * 256 + d] = part;
            __syncthreads();
            if (q == 0) {
                u32 tot = 0;
#pragma unroll
                for (int qq = 0; qq < NT / 256; ++qq) {
                    const u32 x = s_part[qq * 256 + d];
                    s_part[qq * 256 + d] = tot;
                    tot += x;
                }
                u32 incl = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= (u32)o) incl += y;
                }
                if (lane == 31) s_wsum[w] = incl;
                s_dbase[d] = incl - tot;
            }
            __syncthreads();
            {
                u32 base = s_dbase[d] + s_part[q * 256 + d];
                for (u32 ww = 0; ww < (d >> 5); ++ww) base += s_wsum[ww];
#pragma unroll
                for (int k = 0; k < 8; ++k) cnt[(8 * q + k) * 256 + d] = (unsigned short)(base + c[k]);
            }
            __syncthreads();
            if (wact) {
#pragma unroll
                for (int j = 0; j < E; ++j) X[cnt[w * 256 + dig[j]] + pos[j]] = v[j];
            }
            __syncthreads();
            // the counters are free again: zero them for the next pass or leaf
            for (u32 i = tid; i < (u32)NW * 256u; i += NT) cnt[i] = 0;
            if (wact) {
#pragma unroll
                for (int j = 0; j < E; ++j) v[j] = X[wbase + j * 32 + lane];
            }
            __syncthreads();
        }
        // 3. runs of keys equal in the window but not equal: insertion sort (in place).
        //    Thread t scans positions [t*per, (t+1)*per) in order and sorts every run that
        //    starts there (a run may extend into the next thread's range, which skips it).
        if (lo_bit > 0) {
            u32 budget = RADIX_FIX_BUDGET;
            const u32 per = (n + NT - 1) / NT;
            const u32 i0 = tid * per, i1 = i0 + per < n ? i0 + per : n;
            if (i0 < i1) {
                // window of the element before the range: a run entering the range belongs
                // to the previous thread
                u64 wprev = i0 > 0 ? (TR::key(X[i0 - 1]) - kmin) >> lo_bit : ~0ull;
                u32 rs = i0;          // start of the current run
                bool own = false;     // the current run started inside this range
                for (u32 i = i0; i < n; ++i) {
                    const u64 wi = (TR::key(X[i]) - kmin) >> lo_bit;
                    if (wi != wprev) {
                        // run [rs, i) ends: sort it if it is ours and longer than one
                        if (own && i - rs > 1) {
                            for (u32 k = rs + 1; k < i && budget; ++k) {
                                const V x = X[k];
                                u32 q = k;
                                while (q > rs && TR::less(x, X[q - 1]) && budget) {
                                    X[q] = X[q - 1];
                                    --q;
                                    --budget;
                                }
                                X[q] = x;
                            }
                        }
                        if (i >= i1) break;  // runs starting beyond the range are not ours
                        rs = i;
                        own = true;
                        wprev = wi;
                    }
                    if (i + 1 == n && own && n - rs > 1) {
                        for (u32 k = rs + 1; k < n && budget; ++k) {
                            const V x = X[k];
                            u32 q = k;
                            while (q > rs && TR::less(x, X[q - 1]) && budget) {
                                X[q] = X[q - 1];
                                --q;
                                --budget;
                            }
                            X[q] = x;
                        }
                    }
                }
                if (!budget) s_flag = 1;
            }
            __syncthreads();
            if (s_flag) {
                // too much insertion work: hand the untouched leaf to the merge sort
                if (tid == 0) {
                    const u32 q = atomicAdd(fb_count, 1u);
                    if (q < fb_cap) fb_queue[q] = td;
                }
                continue;
            }
            // 4a. write back from the (fixed-up) tile
            for (u32 i = tid; i < n; i += NT) g[i] = X[i];
        } else if (wact) {
            // 4b. the last pass left the sorted leaf in registers (warp-striped)
#pragma unroll
            for (int j = 0; j < E; ++j) {
                const u32 idx = wbase + j * 32 + lane;
                if (idx < n) g[idx] = v[j];
            }
        }
    }
}

template <class TR, int THREADS, int ITEMS>
struct BaseClass {
    static constexpr u32 TILE = THREADS * ITEMS;
    static constexpr size_t smem = (size_t)padidx(TILE) * sizeof(typename TR::V) + 16;
};

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
