// k_cta.cuh -- the single-CTA tier: one CTA sorts a medium subproblem completely, strictly in
// place, with the paper's recursion-free driver (§4.6).
//
// PAPER.md:147-153 (§4 preamble): large problems are partitioned by all processors together;
// "then we assign remaining problems in a balanced way to threads, which sort them
// sequentially".  On the GPU the "thread" of a remaining problem is one CTA (one per SM,
// persistent, problems taken by ticket), and its sequential algorithm is IS4o with the
// strictly in-place driver of §4.6:
//
//     i := lo; j := hi                                   (the whole problem is one bucket)
//     while i < hi:
//         if j - i <= leaf capacity: sort [i, j) in shared memory; i := j
//         else: partition [i, j)       (its buckets' maxima become findable, see below)
//         j := the end of the bucket starting at i      (searchNextLargest)
//
// searchNextLargest(A[i], i+1, hi) finds the first element larger than the bucket's maximum,
// which the partition stored at the bucket's first position.  Two GPU
// refinements keep the common case cheap: the bucket bounds of the latest partition are kept
// in shared memory (its k+1 delimiters -- part of the O(k b) buffer space, not a stack), and
// the maxima are stored only when a bucket is partitioned again before the later buckets of
// its parent are reached (then those later buckets are marked, so that the search can find
// them once the bounds are overwritten).  Nothing of size O(n) or O(log n) is kept: the driver's
// state is (i, j, hi) and one partition's bounds.
//
// A partition of [i, j) by the CTA (the paper's four phases with one "thread" = one CTA):
//   sampling      alpha*k-1 stratified samples sorted in shared memory, equidistant splitters,
//                 duplicates -> equality buckets, classifier in shared memory (as K1);
//   classification the problem is one stripe: k2_stripe (K2's tile machinery),
//                 full blocks flushed to the front, partial buffers kept in shared memory;
//   permutation   with one stripe the full blocks are a prefix, so no Appendix-A moves; the
//                 (w, r) words and reader counts live in shared memory; chains = lanes, blocks
//                 moved by TMA through shared-memory swap buffers (as K3);
//   cleanup       overhangs saved first, then each bucket's empty slots filled from its
//                 overhang, its partial buffer and the overflow block (as K4).
// Leaves (<= NT * CE elements) are sorted by the cell sort of the base case (cell_leaf).
#pragma once
#include "common.cuh"
#include "k_base.cuh"
#include "k_classify.cuh"
#include "k_permute.cuh"
#include "k_sample.cuh"

namespace ips4o {

template <class TR>
struct CtaCfg {
    static constexpr int NT = 512;                 // 128 registers per thread (K2 tiles + cell sort)
    static constexpr int E = 16 / TR::S * 4;       // K2 elements per thread and tile
    static constexpr int CE = TR::S == 8 ? 16 : 8; // cell-sort elements per thread
    static constexpr u32 LEAF = NT * CE;           // leaf capacity (u64: 8192, 16-byte: 4096)
    static constexpr int SAMPLE_ITEMS = 8;         // sample sort: NT * 8 = 4096 keys
    static constexpr u32 SAMPLE = 4096;            // sample capacity
    static constexpr int CHAIN_WARPS = 3, CHAIN_LANES = 16;
    static constexpr int CHAINS = CHAIN_WARPS * CHAIN_LANES;  // permutation chains
    typedef K2Smem<TR, NT, E> SM;
    // stage region (2 K2 tiles, 64 KB) reuse: the sample, the chains' swap buffers / the cleanup's
    // overhang scratch below META_OFF, the partition metadata in the last 8 KB; the leaf tile
    static constexpr size_t META_OFF = SM::stage_bytes - 8 * 1024;
    static constexpr size_t smem = SM::total + 64;  // (+ slack: the leaf tile overlaps the LUT by 16 B)
};

// Partition metadata (in the stage region's last 8 KB).
struct CtaMeta {
    u64 e[MAXK + 1];      // element-exact bucket starts e_0..e_K
    u64 wr[MAXK];         // packed (w:32 | r+2^31:32) block pointers (shared-memory atomics)
    u32 rd[MAXK];         // reader counts
    u32 d[MAXK + 1];      // delimiters (block index from g)
    u32 flag[MAXK];       // cleanup: overhang saved
    u32 done[MAXK / 32];  // permutation: bucket has no unprocessed block left
    u32 ticket;           // cleanup group ticket
    int ovf_owner;
};

__device__ __forceinline__ u64 atoms_add_u64(u64* p, u64 v) {
    return atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// ------------------------------------------------------------------ one partition

// Sampling and the classifier of [tp.lo, tp.hi) into shared memory (tree, spl, lut, tp).
template <class TR>
__device__ void cta_sample(const Mem<TR>& mem, TaskParam& tp, u64* keys, u64* dist, u64* tree, u64* spl,
                           unsigned short* lut, u64* btot_dummy, u64 seed, u32& s_flag, u32& s_nd) {
    typedef CtaCfg<TR> C;
    const u64 lo = tp.lo, n = tp.hi - tp.lo;
    u32 k = 4;
    while ((u64)k * TR::LEAF < n && k < (u32)MAXK) k *= 2;  // adaptive k
    u32 alpha = (u32)llround(0.2 * log2((double)n));
    if (alpha < 1) alpha = 1;
    const u32 amax = (C::SAMPLE - 1) / k;
    if (alpha < amax) alpha = amax;
    const u64 acap = (n + 1) / k;
    if ((u64)alpha > acap) alpha = (u32)(acap > 0 ? acap : 1);
    const u32 m = alpha * k - 1;
    constexpr u32 TILE = C::NT * C::SAMPLE_ITEMS;
    for (u32 j = threadIdx.x; j < TILE; j += C::NT) {
        u64 x = ~0ull;
        if (j < m) {
            const u64 a = lo + n * j / m, b = lo + n * (j + 1) / m;
            const u64 r = mix64(seed ^ mix64(lo * 0x9E3779B97F4A7C15ull + j));
            x = mem.key(a + __umul64hi(r, b - a), tp.part);
        }
        keys[padidx(j)] = x;
    }
    __syncthreads();
    block_sort_smem<TKey, C::NT, C::SAMPLE_ITEMS>(keys, TILE);
    if (threadIdx.x == 0) s_flag = 0;
    __syncthreads();
    for (u32 i = 1 + threadIdx.x; i + 1 < k; i += C::NT)
        if (keys[padidx(i * alpha - 1)] == keys[padidx((i + 1) * alpha - 1)]) s_flag = 1;
    __syncthreads();
    const u32 eq = s_flag;
    if (!eq) {
        for (u32 i = threadIdx.x; i + 1 < k; i += C::NT) dist[i] = keys[padidx((i + 1) * alpha - 1)];
        if (threadIdx.x == 0) s_nd = k - 1;
    } else if (threadIdx.x == 0) {
        // equality buckets: k/2-1 picks, distinct values kept
        const u32 k2 = k / 2, a2 = 2 * alpha;
        u32 nd = 0;
        for (u32 i = 1; i < k2; ++i) {
            const u64 v = keys[padidx(i * a2 - 1)];
            if (nd == 0 || dist[nd - 1] != v) dist[nd++] = v;
        }
        s_nd = nd;
    }
    __syncthreads();
    build_tree_block(dist, s_nd, eq, tree, spl, &tp, btot_dummy, lut, reinterpret_cast<u32*>(keys));
    __syncthreads();
}

template <class TR>
__device__ __forceinline__ void* mem_base(const Mem<TR>& mem) {
    if constexpr (TR::KV) return mem.k;
    else return mem.d;
}

// Block permutation of one stripe's full blocks [0, F) within [g, g + nblocks*B) (PAPER.md:
// 252-304) by the CTA's chains, pointers in shared memory.
template <class TR>
__device__ void cta_permute(const Mem<TR>& mem, const TaskParam& tp, CtaMeta& M, const u64* tree, const u64* spl,
                            char* swap, u64* mbars, char* ovf, u32& phase, u32* err) {
    typedef CtaCfg<TR> C;
    constexpr u32 BB = TR::B * TR::S;
    const u32 tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
    const bool chain = wi < (u32)C::CHAIN_WARPS && lane < (u32)C::CHAIN_LANES;
    if (!chain) return;
    const u32 cid = wi * C::CHAIN_LANES + lane;
    char* const mybuf = swap + (size_t)cid * 2 * BB;
    u64* const mymbar = &mbars[cid];
    char* tbase = reinterpret_cast<char*>(mem_base(mem)) + tp.g * GridStride<TR>::v;
    char* vbase = nullptr;
    if constexpr (TR::KV) vbase = reinterpret_cast<char*>(mem.v) + tp.g * 8;
    auto classify_buf = [&](const char* b) {
        typename TR::V v;
        memcpy(&v, b, sizeof(v));
        return classify_key(TR::key(v, tp.part), tree, spl, tp.logk, tp.kprime, tp.eq);
    };
    // (phase: this chain's mbarrier parity, kept across partitions by the caller)
    u32 st = CH_FREE, xb = 0, dest = 0, slot = 0;
    u32 pb = (cid * 97u) % tp.K;
    u64 guard = 0;
    while (st != CH_DEAD) {
        if (++guard > (1ull << 32)) {  // (a safety net: never expected)
            atomicOr(err, (u32)ERR_PROGRESS);
            break;
        }
        if (st == CH_FREE) {
            const u32 b = next_open_bucket(M.done, pb, tp.K);
            if (b == 0xFFFFFFFFu) {
                st = CH_DEAD;
                continue;
            }
            pb = b;
            // (S18 in shared memory: the reader announcement is ordered before the take)
            atomicAdd(&M.rd[pb], 1u);
            __threadfence_block();
            const u64 old = atoms_add_u64(&M.wr[pb], ~0ull);
            const int ow = (int)(u32)(old >> 32), orr = (int)((u32)old - RBIAS);
            if (orr < ow) {
                atomicSub(&M.rd[pb], 1u);
                atomicOr(&M.done[pb >> 5], 1u << (pb & 31));
            } else {
                bulk_wait_read0();
                fence_proxy_async_smem();
                K3Blk<TR>::load(mybuf + xb * BB, tbase, vbase, (u32)orr, mymbar);
                st = CH_TAKING;
            }
        } else if (st == CH_HELD) {
            const u64 old = atoms_add_u64(&M.wr[dest], 1ull << 32);
            __threadfence_block();
            const int ow = (int)(u32)(old >> 32), orr = (int)((u32)old - RBIAS);
            slot = (u32)ow;
            if (ow <= orr) {
                bulk_wait_read0();
                fence_proxy_async_smem();
                K3Blk<TR>::load(mybuf + (xb ^ 1) * BB, tbase, vbase, (u32)ow, mymbar);
                st = CH_SWAPPING;
            } else {
                st = CH_WAITW;
            }
        }
        if (st == CH_WAITW && *(volatile u32*)&M.rd[dest] == 0u) {
            __threadfence_block();
            if (tp.g + (u64)(slot + 1) * TR::B > tp.hi) {
                // past the end: the overflow block, in shared memory
                const uint4* s = reinterpret_cast<const uint4*>(mybuf + xb * BB);
                uint4* d = reinterpret_cast<uint4*>(ovf);
                for (u32 q = 0; q < BB / 16; ++q) d[q] = s[q];
                M.ovf_owner = (int)dest;
            } else {
                K3Blk<TR>::store(tbase, vbase, slot, mybuf + xb * BB);
                bulk_commit();
            }
            st = CH_FREE;
        }
        if ((st == CH_TAKING || st == CH_SWAPPING) && mbar_test(mymbar, phase)) {
            phase ^= 1u;
            if (st == CH_TAKING) {
                __threadfence_block();
                atomicSub(&M.rd[pb], 1u);  // the block has been read
                dest = classify_buf(mybuf + xb * BB);
                st = CH_HELD;
            } else {
                const u32 od = classify_buf(mybuf + (xb ^ 1) * BB);
                if (od != dest) {
                    K3Blk<TR>::store(tbase, vbase, slot, mybuf + xb * BB);
                    bulk_commit();
                    xb ^= 1u;
                    dest = od;
                }
                st = CH_HELD;
            }
        }
    }
    bulk_wait0();
}

// Cleanup: warps take groups of 4 buckets in order; each group first saves
// the overhangs of its buckets' last blocks (into the next buckets' heads) and publishes them,
// then fills each bucket's empty slots from its overhang, its partial buffer (shared memory)
// and the overflow block.
template <class TR>
__device__ void cta_cleanup(const Mem<TR>& mem, const TaskParam& tp, CtaMeta& M, const u32* fill,
                            const typename TR::V* buf, const char* ovf, typename TR::V* scratch) {
    typedef typename TR::V V;
    constexpr int B = TR::B;
    constexpr u32 G = 4;
    const u32 lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    V* ovh = scratch + (size_t)wi * G * B;
    const u32 ngroups = (tp.K + G - 1) / G;
    for (;;) {
        u32 tk = 0;
        if (lane == 0) tk = atomicAdd(&M.ticket, 1u);
        tk = __shfl_sync(0xffffffffu, tk, 0);
        if (tk >= ngroups) break;
        const u32 b0 = tk * G;
        // 1. overhangs of the group's buckets, saved and published first
        for (u32 gi = 0; gi < G; ++gi) {
            const u32 b = b0 + gi;
            if (b >= tp.K) break;
            const u64 e1 = M.e[b + 1];
            const u64 db = tp.g + (u64)M.d[b] * B;
            const u64 in_end = M.ovf_owner == (int)b ? tp.g + (u64)(tp.nblocks - 1) * B
                                                     : tp.g + (u64)(u32)(M.wr[b] >> 32) * B;
            const u32 ovl = (in_end > db && in_end > e1) ? (u32)(in_end - e1) : 0u;
            for (u32 k = lane; k < ovl; k += 32) ovh[gi * B + k] = mem.ld(e1 + k);
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            for (u32 gi = 0; gi < G && b0 + gi < tp.K; ++gi) *(volatile u32*)&M.flag[b0 + gi] = 1u;
        }
        // 2. each bucket: its sources into its empty slots
        for (u32 gi = 0; gi < G; ++gi) {
            const u32 b = b0 + gi;
            if (b >= tp.K) break;
            const u64 e0 = M.e[b], e1 = M.e[b + 1];
            const u32 d = M.d[b];
            const u64 db = tp.g + (u64)d * B;
            const bool own_ovf = M.ovf_owner == (int)b;
            const u64 in_end = own_ovf ? tp.g + (u64)(tp.nblocks - 1) * B : tp.g + (u64)(u32)(M.wr[b] >> 32) * B;
            const u32 ovl = (in_end > db && in_end > e1) ? (u32)(in_end - e1) : 0u;
            const u32 fb = fill[b];
            const u32 nsrc = ovl + fb + (own_ovf ? (u32)B : 0u);
            const u64 hend = db < e1 ? db : e1;
            const u64 ts = db < e1 ? (in_end < e1 ? in_end : e1) : e1;
            const u64 hl = hend - e0;
            // wait until the bucket owning block d-1 (under our head) has saved its overhang
            if (lane == 0 && hl > 0 && d >= 1) {
                u32 lo = 0, hi = b;  // largest o < b with d_o <= d-1
                while (hi - lo > 1) {
                    const u32 mid = (lo + hi) >> 1;
                    if (M.d[mid] <= d - 1) lo = mid;
                    else hi = mid;
                }
                if (lo < b)
                    while (*(volatile u32*)&M.flag[lo] == 0u) __nanosleep(32);
                __threadfence_block();
            }
            __syncwarp();
            for (u32 k = lane; k < nsrc; k += 32) {
                V val;
                if (k < ovl) val = ovh[gi * B + k];
                else if (k - ovl < fb) val = K2Buf<TR>::get(buf, b * B + (k - ovl));
                else val = ovf_get<TR>(ovf, k - ovl - fb);
                mem.st((u64)k < hl ? e0 + k : ts + (k - hl), val);
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ the driver

template <class TR>
struct CtaShared {
    TaskParam tp;
    StripeDesc sd;
    u32 s_flag, s_nd, s_nflushed, s_bcast;
    u64 s_bcast64;
    u32 K, eq;           // of the latest partition (its bounds are cached in the buffer region)
    u64 clo, chi;        // cached partition range
    CellSh<CtaCfg<TR>::NT / 32> cell;
};

// searchNextLargest: the first position p in (i, hi) whose key exceeds
// the key at i (the bucket's maximum), hi if none -- an exponential search by warp 0's lanes
// (probes i + 2^lane), then 32-way narrowing.  Monotone: the bucket's elements are <= its
// maximum, every later element is larger.  Returns via *out (all threads read it after a barrier).
template <class TR>
__device__ void search_next_largest(const Mem<TR>& mem, u64 i, u64 hi, u32 part, u64* out) {
    if (threadIdx.x >= 32) return;
    const u32 lane = threadIdx.x;
    const u64 mx = mem.key(i, part);
    // exponential phase: the smallest l with key(i + 2^l) > mx
    u64 lo = i, up = hi;  // invariant: key(lo) <= mx (lo = i), answer in (lo, up]
    {
        const u64 off = 1ull << lane;
        const u64 p = i + off;
        const bool gt = p < hi && mem.key(p, part) > mx;
        const u32 bal = __ballot_sync(0xffffffffu, gt);
        const u32 inr = __ballot_sync(0xffffffffu, p < hi);
        if (bal) {
            const u32 l = __ffs(bal) - 1;
            up = i + (1ull << l);
            lo = l ? i + (1ull << (l - 1)) : i;
        } else {
            // every probe in range is <= mx: the answer lies after the last in-range probe
            const u32 l = inr ? 31 - __clz(inr) : 0u;
            lo = inr ? i + (1ull << l) : i;
            up = hi;
        }
    }
    // 32-way narrowing of (lo, up]: key(lo) <= mx, up = hi or key(up) > mx
    while (up - lo > 1) {
        const u64 span = up - lo;
        const u64 p = lo + 1 + (span - 1) * (u64)lane / 32;  // 32 probes in (lo, up)
        const bool gt = mem.key(p, part) > mx;
        const u32 bal = __ballot_sync(0xffffffffu, gt);
        if (bal) {
            const u32 l = __ffs(bal) - 1;
            const u64 pl = lo + 1 + (span - 1) * (u64)l / 32;
            const u64 pprev = l ? lo + 1 + (span - 1) * (u64)(l - 1) / 32 : lo;
            up = pl;
            lo = pprev;
        } else {
            lo = lo + 1 + (span - 1) * 31ull / 32;
        }
    }
    if (lane == 0) *out = up;
}

template <class TR>
__device__ __forceinline__ u64 key_max_pos(const Mem<TR>& mem, u64 a, u64 b, u32 part, u64* s_w, u32* s_wi) {
    // position of a maximal key in [a, b) (CTA-wide)
    typedef CtaCfg<TR> C;
    u64 bk = 0, bp = a;
    for (u64 x = a + threadIdx.x; x < b; x += C::NT) {
        const u64 k = mem.key(x, part);
        if (k > bk || (k == bk && x < bp)) {
            bk = k;
            bp = x;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const u64 k2 = __shfl_xor_sync(0xffffffffu, bk, o), p2 = __shfl_xor_sync(0xffffffffu, bp, o);
        if (k2 > bk || (k2 == bk && p2 < bp)) {
            bk = k2;
            bp = p2;
        }
    }
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        s_w[2 * w] = bk;
        s_w[2 * w + 1] = bp;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 k = s_w[0], p = s_w[1];
        for (u32 q = 1; q < C::NT / 32; ++q)
            if (s_w[2 * q] > k || (s_w[2 * q] == k && s_w[2 * q + 1] < p)) {
                k = s_w[2 * q];
                p = s_w[2 * q + 1];
            }
        s_w[0] = k;
        s_w[1] = p;
    }
    __syncthreads();
    const u64 r = s_w[1];
    __syncthreads();
    return r;
}

template <class TR>
__global__ void __launch_bounds__(CtaCfg<TR>::NT, 1)
    k_cta_sort(LevelArgs A0, const TaskDesc* tasks, const u32* d_ntasks, u32 qcap, u32* ticket) {
    typedef typename TR::V V;
    typedef CtaCfg<TR> C;
    typedef typename C::SM SM;
    constexpr int B = TR::B, NT = C::NT, E = C::E;
    const LevelArgs A = with_dyn(A0);
    extern __shared__ __align__(128) unsigned char smem[];
    V* buf = reinterpret_cast<V*>(smem);
    u64* tree = reinterpret_cast<u64*>(smem + SM::buf_bytes);
    u64* spl = tree + MAXK;
    u32* fill = reinterpret_cast<u32*>(spl + MAXK);
    u32* cnt = fill + MAXK;
    u32* slotb = cnt + MAXK;
    u32* nfl = slotb + MAXK;
    u32* nbl = nfl + MAXK;
    V* stage = reinterpret_cast<V*>(smem + SM::buf_bytes + SM::tree_bytes + SM::arr_bytes + SM::rtree_bytes);
    unsigned short* lut = reinterpret_cast<unsigned short*>(reinterpret_cast<unsigned char*>(stage) + SM::stage_bytes);
    CtaMeta& M = *reinterpret_cast<CtaMeta*>(reinterpret_cast<unsigned char*>(stage) + C::META_OFF);
    char* ovf = reinterpret_cast<char*>(stage) + C::META_OFF + ((sizeof(CtaMeta) + 127) & ~(size_t)127);
    u64* bcache = reinterpret_cast<u64*>(smem + 96 * 1024);   // cached bounds (buffer region, past the cell counters)
    u64* dist = reinterpret_cast<u64*>(smem + 64 * 1024);     // sampling scratch (buffer region)
    static_assert(SM::buf_bytes >= 96 * 1024 + (MAXK + 1) * 8, "bounds cache in the buffer region");
    u64* btot_dummy = dist + MAXK;
    __shared__ CtaShared<TR> S;
    __shared__ __align__(8) u64 s_mbar[2];
    __shared__ __align__(8) u64 c_mbar[C::CHAINS];
    __shared__ u64 s_red[2 * (NT / 32)];
    static_assert(((sizeof(CtaMeta) + 127) & ~(size_t)127) + TR::B * TR::S <= 8 * 1024,
                  "partition metadata and the overflow block fit the stage region's tail");
    static_assert(SM::stage_bytes >= (size_t)C::LEAF * sizeof(V) && SM::stage_bytes >= padidx(NT * C::SAMPLE_ITEMS) * 8,
                  "stage region reuse");
    static_assert((size_t)C::CHAINS * 2 * TR::B * TR::S <= C::META_OFF, "swap buffers");
    static_assert((size_t)(C::CE + 4) * NT * 4 + 8 <= 64 * 1024, "cell counters below the sampling scratch");
    static_assert((size_t)NT / 32 * 4 * TR::B * sizeof(V) <= C::META_OFF, "cleanup overhang scratch");
    const u32 tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&s_mbar[0], 1);
        mbar_init(&s_mbar[1], 1);
    }
    if (tid < (u32)C::CHAINS) mbar_init(&c_mbar[tid], 1);
    mbar_fence_init();
    __syncthreads();
    u32 kphase = 0;      // K2 stage mbarrier parities
    u32 cphase = 0;      // this thread's chain mbarrier parity (chains: cta_permute)
    const Mem<TR> mem(A.data, A.vals);
    V* data = reinterpret_cast<V*>(A.data);
    const u32 ntasks = min(*d_ntasks, qcap);
    u64 nparts = 0, nmarks = 0, nleaves = 0;
    for (;;) {
        if (tid == 0) S.s_bcast = atomicAdd(ticket, 1u);
        __syncthreads();
        const u32 tk = S.s_bcast;
        __syncthreads();
        if (tk >= ntasks) break;
        const TaskDesc task = tasks[tk];
        const u64 lo = task.lo, hi = task.hi;
        const u32 part = 0;
        u64 i = lo, j = hi;
        if (tid == 0) {
            S.K = 0;
            S.clo = S.chi = 0;
        }
        __syncthreads();
        u64 iters = 0;
        while (i < hi) {
            if (++iters > 4 * (hi - lo) + 64) {  // (a safety net: the driver advances every step)
                if (tid == 0) atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_PROGRESS);
                break;
            }
            if (j <= i) {
                if (tid == 0) atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_PROGRESS);
                break;
            }
            if (j - i <= (u64)C::LEAF) {
                // ---- leaf: the cell sort in shared memory (clustered keys: partition instead)
                const TaskDesc td{i, j, 0u, 0u};
                int r = 0;
                if (j - i > 1) r = cell_leaf<TR, NT, C::CE>(td, mem, data, stage, reinterpret_cast<u32*>(smem), S.cell, []() {});
                if (IPS4O_BASE_TMA_WB && tid == 0) bulk_wait0();
                fence_proxy_async_global();  // (plain write-back stores before later TMA reads)
                __syncthreads();
                if (r == 0) {
                    ++nleaves;
                    i = j;
                    goto next_bucket;
                }
            }
            {
                // an equality bucket of the cached partition, or all keys equal: nothing to do
                bool alleq = false;
                {
                    const u64 k0 = mem.key(i, part);
                    bool ne = false;
                    for (u64 x = i + tid; x < j && !ne; x += NT) ne = mem.key(x, part) != k0;
                    alleq = !__syncthreads_or(ne);
                }
                if (alleq) {
                    i = j;
                    goto next_bucket;
                }
                // ---- partition [i, j).  The later buckets of the cached partition are marked
                //      first (their maxima to their first positions), so that
                //      searchNextLargest finds them after the cache is overwritten.
                if (S.K && j < S.chi) {
                    for (u32 b = 0; b < S.K; ++b) {
                        const u64 a = bcache[b], z = bcache[b + 1];
                        if (a < j || z - a < 2) continue;
                        const u64 pm = key_max_pos<TR>(mem, a, z, part, s_red, nullptr);
                        if (tid == 0 && pm != a) {
                            const V x = mem.ld(a), y = mem.ld(pm);
                            mem.st(a, y);
                            mem.st(pm, x);
                        }
                        __syncthreads();
                        ++nmarks;
                    }
                }
                ++nparts;
                // sampling + classifier
                if (tid == 0) {
                    TaskParam& tp = S.tp;
                    memset(&tp, 0, sizeof tp);
                    tp.lo = i;
                    tp.hi = j;
                    u64 g = i;
                    const uintptr_t base = reinterpret_cast<uintptr_t>(mem_base(mem));
                    while (((base + g * GridStride<TR>::v) & 15u) != 0 && g < j) ++g;
                    tp.g = g;
                    tp.nblocks = (u32)((j - g + B - 1) / B);
                    tp.part = part;
                    StripeDesc& sd = S.sd;
                    sd.begin = i;
                    sd.end = j;
                    sd.task = 0;
                    sd.sb = 0;
                    sd.se = tp.nblocks;
                    sd.first = 1;
                }
                __syncthreads();
                cta_sample<TR>(mem, S.tp, reinterpret_cast<u64*>(stage), dist, tree, spl, lut, btot_dummy,
                               A.seed ^ mix64(i), S.s_flag, S.s_nd);
                const TaskParam tp = S.tp;
                // classification (one stripe)
                if (tid < (u32)MAXK) {
                    fill[tid] = 0;
                    cnt[tid] = 0;
                    nbl[tid] = 0;
                }
                if (tid == 0) S.s_nflushed = 0;
                __syncthreads();
                k2_stripe<TR, NT, E>(mem, S.sd, tp, buf, nullptr, spl, fill, cnt, slotb, nfl, nbl, stage, lut,
                                     &S.s_nflushed, s_mbar, kphase);
                if (tid < (u32)MAXK) bulk_wait0();  // the flushes have left the buffers
                __syncthreads();
                // bounds, delimiters, (w, r) words (one stripe: the full blocks are [0, F))
                {
                    const u32 F = S.s_nflushed;
                    const u32 lane = tid & 31, w = tid >> 5;
                    const u64 c = tid < (u32)MAXK ? (u64)nbl[tid] * B + cnt[tid] : 0ull;
                    u64 incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const u64 y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= (u32)o) incl += y;
                    }
                    if (lane == 31) s_red[w] = incl;
                    __syncthreads();
                    u64 off = 0;
                    for (u32 ww = 0; ww < w; ++ww) off += s_red[ww];
                    if (tid < (u32)MAXK) {
                        const u64 e = tp.lo + off + incl - c;
                        M.e[tid] = e;
                        M.d[tid] = e > tp.g ? (u32)((e - tp.g + B - 1) / B) : 0u;
                        if (tid == MAXK - 1) {
                            M.e[MAXK] = tp.hi;
                            M.d[MAXK] = tp.nblocks;
                        }
                        M.rd[tid] = 0;
                        M.flag[tid] = 0;
                    }
                    if (tid < MAXK / 32) M.done[tid] = 0;
                    if (tid == 0) {
                        M.ticket = 0;
                        M.ovf_owner = -1;
                    }
                    __syncthreads();
                    if (tid < (u32)MAXK) {
                        const u32 d = M.d[tid], dn = M.d[tid + 1];
                        const u32 nf = F > d ? min(dn, F) - d : 0u;
                        const bool all_here = c == tp.hi - tp.lo;
                        const u32 w0 = all_here ? d + nf : d;
                        M.wr[tid] = ((u64)w0 << 32) | (u64)(u32)(d + nf - 1u + RBIAS);
                        if (tid >= tp.K || nf == 0 || all_here) atomicOr(&M.done[tid >> 5], 1u << (tid & 31));
                    }
                    __syncthreads();
                }
                // permutation (swap buffers in the stage region)
                cta_permute<TR>(mem, tp, M, tree, spl, reinterpret_cast<char*>(stage), c_mbar, ovf, cphase,
                                &A.ctr[CTR_ERROR]);
                __syncthreads();
                // cleanup (overhang scratch in the stage region)
                cta_cleanup<TR>(mem, tp, M, fill, buf, ovf, stage);
                __syncthreads();
                // cache the bounds of this partition (the buffer region: the partial buffers are consumed)
                for (u32 b = tid; b <= tp.K; b += NT) bcache[b] = b < tp.K ? M.e[b] : tp.hi;
                if (tid == 0) {
                    S.K = tp.K;
                    S.eq = tp.eq;
                    S.clo = tp.lo;
                    S.chi = tp.hi;
                }
                __syncthreads();
            }
        next_bucket:
            if (i >= hi) break;
            // the end of the bucket starting at i: from the cached bounds of the latest
            // partition (equality buckets skipped: their keys are all equal), else
            // searchNextLargest (the bucket's maximum is at i)
            {
                u64 jn = 0;
                bool cached = false;
                const u32 K = S.K;
                while (K && i >= S.clo && i < S.chi) {
                    u32 lo2 = 0, hi2 = K;  // the last b with bcache[b] <= i: i's (non-empty) bucket
                    while (hi2 - lo2 > 1) {
                        const u32 mid = (lo2 + hi2) >> 1;
                        if (bcache[mid] <= i) lo2 = mid;
                        else hi2 = mid;
                    }
                    jn = bcache[lo2 + 1];
                    if (S.eq && (lo2 & 1u)) {
                        i = jn;  // an equality bucket: done
                        continue;
                    }
                    cached = true;
                    break;
                }
                if (i >= hi) break;
                if (!cached) {
                    search_next_largest<TR>(mem, i, hi, part, &S.s_bcast64);
                    __syncthreads();
                    jn = S.s_bcast64;
                    __syncthreads();
                }
                j = jn;
            }
        }
    }
    if (tid == 0) {
        atomicAdd((unsigned long long*)&A.dstats[DS_MED_PARTS], (unsigned long long)nparts);
        atomicAdd((unsigned long long*)&A.dstats[DS_MED_MARKS], (unsigned long long)nmarks);
        atomicAdd((unsigned long long*)&A.dstats[DS_MED_LEAVES], (unsigned long long)nleaves);
    }
}

}  // namespace ips4o
