// k_classify.cuh -- K2: local classification with block-buffered flushes (§4.1).
//
// Persistent CTAs (one per SM, 512 threads) take stripes from an LPT-ordered list.  Per
// tile of 512*E elements:
//   1. 128-bit coalesced loads, branchless tree descent per element (tree in smem);
//   2. warp-aggregated ranking with MATCH.ANY: every element gets its position in its
//      bucket's stream without per-element shared atomics;
//   3. one thread per bucket turns per-warp counts into offsets and claims flush slots;
//   4. elements land in the bucket's shared buffer block (b elements); blocks that
//      complete inside the tile beyond the first are written straight to the stripe;
//   5. full buffers are flushed as whole blocks with TMA bulk copies (UBLKCP) into the
//      already-consumed front of the stripe (there is room: at least b more elements
//      were read than written back);
//   6. the remainders start the next buffer fill.
// At the end of a stripe the counts, the number of flushed blocks and the partially
// filled buffers (spilled to the auxiliary area) are published for K3/K4.
#pragma once
#include "common.cuh"

namespace ips4o {

#ifndef IPS4O_K2_PRED_SPL  // the bucket-hint classifier loads a splitter only for cells that hold one (measured: no gain)
#define IPS4O_K2_PRED_SPL 0
#endif
template <class TR, int NT, int E, int ST = K2_STAGES>
struct K2Smem {
    typedef typename TR::V V;
    static constexpr int B = TR::B;
    static constexpr int NW = NT / 32;
    static constexpr size_t buf_bytes = (size_t)MAXK * B * sizeof(V);
    static constexpr size_t wcnt_bytes = 0;
    static constexpr size_t tree_bytes = 2 * MAXK * 8;
    static constexpr size_t arr_bytes = 5 * MAXK * 4;
    static constexpr size_t rtree_bytes = IPS4O_K2_LUT ? 0 : (size_t)MAXK * TREE_COPIES * 8;  // tree copies
    static constexpr size_t stage_bytes = (size_t)ST * NT * E * TR::S;  // staged tiles
    static constexpr size_t lut_bytes = IPS4O_K2_LUT ? (size_t)LUT_STRIDE * 2 : 0;  // bucket hints
    static constexpr size_t total =
        buf_bytes + wcnt_bytes + tree_bytes + arr_bytes + rtree_bytes + stage_bytes + lut_bytes;
};

// Loads one tile (<= NT*E elements from tb, len valid) into raw 16-byte registers; bit e of
// the returned mask is set for valid elements.  128-bit coalesced loads (read-only path:
// every element is read before anything is written to its address in this kernel).  The
// registers are only consumed when the tile is processed, so the loads of the next tile
// stay in flight while the current one is classified.
template <class TR, int NT, int E>
__device__ __forceinline__ u32 k2_load(const Mem<TR>& mem, u64 tb, u32 len, uint4 (&raw)[E / TR::VEC]) {
    typedef typename TR::V V;
    constexpr int VEC = TR::VEC, NV = E / VEC;
    const u32 tid = threadIdx.x;
    u32 valid = 0;
    if constexpr (TR::KV) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const u32 e0 = (u32)(i * NT + tid);
            V x = TR::pad();
            if (e0 < len) {
                x = mem.ld(tb + e0);
                valid |= 1u << i;
            }
            memcpy(&raw[i], &x, 16);
        }
        return valid;
    } else {
    const V* data = mem.d;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const u32 e0 = (u32)(i * NT + tid) * VEC;
        if (e0 + VEC <= len) {
            raw[i] = ld_nc_v4(data + tb + e0);
            valid |= ((1u << VEC) - 1u) << (i * VEC);
        } else {
            V tmp[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                if (e0 + q < len) {
                    tmp[q] = data[tb + e0 + q];
                    valid |= 1u << (i * VEC + q);
                } else {
                    tmp[q] = TR::pad();
                }
            }
            memcpy(&raw[i], tmp, 16);
        }
    }
    return valid;
    }
}

// A tile of NT*E elements from element idx into a shared-memory stage by TMA bulk copies
// completing on mbar (KV: the key tile, then the value tile).
template <class TR, int NT, int E>
__device__ __forceinline__ void k2_stage_load(typename TR::V* stage, const Mem<TR>& mem, u64 idx, u64* mbar) {
    constexpr u32 TILE = NT * E;
    if constexpr (TR::KV) {
        u64* sk = reinterpret_cast<u64*>(stage);
        mbar_expect_tx(mbar, TILE * 16u);
        bulk_g2s_tx(sk, mem.k + idx, TILE * 8u, mbar);
        bulk_g2s_tx(sk + TILE, mem.v + idx, TILE * 8u, mbar);
    } else {
        bulk_g2s(stage, mem.d + idx, TILE * (u32)sizeof(typename TR::V), mbar);
    }
}
// this thread's elements (i*NT + tid) of a staged tile, as raw 16-byte registers
template <class TR, int NT, int E>
__device__ __forceinline__ void k2_stage_read(const typename TR::V* stage, uint4 (&raw)[E / TR::VEC]) {
    if constexpr (TR::KV) {
        const u64* sk = reinterpret_cast<const u64*>(stage);
        const u64* sv = sk + NT * E;
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const u64 k = sk[i * NT + threadIdx.x], v = sv[i * NT + threadIdx.x];
            raw[i] = make_uint4((u32)k, (u32)(k >> 32), (u32)v, (u32)(v >> 32));
        }
    } else {
        const uint4* sp = reinterpret_cast<const uint4*>(stage);
#pragma unroll
        for (int i = 0; i < E / TR::VEC; ++i) raw[i] = sp[i * NT + threadIdx.x];
    }
}
// K2's shared-memory bucket buffers: K*B element slots (KV: a key half and a value half, so
// that a full block leaves as one key block and one value block)
template <class TR>
struct K2Buf {
    typedef typename TR::V V;
    __device__ __forceinline__ static void put(V* buf, u32 idx, const V& v) {
        if constexpr (TR::KV) {
            u64* b = reinterpret_cast<u64*>(buf);
            b[idx] = v.x;
            b[(u32)MAXK * TR::B + idx] = v.y;
        } else {
            buf[idx] = v;
        }
    }
    __device__ __forceinline__ static V get(const V* buf, u32 idx) {
        if constexpr (TR::KV) {
            const u64* b = reinterpret_cast<const u64*>(buf);
            return make_ulonglong2(b[idx], b[(u32)MAXK * TR::B + idx]);
        } else {
            return buf[idx];
        }
    }
    // block of bucket b to element gidx by TMA bulk stores (bulk-group completion)
    __device__ __forceinline__ static void flush(const Mem<TR>& mem, u64 gidx, V* buf, u32 b) {
        if constexpr (TR::KV) {
            u64* bk = reinterpret_cast<u64*>(buf);
            bulk_s2g(mem.k + gidx, bk + b * TR::B, TR::B * 8u);
            bulk_s2g(mem.v + gidx, bk + (u32)MAXK * TR::B + b * TR::B, TR::B * 8u);
        } else {
            bulk_s2g(mem.d + gidx, buf + b * TR::B, TR::B * (u32)sizeof(V));
        }
    }
};

// Branchless descent for all E elements of the thread, level by level so that the E
// independent shared-memory lookups of a level are in flight together.  LOGK = 8 is the
// k' = 256 case of the big levels; LOGK = 0 takes the depth at run time.
// The comparison outcome of level l is bit (logk-1-l) of the leaf index i, so a ballot of
// it per level gives, at the end, the set of lanes whose element fell into the same leaf
// ("peers", the warp-aggregation mask) without a separate MATCH.ANY; the equality test
// and the validity of the element add one ballot each.
template <int E, int LOGK>
__device__ __forceinline__ void k2_classify_keys(const u64 (&key)[E], u32 valid, bool full,
                                                 const u64* tree, const u64* spl, u32 logk,
                                                 u32 kprime, u32 eq, u32 (&bk)[E], u32 (&peers)[E]);

template <class TR, int E, int LOGK>
__device__ __forceinline__ void k2_classify(const typename TR::V (&v)[E], u32 valid, bool full,
                                            const u64* tree, const u64* spl, u32 logk, u32 kprime,
                                            u32 eq, u32 (&bk)[E], u32 (&peers)[E]) {
    u64 key[E];
#pragma unroll
    for (int e = 0; e < E; ++e) key[e] = TR::key(v[e], 0);
    k2_classify_keys<E, LOGK>(key, valid, full, tree, spl, logk, kprime, eq, bk, peers);
}

// One level of the branchless descent for one key: node = a[j];
// p = [node <= key]; j <- 2j + p (as a byte offset in this lane's tree copy:
// a <- 2a + (p ? t1 : t0)), and the ballot of p refines the key's peer mask.  Written in
// PTX so that the comparison is evaluated once and feeds the ballot, the mask update and
// the index update (8 SASS instructions per level and key).
__device__ __forceinline__ void descend_step(u64 key, u32 sbase, u32& a, u32& peers, u32 t0, u32 t1) {
    asm("{\n\t"
        ".reg .pred p;\n\t"
        ".reg .b32 x, m, t, ad;\n\t"
        ".reg .b64 nd;\n\t"
        "add.u32 ad, %2, %0;\n\t"
        "ld.shared.u64 nd, [ad];\n\t"
        "setp.ge.u64 p, %3, nd;\n\t"
        "vote.sync.ballot.b32 x, p, 0xffffffff;\n\t"
        "selp.b32 m, 0, 0xffffffff, p;\n\t"
        "xor.b32 x, x, m;\n\t"
        "and.b32 %1, %1, x;\n\t"
        "selp.b32 t, %5, %4, p;\n\t"
        "mad.lo.u32 %0, %0, 2, t;\n\t"
        "}"
        : "+r"(a), "+r"(peers)
        : "r"(sbase), "l"(key), "r"(t0), "r"(t1));
}

template <int E, int LOGK>
__device__ __forceinline__ void k2_classify_keys(const u64 (&key)[E], u32 valid, bool full,
                                                 const u64* tree, const u64* spl, u32 logk,
                                                 u32 kprime, u32 eq, u32 (&bk)[E], u32 (&peers)[E]) {
    // tree: the replicated layout of rtree_fill (node j of copy c at byte 128*j + 8*c); lane
    // l reads copy l % 16, so the 16 lanes of a half-warp never share a bank pair: every
    // lookup is one conflict-free 64-bit load whatever nodes the keys lead to.
    u32 a[E];  // byte offset of the current node in this lane's copy
    const u32 cofs = (threadIdx.x & (TREE_COPIES - 1)) * 8u;
    const u32 t0 = 0u - cofs, t1 = TREE_NODE_BYTES - cofs;  // a' = 2a + (p ? t1 : t0)
    const u64 root = tree[cofs / 8 + TREE_COPIES];           // node 1 (any copy)
    const char* tb = reinterpret_cast<const char*>(tree);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const bool p = key[e] >= root;  // level 0 from a register: j = 2 + [root <= e]
        const u32 x = __ballot_sync(0xffffffffu, p);
        peers[e] = p ? x : ~x;
        a[e] = (p ? 3u : 2u) * TREE_NODE_BYTES + cofs;
    }
    const u32 sb = (u32)__cvta_generic_to_shared(tb);
    if (LOGK == 8) {
#pragma unroll
        for (int l = 1; l < 8; ++l)
#pragma unroll
            for (int e = 0; e < E; ++e) descend_step(key[e], sb, a[e], peers[e], t0, t1);
    } else {
        for (u32 l = 1; l < logk; ++l)
#pragma unroll
            for (int e = 0; e < E; ++e) descend_step(key[e], sb, a[e], peers[e], t0, t1);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        u32 i = (a[e] - cofs) / TREE_NODE_BYTES - kprime;
        if (eq) {
            const u32 ii = i ? i : 1u;
            const bool isq = i >= 1u && spl[ii] >= key[e];
            const u32 x = __ballot_sync(0xffffffffu, isq);
            peers[e] &= isq ? x : ~x;
            i = 2 * i - (isq ? 1u : 0u);
        }
        const bool ok = (valid >> e) & 1u;
        if (!full) {
            const u32 x = __ballot_sync(0xffffffffu, ok);
            peers[e] &= ok ? x : ~x;
        }
        bk[e] = ok ? i : INV_BUCKET;
    }
}

// Fill the replicated tree (TREE_COPIES interleaved copies of the 256-node BFS array) from
// the task's tree in global memory.  Block-wide; the caller synchronises.
__device__ __forceinline__ void rtree_fill(u64* rtree, const u64* gtree, u32 tid, u32 nthreads) {
    for (u32 i = tid; i < (u32)MAXK * TREE_COPIES; i += nthreads) rtree[i] = gtree[i / TREE_COPIES];
}

// One level of the branchless descent without a peer mask (the ranks come from shared-
// memory atomics): 5 SASS instructions per level and key.
__device__ __forceinline__ void descend_step_nb(u64 key, u32 sbase, u32& a, u32 t0, u32 t1) {
    asm("{\n\t"
        ".reg .pred p;\n\t"
        ".reg .b32 t, ad;\n\t"
        ".reg .b64 nd;\n\t"
        "add.u32 ad, %1, %0;\n\t"
        "ld.shared.u64 nd, [ad];\n\t"
        "setp.ge.u64 p, %2, nd;\n\t"
        "selp.b32 t, %4, %3, p;\n\t"
        "mad.lo.u32 %0, %0, 2, t;\n\t"
        "}"
        : "+r"(a)
        : "r"(sbase), "l"(key), "r"(t0), "r"(t1));
}

// Branchless classification of E keys through the replicated tree,
// level by level so that the E lookups of a level are in flight together.
template <int E, int LOGK>
__device__ __forceinline__ void k2_bucket_keys(const u64 (&key)[E], u32 valid, const u64* tree, const u64* spl,
                                               u32 logk, u32 kprime, u32 eq, u32 (&bk)[E]) {
    u32 a[E];
    const u32 cofs = (threadIdx.x & (TREE_COPIES - 1)) * 8u;
    const u32 t0 = 0u - cofs, t1 = TREE_NODE_BYTES - cofs;
    const u32 sb = (u32)__cvta_generic_to_shared(tree);
    if (LOGK == 8) {
        // levels 0-2 from registers (nodes 1..7, the same for every lane), then 3-7 from
        // the replicated tree in shared memory
        const u64 n1 = tree[1 * TREE_COPIES], n2 = tree[2 * TREE_COPIES], n3 = tree[3 * TREE_COPIES];
        const u64 n4 = tree[4 * TREE_COPIES], n5 = tree[5 * TREE_COPIES], n6 = tree[6 * TREE_COPIES],
                  n7 = tree[7 * TREE_COPIES];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const bool p0 = key[e] >= n1;
            const bool p1 = key[e] >= (p0 ? n3 : n2);
            const u64 m2 = p0 ? (p1 ? n7 : n6) : (p1 ? n5 : n4);
            const bool p2 = key[e] >= m2;
            const u32 j = 8u + (p0 ? 4u : 0u) + (p1 ? 2u : 0u) + (p2 ? 1u : 0u);
            a[e] = j * TREE_NODE_BYTES + cofs;
        }
#pragma unroll
        for (int l = 3; l < 8; ++l)
#pragma unroll
            for (int e = 0; e < E; ++e) descend_step_nb(key[e], sb, a[e], t0, t1);
    } else {
        const u64 root = tree[cofs / 8 + TREE_COPIES];
#pragma unroll
        for (int e = 0; e < E; ++e) a[e] = (key[e] >= root ? 3u : 2u) * TREE_NODE_BYTES + cofs;
        for (u32 l = 1; l < logk; ++l)
#pragma unroll
            for (int e = 0; e < E; ++e) descend_step_nb(key[e], sb, a[e], t0, t1);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        u32 i = (a[e] - cofs) / TREE_NODE_BYTES - kprime;
        if (eq) {
            const u32 ii = i ? i : 1u;
            const bool isq = i >= 1u && spl[ii] >= key[e];
            i = 2 * i - (isq ? 1u : 0u);
        }
        bk[e] = ((valid >> e) & 1u) ? i : INV_BUCKET;
    }
}

// Classification through the bucket-hint table (common.cuh): the leaf a key reaches in the
// splitter tree (the number of padded splitters <= key, ties right) is
// A + #{j in 1..d : s_{A+j} <= key} for the entry (A, d) of the key's cell.  Nearly every cell
// holds at most one splitter, so one comparison settles the key; cells with several
// splitters finish with a binary search over them (all lanes of a warp wait for it only when
// one of them needs it).  Equality buckets as in k2_bucket_keys.
template <int E, bool FULL = false, bool HI32 = false>
__device__ __forceinline__ void k2_bucket_keys_lut(const u64 (&key)[E], u32 valid, const unsigned short* lut,
                                                   const u64* spl, u64 lut_lo, u32 lut_sh, u32 eq, u32 (&bk)[E]) {
    u32 cnt[E], en[E], more = 0;
    // HI32 (lut_sh >= 32; lut_lo is a multiple of 2^lut_sh): the cell from the keys' high words
    const u32 lo_hi = (u32)(lut_lo >> 32) >> (lut_sh - 32u);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        u32 c;
        if constexpr (HI32) {
            const u32 kh = (u32)(key[e] >> 32) >> (lut_sh - 32u);
            c = kh < lo_hi ? LUT_N : min(kh - lo_hi, LUT_N - 1u);
        } else {
            const u64 y = (key[e] - lut_lo) >> lut_sh;
            c = (y >> LUT_LOG) != 0ull ? LUT_N - 1u : (u32)y;
            c = key[e] < lut_lo ? LUT_N : c;
        }
        en[e] = lut[c];
        const u32 A = en[e] & 0xFFu, d = en[e] >> 8;
#if IPS4O_K2_PRED_SPL
        // only keys whose cell holds a splitter (d > 0; ~6 % of the cells at k = 256) load
        // its first splitter: a predicated load (branch-free), so the other lanes add no
        // shared-memory wavefronts
        u64 s1 = ~0ull;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.u64 %0, [%1];\n\t}"
                     : "+l"(s1)
                     : "r"((u32)__cvta_generic_to_shared(spl + min(A + 1u, (u32)MAXK - 1u))), "r"(d));
#else
        // (branch-free: every key loads its cell's first splitter, used only if d > 0)
        const u64 s1 = spl[min(A + 1u, (u32)MAXK - 1u)];
#endif
        const u32 ge = (u32)(key[e] >= s1) & (u32)(d != 0u);
        cnt[e] = A + ge;
        more |= (ge & (u32)(d > 1u)) << e;
    }
    if (__any_sync(0xffffffffu, more != 0u)) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (more & (1u << e)) {
                // s_l <= key for l = A+1; candidates s_{l+1} .. s_{l+n}
                u32 l = cnt[e], n = (en[e] >> 8) - 1u;
                while (n) {
                    const u32 h = (n + 1u) >> 1;
                    if (key[e] >= spl[l + h]) {
                        l += h;
                        n -= h;
                    } else {
                        n = h - 1u;
                    }
                }
                cnt[e] = l;
            }
        }
    }
    if (eq) {  // (one uniform branch for all E keys)
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const u32 i = cnt[e];
            const u32 ii = i ? i : 1u;
            const bool isq = i >= 1u && spl[ii] >= key[e];
            cnt[e] = 2 * i - (isq ? 1u : 0u);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) bk[e] = (FULL || ((valid >> e) & 1u)) ? cnt[e] : INV_BUCKET;
}

// Elements of a tile that start a bucket's next buffer block while the buffer's completed
// block is still being flushed: kept in registers and written into the buffer during the
// next tile's placement, after the flush has read the buffer (so the TMA read latency
// overlaps the next tile's classification instead of stalling a barrier).
template <class TR, int E>
struct K2Defer {
    typename TR::V v[E];
    u32 idx[E];  // buffer slot: bucket * B + offset
    u32 mask;
};

template <class TR, int NT, int E, int LOGK, bool AGG, bool FULL = false, bool HI32 = false>
__device__ __forceinline__ void k2_tile(const Mem<TR>& mem, const uint4 (&raw)[E / TR::VEC],
                                        u32 valid, bool final_tile, u64 mb, u32 cap,
                                        typename TR::V* buf, u32* nbl,
                                        const u64* tree, const u64* spl, u32* fill, u32* cnt,
                                        u32* slotb, u32* nfl, u32* s_nflushed, u32 logk,
                                        u32 kprime, u32 eq, u64 refill,
                                        typename TR::V* refill_stage, u64* refill_mbar, K2Defer<TR, E>& df,
                                        bool& agg, const unsigned short* lut, u64 lut_lo, u32 lut_sh) {
    typedef typename TR::V V;
    constexpr int B = TR::B;
    const u32 tid = threadIdx.x;
    V v[E];
#pragma unroll
    for (int i = 0; i < E / TR::VEC; ++i) memcpy(&v[i * TR::VEC], &raw[i], 16);
    // 1. classify; 2. rank: the position of the element in its bucket's stream of this
    //    stripe is the value a shared-memory atomic increment of the bucket count returns
    //    (elements of a bucket may take any order)
    u32 bk[E], pos[E];
    {
        u64 key[E];
#pragma unroll
        for (int e = 0; e < E; ++e) key[e] = TR::key(v[e], 0);
#if IPS4O_K2_LUT
        k2_bucket_keys_lut<E, FULL, HI32>(key, valid, lut, spl, lut_lo, lut_sh, eq, bk);
#else
        k2_bucket_keys<E, LOGK>(key, valid, tree, spl, logk, kprime, eq, bk);
#endif
    }
    // (skewed tiles -- sorted runs, equal keys: the previous tile put more than 1/8 of its
    // elements into one bucket -- check each slot for a warp whose 32 elements share a
    // bucket; such a warp takes its 32 positions with one atomic instead of 32 serialised)
    const u32 lane = tid & 31;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        bool done = false;
        if (AGG) {
            const u32 b0 = __shfl_sync(0xffffffffu, bk[j], 0);
            if (__all_sync(0xffffffffu, bk[j] == b0) && (FULL || b0 != INV_BUCKET)) {
                u32 base = 0;
                if (lane == 0) base = atomicAdd(&cnt[b0], 32u);
                pos[j] = __shfl_sync(0xffffffffu, base, 0) + lane;
                done = true;
            }
        }
        if (!done && (FULL || bk[j] != INV_BUCKET)) pos[j] = atomicAdd(&cnt[bk[j]], 1u);
        // bucket (< 2^16) and position (< B + tile < 2^16) in one register until placement
        if (FULL || bk[j] != INV_BUCKET) bk[j] |= pos[j] << 16;
    }
    __syncthreads();
    if (refill != ~0ull && tid == 0) {
        // every thread has read the stage: load the tile two ahead into it (WAR across the
        // generic and async proxies: fence first)
        fence_proxy_async_smem();
        k2_stage_load<TR, NT, E>(refill_stage, mem, refill, refill_mbar);
    }
    // 3. per bucket: the previous tile's flush has read the buffer; blocks completed in
    //    this tile and their flush slots.  cnt[b] counts the bucket's stream from the first
    //    element of its buffer (the atomics above returned buffer-relative positions); it is
    //    rebased past the blocks flushed now, nbl[b] counts the flushed blocks.
    bool hot = false;
    if (tid < (u32)MAXK) {
        if (!IPS4O_K2_WFLUSH) bulk_wait_read0();
        const u32 b = tid;
        const u32 run = cnt[b];  // buffered (incl. deferred) + new elements
        hot = run - fill[b] > (u32)(NT * E / 8);
        u32 nf = run / B, slot = 0;
        if (nf) {
            if (final_tile) {
                // head elements of the first stripe (< one 16-byte vector): at most one
                // bucket completes a block; keep it buffered if the stripe has no room.
                if (*s_nflushed + nf <= cap) {
                    slot = *s_nflushed;
                    *s_nflushed += nf;
                } else {
                    nf = 0;
                }
            } else {
                slot = atomicAdd(s_nflushed, nf);
            }
        }
        nfl[b] = nf;
        slotb[b] = slot;
        cnt[b] = run - nf * B;
        fill[b] = run - nf * B;
        nbl[b] += nf;
    }
    if (AGG || LOGK == 8) agg = __syncthreads_or(hot);
    else __syncthreads();
    // 4. place: the previous tile's deferred elements, then this tile's: first block ->
    //    smem buffer, later complete blocks -> straight to the stripe, the start of the
    //    next block -> deferred
#pragma unroll
    for (int j = 0; j < E; ++j)
        if (df.mask & (1u << j)) K2Buf<TR>::put(buf, df.idx[j], df.v[j]);
    u32 defer = 0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        if (!FULL && bk[j] == INV_BUCKET) continue;
        const u32 b = bk[j] & 0xFFFFu;
        const u32 p = bk[j] >> 16;
        const u32 q = p / B, off = p % B;
        if (q == 0) {
            K2Buf<TR>::put(buf, b * B + off, v[j]);
        } else {
            const u32 nf = nfl[b];
            if (q < nf) {
                mem.st(mb + (u64)(slotb[b] + q) * B + off, v[j]);
            } else {
                df.v[j] = v[j];
                df.idx[j] = b * B + (p - nf * B);
                defer |= 1u << j;
            }
        }
    }
    df.mask = defer;
#if IPS4O_K2_WFLUSH
    static_assert(!TR::KV, "warp flushes: AoS element types only");
    typename TR::V* data = mem.d;
    __syncthreads();
    // 5. flush complete buffer blocks: warp w copies the blocks of buckets w, w + NT/32, ...
    //    (one 16-byte vector per lane and block, two blocks in flight); the next tile's
    //    barriers order these reads before the buffers are refilled
    {
        constexpr u32 NWP = NT / 32, NV = B * sizeof(V) / 16;
        static_assert(NV <= 32, "a block is one vector per lane");
        const u32 w = tid >> 5;
        const u32 bl = w + NWP * lane;
        u32 m = __ballot_sync(0xffffffffu, bl < (u32)MAXK && nfl[bl] != 0u);
        while (m) {
            const u32 b0 = w + NWP * (u32)(__ffs(m) - 1);
            m &= m - 1;
            const bool two = m != 0u;
            const u32 b1 = two ? w + NWP * (u32)(__ffs(m) - 1) : b0;
            if (two) m &= m - 1;
            if (lane < NV) {
                const uint4 x0 = reinterpret_cast<const uint4*>(buf + b0 * B)[lane];
                const uint4 x1 = reinterpret_cast<const uint4*>(buf + b1 * B)[lane];
                reinterpret_cast<uint4*>(data + mb + (u64)slotb[b0] * B)[lane] = x0;
                if (two) reinterpret_cast<uint4*>(data + mb + (u64)slotb[b1] * B)[lane] = x1;
            }
        }
    }
#else
    fence_proxy_async_smem();
    __syncthreads();
    // 5. flush complete buffer blocks with TMA bulk copies (their reads are awaited at the
    //    next tile's step 3)
    if (tid < (u32)MAXK && nfl[tid]) {
        K2Buf<TR>::flush(mem, mb + (u64)slotb[tid] * B, buf, tid);
        bulk_commit();
    }
#endif
}

// End of a stripe: the last flushes have read their buffers; deferred elements join the
// buffers (which then hold every partial block).
template <class TR, int E>
__device__ __forceinline__ void k2_drain(typename TR::V* buf, K2Defer<TR, E>& df) {
    if (threadIdx.x < (u32)MAXK) bulk_wait_read0();
    __syncthreads();
#pragma unroll
    for (int j = 0; j < E; ++j)
        if (df.mask & (1u << j)) K2Buf<TR>::put(buf, df.idx[j], df.v[j]);
    df.mask = 0;
    __syncthreads();
}

// Local classification of one stripe by the whole CTA: the stripe's front
// receives s_nflushed full blocks; per bucket fill / cnt / nbl count its buffered elements,
// flushed blocks and total; the partially filled buffers stay in buf (deferred elements
// joined).  The task's classifier is in shared memory (spl, lut, rtree); fill, cnt, nbl and
// *s_nflushed are zero on entry.  s_mbar: two initialised mbarriers with their phase bits.
template <class TR, int NT, int E, int ST = K2_STAGES>
__device__ __forceinline__ void k2_stripe(const Mem<TR>& mem, const StripeDesc& sd, const TaskParam& tp,
                                          typename TR::V* buf, u64* rtree, u64* spl, u32* fill, u32* cnt, u32* slotb,
                                          u32* nfl, u32* nbl, typename TR::V* stage, unsigned short* lut,
                                          u32* s_nflushed_p, u64* s_mbar, u32& phase) {
    constexpr int B = TR::B;
    constexpr u32 TILE = NT * E;
    const u32 tid = threadIdx.x;
    u32& s_nflushed = *s_nflushed_p;
    const u64 mb = sd.begin > tp.g ? sd.begin : tp.g;  // stripe main region start (block aligned)
    const u64 me = sd.end;
    K2Defer<TR, E> df;
    df.mask = 0;
    bool agg = false;  // skewed tiles: aggregate the atomics of uniform warps
    const u32 cap = me > mb ? (u32)((me - mb) / B) : 0u;
    if (mb < me) {
        // full tiles: staged in shared memory by TMA bulk loads two tiles ahead (a tile
        // is contiguous: one cp.async.bulk each, completion on the stage's mbarrier);
        // then the (single) partial tail tile by direct 128-bit loads
        const u64 nft = (me - mb) / TILE;
        uint4 cur[E / TR::VEC];
        constexpr u32 ALL = (E >= 32) ? 0xFFFFFFFFu : ((1u << E) - 1u);
        if (tid == 0) {
            for (u64 k = 0; k < (u64)ST && k < nft; ++k)
                k2_stage_load<TR, NT, E>(stage + k * TILE, mem, mb + k * TILE, &s_mbar[k]);
        }
        for (u64 ti = 0; ti < nft; ++ti) {
            const u32 st = ST == 2 ? (u32)(ti & 1) : 0u;
            mbar_wait(&s_mbar[st], (phase >> st) & 1u);
            phase ^= 1u << st;
            k2_stage_read<TR, NT, E>(stage + st * TILE, cur);
            // two stages: the tile's first barrier follows every thread's reads of the
            // stage, and the refill for tile ti+2 is issued after it, inside k2_tile; one
            // stage: an extra barrier here, then the load of tile ti+1
            u64 refill = ~0ull;
            if (ST == 2) {
                refill = ti + 2 < nft ? mb + (ti + 2) * TILE : ~0ull;
            } else {
                __syncthreads();
                if (tid == 0 && ti + 1 < nft) {
                    fence_proxy_async_smem();
                    k2_stage_load<TR, NT, E>(stage, mem, mb + (ti + 1) * TILE, &s_mbar[0]);
                }
            }
            if (tp.logk == 8 && !agg && tp.lut_sh >= 32u)
                k2_tile<TR, NT, E, 8, false, true, true>(mem, cur, ALL, false, mb, cap, buf, nbl, rtree, spl, fill, cnt,
                                                         slotb, nfl, s_nflushed_p, tp.logk, tp.kprime, tp.eq,
                                                         refill, stage + st * TILE, &s_mbar[st], df, agg, lut, tp.lut_lo, tp.lut_sh);
            else if (tp.logk == 8 && !agg)
                k2_tile<TR, NT, E, 8, false, true>(mem, cur, ALL, false, mb, cap, buf, nbl, rtree, spl, fill, cnt,
                                             slotb, nfl, s_nflushed_p, tp.logk, tp.kprime, tp.eq,
                                             refill, stage + st * TILE, &s_mbar[st], df, agg, lut, tp.lut_lo, tp.lut_sh);
            else
                k2_tile<TR, NT, E, 0, true, true>(mem, cur, ALL, false, mb, cap, buf, nbl, rtree, spl, fill, cnt,
                                            slotb, nfl, s_nflushed_p, tp.logk, tp.kprime, tp.eq,
                                            refill, stage + st * TILE, &s_mbar[st], df, agg, lut, tp.lut_lo, tp.lut_sh);
        }
        const u64 tb = mb + nft * TILE;
        if (tb < me) {
            const u32 vt = k2_load<TR, NT, E>(mem, tb, (u32)(me - tb), cur);
            k2_tile<TR, NT, E, 0, true>(mem, cur, vt, false, mb, cap, buf, nbl, rtree, spl, fill, cnt,
                                  slotb, nfl, s_nflushed_p, tp.logk, tp.kprime, tp.eq,
                                  ~0ull, nullptr, nullptr, df, agg, lut, tp.lut_lo, tp.lut_sh);
        }
    }
    if (sd.first && tp.lo < tp.g) {
        // head elements [lo, g) of the task, processed last so that every write stays
        // behind the read frontier (their block grid starts at g)
        const u64 hend = tp.g < tp.hi ? tp.g : tp.hi;
        uint4 hv[E / TR::VEC];
        const u32 hval = k2_load<TR, NT, E>(mem, tp.lo, (u32)(hend - tp.lo), hv);
        k2_tile<TR, NT, E, 0, true>(mem, hv, hval, true, mb, cap, buf, nbl, rtree, spl, fill, cnt, slotb, nfl,
                       s_nflushed_p, tp.logk, tp.kprime, tp.eq, ~0ull, nullptr, nullptr, df, agg, lut, tp.lut_lo, tp.lut_sh);
    }
    k2_drain<TR, E>(buf, df);
}

template <class TR, int NT, int E, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_classify(LevelArgs A0) {
    const LevelArgs A = with_dyn(A0);
    typedef typename TR::V V;
    typedef K2Smem<TR, NT, E, K2_MAIN_STAGES> SM;
    constexpr int B = TR::B;
    constexpr u32 TILE = NT * E;
    extern __shared__ __align__(128) unsigned char smem[];
    V* buf = reinterpret_cast<V*>(smem);
    u64* tree = reinterpret_cast<u64*>(smem + SM::buf_bytes + SM::wcnt_bytes);
    u64* spl = tree + MAXK;
    u32* fill = reinterpret_cast<u32*>(spl + MAXK);
    u32* cnt = fill + MAXK;
    u32* slotb = cnt + MAXK;
    u32* nfl = slotb + MAXK;
    u32* nbl = nfl + MAXK;
    u64* rtree = reinterpret_cast<u64*>(smem + SM::buf_bytes + SM::wcnt_bytes + SM::tree_bytes + SM::arr_bytes);
    V* stage = reinterpret_cast<V*>(smem + SM::buf_bytes + SM::wcnt_bytes + SM::tree_bytes + SM::arr_bytes +
                                    SM::rtree_bytes);
    unsigned short* lut = reinterpret_cast<unsigned short*>(reinterpret_cast<unsigned char*>(stage) + SM::stage_bytes);
    __shared__ u32 s_stripe, s_nflushed, s_wsum[NT / 32];
    __shared__ u64 s_spbase;
    __shared__ __align__(8) u64 s_mbar[2];
    u32 phase = 0;  // parity of the next completion of each stage's mbarrier (bits 0, 1)
    if (threadIdx.x == 0) {
        mbar_init(&s_mbar[0], 1);
        mbar_init(&s_mbar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const Mem<TR> mem(A.data, A.vals);

    for (;;) {
        if (tid == 0) {
            u32 tk = atomicAdd(&A.ctr[CTR_STRIPE], 1u);
            s_stripe = tk < A.nstripes ? A.stripe_order[tk] : 0xFFFFFFFFu;
        }
        __syncthreads();
        const u32 sidx = s_stripe;
        if (sidx == 0xFFFFFFFFu) return;
        const StripeDesc sd = A.sd[sidx];
        const TaskParam tp = A.tp[sd.task];
        if (tid < (u32)MAXK) {
            tree[tid] = A.tree[(u64)sd.task * MAXK + tid];
            spl[tid] = A.spl[(u64)sd.task * MAXK + tid];
            fill[tid] = 0;
            cnt[tid] = 0;
            nbl[tid] = 0;
        }
        if (!IPS4O_K2_LUT) rtree_fill(rtree, A.tree + (u64)sd.task * MAXK, tid, NT);
        if (IPS4O_K2_LUT) {
            const uint4* gl = reinterpret_cast<const uint4*>(A.lut + (u64)sd.task * LUT_STRIDE);
            for (u32 i = tid; i < LUT_STRIDE * 2 / 16; i += NT) reinterpret_cast<uint4*>(lut)[i] = gl[i];
        }
        if (tid == 0) s_nflushed = 0;
        __syncthreads();
        k2_stripe<TR, NT, E, K2_MAIN_STAGES>(mem, sd, tp, buf, rtree, spl, fill, cnt, slotb, nfl, nbl, stage, lut, &s_nflushed, s_mbar,
                             phase);
        // ---- publish counts; spill partial buffers (compacted) to the auxiliary area
        u32 f = tid < (u32)MAXK ? fill[tid] : 0u;
        u32 incl = f;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (u32)o) incl += y;
        }
        if (lane == 31) s_wsum[w] = incl;
        __syncthreads();
        u32 woff = 0, total = 0;
        for (u32 ww = 0; ww < (u32)MAXK / 32; ++ww) {
            if (ww < w) woff += s_wsum[ww];
            total += s_wsum[ww];
        }
        const u32 excl = woff + incl - f;
        if (tid == 0) s_spbase = atomicAdd((unsigned long long*)A.spill_ctr, (unsigned long long)total);
        __syncthreads();
        if (tid < (u32)MAXK) {
            const u32 cb = nbl[tid] * (u32)B + cnt[tid];
            A.s_count[(u64)sidx * MAXK + tid] = cb;
            if (cb) atomicAdd((unsigned long long*)&A.btot[(u64)sd.task * MAXK + tid], (unsigned long long)cb);
            A.s_fill[(u64)sidx * MAXK + tid] = f;
            A.s_spoff[(u64)sidx * MAXK + tid] = excl;
            slotb[tid] = excl;
        }
        if (tid == 0) {
            A.s_spbase[sidx] = s_spbase;
            A.s_nfull[sidx] = s_nflushed;
            if (s_spbase + total > A.spill_cap) atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_SPILL);
        }
        __syncthreads();
        if (s_spbase + total <= A.spill_cap) {
            V* sp = reinterpret_cast<V*>(A.spill) + s_spbase;
            for (u32 b = w; b < (u32)MAXK; b += NT / 32) {
                const u32 fb = fill[b], ob = slotb[b];
                for (u32 j = lane; j < fb; j += 32) sp[ob + j] = K2Buf<TR>::get(buf, b * B + j);
            }
        }
        if (tid < (u32)MAXK) bulk_wait0();
        __syncthreads();
    }
}

}  // namespace ips4o
