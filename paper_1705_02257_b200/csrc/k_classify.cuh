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

template <class TR>
struct K2Smem {
    typedef typename TR::V V;
    static constexpr int B = TR::B;
    static constexpr int NW = K2_THREADS / 32;
    static constexpr size_t buf_bytes = (size_t)MAXK * B * sizeof(V);
    static constexpr size_t wcnt_bytes = (size_t)NW * MAXK * 2;
    static constexpr size_t tree_bytes = 2 * MAXK * 8;
    static constexpr size_t arr_bytes = 4 * MAXK * 4;
    static constexpr size_t total = buf_bytes + wcnt_bytes + tree_bytes + arr_bytes;
};

template <class TR>
__device__ __forceinline__ void k2_tile(typename TR::V* __restrict__ data, u64 tb, u32 len,
                                        bool final_tile, u64 mb, u32 cap,
                                        typename TR::V* buf, unsigned short* wcnt,
                                        const u64* tree, const u64* spl, u32* fill, u32* cnt,
                                        u32* slotb, u32* nfl, u32* s_nflushed, u32 logk,
                                        u32 kprime, u32 eq) {
    typedef typename TR::V V;
    constexpr int B = TR::B, E = TR::E2, VEC = TR::VEC, NV = E / VEC;
    const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

    V v[E];
    u32 bk[E];
    u32 pos[E];
    // 1. load + classify
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const u32 e0 = (u32)(i * K2_THREADS + tid) * VEC;
        if (e0 + VEC <= len) {
            uint4 x = ld_nc_v4(data + tb + e0);
            V tmp[VEC];
            memcpy(tmp, &x, 16);
#pragma unroll
            for (int q = 0; q < VEC; ++q) v[i * VEC + q] = tmp[q];
#pragma unroll
            for (int q = 0; q < VEC; ++q)
                bk[i * VEC + q] = classify_key(TR::key(v[i * VEC + q]), tree, spl, logk, kprime, eq);
        } else {
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                if (e0 + q < len) {
                    v[i * VEC + q] = data[tb + e0 + q];
                    bk[i * VEC + q] = classify_key(TR::key(v[i * VEC + q]), tree, spl, logk, kprime, eq);
                } else {
                    v[i * VEC + q] = TR::pad();
                    bk[i * VEC + q] = INV_BUCKET;
                }
            }
        }
    }
    // 2. warp-aggregated ranking
    const u32 lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const u32 b = bk[j];
        const u32 peers = __match_any_sync(0xffffffffu, b);
        const u32 leader = __ffs(peers) - 1;
        u32 base = 0;
        if (lane == leader && b != INV_BUCKET) {
            base = wcnt[w * MAXK + b];
            wcnt[w * MAXK + b] = (unsigned short)(base + __popc(peers));
        }
        base = __shfl_sync(0xffffffffu, base, leader);
        pos[j] = base + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();
    // 3. per bucket: offsets over warps, completed blocks, flush slots
    if (tid < (u32)MAXK) {
        const u32 b = tid;
        const u32 f = fill[b];
        u32 run = f;
#pragma unroll
        for (int ww = 0; ww < K2_THREADS / 32; ++ww) {
            u32 c = wcnt[ww * MAXK + b];
            wcnt[ww * MAXK + b] = (unsigned short)run;
            run += c;
        }
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
        cnt[b] += run - f;
        fill[b] = run - nf * B;
    }
    __syncthreads();
    // 4. place: first block -> smem buffer, later complete blocks -> straight to the stripe
    u32 defer = 0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const u32 b = bk[j];
        if (b == INV_BUCKET) continue;
        const u32 p = (u32)wcnt[w * MAXK + b] + pos[j];
        const u32 q = p / B, off = p % B, nf = nfl[b];
        if (q == 0) {
            buf[b * B + off] = v[j];
        } else if (q < nf) {
            data[mb + (u64)(slotb[b] + q) * B + off] = v[j];
        } else {
            pos[j] = p - nf * B;
            defer |= 1u << j;
        }
    }
    fence_proxy_async_smem();
    __syncthreads();
    // 5. flush complete buffer blocks with TMA bulk copies
    if (tid < (u32)MAXK && nfl[tid]) {
        bulk_s2g(data + mb + (u64)slotb[tid] * B, buf + tid * B, B * sizeof(V));
        bulk_commit();
        bulk_wait_read0();
    }
    __syncthreads();
    // 6. remainders start the next buffer; reset per-warp counters
#pragma unroll
    for (int j = 0; j < E; ++j)
        if (defer & (1u << j)) buf[bk[j] * B + pos[j]] = v[j];
    if (tid < (u32)MAXK) {
#pragma unroll
        for (int ww = 0; ww < K2_THREADS / 32; ++ww) wcnt[ww * MAXK + tid] = 0;
    }
    __syncthreads();
}

template <class TR>
__global__ void __launch_bounds__(K2_THREADS, 1) k_classify(LevelArgs A) {
    typedef typename TR::V V;
    typedef K2Smem<TR> SM;
    constexpr int B = TR::B, E = TR::E2;
    constexpr u32 TILE = K2_THREADS * E;
    extern __shared__ __align__(128) unsigned char smem[];
    V* buf = reinterpret_cast<V*>(smem);
    unsigned short* wcnt = reinterpret_cast<unsigned short*>(smem + SM::buf_bytes);
    u64* tree = reinterpret_cast<u64*>(smem + SM::buf_bytes + SM::wcnt_bytes);
    u64* spl = tree + MAXK;
    u32* fill = reinterpret_cast<u32*>(spl + MAXK);
    u32* cnt = fill + MAXK;
    u32* slotb = cnt + MAXK;
    u32* nfl = slotb + MAXK;
    __shared__ u32 s_stripe, s_nflushed, s_wsum[K2_THREADS / 32];
    __shared__ u64 s_spbase;
    const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    V* data = reinterpret_cast<V*>(A.data);

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
#pragma unroll
            for (int ww = 0; ww < K2_THREADS / 32; ++ww) wcnt[ww * MAXK + tid] = 0;
        }
        if (tid == 0) s_nflushed = 0;
        __syncthreads();
        const u64 mb = sd.begin > tp.g ? sd.begin : tp.g;  // stripe main region start (block aligned)
        const u64 me = sd.end;
        const u32 cap = me > mb ? (u32)((me - mb) / B) : 0u;
        for (u64 tb = mb; tb < me; tb += TILE) {
            const u32 len = (u32)((me - tb) < TILE ? (me - tb) : TILE);
            k2_tile<TR>(data, tb, len, false, mb, cap, buf, wcnt, tree, spl, fill, cnt, slotb, nfl,
                        &s_nflushed, tp.logk, tp.kprime, tp.eq);
        }
        if (sd.first && tp.lo < tp.g) {
            // head elements [lo, g) of the task, processed last so that every write stays
            // behind the read frontier (their block grid starts at g)
            const u64 hend = tp.g < tp.hi ? tp.g : tp.hi;
            k2_tile<TR>(data, tp.lo, (u32)(hend - tp.lo), true, mb, cap, buf, wcnt, tree, spl,
                        fill, cnt, slotb, nfl, &s_nflushed, tp.logk, tp.kprime, tp.eq);
        }
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
            A.s_count[(u64)sidx * MAXK + tid] = cnt[tid];
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
            for (u32 b = w; b < (u32)MAXK; b += K2_THREADS / 32) {
                const u32 fb = fill[b], ob = slotb[b];
                for (u32 j = lane; j < fb; j += 32) sp[ob + j] = buf[b * B + j];
            }
        }
        if (tid < (u32)MAXK) bulk_wait0();
        __syncthreads();
    }
}

}  // namespace ips4o
