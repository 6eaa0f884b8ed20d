// k_classify_rec.cuh -- K2 for 100-byte records (local classification).
//
// Same algorithm as k_classify.cuh with records: a tile of NT records is staged in shared
// memory by coalesced 4-byte loads (records are only 4-byte aligned), each thread
// classifies one record on the task's key part (branchless descent + ballot peers), the
// record is copied into its bucket's 4-record buffer block (400 B), and full buffers are
// written back to the consumed front of the stripe by warp-cooperative coalesced copies.
// The block grid of a record task starts at lo (no 16-byte alignment requirement).
#pragma once
#include "common.cuh"
#include "k_classify.cuh"

namespace ips4o {

template <int NT>
struct K2RecSmem {
    static constexpr int NW = NT / 32;
    static constexpr size_t buf_bytes = (size_t)MAXK * TRec::B * 100;
    static constexpr size_t stage_bytes = (size_t)NT * 100;
    static constexpr size_t wcnt_bytes = (size_t)NW * MAXK * 2;
    static constexpr size_t tree_bytes = 2 * MAXK * 8;
    static constexpr size_t arr_bytes = 4 * MAXK * 4;
    static constexpr size_t rtree_bytes = (size_t)MAXK * TREE_COPIES * 8;
    static constexpr size_t total = buf_bytes + stage_bytes + wcnt_bytes + tree_bytes + arr_bytes + rtree_bytes;
};

__device__ __forceinline__ void copy_rec(u32* dst, const u32* src) {
#pragma unroll
    for (int i = 0; i < 25; ++i) dst[i] = src[i];
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_classify_rec(LevelArgs A) {
    typedef K2RecSmem<NT> SM;
    constexpr int B = TRec::B;     // records per block
    constexpr int NW = NT / 32;
    constexpr u32 RW = 25;         // words per record
    extern __shared__ __align__(128) unsigned char smem[];
    u32* buf = reinterpret_cast<u32*>(smem);                                   // [256][B][25]
    u32* stage = reinterpret_cast<u32*>(smem + SM::buf_bytes);                 // [NT][25]
    unsigned short* wcnt = reinterpret_cast<unsigned short*>(smem + SM::buf_bytes + SM::stage_bytes);
    u64* tree = reinterpret_cast<u64*>(smem + SM::buf_bytes + SM::stage_bytes + SM::wcnt_bytes);
    u64* spl = tree + MAXK;
    u32* fill = reinterpret_cast<u32*>(spl + MAXK);
    u32* cnt = fill + MAXK;
    u32* slotb = cnt + MAXK;
    u32* nfl = slotb + MAXK;
    u64* rtree = reinterpret_cast<u64*>(smem + SM::buf_bytes + SM::stage_bytes + SM::wcnt_bytes + SM::tree_bytes +
                                        SM::arr_bytes);
    __shared__ u32 s_stripe, s_nflushed, s_wsum[NW];
    __shared__ u64 s_spbase;
    const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    u32* gw = reinterpret_cast<u32*>(A.data);

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
        for (u32 b = tid; b < (u32)MAXK; b += NT) {
            tree[b] = A.tree[(u64)sd.task * MAXK + b];
            spl[b] = A.spl[(u64)sd.task * MAXK + b];
            fill[b] = 0;
            cnt[b] = 0;
            for (int ww = 0; ww < NW; ++ww) wcnt[ww * MAXK + b] = 0;
        }
        rtree_fill(rtree, A.tree + (u64)sd.task * MAXK, tid, NT);
        if (tid == 0) s_nflushed = 0;
        __syncthreads();
        const u64 mb = sd.begin, me = sd.end;  // g == lo for records: no head region
        for (u64 tb = mb; tb < me; tb += NT) {
            const u32 len = (u32)((me - tb) < NT ? (me - tb) : NT);
            // stage the tile (coalesced 4-byte words)
            const u32* src = gw + tb * RW;
            for (u32 i = tid; i < len * RW; i += NT) stage[i] = src[i];
            __syncthreads();
            const bool valid = tid < len;
            const u32* my = stage + tid * RW;
            u64 key[1];
            key[0] = valid ? (tp.part ? TRec::lo_of(my[2]) : TRec::hi_of(my[0], my[1])) : 0ull;
            u32 bk[1], peers[1];
            const bool full = __all_sync(0xffffffffu, valid);
            if (tp.logk == 8)
                k2_classify_keys<1, 8>(key, valid ? 1u : 0u, full, rtree, spl, tp.logk, tp.kprime, tp.eq, bk, peers);
            else
                k2_classify_keys<1, 0>(key, valid ? 1u : 0u, full, rtree, spl, tp.logk, tp.kprime, tp.eq, bk, peers);
            // warp-aggregated ranking
            const u32 b = bk[0];
            const u32 leader = __ffs(peers[0]) - 1;
            u32 base = 0;
            if (lane == leader && b != INV_BUCKET) {
                base = wcnt[w * MAXK + b];
                wcnt[w * MAXK + b] = (unsigned short)(base + __popc(peers[0]));
            }
            base = __shfl_sync(0xffffffffu, base, leader);
            u32 pos = base + __popc(peers[0] & lanemask_lt());
            __syncthreads();
            for (u32 bb = tid; bb < (u32)MAXK; bb += NT) {
                const u32 f = fill[bb];
                u32 run = f;
                for (int ww = 0; ww < NW; ++ww) {
                    u32 c = wcnt[ww * MAXK + bb];
                    wcnt[ww * MAXK + bb] = (unsigned short)run;
                    run += c;
                }
                const u32 nf = run / B;
                nfl[bb] = nf;
                slotb[bb] = nf ? atomicAdd(&s_nflushed, nf) : 0u;
                cnt[bb] += run - f;
                fill[bb] = run - nf * B;
            }
            __syncthreads();
            bool defer = false;
            if (b != INV_BUCKET) {
                const u32 p = (u32)wcnt[w * MAXK + b] + pos;
                const u32 q = p / B, off = p % B, nf = nfl[b];
                if (q == 0) {
                    copy_rec(buf + (b * B + off) * RW, my);
                } else if (q < nf) {
                    copy_rec(gw + (mb + (u64)(slotb[b] + q) * B + off) * RW, my);
                } else {
                    pos = p - nf * B;
                    defer = true;
                }
            }
            __syncthreads();
            // flush complete buffer blocks: warp w handles buckets w, w+NW, ...
            for (u32 bb = w; bb < (u32)MAXK; bb += NW) {
                if (nfl[bb]) {
                    u32* dst = gw + (mb + (u64)slotb[bb] * B) * RW;
                    const u32* sb = buf + bb * B * RW;
                    for (u32 i = lane; i < B * RW; i += 32) dst[i] = sb[i];
                }
            }
            __syncthreads();
            if (defer) copy_rec(buf + (b * B + pos) * RW, my);
            for (u32 bb = tid; bb < (u32)MAXK; bb += NT)
                for (int ww = 0; ww < NW; ++ww) wcnt[ww * MAXK + bb] = 0;
            __syncthreads();
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
        for (u32 ww = 0; ww < (u32)NW; ++ww) {
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
            u32* sp = reinterpret_cast<u32*>(A.spill) + s_spbase * RW;
            for (u32 bb = w; bb < (u32)MAXK; bb += NW) {
                const u32 fb = fill[bb], ob = slotb[bb];
                for (u32 i = lane; i < fb * RW; i += 32) sp[ob * RW + i] = buf[bb * B * RW + i];
            }
        }
        __syncthreads();
    }
}

}  // namespace ips4o
