// k_classify_rec.cuh -- K2 for wide elements moved as 32-bit words: the 100-byte records
// and the 32-byte quartets (local classification).
//
// Same algorithm as k_classify.cuh: a tile of elements is staged in shared memory by a TMA
// bulk copy (records are only 4-byte aligned: the < 16 bytes around the aligned body by
// plain loads), each thread classifies its elements on the task's key part, the element's
// words are copied into its bucket's buffer block (records: 4 x 100 B, quartets: 16 x 32 B),
// and full buffers leave by TMA bulk stores into the consumed front of the stripe.
#pragma once
#include "common.cuh"
#include "k_classify.cuh"

namespace ips4o {

// threads and elements per thread and tile: records 256 x 2 (a 51 KB tile), quartets
// IPS4O_K2Q_NT x (1024 / IPS4O_K2Q_NT) (32 KB)
#ifndef IPS4O_K2Q_NT
#define IPS4O_K2Q_NT 256
#endif
#ifndef IPS4O_K2R_NT  // records: threads per K2 CTA (tile 512 records)
#define IPS4O_K2R_NT 512
#endif
template <class TR>
struct K2RecRpt {
    static constexpr int NT = TR::S >= 64 ? IPS4O_K2R_NT : IPS4O_K2Q_NT;
    static constexpr int v = TR::S >= 64 ? 512 / IPS4O_K2R_NT : 1024 / IPS4O_K2Q_NT;
};
#ifndef IPS4O_K2REC_STAGES  // tiles staged ahead by TMA (2: the next tile loads while this one is placed)
#define IPS4O_K2REC_STAGES 2
#endif
constexpr int K2REC_STAGES = IPS4O_K2REC_STAGES;

template <class TR, int NT>
struct K2RecSmem {
    static constexpr int NW = NT / 32;
    static constexpr size_t buf_bytes = (size_t)MAXK * TR::B * TR::S;
    static constexpr size_t stage1 = ((size_t)NT * K2RecRpt<TR>::v * TR::S + 16 + 15) / 16 * 16;  // one stage
    static constexpr size_t stage_bytes = stage1 * K2REC_STAGES;
    static constexpr size_t wcnt_bytes = 0;
    static constexpr size_t tree_bytes = 2 * MAXK * 8;
    static constexpr size_t arr_bytes = 5 * MAXK * 4;
    static constexpr size_t rtree_bytes = IPS4O_K2_LUT ? 0 : (size_t)MAXK * TREE_COPIES * 8;
    static constexpr size_t lut_bytes = IPS4O_K2_LUT ? (size_t)LUT_STRIDE * 2 : 0;  // bucket hints
    static constexpr size_t total =
        buf_bytes + stage_bytes + wcnt_bytes + tree_bytes + arr_bytes + rtree_bytes + lut_bytes;
};

// one element's words (quartets: 16-byte vectors -- their stage, buffer and block-grid
// addresses are 16-byte aligned; records: 4-byte words)
template <int RW>
__device__ __forceinline__ void copy_rec(u32* dst, const u32* src) {
    if constexpr (RW % 4 == 0) {
#pragma unroll
        for (int i = 0; i < RW / 4; ++i) reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    } else {
#pragma unroll
        for (int i = 0; i < RW; ++i) dst[i] = src[i];
    }
}

template <class TR, int NT>
__global__ void __launch_bounds__(NT, 1) k_classify_rec(LevelArgs A0) {
    const LevelArgs A = with_dyn(A0);
    typedef K2RecSmem<TR, NT> SM;
    constexpr int B = TR::B;       // elements per block
    constexpr int NW = NT / 32;
    constexpr u32 RW = TR::RW;     // words per element
    extern __shared__ __align__(128) unsigned char smem[];
    u32* buf = reinterpret_cast<u32*>(smem);                                   // [256][B][25]
    u32* stage = reinterpret_cast<u32*>(smem + SM::buf_bytes);                 // [stages][NT*RPT][RW]
    u64* tree = reinterpret_cast<u64*>(smem + SM::buf_bytes + SM::stage_bytes + SM::wcnt_bytes);
    u64* spl = tree + MAXK;
    u32* fill = reinterpret_cast<u32*>(spl + MAXK);
    u32* cnt = fill + MAXK;
    u32* slotb = cnt + MAXK;
    u32* nfl = slotb + MAXK;
    u32* nbl = nfl + MAXK;
    constexpr int RPT = K2RecRpt<TR>::v;
    constexpr int RS = RPT;  // record slots per thread
    constexpr u32 STW = (u32)(SM::stage1 / 4);  // words per stage
    __shared__ u32 s_head[3 * RW], s_hb[3];
    __shared__ __align__(8) u64 s_mbar[K2REC_STAGES];
    u32 sphase = 0;  // bit s: parity of stage s's next completion
    if (threadIdx.x == 0) {
        for (int i = 0; i < K2REC_STAGES; ++i) mbar_init(&s_mbar[i], 1);
        mbar_fence_init();
    }
    constexpr u32 RT = NT * RPT;  // records per tile
    u64* rtree = reinterpret_cast<u64*>(smem + SM::buf_bytes + SM::stage_bytes + SM::wcnt_bytes + SM::tree_bytes +
                                        SM::arr_bytes);
    unsigned short* lut = reinterpret_cast<unsigned short*>(reinterpret_cast<unsigned char*>(rtree) + SM::rtree_bytes);
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
        if (sidx == 0xFFFFFFFFu) {
            bulk_wait0();  // the block stores are complete before the CTA exits
            return;
        }
        const StripeDesc sd = A.sd[sidx];
        const TaskParam tp = A.tp[sd.task];
        for (u32 b = tid; b < (u32)MAXK; b += NT) {
            tree[b] = A.tree[(u64)sd.task * MAXK + b];
            spl[b] = A.spl[(u64)sd.task * MAXK + b];
            fill[b] = 0;
            cnt[b] = 0;
            nbl[b] = 0;
        }
        if (!IPS4O_K2_LUT) rtree_fill(rtree, A.tree + (u64)sd.task * MAXK, tid, NT);
        if (IPS4O_K2_LUT) {
            const uint4* gl = reinterpret_cast<const uint4*>(A.lut + (u64)sd.task * LUT_STRIDE);
            for (u32 i = tid; i < LUT_STRIDE * 2 / 16; i += NT) reinterpret_cast<uint4*>(lut)[i] = gl[i];
        }
        if (tid == 0) s_nflushed = 0;
        __syncthreads();
        // the block grid starts at g, the first 16-byte aligned record >= lo (TMA block
        // moves); the < 4 head records [lo, g) of a task's first stripe are classified after
        // its tiles and go straight to the spill with the partial buffers (they never
        // complete a block, so no flush can outrun the read frontier)
        const u64 mb = sd.begin > tp.g ? sd.begin : tp.g, me = sd.end;
        const u32 nhead = sd.first ? (u32)(tp.g - tp.lo) : 0u;
        if (tid < nhead * RW) s_head[tid] = gw[tp.lo * RW + tid];
        if (tid < 3) s_hb[tid] = INV_BUCKET;
        // stage tile ti into stage st: the 16-byte aligned body of its bytes by one TMA bulk
        // copy (mbarrier completion), the < 16 bytes before / after it by plain loads; record
        // r of the tile then starts at stage word dw + RW r.  The plain stores are ordered
        // before the tile's processing by the barriers in between.
        const u64 ntiles = mb < me ? (me - mb + RT - 1) / RT : 0ull;
        auto tile_geom = [&](u64 ti, uintptr_t& p0, uintptr_t& p1, uintptr_t& a0, uintptr_t& a1, uintptr_t& w0, u32& len) {
            const u64 tb = mb + ti * RT;
            len = (u32)((me - tb) < RT ? (me - tb) : RT);
            p0 = (uintptr_t)(gw + tb * RW);
            p1 = p0 + (uintptr_t)len * (u32)TR::S;
            a0 = (p0 + 15) & ~(uintptr_t)15;
            a1 = p1 & ~(uintptr_t)15;
            w0 = p0 & ~(uintptr_t)15;  // stage byte 0
        };
        auto stage_tile = [&](u64 ti, u32 st) {
            uintptr_t p0, p1, a0, a1, w0;
            u32 len;
            tile_geom(ti, p0, p1, a0, a1, w0, len);
            u32* sg = stage + st * STW;
            const u32 dw = (u32)((p0 - w0) / 4);
            if (tid == 0) {
                fence_proxy_async_smem();  // earlier generic accesses of the stage before the TMA write
                if (a1 > a0) bulk_g2s(reinterpret_cast<char*>(sg) + (a0 - w0), reinterpret_cast<const void*>(a0),
                                      (u32)(a1 - a0), &s_mbar[st]);
                else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((u32)__cvta_generic_to_shared(&s_mbar[st])) : "memory");
            }
            // head words [p0, min(a0, p1)) and tail words [max(a1, a0), p1)
            const u32 nh = (u32)(((a0 < p1 ? a0 : p1) - p0) / 4);
            const uintptr_t t0 = a1 > a0 ? a1 : (a0 < p1 ? a0 : p1);
            const u32 nt = (u32)((p1 - t0) / 4);
            if (tid < nh) sg[dw + tid] = reinterpret_cast<const u32*>(p0)[tid];
            if (tid >= 32 && tid - 32 < nt) sg[(t0 - w0) / 4 + (tid - 32)] = reinterpret_cast<const u32*>(t0)[tid - 32];
        };
        for (u64 ti = 0; ti < (u64)K2REC_STAGES && ti < ntiles; ++ti) stage_tile(ti, (u32)ti);
        for (u64 ti = 0; ti < ntiles; ++ti) {
            const u32 st = K2REC_STAGES == 2 ? (u32)(ti & 1) : 0u;
            uintptr_t p0, p1, a0, a1, w0;
            u32 len;
            tile_geom(ti, p0, p1, a0, a1, w0, len);
            const u32 dw = (u32)((p0 - w0) / 4);
            const u32* sg = stage + st * STW;
            constexpr bool with_head = false;
            mbar_wait(&s_mbar[st], (sphase >> st) & 1u);
            sphase ^= 1u << st;
            __syncthreads();
            // classify this thread's records (branchless descent) and rank
            // them in their buckets' buffer streams by shared-memory atomics (any order
            // inside a bucket)
            auto rec_ptr = [&](int r) -> const u32* {
                return r < RPT ? sg + dw + (tid + r * NT) * RW : s_head + tid * RW;
            };
            u64 key[RS];
            u32 valid = 0;
#pragma unroll
            for (int r = 0; r < RS; ++r) {
                const u32* my = rec_ptr(r);
                const bool ok = r < RPT ? tid + r * NT < len : (with_head && tid < nhead);
                key[r] = ok ? TR::key_w(my, tp.part) : 0ull;
                valid |= (ok ? 1u : 0u) << r;
            }
            u32 bk[RS], pos[RS];
#if IPS4O_K2_LUT
            k2_bucket_keys_lut<RS>(key, valid, lut, spl, tp.lut_lo, tp.lut_sh, tp.eq, bk);
#else
            if (tp.logk == 8) k2_bucket_keys<RS, 8>(key, valid, rtree, spl, tp.logk, tp.kprime, tp.eq, bk);
            else k2_bucket_keys<RS, 0>(key, valid, rtree, spl, tp.logk, tp.kprime, tp.eq, bk);
#endif
#pragma unroll
            for (int r = 0; r < RS; ++r)
                if (bk[r] != INV_BUCKET) pos[r] = atomicAdd(&cnt[bk[r]], 1u);
            __syncthreads();
            // per bucket: completed blocks, flush slots; rebase the buffer-relative counts
            for (u32 bb = tid; bb < (u32)MAXK; bb += NT) {
                const u32 run = cnt[bb];
                const u32 nf = run / B;
                nfl[bb] = nf;
                slotb[bb] = nf ? atomicAdd(&s_nflushed, nf) : 0u;
                cnt[bb] = run - nf * B;
                fill[bb] = run - nf * B;
                nbl[bb] += nf;
            }
            __syncthreads();
            u32 defer = 0;
#pragma unroll
            for (int r = 0; r < RS; ++r) {
                const u32 b = bk[r];
                if (b == INV_BUCKET) continue;
                const u32* my = rec_ptr(r);
                const u32 p = pos[r];
                const u32 q = p / B, off = p % B, nf = nfl[b];
                if (q == 0) {
                    copy_rec<RW>(buf + (b * B + off) * RW, my);
                } else if (q < nf) {
                    copy_rec<RW>(gw + (mb + (u64)(slotb[b] + q) * B + off) * RW, my);
                } else {
                    pos[r] = p - nf * B;
                    defer |= 1u << r;
                }
            }
            fence_proxy_async_smem();  // the buffers' generic writes before the TMA reads them
            __syncthreads();
            // flush complete buffer blocks by TMA bulk stores (400-byte blocks: 16-byte aligned
            // in the block grid and in shared memory); read before the deferred records land
            for (u32 bb = tid; bb < (u32)MAXK; bb += NT) {
                if (nfl[bb]) {
                    bulk_s2g(gw + (mb + (u64)slotb[bb] * B) * RW, buf + bb * B * RW, B * RW * 4);
                    bulk_commit();
                }
            }
            if (tid < (u32)MAXK) bulk_wait_read0();
            __syncthreads();
#pragma unroll
            for (int r = 0; r < RS; ++r)
                if (defer & (1u << r)) copy_rec<RW>(buf + (bk[r] * B + pos[r]) * RW, rec_ptr(r));
            __syncthreads();  // every read of this stage is done: it takes the tile K2REC_STAGES ahead
            if (ti + K2REC_STAGES < ntiles) stage_tile(ti + K2REC_STAGES, st);
        }
        // head records: classified now, spilled with the bucket's partial buffer
        if (tid < nhead) {
            const u32* my = s_head + tid * RW;
            u64 hk[1] = {TR::key_w(my, tp.part)};
            s_hb[tid] = classify_key(hk[0], tree, spl, tp.logk, tp.kprime, tp.eq);  // (a partial warp)
        }
        __syncthreads();
        // ---- publish counts; spill partial buffers (compacted) to the auxiliary area
        u32 nh_b = 0;  // head records of this bucket
        if (tid < (u32)MAXK)
            for (u32 i = 0; i < 3; ++i) nh_b += s_hb[i] == tid ? 1u : 0u;
        u32 f = tid < (u32)MAXK ? fill[tid] + nh_b : 0u;
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
            const u32 cb = nbl[tid] * (u32)B + cnt[tid] + nh_b;
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
            u32* sp = reinterpret_cast<u32*>(A.spill) + s_spbase * RW;
            for (u32 bb = w; bb < (u32)MAXK; bb += NW) {
                const u32 fb = fill[bb], ob = slotb[bb];
                for (u32 i = lane; i < fb * RW; i += 32) sp[ob * RW + i] = buf[bb * B * RW + i];
                u32 o2 = ob + fb;  // then the bucket's head records
                for (u32 h = 0; h < 3; ++h) {
                    if (s_hb[h] != bb) continue;
                    for (u32 i = lane; i < RW; i += 32) sp[o2 * RW + i] = s_head[h * RW + i];
                    ++o2;
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace ips4o
