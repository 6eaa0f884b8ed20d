// k_permute.cuh -- K3: delimiters, empty-block movement and the block permutation.
//
// k_prepare (one CTA per task): bucket sizes (summed by K2's stripes) -> element-exact
//   bucket starts e_i; delimiters d_i = e_i rounded up to the block grid;
//   full-block counts per bucket; initial (w_i, r_i).
// k_moves: Appendix A -- make every bucket read "full blocks, then
//   empty blocks" by moving the last full blocks of a bucket into its first empty
//   blocks.  On the GPU every (bucket, hole) pair is an independent warp task.
// k_permute (persistent, co-resident): the block permutation of PAPER.md:252-304.  Each
//   warp is one "thread" of the paper: it takes a block from its primary bucket by an
//   atomic fetch-and-add on r, classifies the block's first element, claims w_dest by an
//   atomic fetch-and-add, and either swaps (w <= r) or writes into an empty block
//   (w > r), waiting for the bucket's readers at the crossing.  (w, r)
//   live in one 64-bit word, so both updates see a consistent
//   pair.  Swap buffers are the warp's registers: a 512-byte block is 16 B per lane.
#pragma once
#include "common.cuh"

namespace ips4o {

#ifndef IPS4O_K3_RELAXED  // 1: the pointer atomics without release / acquire semantics (measurement)
#define IPS4O_K3_RELAXED 0
#endif
#ifndef IPS4O_K3_IDLE_NS  // back-off of a K3 warp whose chains all wait
#define IPS4O_K3_IDLE_NS 32
#endif
constexpr int K2P_MAXST = 1024;  // stripes of one task staged in shared memory by k_prepare

template <class TR>
__global__ void __launch_bounds__(MAXK) k_prepare(LevelArgs A0) {
    const LevelArgs A = with_dyn(A0);
    constexpr int B = TR::B;
    __shared__ u32 s_d[MAXK + 1];
    __shared__ u32 s_wsum[MAXK / 32];
    __shared__ u64 s_wsum64[MAXK / 32];
    const u32 t = blockIdx.x, b = threadIdx.x, lane = b & 31, w = b >> 5;
    if (t >= A.ntasks) return;  // (grid = the workspace's task capacity)
    const TaskParam tp = A.tp[t];
    const u32 S0 = tp.stripe_begin, NS = tp.nstripes;

    // bucket size = sum over this task's stripes; the stripes' block
    // ranges are staged in shared memory for the loops below
    __shared__ u32 s_sb[K2P_MAXST], s_fe[K2P_MAXST];
    const bool staged = NS <= (u32)K2P_MAXST;
    if (staged) {
        for (u32 j = b; j < NS; j += MAXK) {
            s_sb[j] = A.sd[S0 + j].sb;
            s_fe[j] = A.sd[S0 + j].sb + A.s_nfull[S0 + j];
        }
    }
    const u64 c = A.btot[(u64)t * MAXK + b];  // summed by K2 over the task's stripes (64-bit)
    __syncthreads();  // staged stripe ranges
    // exclusive scan over the 256 buckets (64-bit: a task may exceed 2^32 elements)
    u64 incl64 = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u64 y = __shfl_up_sync(0xffffffffu, incl64, o);
        if (lane >= (u32)o) incl64 += y;
    }
    if (lane == 31) s_wsum64[w] = incl64;
    __syncthreads();
    u64 woff64 = 0;
    for (u32 ww = 0; ww < w; ++ww) woff64 += s_wsum64[ww];
    const u64 e = tp.lo + woff64 + incl64 - c;
    A.bnd[(u64)t * (MAXK + 1) + b] = e;
    if (b == MAXK - 1) A.bnd[(u64)t * (MAXK + 1) + MAXK] = e + c;  // == hi
    // delimiter: e rounded up to the block grid of origin g (e < g only for e = lo)
    const u32 d = e > tp.g ? (u32)((e - tp.g + B - 1) / B) : 0u;
    s_d[b] = d;
    if (b == 0) s_d[MAXK] = tp.nblocks;
    __syncthreads();
    const u32 dn = s_d[b + 1];
    A.dblk[(u64)t * (MAXK + 1) + b] = d;
    if (b == 0) A.dblk[(u64)t * (MAXK + 1) + MAXK] = tp.nblocks;
    // full blocks inside [d, dn): every stripe holds full blocks [sb, sb+F) then empty ones
    auto fs_of = [&](u32 j) { return staged ? s_sb[j] : A.sd[S0 + j].sb; };
    auto fe_of = [&](u32 j) { return staged ? s_fe[j] : A.sd[S0 + j].sb + A.s_nfull[S0 + j]; };
    // stripes are in block order: only those from the one containing d onwards overlap
    // [d, dn) (a level-1 bucket spans a few of the ~444 stripes)
    u32 j0 = 0;
    {
        u32 lo2 = 0, hi2 = NS;  // last stripe with sb <= d
        while (hi2 - lo2 > 1) {
            const u32 mid = (lo2 + hi2) >> 1;
            if (fs_of(mid) <= d) lo2 = mid;
            else hi2 = mid;
        }
        j0 = lo2;
    }
    u32 nf = 0;
    for (u32 j = j0; j < NS; ++j) {
        const u32 fs = fs_of(j), fe = fe_of(j);
        if (fs >= dn) break;
        const u32 lo2 = fs > d ? fs : d, hi2 = fe < dn ? fe : dn;
        if (hi2 > lo2) nf += hi2 - lo2;
    }
    // Appendix A: holes (empty blocks) inside [d, d+nf) must be filled
    u32 fullpre = 0;
    for (u32 j = j0; j < NS; ++j) {
        const u32 fs = fs_of(j), fe = fe_of(j);
        if (fs >= d + nf) break;
        const u32 lo2 = fs > d ? fs : d, hi2 = fe < d + nf ? fe : d + nf;
        if (hi2 > lo2) fullpre += hi2 - lo2;
    }
    const u32 moves = nf - fullpre;
    A.nfb[(u64)t * MAXK + b] = nf;
    __syncthreads();
    u32 incl = moves;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (u32)o) incl += y;
    }
    if (lane == 31) s_wsum[w] = incl;
    __syncthreads();
    u32 woff = 0;
    for (u32 ww = 0; ww < w; ++ww) woff += s_wsum[ww];
    A.mov[(u64)t * (MAXK + 1) + b] = woff + incl - moves;
    if (b == MAXK - 1) {
        A.mov[(u64)t * (MAXK + 1) + MAXK] = woff + incl;
        if (woff + incl) atomicAdd(&A.ctr[CTR_AMOVES], woff + incl);
    }
    // w_i = d_i, r_i = d_i + nf_i - 1 (block indices; r biased).  A task whose
    // elements all fell into this one bucket (equal keys) has, after the Appendix-A moves,
    // only blocks of this bucket in [d, d+nf): every block is in place, w_i = d_i + nf_i.
    const bool all_here = c == tp.hi - tp.lo;
    const u32 w0 = all_here ? d + nf : d;
    *ctl_wr(A.wr, t, b) = ((u64)w0 << 32) | (u64)(u32)(d + nf - 1u + RBIAS);
    *ctl_readers(A.wr, t, b) = 0;
    A.cflag[(u64)t * MAXK + b] = 0;
    const u32 dn_bit = (b >= tp.K || nf == 0 || all_here) ? 1u : 0u;
    const u32 bal = __ballot_sync(0xffffffffu, dn_bit);
    if (lane == 0) A.done[(u64)t * (MAXK / 32) + w] = bal;
    if (b == 0) {
        A.ovf_owner[t] = -1;
    }
    // per-task stripe prefixes of full / empty block counts (for k_moves): block-wide scans
    // over the stripes, 256 at a time
    __shared__ u32 s_wf[MAXK / 32], s_we[MAXK / 32];
    u32 pf = 0, pe = 0;
    for (u32 base = 0; base < NS; base += MAXK) {
        const u32 j = base + b;
        u32 F = 0, Em = 0;
        if (j < NS) {
            const StripeDesc sd = A.sd[S0 + j];
            F = A.s_nfull[S0 + j];
            Em = (sd.se - sd.sb) - F;
        }
        u32 iF = F, iE = Em;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 yF = __shfl_up_sync(0xffffffffu, iF, o), yE = __shfl_up_sync(0xffffffffu, iE, o);
            if (lane >= (u32)o) {
                iF += yF;
                iE += yE;
            }
        }
        __syncthreads();
        if (lane == 31) {
            s_wf[w] = iF;
            s_we[w] = iE;
        }
        __syncthreads();
        u32 oF = 0, oE = 0, tF = 0, tE = 0;
        for (u32 ww = 0; ww < MAXK / 32; ++ww) {
            if (ww < w) {
                oF += s_wf[ww];
                oE += s_we[ww];
            }
            tF += s_wf[ww];
            tE += s_we[ww];
        }
        if (j < NS) {
            A.prefF[S0 + j] = pf + oF + iF - F;
            A.prefE[S0 + j] = pe + oE + iE - Em;
        }
        pf += tF;
        pe += tE;
    }
}

// last j in [0, n) with key(j) <= x (key non-decreasing, key(0) <= x)
template <class F>
__device__ __forceinline__ u32 last_le(u32 n, u64 x, F key) {
    u32 lo = 0, hi = n;  // invariant: key(lo) <= x
    while (hi - lo > 1) {
        u32 mid = (lo + hi) >> 1;
        if (key(mid) <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

template <class TR>
__global__ void __launch_bounds__(256) k_moves(LevelArgs A0) {
    const LevelArgs A = with_dyn(A0);
    constexpr int B = TR::B;
    // the task's per-stripe block counts and the per-bucket move ranges, staged in shared
    // memory: the searches below are then shared-memory lookups
    __shared__ u32 s_sb[K2P_MAXST], s_se[K2P_MAXST], s_F[K2P_MAXST], s_pE[K2P_MAXST], s_pF[K2P_MAXST];
    __shared__ u32 s_mov[MAXK + 1], s_d[MAXK + 1], s_nf[MAXK];
    // work items (task t, part bx of gx): grid-stride (the grid is fixed; gx from the plan)
    const u32 gx = A0.dyn->moves_gx;
    for (u32 item = blockIdx.x; item < A.ntasks * gx; item += gridDim.x) {
    const u32 t = item / gx, bx = item % gx;
    __syncthreads();  // the previous item's shared tables are no longer read
    const u32 lane = threadIdx.x & 31;
    const u32 wib = threadIdx.x >> 5;
    const TaskParam tp = A.tp[t];
    const u32 S0 = tp.stripe_begin, NS = tp.nstripes;
    const u32* mov = A.mov + (u64)t * (MAXK + 1);
    const u32 M = mov[MAXK];
    if (M == 0 || bx * (blockDim.x >> 5) * 32u >= M) continue;
    const bool staged = NS <= (u32)K2P_MAXST;
    for (u32 i = threadIdx.x; i <= (u32)MAXK; i += blockDim.x) {
        s_mov[i] = mov[i];
        s_d[i] = A.dblk[(u64)t * (MAXK + 1) + i];
        if (i < (u32)MAXK) s_nf[i] = A.nfb[(u64)t * MAXK + i];
    }
    if (staged) {
        for (u32 j = threadIdx.x; j < NS; j += blockDim.x) {
            const StripeDesc sd = A.sd[S0 + j];
            s_sb[j] = sd.sb;
            s_se[j] = sd.se;
            s_F[j] = A.s_nfull[S0 + j];
            s_pE[j] = A.prefE[S0 + j];
            s_pF[j] = A.prefF[S0 + j];
        }
    }
    __syncthreads();
    auto sb_of = [&](u32 j) { return staged ? s_sb[j] : A.sd[S0 + j].sb; };
    auto se_of = [&](u32 j) { return staged ? s_se[j] : A.sd[S0 + j].se; };
    auto F_of = [&](u32 j) { return staged ? s_F[j] : A.s_nfull[S0 + j]; };
    auto pE_of = [&](u32 j) { return staged ? s_pE[j] : A.prefE[S0 + j]; };
    auto pF_of = [&](u32 j) { return staged ? s_pF[j] : A.prefF[S0 + j]; };
    const u32 nwarps = gx * (blockDim.x >> 5);
    char* base = reinterpret_cast<char*>(A.data) + tp.g * GridStride<TR>::v;
    char* vbase = TR::KV ? reinterpret_cast<char*>(A.vals) + tp.g * 8 : nullptr;
    // a block in registers (16 B per lane; KV: lanes 0-15 the key block, 16-31 the value block)
    auto blk_load = [&](u32 x) -> BlockRegs {
        if constexpr (TR::KV) {
            BlockRegs r;
            const char* p = (lane < 16 ? base + (u64)x * (B * 8) + 16 * lane : vbase + (u64)x * (B * 8) + 16 * (lane - 16));
            asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]) : "l"(p) : "memory");
            return r;
        } else {
            return BlockIO<TR>::load(base + (u64)x * (B * TR::S), lane);
        }
    };
    auto blk_store = [&](u32 x, const BlockRegs& r) {
        if constexpr (TR::KV) {
            char* p = (lane < 16 ? base + (u64)x * (B * 8) + 16 * lane : vbase + (u64)x * (B * 8) + 16 * (lane - 16));
            asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(r.w[0]), "r"(r.w[1]), "r"(r.w[2]),
                         "r"(r.w[3])
                         : "memory");
        } else {
            BlockIO<TR>::store(base + (u64)x * (B * TR::S), lane, r);
        }
    };
    // every lane locates one move (five binary searches), then the warp copies the 32
    // blocks two at a time (the moves are independent: sources are full blocks, targets
    // empty ones)
    for (u32 m0 = (bx * (blockDim.x >> 5) + wib) * 32u; m0 < M; m0 += nwarps * 32u) {
        const u32 m = m0 + lane;
        u32 src = 0, dst = 0;
        if (m < M) {
            const u32 b = last_le(MAXK, m, [&](u32 i) { return (u64)s_mov[i]; });
            const u32 k = m - s_mov[b];
            const u32 d = s_d[b];
            const u32 nf = s_nf[b];
            // k-th empty block at or after d
            const u32 jd = last_le(NS, d, [&](u32 i) { return (u64)sb_of(i); });
            const u32 sbd = sb_of(jd), Fd = F_of(jd), sed = se_of(jd);
            const u32 se_d = d < sed ? d : sed;
            const u32 eb = pE_of(jd) + (se_d > sbd + Fd ? se_d - (sbd + Fd) : 0u) + k;
            const u32 je = last_le(NS, eb, [&](u32 i) { return (u64)pE_of(i); });
            dst = sb_of(je) + F_of(je) + (eb - pE_of(je));
            // k-th full block at or after d + nf
            const u32 x = d + nf;
            const u32 jx = last_le(NS, x, [&](u32 i) { return (u64)sb_of(i); });
            const u32 sbx = sb_of(jx), Fx = F_of(jx);
            const u32 fb = pF_of(jx) + (x - sbx < Fx ? x - sbx : Fx) + k;
            const u32 jf = last_le(NS, fb, [&](u32 i) { return (u64)pF_of(i); });
            src = sb_of(jf) + (fb - pF_of(jf));
        }
        const u32 cnt = M - m0 < 32u ? M - m0 : 32u;
        for (u32 i = 0; i < cnt; i += 2) {
            const bool two = i + 1 < cnt;
            const u32 s0 = __shfl_sync(0xffffffffu, src, i), d0 = __shfl_sync(0xffffffffu, dst, i);
            const u32 s1 = __shfl_sync(0xffffffffu, src, two ? i + 1 : i), d1 = __shfl_sync(0xffffffffu, dst, two ? i + 1 : i);
            const BlockRegs v0 = blk_load(s0);
            BlockRegs v1;
            if (two) v1 = blk_load(s1);
            blk_store(d0, v0);
            if (two) blk_store(d1, v1);
        }
    }
    }
}

// ------------------------------------------------------------------ permutation

// Warp-cooperative classification of one key held by every lane (the first element of a
// block): the number of padded splitters <= key.  That count is exactly the leaf the
// branchless descent of PAPER.md:138-142 reaches (j <- 2j + [a_j <= e] over a complete BST
// of the sorted splitters computes this rank; ties go right), found here with
// two ballots over groups of 8 splitters instead of 8 dependent lookups by every lane.
// slot[p] = s_{p+1} (p < nsl = k'-1, padded); glast = slot[8*lane+7] when valid.  With
// equality buckets one more comparison against the lower splitter.
__device__ __forceinline__ u32 warp_classify(u64 key, const u64* slot, u32 nsl, u32 eq, u32 lane,
                                             u64 glast, bool gok) {
    const u32 c1 = __popc(__ballot_sync(0xffffffffu, gok && key >= glast));
    const u32 p = 8 * c1 + (lane & 7u);
    const bool ok = lane < 8u && p < nsl && key >= slot[p < nsl ? p : 0u];
    const u32 i = 8 * c1 + __popc(__ballot_sync(0xffffffffu, ok));
    if (eq) {
        const bool isq = i >= 1u && slot[i >= 1u ? i - 1u : 0u] >= key;
        return 2 * i - (isq ? 1u : 0u);
    }
    return i;
}

// next bucket (cyclic over nwords*32 buckets, starting at gb inclusive) whose bit in
// `bits` is clear; ~0u if none.  Warp-cooperative: 32 words per probe.
__device__ __forceinline__ u32 next_clear_bit(const u32* bits, u32 nwords, u32 gb, u32 lane) {
    const u32 w0 = gb >> 5;
    for (u32 base = 0; base <= nwords; base += 32) {
        const u32 off = base + lane;
        u32 word = 0xFFFFFFFFu;
        u32 widx = 0;
        if (off <= nwords) {
            widx = (w0 + off) % nwords;
            word = *(volatile const u32*)(bits + widx);
            if (off == 0) word |= (1u << (gb & 31)) - 1u;          // first pass: bits >= gb
            if (off == nwords) word |= ~((1u << (gb & 31)) - 1u);  // wrap-around: bits < gb
        }
        const u32 bal = __ballot_sync(0xffffffffu, word != 0xFFFFFFFFu);
        if (bal) {
            const u32 src = __ffs(bal) - 1;
            const u32 wsel = __shfl_sync(0xffffffffu, widx, src);
            const u32 wv = __shfl_sync(0xffffffffu, word, src);
            return wsel * 32 + (__ffs(~wv) - 1);
        }
    }
    return 0xFFFFFFFFu;
}

// first not-done bucket at or after b (cyclic over K buckets); ~0u if every bucket is done.
// Serial scan by one lane over the task's done words (rare: once per exhausted bucket).
__device__ __forceinline__ u32 next_open_bucket(const u32* done, u32 b, u32 K) {
    const u32 nw = (K + 31) / 32;
    for (u32 i = 0; i <= nw; ++i) {
        const u32 wi = ((b >> 5) + i) % nw;
        u32 word = *(volatile const u32*)(done + wi);
        if (i == 0) word |= (1u << (b & 31)) - 1u;             // bits >= b in the first word
        if (i == nw) word |= ~((1u << (b & 31)) - 1u);         // wrap-around: bits < b
        if (wi == nw - 1 && (K & 31)) word |= ~((1u << (K & 31)) - 1u);
        if (word != 0xFFFFFFFFu) return wi * 32 + (__ffs(~word) - 1);
    }
    return 0xFFFFFFFFu;
}

// Block permutation.  Each CTA works on one task at a time (its
// splitters in shared memory) and moves on to the next unfinished task when none of the
// task's buckets has an unprocessed block left.  Each warp runs K3_SLOTS independent
// chains (the paper's threads) in lock step, so that their atomic round trips and block
// loads overlap: lane c performs the pointer atomics of chain c, all 32 lanes move the
// blocks (16 B per lane of a 512-B block), and each chain's swap buffer lives in registers.
// Per round:
//   (a) chains without a block take one from their primary bucket: readers++ (release),
//       then r <- r-1 on the packed (w, r) word; a failed take (r < w) marks the bucket
//       done and the chain moves to the next open bucket;
//   (b) every held block is classified by its first element; w_dest <- w_dest+1;
//       if the old w <= old r the target is an unprocessed block: read it, and unless it
//       already belongs to dest (skip) write ours there and carry it on;
//       otherwise the target is empty: wait for the bucket's readers at the crossing
//       (PAPER.md:298-302), write (or use the overflow block past the end,
//       PAPER.md:220-221) and the chain is free again.
#ifdef IPS4O_K3_TIMELINE
__device__ unsigned int g_k3_hist[4096];
__device__ unsigned long long g_k3_t0;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void k_timer_start() { g_k3_t0 = gtimer(); }
#define K3_TL_EVENT(kind)                                                                      \
    do {                                                                                       \
        const unsigned long long dt_ = (gtimer() - g_k3_t0) / 1000ull;                         \
        atomicAdd(&g_k3_hist[(kind) * 2048 + (dt_ < 2047 ? dt_ : 2047)], 1u);                   \
    } while (0)
#else
#define K3_TL_EVENT(kind) do {} while (0)
#endif

template <class TR>
__global__ void __launch_bounds__(K3_THREADS, K3_MINB) k_permute(LevelArgs A0) {
    const LevelArgs A = with_dyn(A0);
    if (A.ntasks == 0) return;
    u32 nmoves = 0;  // block writes of this warp (lane 0)
    constexpr int B = TR::B;
    constexpr u32 BB = B * TR::S;  // block bytes
    constexpr int C = K3_SLOTS;
    constexpr u32 CM = (1u << C) - 1u;
    __shared__ u64 s_spl[MAXK];
    __shared__ u32 s_next;
    const u32 tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
    const u32 nw = blockDim.x >> 5;
    const u32 T = A.ntasks;
    char* const data = reinterpret_cast<char*>(A.data);
    u32 t = (u32)((u64)blockIdx.x * T / gridDim.x);
    const u32 tnwords = (T + 31) / 32;

    for (;;) {
        // next unfinished task (cyclic from t); exit when every task is finished
        if (tid < 32) {
            const u32 nt = next_clear_bit(A.tdone, tnwords, t, lane);
            if (lane == 0) s_next = nt;
        }
        __syncthreads();
        const u32 nt = s_next;
        if (nt == 0xFFFFFFFFu || nt >= T) break;
        t = nt;
        if (tid < (u32)MAXK) s_spl[tid] = A.spl[(u64)t * MAXK + tid];
        __syncthreads();
        const TaskParam tp = A.tp[t];
        u32* done = A.done + (u64)t * (MAXK / 32);
        char* tbase = data + tp.g * TR::S;
        const u64* slot = s_spl + 1;
        const u32 nsl = tp.kprime - 1u;
        const bool gok = 8 * lane + 7 < nsl;
        const u64 glast = gok ? slot[8 * lane + 7] : 0ull;

        // per-chain scalars live in lane c (c < C); block registers in every lane
        u32 my_pb = (u32)((((u64)blockIdx.x * nw + wi) * C + lane) * 97u % tp.K);
        bool my_alive = lane < (u32)C;
        u32 my_dest = 0;
        u32 held = 0;  // warp-uniform: chains holding a block (classified, my_dest valid)
        BlockRegs cur[C];

        for (;;) {
            // ---- 1. one pointer atomic per chain: free chains take (r <- r-1 on their
            //         primary bucket, after announcing themselves as readers), chains with a
            //         block claim their destination slot (w <- w+1)
            const bool my_held = lane < (u32)C && ((held >> lane) & 1u);
            bool my_take = my_alive && !my_held;
            if (my_take) {
                const u32 b = next_open_bucket(done, my_pb, tp.K);
                if (b == 0xFFFFFFFFu) {
                    my_alive = false;
                    my_take = false;
                } else {
                    my_pb = b;
                }
            }
            u64 my_old = 0;
            if (my_take || my_held) {
                u64 op = 1ull << 32;
                u64* wp = ctl_wr(A.wr, t, my_dest);
                if (my_take) {
                    // the reader announcement is performed before the take: the take's operand
                    // depends on the value the announcement returns (the count never reaches
                    // 2^31, so the added term is 0)
#if IPS4O_K3_ACQUIRE
                    atom_add_acquire_u32(ctl_readers(A.wr, t, my_pb), 1u);
                    op = ~0ull;
#else
                    const u32 r0 = atomicAdd(ctl_readers(A.wr, t, my_pb), 1u);
                    op = ~0ull + (u64)(r0 >> 31);
#endif
                    wp = ctl_wr(A.wr, t, my_pb);
                }
                my_old = atomicAdd((unsigned long long*)wp, op);
            }
            const int my_ow = (int)(u32)(my_old >> 32);
            const int my_orr = (int)((u32)my_old - RBIAS);
            if (my_held) K3_TL_EVENT(0);   // a placement attempt (1 us bins)
            if (my_take) K3_TL_EVENT(1);   // a take attempt
            // 2. decode: source block of this round's load (taken block / swap target)
            int my_src = -1;
            bool my_write = false;
            if (my_take) {
                if (my_orr < my_ow) {  // nothing left to take in this bucket
                    atomicSub(ctl_readers(A.wr, t, my_pb), 1u);
                    atomicOr(&done[my_pb >> 5], 1u << (my_pb & 31));
                } else {
                    my_src = my_orr;
                }
            } else if (my_held) {
                if (my_ow <= my_orr) my_src = my_ow;  // unprocessed block at w: swap
                else my_write = true;                 // empty block at w: write
            }
            const u32 ld = __ballot_sync(0xffffffffu, my_src >= 0) & CM;
            const u32 wrt = __ballot_sync(0xffffffffu, my_write) & CM;
            const u32 tk = __ballot_sync(0xffffffffu, my_take && my_src >= 0) & CM;
            const u32 alive = __ballot_sync(0xffffffffu, my_alive) & CM;
            if (!ld && !wrt && !held) {
                if (!alive) break;
                continue;
            }
            // 3. all block loads of the round in flight together
            BlockRegs nxt[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int src = __shfl_sync(0xffffffffu, my_src, c);
                if ((ld >> c) & 1u) nxt[c] = BlockIO<TR>::load(tbase + (u64)src * BB, lane);
            }
            // 4. taken blocks: release the readers once every lane's read has completed (before
            //    any wait below: a chain of this warp may be the reader another one waits for)
            if (tk) {
                u32 x = 0;
#pragma unroll
                for (int c = 0; c < C; ++c)
                    if ((tk >> c) & 1u) x |= nxt[c].w[0] | nxt[c].w[1] | nxt[c].w[2] | nxt[c].w[3];
                if (__any_sync(0xffffffffu, x == 0x9E3779B9u)) __nanosleep(0);  // forces the loads
                if (my_take && my_src >= 0) atomicSub(ctl_readers(A.wr, t, my_pb), 1u);
            }
            // 5. writes into empty blocks: wait for the bucket's readers at the crossing
            //    (PAPER.md:298-302), then write (past the end: the overflow block)
            if (wrt) {
                if (my_write) {
                    while (*(volatile u32*)ctl_readers(A.wr, t, my_dest) != 0u) __nanosleep(64);
                }
                __syncwarp();
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const int ow = __shfl_sync(0xffffffffu, my_ow, c);
                    const u32 dc = __shfl_sync(0xffffffffu, my_dest, c);
                    if ((wrt >> c) & 1u) {
                        if (tp.g + (u64)(ow + 1) * B > tp.hi) {
                            char* ob = reinterpret_cast<char*>(A.ovf) + (u64)t * BB;
                            BlockIO<TR>::store(ob, lane, cur[c]);
                            if (lane == 0) A.ovf_owner[t] = (int)dc;
                        } else {
                            BlockIO<TR>::store(tbase + (u64)ow * BB, lane, cur[c]);
                        }
                    }
                }
                held &= ~wrt;
                if (lane == 0) nmoves += __popc(wrt);
            }
            // 6. consume the loads: taken blocks become held; swap targets are classified -- already in
            //    place: skip, else ours is written there and we carry on
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (!((ld >> c) & 1u)) continue;
                const u32 d = warp_classify(BlockIO<TR>::first_key(nxt[c], tp.part), slot, nsl, tp.eq, lane,
                                            glast, gok);
                if ((tk >> c) & 1u) {
                    cur[c] = nxt[c];
                    if (lane == (u32)c) my_dest = d;
                } else {
                    const u32 dc = __shfl_sync(0xffffffffu, my_dest, c);
                    if (d != dc) {
                        const int ow = __shfl_sync(0xffffffffu, my_ow, c);
                        BlockIO<TR>::store(tbase + (u64)ow * BB, lane, cur[c]);
                        if (lane == 0) ++nmoves;
                        cur[c] = nxt[c];
                        if (lane == (u32)c) my_dest = d;
                    }
                }
            }
            held |= tk;
        }
        __syncthreads();
        if (tid == 0) atomicOr(&A.tdone[t >> 5], 1u << (t & 31));
    }
    if (lane == 0 && nmoves) atomicAdd(&A.ctr[CTR_BMOVES], nmoves);
}


// ------------------------------------------------------------------ permutation, TMA version
//
// The same protocol with the swap buffers in shared memory (the paper's per-thread swap
// buffers) and the blocks moved by TMA bulk copies: every lane of a warp
// runs its own chain (K3T_CHAINS per warp), so a chain waits only for its own atomic and
// its own block load, and the loads of up to K3T_CHAINS chains per warp are in flight
// together without occupying registers.  Chain states:
//   FREE      take a block from the primary bucket (readers++, then r <- r-1) and load it;
//   TAKING    the taken block is arriving (mbarrier): release the reader count, classify;
//   HELD      claim the destination slot (w <- w+1): an unprocessed block there is loaded
//             (SWAPPING), an empty one is written once the bucket's readers are gone (WAITW);
//   SWAPPING  the displaced block is arriving: if it already belongs to the destination it
//             stays (skip), else ours is written over it and the displaced one is carried on.
// Used for the 8/16-byte types (block grid 16-byte aligned); records use k_permute.
#ifndef IPS4O_K3_PF  // L2 prefetch of the blocks later claims / takes of a bucket will load (0: off; n: n x the default distance)
#define IPS4O_K3_PF 1
#endif
#ifndef IPS4O_K3_DEFER  // the atomics' return values consumed after the round's arrived blocks have been served
#define IPS4O_K3_DEFER 0
#endif
#ifndef IPS4O_K3_SKIPSCAN  // a chain takes from its last bucket again without scanning the done bits first
#define IPS4O_K3_SKIPSCAN 0
#endif
#ifndef IPS4O_K3_PF_DEN
#define IPS4O_K3_PF_DEN 1
#endif
#ifndef IPS4O_K3_PF_MIN
#define IPS4O_K3_PF_MIN 1
#endif
#ifndef IPS4O_K3T_WARPS
#define IPS4O_K3T_WARPS 4
#endif
#ifndef IPS4O_K3T_CHAINS
#define IPS4O_K3T_CHAINS 16
#endif
constexpr int K3T_WARPS = IPS4O_K3T_WARPS;      // warps per CTA
constexpr int K3T_CHAINS = IPS4O_K3T_CHAINS;    // chains (lanes) per warp
constexpr int K3T_THREADS = 32 * K3T_WARPS;
enum { CH_FREE = 0, CH_TAKING = 1, CH_HELD = 2, CH_SWAPPING = 3, CH_WAITW = 4, CH_DEAD = 5 };

template <class TR>
struct K3TSmem {
    static constexpr u32 BB = TR::B * TR::S;
    static constexpr size_t buf_bytes = (size_t)K3T_WARPS * K3T_CHAINS * 2 * BB;
    static constexpr size_t total = buf_bytes;
};

__device__ __forceinline__ bool mbar_test(u64* mbar, u32 parity) {
    u32 ok;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"((u32)__cvta_generic_to_shared(mbar)), "r"(parity)
                 : "memory");
    return ok != 0;
}

// A block's TMA moves between global memory and a chain's shared-memory swap buffer (KV: the
// key block and the value block, kept as [keys | values] in shared memory and in the overflow
// block).
template <class TR>
struct K3Blk {
    static constexpr u32 BB = TR::B * TR::S;
    __device__ __forceinline__ static void load(char* sbuf, char* kb, char* vb, u32 x, u64* mbar) {
        if constexpr (TR::KV) {
            constexpr u32 H = TR::B * 8;
            mbar_expect_tx(mbar, 2 * H);
            bulk_g2s_tx(sbuf, kb + (u64)x * H, H, mbar);
            bulk_g2s_tx(sbuf + H, vb + (u64)x * H, H, mbar);
        } else {
            bulk_g2s(sbuf, kb + (u64)x * BB, BB, mbar);
        }
    }
    __device__ __forceinline__ static void prefetch(const char* kb, const char* vb, u32 x) {
        if constexpr (TR::KV) {
            constexpr u32 H = TR::B * 8;
            bulk_prefetch_l2(kb + (u64)x * H, H);
            bulk_prefetch_l2(vb + (u64)x * H, H);
        } else {
            bulk_prefetch_l2(kb + (u64)x * BB, BB);
        }
    }
    __device__ __forceinline__ static void store(char* kb, char* vb, u32 x, const char* sbuf) {
        if constexpr (TR::KV) {
            constexpr u32 H = TR::B * 8;
            bulk_s2g(kb + (u64)x * H, sbuf, H);
            bulk_s2g(vb + (u64)x * H, sbuf + H, H);
        } else {
            bulk_s2g(kb + (u64)x * BB, sbuf, BB);
        }
    }
};

template <class TR>
__global__ void __launch_bounds__(K3T_THREADS) k_permute_tma(LevelArgs A0) {
    const LevelArgs A = with_dyn(A0);
    if (A.ntasks == 0) return;
    u32 nmoves = 0;  // block writes of this chain
    typedef K3TSmem<TR> SM;
    constexpr u32 BB = SM::BB;
    extern __shared__ __align__(128) unsigned char smk3[];
    __shared__ u64 s_tree[MAXK], s_spl[MAXK];
    __shared__ __align__(8) u64 s_mbar[K3T_WARPS * K3T_CHAINS];
    __shared__ u32 s_next;
    const u32 tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
    const u32 T = A.ntasks;
    char* const data = reinterpret_cast<char*>(A.data);
    const bool chain = lane < (u32)K3T_CHAINS;
    const u32 cid = wi * K3T_CHAINS + lane;  // chain index in the CTA
    char* const mybuf = reinterpret_cast<char*>(smk3) + (size_t)(chain ? cid : 0) * 2 * BB;
    u64* const mymbar = &s_mbar[chain ? cid : 0];
    if (chain) mbar_init(mymbar, 1);
    mbar_fence_init();
    __syncthreads();
    u32 phase = 0;  // parity of this chain's next mbarrier completion
    // first task: CTAs spread in proportion to the tasks' block counts (the position of
    // this CTA's share in the concatenation of the tasks' blocks), so that tasks of
    // different sizes finish together
    u32 t = 0;
    if (tid < 32) {
        u64 total = 0;
        for (u32 q = lane; q < T; q += 32) total += A.tp[q].nblocks;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
        const u64 target = (u64)blockIdx.x * total / gridDim.x;
        u64 acc = 0;
        u32 found = T - 1;
        for (u32 q0 = 0; q0 < T; q0 += 32) {
            const u32 q = q0 + lane;
            const u64 nb = q < T ? A.tp[q].nblocks : 0;
            u64 incl = nb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u64 y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (u32)o) incl += y;
            }
            const u32 hit = __ballot_sync(0xffffffffu, q < T && acc + incl > target);
            if (hit) {
                found = q0 + __ffs(hit) - 1;
                break;
            }
            acc += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_next = found;
    }
    __syncthreads();
    t = s_next;
    __syncthreads();
    bool first = true;
    const u32 tnwords = (T + 31) / 32;

    for (;;) {
        if (tid < 32) {
            // (after the first task, helpers start their search at spread positions, so
            // that they do not all pile onto the task next to the one they finished)
            const u32 from = first ? t : (u32)((t + 1u + (u64)blockIdx.x * 61u) % T);
            const u32 nt = next_clear_bit(A.tdone, tnwords, from, lane);
            if (lane == 0) s_next = nt;
        }
        __syncthreads();
        first = false;
        const u32 nt = s_next;
        if (nt == 0xFFFFFFFFu || nt >= T) break;
        t = nt;
        if (tid < (u32)MAXK) {
            s_tree[tid] = A.tree[(u64)t * MAXK + tid];
            s_spl[tid] = A.spl[(u64)t * MAXK + tid];
        }
        for (u32 i = tid + K3T_THREADS; i < (u32)MAXK; i += K3T_THREADS) {
            s_tree[i] = A.tree[(u64)t * MAXK + i];
            s_spl[i] = A.spl[(u64)t * MAXK + i];
        }
        __syncthreads();
        const TaskParam tp = A.tp[t];
        u32* done = A.done + (u64)t * (MAXK / 32);
        char* tbase = data + tp.g * GridStride<TR>::v;
        char* vbase = TR::KV ? reinterpret_cast<char*>(A.vals) + tp.g * 8 : nullptr;
        auto classify_buf = [&](const char* b) {
            typename TR::V v;
            memcpy(&v, b, sizeof(v));
            return classify_key(TR::key(v, tp.part), s_tree, s_spl, tp.logk, tp.kprime, tp.eq);
        };

#if IPS4O_K3_PF
        // L2 prefetch distance: the block a later claim / take of the same bucket will load, about
        // half the chains working on the bucket ahead (a bucket's unprocessed blocks [w, r] are
        // consumed in order from both ends)
        const int pfd = (int)max((u32)IPS4O_K3_PF_MIN, (u32)(gridDim.x * (K3T_WARPS * K3T_CHAINS)) / max(1u, T * tp.K * 2u) *
                                                            (u32)IPS4O_K3_PF / (u32)IPS4O_K3_PF_DEN);
#endif
        u32 st = chain ? CH_FREE : CH_DEAD;
        u32 pb = (u32)(((u64)blockIdx.x * (K3T_WARPS * K3T_CHAINS) + cid) * 97u % tp.K);
        u32 xb = 0;       // buffer holding our block (the other one receives loads)
        u32 dest = 0, slot = 0;
        bool pb_ok = false;  // the last take from pb succeeded
        while (__any_sync(0xffffffffu, st != CH_DEAD)) {
#if IPS4O_K3_DEFER
            // The same steps with the atomics' results consumed late: takes and claims are issued,
            // then the chains whose blocks have arrived are served, and only then the warp waits
            // for the atomics' return values (a chain is in one state per round, so every chain's
            // own sequence of operations is unchanged).
            bool progressed = false;
            u32 pend = 0;  // 1: take issued, 2: claim issued (result in old)
            u64 old = 0;
            if (st == CH_FREE) {
                const u32 b = next_open_bucket(done, pb, tp.K);
                if (b == 0xFFFFFFFFu) {
                    st = CH_DEAD;
                } else {
                    pb = b;
                    K3_TL_EVENT(1);
                    atomicAdd(ctl_readers(A.wr, t, pb), 1u);  // (S18: announced before the take's release)
                    old = atom_add_release_u64(ctl_wr(A.wr, t, pb), ~0ull);
                    pend = 1;
                    progressed = true;
                }
            } else if (st == CH_HELD) {
                K3_TL_EVENT(0);
                old = atom_add_acquire_u64(ctl_wr(A.wr, t, dest), 1ull << 32);
                pend = 2;
                progressed = true;
            }
            // ---- arrived blocks
            if ((st == CH_TAKING || st == CH_SWAPPING) && mbar_test(mymbar, phase)) {
                phase ^= 1u;
                if (st == CH_TAKING) {
                    red_add_release_u32(ctl_readers(A.wr, t, pb), ~0u);  // the block has been read (release)
                    dest = classify_buf(mybuf + xb * BB);
                    st = CH_HELD;
                } else {
                    const u32 od = classify_buf(mybuf + (xb ^ 1) * BB);
                    if (od != dest) {
                        K3Blk<TR>::store(tbase, vbase, slot, mybuf + xb * BB);
                        bulk_commit();
                        ++nmoves;
                        xb ^= 1u;
                        dest = od;
                    }  // else: already in place, skip it and keep ours
                    st = CH_HELD;
                }
                progressed = true;
            }
            // ---- the atomics' results
            if (pend == 1) {
                const int ow = (int)(u32)(old >> 32), orr = (int)((u32)old - RBIAS);
                if (orr < ow) {
                    atomicSub(ctl_readers(A.wr, t, pb), 1u);
                    atomicOr(&done[pb >> 5], 1u << (pb & 31));
                } else {
                    bulk_wait_read0();  // our earlier stores have read this buffer
                    fence_proxy_async_smem();
                    K3Blk<TR>::load(mybuf + xb * BB, tbase, vbase, (u32)orr, mymbar);
#if IPS4O_K3_PF
                    if (orr - pfd >= ow) K3Blk<TR>::prefetch(tbase, vbase, (u32)(orr - pfd));
#endif
                    st = CH_TAKING;
                }
            } else if (pend == 2) {
                const int ow = (int)(u32)(old >> 32), orr = (int)((u32)old - RBIAS);
                slot = (u32)ow;
                if (ow <= orr) {
                    bulk_wait_read0();
                    fence_proxy_async_smem();
                    K3Blk<TR>::load(mybuf + (xb ^ 1) * BB, tbase, vbase, (u32)ow, mymbar);
#if IPS4O_K3_PF
                    if (ow + pfd <= orr) K3Blk<TR>::prefetch(tbase, vbase, (u32)(ow + pfd));
#endif
                    st = CH_SWAPPING;
                } else {
                    st = CH_WAITW;  // empty block: written once the bucket has no readers
                }
            }
            if (st == CH_WAITW && ld_acquire_u32(ctl_readers(A.wr, t, dest)) == 0u) {
                if (tp.g + (u64)(slot + 1) * TR::B > tp.hi) {
                    bulk_s2g(reinterpret_cast<char*>(A.ovf) + (u64)t * BB, mybuf + xb * BB, BB);
                    A.ovf_owner[t] = (int)dest;
                } else {
                    K3Blk<TR>::store(tbase, vbase, slot, mybuf + xb * BB);
                }
                bulk_commit();
                ++nmoves;
                st = CH_FREE;
                progressed = true;
            }
#else
            bool progressed = false;
            // ---- atomics: takes (FREE) and claims (HELD), one round trip for all chains
            if (st == CH_FREE) {
#if IPS4O_K3_SKIPSCAN
                // (the bucket the last take succeeded in is tried again without reading the done bits)
                const u32 b = pb_ok ? pb : next_open_bucket(done, pb, tp.K);
#else
                const u32 b = next_open_bucket(done, pb, tp.K);
#endif
                if (b == 0xFFFFFFFFu) {
                    st = CH_DEAD;
                } else {
                    pb = b;
                    K3_TL_EVENT(1);
                    // the reader announcement is ordered before the take by the
                    // take's release semantics; a writer's claim (acquire) that observes this
                    // take then also observes the announcement
                    atomicAdd(ctl_readers(A.wr, t, pb), 1u);
#if IPS4O_K3_RELAXED
                    const u64 old = atomicAdd((unsigned long long*)ctl_wr(A.wr, t, pb), ~0ull);
#else
                    const u64 old = atom_add_release_u64(ctl_wr(A.wr, t, pb), ~0ull);
#endif
                    const int ow = (int)(u32)(old >> 32), orr = (int)((u32)old - RBIAS);
                    pb_ok = orr >= ow;
                    if (orr < ow) {
                        atomicSub(ctl_readers(A.wr, t, pb), 1u);
                        atomicOr(&done[pb >> 5], 1u << (pb & 31));
                    } else {
                        bulk_wait_read0();  // our earlier stores have read this buffer
                        fence_proxy_async_smem();
                        K3Blk<TR>::load(mybuf + xb * BB, tbase, vbase, (u32)orr, mymbar);
#if IPS4O_K3_PF
                        if (orr - pfd >= ow) K3Blk<TR>::prefetch(tbase, vbase, (u32)(orr - pfd));
#endif
                        st = CH_TAKING;
                    }
                    progressed = true;
                }
            } else if (st == CH_HELD) {
                K3_TL_EVENT(0);
#if IPS4O_K3_RELAXED
                const u64 old = atomicAdd((unsigned long long*)ctl_wr(A.wr, t, dest), 1ull << 32);
#else
                const u64 old = atom_add_acquire_u64(ctl_wr(A.wr, t, dest), 1ull << 32);
#endif
                const int ow = (int)(u32)(old >> 32), orr = (int)((u32)old - RBIAS);
                slot = (u32)ow;
                if (ow <= orr) {
                    bulk_wait_read0();
                    fence_proxy_async_smem();
                    K3Blk<TR>::load(mybuf + (xb ^ 1) * BB, tbase, vbase, (u32)ow, mymbar);
#if IPS4O_K3_PF
                    if (ow + pfd <= orr) K3Blk<TR>::prefetch(tbase, vbase, (u32)(ow + pfd));
#endif
                    st = CH_SWAPPING;
                } else {
                    st = CH_WAITW;  // empty block: written once the bucket has no readers
                }
                progressed = true;
            }
            if (st == CH_WAITW && ld_acquire_u32(ctl_readers(A.wr, t, dest)) == 0u) {
                // no reader left at the crossing: write into the empty block
                // (past the task end: the overflow block).  (Never spin here:
                // the reader may be a chain of this warp.)
                if (tp.g + (u64)(slot + 1) * TR::B > tp.hi) {
                    bulk_s2g(reinterpret_cast<char*>(A.ovf) + (u64)t * BB, mybuf + xb * BB, BB);
                    A.ovf_owner[t] = (int)dest;
                } else {
                    K3Blk<TR>::store(tbase, vbase, slot, mybuf + xb * BB);
                }
                bulk_commit();
                ++nmoves;
                st = CH_FREE;
                progressed = true;
            }
            // ---- arrived blocks
            if ((st == CH_TAKING || st == CH_SWAPPING) && mbar_test(mymbar, phase)) {
                phase ^= 1u;
                if (st == CH_TAKING) {
                    red_add_release_u32(ctl_readers(A.wr, t, pb), ~0u);  // the block has been read (release)
                    dest = classify_buf(mybuf + xb * BB);
                    st = CH_HELD;
                } else {
                    const u32 od = classify_buf(mybuf + (xb ^ 1) * BB);
                    if (od != dest) {
                        K3Blk<TR>::store(tbase, vbase, slot, mybuf + xb * BB);
                        bulk_commit();
                        ++nmoves;
                        xb ^= 1u;
                        dest = od;
                    }  // else: already in place, skip it and keep ours
                    st = CH_HELD;
                }
                progressed = true;
            }
#endif
            if (!__any_sync(0xffffffffu, progressed)) __nanosleep(IPS4O_K3_IDLE_NS);
        }
        __syncthreads();
        if (tid == 0) atomicOr(&A.tdone[t >> 5], 1u << (t & 31));
    }
    bulk_wait0();  // every block store is complete before the kernel ends
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nmoves += __shfl_xor_sync(0xffffffffu, nmoves, o);
    if (lane == 0 && nmoves) atomicAdd(&A.ctr[CTR_BMOVES], nmoves);
}

}  // namespace ips4o
