// k_permute.cuh -- K3: delimiters, empty-block movement and the block permutation.
//
// k_prepare (one CTA per task): prefix sum of the stripes' bucket counts -> element-exact
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

template <class TR>
__global__ void __launch_bounds__(MAXK) k_prepare(LevelArgs A) {
    constexpr int B = TR::B;
    __shared__ u32 s_d[MAXK + 1];
    __shared__ u32 s_wsum[MAXK / 32];
    const u32 t = blockIdx.x, b = threadIdx.x, lane = b & 31, w = b >> 5;
    const TaskParam tp = A.tp[t];
    const u32 S0 = tp.stripe_begin, NS = tp.nstripes;

    // bucket size = sum over this task's stripes
    u32 c = 0;
    for (u32 j = 0; j < NS; ++j) c += A.s_count[(u64)(S0 + j) * MAXK + b];
    // exclusive scan over the 256 buckets
    u32 incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (u32)o) incl += y;
    }
    if (lane == 31) s_wsum[w] = incl;
    __syncthreads();
    u32 woff = 0;
    for (u32 ww = 0; ww < w; ++ww) woff += s_wsum[ww];
    const u64 e = tp.lo + woff + incl - c;
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
    u32 nf = 0;
    for (u32 j = 0; j < NS; ++j) {
        const StripeDesc sd = A.sd[S0 + j];
        const u32 fs = sd.sb, fe = sd.sb + A.s_nfull[S0 + j];
        const u32 lo2 = fs > d ? fs : d, hi2 = fe < dn ? fe : dn;
        if (hi2 > lo2) nf += hi2 - lo2;
    }
    // Appendix A: holes (empty blocks) inside [d, d+nf) must be filled
    u32 fullpre = 0;
    for (u32 j = 0; j < NS; ++j) {
        const StripeDesc sd = A.sd[S0 + j];
        const u32 fs = sd.sb, fe = sd.sb + A.s_nfull[S0 + j];
        const u32 lo2 = fs > d ? fs : d, hi2 = fe < d + nf ? fe : d + nf;
        if (hi2 > lo2) fullpre += hi2 - lo2;
    }
    const u32 moves = nf - fullpre;
    A.nfb[(u64)t * MAXK + b] = nf;
    __syncthreads();
    incl = moves;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (u32)o) incl += y;
    }
    if (lane == 31) s_wsum[w] = incl;
    __syncthreads();
    woff = 0;
    for (u32 ww = 0; ww < w; ++ww) woff += s_wsum[ww];
    A.mov[(u64)t * (MAXK + 1) + b] = woff + incl - moves;
    if (b == MAXK - 1) A.mov[(u64)t * (MAXK + 1) + MAXK] = woff + incl;
    // w_i = d_i, r_i = d_i + nf_i - 1 (block indices; r biased)
    A.wr[(u64)t * MAXK + b] = ((u64)d << 32) | (u64)(u32)(d + nf - 1u + RBIAS);
    A.readers[(u64)t * MAXK + b] = 0;
    A.cflag[(u64)t * MAXK + b] = 0;
    const u32 dn_bit = (b >= tp.K || nf == 0) ? 1u : 0u;
    const u32 bal = __ballot_sync(0xffffffffu, dn_bit);
    if (lane == 0) A.done[(u64)t * (MAXK / 32) + w] = bal;
    if (b == 0) {
        A.ovf_owner[t] = -1;
        // per-task stripe prefixes of full / empty block counts (for k_moves)
        u32 pf = 0, pe = 0;
        for (u32 j = 0; j < NS; ++j) {
            const StripeDesc sd = A.sd[S0 + j];
            const u32 F = A.s_nfull[S0 + j];
            A.prefF[S0 + j] = pf;
            A.prefE[S0 + j] = pe;
            pf += F;
            pe += (sd.se - sd.sb) - F;
        }
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
__global__ void __launch_bounds__(256) k_moves(LevelArgs A) {
    constexpr int B = TR::B;
    const u32 t = blockIdx.y;
    const u32 lane = threadIdx.x & 31;
    const u32 wib = threadIdx.x >> 5;
    const TaskParam tp = A.tp[t];
    const u32 S0 = tp.stripe_begin, NS = tp.nstripes;
    const u32* mov = A.mov + (u64)t * (MAXK + 1);
    const u32 M = mov[MAXK];
    const u32 nwarps = gridDim.x * (blockDim.x >> 5);
    char* base = reinterpret_cast<char*>(A.data) + tp.g * TR::S;
    for (u32 m = blockIdx.x * (blockDim.x >> 5) + wib; m < M; m += nwarps) {
        u64 src = 0, dst = 0;
        if (lane == 0) {
            const u32 b = last_le(MAXK, m, [&](u32 i) { return (u64)mov[i]; });
            const u32 k = m - mov[b];
            const u32 d = A.dblk[(u64)t * (MAXK + 1) + b];
            const u32 nf = A.nfb[(u64)t * MAXK + b];
            // k-th empty block at or after d
            const u32 jd = last_le(NS, d, [&](u32 i) { return (u64)A.sd[S0 + i].sb; });
            const StripeDesc sdd = A.sd[S0 + jd];
            const u32 Fd = A.s_nfull[S0 + jd];
            const u32 se_d = d < sdd.se ? d : sdd.se;
            const u32 eb = A.prefE[S0 + jd] + (se_d > sdd.sb + Fd ? se_d - (sdd.sb + Fd) : 0u) + k;
            const u32 je = last_le(NS, eb, [&](u32 i) { return (u64)A.prefE[S0 + i]; });
            const StripeDesc sde = A.sd[S0 + je];
            dst = sde.sb + A.s_nfull[S0 + je] + (eb - A.prefE[S0 + je]);
            // k-th full block at or after d + nf
            const u32 x = d + nf;
            const u32 jx = last_le(NS, x, [&](u32 i) { return (u64)A.sd[S0 + i].sb; });
            const StripeDesc sdx = A.sd[S0 + jx];
            const u32 Fx = A.s_nfull[S0 + jx];
            const u32 fb = A.prefF[S0 + jx] + (x - sdx.sb < Fx ? x - sdx.sb : Fx) + k;
            const u32 jf = last_le(NS, fb, [&](u32 i) { return (u64)A.prefF[S0 + i]; });
            src = A.sd[S0 + jf].sb + (fb - A.prefF[S0 + jf]);
        }
        src = __shfl_sync(0xffffffffu, src, 0);
        dst = __shfl_sync(0xffffffffu, dst, 0);
        const BlockRegs v = BlockIO<TR>::load(base + src * (B * TR::S), lane);
        BlockIO<TR>::store(base + dst * (B * TR::S), lane, v);
    }
}

// ------------------------------------------------------------------ permutation

// destination bucket of a block: classify its first element (warp-collective key fetch,
// the classification itself by every lane on the same value)
template <class TR>
__device__ __forceinline__ u32 block_dest(const BlockRegs& r, const u64* tree, const u64* spl,
                                          u32 logk, u32 kprime, u32 eq, u32 part) {
    return classify_key(BlockIO<TR>::first_key(r, part), tree, spl, logk, kprime, eq);
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

// Block permutation.  Each CTA works on one task at a time (its classifier in shared
// memory), starting from a task chosen by its index so that CTAs spread over the tasks;
// when the task has no unprocessed block left it moves to the next unfinished task.
template <class TR>
__global__ void __launch_bounds__(K3_THREADS, 8) k_permute(LevelArgs A) {
    constexpr int B = TR::B;
    constexpr u32 BB = B * TR::S;  // block bytes
    __shared__ u64 s_tree[MAXK], s_spl[MAXK];
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
            if (lane == 0) s_tree[0] = nt;  // slot 0 of the tree is unused: borrow it
        }
        __syncthreads();
        const u32 nt = (u32)s_tree[0];
        __syncthreads();
        if (nt == 0xFFFFFFFFu || nt >= T) return;
        t = nt;
        if (tid < (u32)MAXK) {
            s_tree[tid] = A.tree[(u64)t * MAXK + tid];
            s_spl[tid] = A.spl[(u64)t * MAXK + tid];
        }
        __syncthreads();
        const TaskParam tp = A.tp[t];
        const u32* done = A.done + (u64)t * (MAXK / 32);
        char* tbase = data + tp.g * TR::S;
        // primary buckets spread over the task's buckets
        u32 b = (u32)(((u64)blockIdx.x * nw + wi) * 97u % tp.K);

        for (;;) {
            // ---- take an unprocessed block from the primary bucket (r <- r-1)
            b = next_clear_bit(done, MAXK / 32, b, lane);
            if (b == 0xFFFFFFFFu) break;
            const u32 gb = t * MAXK + b;
            int blk = 0, ok = 0;
            if (lane == 0) {
                atomicAdd(&A.readers[gb], 1u);
                __threadfence();
                const u64 old = atomicAdd((unsigned long long*)&A.wr[gb], ~0ull);  // r -= 1
                const int ow = (int)(u32)(old >> 32);
                const int orr = (int)((u32)old - RBIAS);
                if (orr < ow) {
                    atomicSub(&A.readers[gb], 1u);
                    atomicOr(&A.done[(u64)t * (MAXK / 32) + (b >> 5)], 1u << (b & 31));
                } else {
                    ok = 1;
                    blk = orr;
                }
            }
            ok = __shfl_sync(0xffffffffu, ok, 0);
            if (!ok) continue;
            blk = __shfl_sync(0xffffffffu, blk, 0);
            BlockRegs cur = BlockIO<TR>::load(tbase + (u64)blk * BB, lane);
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicSub(&A.readers[gb], 1u);
            // ---- chain: place the block, swapping with unprocessed blocks on the way
            for (;;) {
                const u32 dest = block_dest<TR>(cur, s_tree, s_spl, tp.logk, tp.kprime, tp.eq, tp.part);
                const u32 gbd = t * MAXK + dest;
                u64 old = 0;
                if (lane == 0) old = atomicAdd((unsigned long long*)&A.wr[gbd], 1ull << 32);  // w += 1
                old = __shfl_sync(0xffffffffu, old, 0);
                const int ow = (int)(u32)(old >> 32);
                const int orr = (int)((u32)old - RBIAS);
                if (ow <= orr) {
                    // case 1: w_dest points to an unprocessed block -> swap
                    const BlockRegs oth = BlockIO<TR>::load(tbase + (u64)ow * BB, lane);
                    const u32 od = block_dest<TR>(oth, s_tree, s_spl, tp.logk, tp.kprime, tp.eq, tp.part);
                    if (od == dest) continue;  // already in place: skip it
                    BlockIO<TR>::store(tbase + (u64)ow * BB, lane, cur);
                    cur = oth;
                } else {
                    // case 2: w_dest points to an empty block -> wait for readers, write, refill
                    if (lane == 0) {
                        while (*(volatile u32*)&A.readers[gbd] != 0u) __nanosleep(64);
                        __threadfence();
                    }
                    __syncwarp();
                    if (tp.g + (u64)(ow + 1) * B > tp.hi) {
                        // the block would reach past the task end: overflow block
                        char* ob = reinterpret_cast<char*>(A.ovf) + (u64)t * BB;
                        BlockIO<TR>::store(ob, lane, cur);
                        if (lane == 0) A.ovf_owner[t] = (int)dest;
                    } else {
                        BlockIO<TR>::store(tbase + (u64)ow * BB, lane, cur);
                    }
                    break;
                }
            }
        }
        __syncthreads();
        if (tid == 0) atomicOr(&A.tdone[t >> 5], 1u << (t & 31));
    }
}

}  // namespace ips4o
