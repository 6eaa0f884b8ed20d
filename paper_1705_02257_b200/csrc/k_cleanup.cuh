// k_cleanup.cuh -- K4: cleanup of partial blocks (§4.3) and task emission.
//
// One warp per (task, bucket), taken in order through an atomic ticket so that a bucket's
// predecessor is always already running.  For bucket i:
//   empty slots  = its head [e_i, min(d_i, e_{i+1})) and [min(w_i, e_{i+1}), e_{i+1});
//   sources      = the overhang of its last written block into the next bucket's head
//                  [e_{i+1}, w_i), every stripe's partially filled buffer for
//                  i, and the overflow block if it belongs to i.
// The overhang is read into shared memory first and published with a flag; a bucket
// writes its head only after the bucket owning the block under that head has
// published (the paper's "reads the head of the first bucket of the next thread into one
// of its swap buffers").  Then the bucket is emitted to the next
// level, to the base case, or dropped (equality buckets; size <= 1).
#pragma once
#include "common.cuh"

namespace ips4o {

constexpr int K4_MAXSTRIPES = 512;  // >= stripes per level batch (MAXS)
constexpr int K4_WARPS = K4_THREADS / 32;

// element i of a task's overflow block (KV types: stored as [B keys | B values], the layout
// of K3's swap buffers)
template <class TR>
__device__ __forceinline__ typename TR::V ovf_get(const void* ovf_block, u32 i) {
    if constexpr (TR::KV) {
        const u64* p = reinterpret_cast<const u64*>(ovf_block);
        return make_ulonglong2(p[i], p[TR::B + i]);
    } else {
        return reinterpret_cast<const typename TR::V*>(ovf_block)[i];
    }
}

// Emission decision for bucket b of task tp (PAPER.md:342 for equality buckets): returns
// 0..3 = base-case class, 4 = next-level task, 5 = nothing, 6 = the single-CTA tier (medium
// tasks: "assign remaining problems ... which sort them sequentially");
// *td = the task.
template <class TR>
__device__ __forceinline__ u32 emit_kind(const LevelArgs& A, const TaskParam& tp, u32 b, u64 e0, u64 e1,
                                         TaskDesc* td) {
    const u64 sz = e1 - e0;
    const bool eqb = tp.eq && (b & 1u);
    u32 part = tp.part;
    bool emit = sz > 1;
    if (eqb) {
        if (part + 1 < (u32)TR::PARTS) ++part;
        else emit = false;
    }
    if (emit && !eqb && sz == tp.hi - tp.lo) {
        // no progress: a splitter choice that leaves the whole task in one
        // interval bucket would recurse forever -- report instead of looping
        atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_PROGRESS);
        emit = false;
    }
    if (!emit) return 5u;
    if (sz <= A.base_cap) {
        *td = TaskDesc{e0, e1, 0u, 0u};
        return base_class<TR>(sz);
    }
    *td = TaskDesc{e0, e1, part, 0u};
    if constexpr (!TR::WIDE) {
        if (sz <= A.medium_max) return 6u;
    }
    return 4u;
}

// One warp per group of K4_GROUP consecutive buckets of a task, groups taken in order
// through an atomic ticket (a bucket's predecessor is in an earlier group or earlier in the
// same group, so it is already running or done).  The group's emitted tasks take their
// queue slots with one atomic per queue, and the base-case element count is summed per warp:
// tens of thousands of buckets would otherwise serialise on a few counter words.
#ifndef IPS4O_K4_GROUP
#define IPS4O_K4_GROUP 4
#endif
constexpr u32 K4_GROUP = IPS4O_K4_GROUP;
template <class TR>
__global__ void __launch_bounds__(K4_THREADS) k_cleanup(LevelArgs A0) {
    if (A0.dyn->k4_cta) return;  // this batch is cleaned up by k_cleanup_cta
    const LevelArgs A = with_dyn(A0);
    typedef typename TR::V V;
    constexpr int B = TR::B;
    static_assert(MAXK % K4_GROUP == 0, "groups never span tasks");
    __shared__ V s_ovh_all[K4_WARPS][K4_GROUP][B];
    __shared__ u32 s_pref_all[K4_WARPS][K4_MAXSTRIPES + 1];
    __shared__ TaskDesc s_td_all[K4_WARPS][K4_GROUP];
    __shared__ u32 s_kind_all[K4_WARPS][K4_GROUP];
    const u32 lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    u32* s_pref = s_pref_all[wi];
    TaskDesc* s_td = s_td_all[wi];
    u32* s_kind = s_kind_all[wi];
    const u32 ngroups = A.ntasks * (MAXK / K4_GROUP);
    const Mem<TR> mem(A.data, A.vals);
    const V* spill = reinterpret_cast<const V*>(A.spill);
    u64 base_elems = 0;  // lane 0: elements of this warp's emitted base-case tasks
    for (;;) {
        u32 ticket = 0;
        if (lane == 0) ticket = atomicAdd(&A.ctr[CTR_TICKET], 1u);
        ticket = __shfl_sync(0xffffffffu, ticket, 0);
        if (ticket >= ngroups) break;
        const u32 t = ticket / (MAXK / K4_GROUP), b0 = (ticket % (MAXK / K4_GROUP)) * K4_GROUP;
        const TaskParam tp = A.tp[t];
        u32* flag = A.cflag + (u64)t * MAXK;
        const u64* bnd = A.bnd + (u64)t * (MAXK + 1);
        const u32* dbl = A.dblk + (u64)t * (MAXK + 1);
        const int ovf_owner = A.ovf_owner[t];
        const u32 S0 = tp.stripe_begin, NS = tp.nstripes;
        // the group's bucket bounds, delimiters and final write pointers, one lane each
        u64 g_e = 0;
        u32 g_d = 0, g_w = 0;
        if (lane <= K4_GROUP) g_e = bnd[b0 + lane];
        if (lane < K4_GROUP) {
            g_d = dbl[b0 + lane];
            g_w = b0 + lane < tp.K ? (u32)(*ctl_wr(A.wr, t, b0 + lane) >> 32) : 0u;
        }
        // 1. the overhangs of the group's last written blocks into the next buckets' heads
        //    are saved and published first, so that no bucket of a later
        //    group waits for this group's earlier buckets to finish
#pragma unroll 1
        for (u32 gi = 0; gi < K4_GROUP; ++gi) {
            const u32 b = b0 + gi;
            if (b < tp.K) {
                const u64 e1 = __shfl_sync(0xffffffffu, g_e, gi + 1);
                const u32 d = __shfl_sync(0xffffffffu, g_d, gi);
                const u32 wfin = __shfl_sync(0xffffffffu, g_w, gi);
                const u64 db_el = tp.g + (u64)d * B;
                const u64 in_end = ovf_owner == (int)b ? tp.g + (u64)(tp.nblocks - 1) * B : tp.g + (u64)wfin * B;
                const u32 ovl = (in_end > db_el && in_end > e1) ? (u32)(in_end - e1) : 0u;
                for (u32 k = lane; k < ovl; k += 32) s_ovh_all[wi][gi][k] = mem.ld(e1 + k);
            }
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            for (u32 gi = 0; gi < K4_GROUP; ++gi) st_release_u32(flag + b0 + gi, 1u);
        }
        // the group's partial-buffer lengths and spill positions, one round trip: lane
        // 8g + j holds stripe j of bucket b0 + g (tasks of at most 8 stripes -- the lower
        // levels); g_excl = its offset among the bucket's spilled elements
        const bool few = NS <= 8u;
        u32 g_excl = 0, g_incl = 0;
        u64 g_src = 0;
        if (few) {
            const u32 gg = lane >> 3, j = lane & 7u;
            u32 len = 0;
            if (j < NS && b0 + gg < tp.K) {
                len = A.s_fill[(u64)(S0 + j) * MAXK + b0 + gg];
                g_src = A.s_spbase[S0 + j] + A.s_spoff[(u64)(S0 + j) * MAXK + b0 + gg];
            }
            g_incl = len;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                const u32 y = __shfl_up_sync(0xffffffffu, g_incl, o, 8);
                if (j >= (u32)o) g_incl += y;
            }
            g_excl = g_incl - len;
        }
        // 2. each bucket: gather its partial blocks into its empty slots, then emit it
#pragma unroll 1
        for (u32 gi = 0; gi < K4_GROUP; ++gi) {
            const u32 b = b0 + gi;
            if (lane == 0) s_kind[gi] = 5u;
            if (b >= tp.K) continue;
            const V* s_ovh = s_ovh_all[wi][gi];
            const u64 e0 = __shfl_sync(0xffffffffu, g_e, gi), e1 = __shfl_sync(0xffffffffu, g_e, gi + 1);
            const u32 d = __shfl_sync(0xffffffffu, g_d, gi);
            const u32 wfin = __shfl_sync(0xffffffffu, g_w, gi);
            const bool own_ovf = ovf_owner == (int)b;
            const u64 db_el = tp.g + (u64)d * B;
            const u64 in_end = own_ovf ? tp.g + (u64)(tp.nblocks - 1) * B : tp.g + (u64)wfin * B;
            const u32 ovl = (in_end > db_el && in_end > e1) ? (u32)(in_end - e1) : 0u;
            // spilled partial buffers of every stripe of this task for bucket b
            u32 sp_total = few ? __shfl_sync(0xffffffffu, g_incl, 8 * gi + 7) : 0u;
            for (u32 base = 0; !few && base < NS; base += 32) {
                const u32 j = base + lane;
                const u32 len = j < NS ? A.s_fill[(u64)(S0 + j) * MAXK + b] : 0u;
                u32 incl = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= (u32)o) incl += y;
                }
                if (j < NS) s_pref[j] = sp_total + incl - len;
                sp_total += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0 && !few) s_pref[NS] = sp_total;
            __syncwarp();
            const u32 nsrc = ovl + sp_total + (own_ovf ? (u32)B : 0u);
            const u64 hend = db_el < e1 ? db_el : e1;
            const u64 ts = db_el < e1 ? (in_end < e1 ? in_end : e1) : e1;
            const u64 hl = hend - e0;
            const u64 nslots = hl + (e1 - ts);
            if ((u64)nsrc != nslots) {
                if (lane == 0) atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_CONSERVE);
                continue;
            }
            // wait until the bucket owning block d-1 (which holds our head) saved its overhang
            if (lane == 0 && hl > 0 && d >= 1) {
                const u32 x = d - 1;
                u32 lo = 0, hi = b;  // largest o < b with dbl[o] <= x
                while (hi - lo > 1) {
                    const u32 mid = (lo + hi) >> 1;
                    if (dbl[mid] <= x) lo = mid;
                    else hi = mid;
                }
                if (lo < b) {
                    while (ld_acquire_u32(flag + lo) == 0u) __nanosleep(100);
                }
            }
            __syncwarp();
            const char* ovf = reinterpret_cast<const char*>(A.ovf) + (u64)t * B * TR::S;
            if (few) {
                // stripe of each spilled source from the lanes of this bucket's segment
                for (u32 k0 = 0; k0 < nsrc; k0 += 32) {
                    const u32 k = k0 + lane, kk = k - ovl;
                    u32 lo = 0;
                    for (u32 j = 1; j < NS; ++j)
                        if (kk >= __shfl_sync(0xffffffffu, g_excl, 8 * gi + j)) lo = j;
                    const u64 sbase = __shfl_sync(0xffffffffu, g_src, 8 * gi + lo);
                    const u32 pre = __shfl_sync(0xffffffffu, g_excl, 8 * gi + lo);
                    if (k < nsrc) {
                        V val;
                        if (k < ovl) val = s_ovh[k];
                        else if (kk < sp_total) val = spill[sbase + (kk - pre)];
                        else val = ovf_get<TR>(ovf, kk - sp_total);
                        mem.st((u64)k < hl ? e0 + k : ts + (k - hl), val);
                    }
                }
            }
            u32 jcur = 0;  // stripe of the previous source (sources are visited in order)
            for (u32 k = few ? nsrc : lane; k < nsrc; k += 32) {
                V val;
                if (k < ovl) {
                    val = s_ovh[k];
                } else if (k - ovl < sp_total) {
                    const u32 kk = k - ovl;
                    u32 lo = jcur, hi = NS;  // last j with s_pref[j] <= kk
                    while (hi - lo > 1) {
                        const u32 mid = (lo + hi) >> 1;
                        if (s_pref[mid] <= kk) lo = mid;
                        else hi = mid;
                    }
                    jcur = lo;
                    const u64 at = A.s_spbase[S0 + lo] + A.s_spoff[(u64)(S0 + lo) * MAXK + b] + (kk - s_pref[lo]);
                    val = spill[at];
                } else {
                    val = ovf_get<TR>(ovf, k - ovl - sp_total);
                }
                const u64 dst = (u64)k < hl ? e0 + k : ts + (k - hl);
                mem.st(dst, val);
            }
            // emit the bucket.  Equality buckets are never recursed into; for
            // records an equality bucket of key part 0 (equal first 8 key bytes) still has to
            // be ordered by part 1, so it becomes a task on the next part.
            if (lane == 0 && A.emit) {
                TaskDesc td;
                const u32 kd = emit_kind<TR>(A, tp, b, e0, e1, &td);
                s_kind[gi] = kd;
                s_td[gi] = td;
                if (kd < 4u) base_elems += e1 - e0;
            }
        }
        __syncwarp();
        // the group's tasks: lane q (queue q: 0-3 base classes, 4 next level, 6 medium)
        // reserves the queue's slots with one atomic
        if (A.emit && lane < 7u && lane != 5u) {
            u32 cntq = 0;
#pragma unroll
            for (u32 gi = 0; gi < K4_GROUP; ++gi) cntq += s_kind[gi] == lane ? 1u : 0u;
            if (cntq) {
                u32* ctr = lane < 4u ? &A.ctr[CTR_BASE0 + lane] : lane == 4u ? &A.ctr[CTR_NEXT] : &A.ctr[CTR_MED];
                TaskDesc* q = lane < 4u ? A.q_base + A.qb_off[lane] : lane == 4u ? A.q_next : A.q_med;
                const u32 cap = lane < 4u ? A.qb_cap[lane] : lane == 4u ? A.qn_cap : A.qm_cap;
                u32 i = atomicAdd(ctr, cntq);
                for (u32 gi = 0; gi < K4_GROUP; ++gi) {
                    if (s_kind[gi] != lane) continue;
                    if (i < cap) q[i] = s_td[gi];
                    else atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_QUEUE);
                    ++i;
                }
            }
        }
        __syncwarp();
    }
    if (lane == 0 && base_elems) atomicAdd((unsigned long long*)A.base_elems, (unsigned long long)base_elems);
}

// Few buckets with many stripes each (the top level): one CTA per bucket, buckets taken in
// ticket order by a persistent grid (a bucket's predecessor always has an earlier ticket, so
// it is held by a running CTA: the wait below cannot deadlock).
template <class TR>
__global__ void __launch_bounds__(K4_THREADS) k_cleanup_cta(LevelArgs A0) {
    if (!A0.dyn->k4_cta) return;  // this batch is cleaned up by the warp kernel
    const LevelArgs A = with_dyn(A0);
    typedef typename TR::V V;
    constexpr int B = TR::B;
    __shared__ V s_ovh[B];
    __shared__ u32 s_pref[K4_MAXSTRIPES + 1];
    __shared__ u64 s_src[K4_MAXSTRIPES];  // spill position of stripe j's partial buffer for b
    __shared__ u32 s_wsum[K4_THREADS / 32];
    __shared__ u32 s_ticket;
    const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const u32 nticket = A.ntasks * MAXK;
    for (;;) {
    __syncthreads();  // the previous bucket's shared state is no longer read
    if (tid == 0) s_ticket = atomicAdd(&A.ctr[CTR_TICKET], 1u);
    __syncthreads();
    const u32 ticket = s_ticket;
    if (ticket >= nticket) break;
    const u32 t = ticket / MAXK, b = ticket % MAXK;
    const TaskParam tp = A.tp[t];
    u32* flag = A.cflag + (u64)t * MAXK;
    if (b >= tp.K) {
        if (tid == 0) st_release_u32(flag + b, 1u);
        continue;
    }
    const Mem<TR> mem(A.data, A.vals);
    const u64* bnd = A.bnd + (u64)t * (MAXK + 1);
    const u32* dbl = A.dblk + (u64)t * (MAXK + 1);
    const u64 e0 = bnd[b], e1 = bnd[b + 1];
    const u32 d = dbl[b];
    const u32 wfin = (u32)(*ctl_wr(A.wr, t, b) >> 32);
    const bool own_ovf = A.ovf_owner[t] == (int)b;
    const u64 db_el = tp.g + (u64)d * B;
    const u64 in_end = own_ovf ? tp.g + (u64)(tp.nblocks - 1) * B : tp.g + (u64)wfin * B;
    const u32 ovl = (in_end > db_el && in_end > e1) ? (u32)(in_end - e1) : 0u;
    for (u32 k = tid; k < ovl; k += blockDim.x) s_ovh[k] = mem.ld(e1 + k);
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        st_release_u32(flag + b, 1u);
    }
    // spilled partial buffers of every stripe of this task for bucket b
    const u32 S0 = tp.stripe_begin, NS = tp.nstripes;
    u32 sp_total = 0;
    for (u32 base = 0; base < NS; base += K4_THREADS) {
        const u32 j = base + tid;
        const u32 len = j < NS ? A.s_fill[(u64)(S0 + j) * MAXK + b] : 0u;
        u32 incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (u32)o) incl += y;
        }
        if (lane == 31) s_wsum[w] = incl;
        __syncthreads();
        u32 woff = 0, tot = 0;
        for (u32 ww = 0; ww < K4_THREADS / 32; ++ww) {
            if (ww < w) woff += s_wsum[ww];
            tot += s_wsum[ww];
        }
        if (j < NS) {
            s_pref[j] = sp_total + woff + incl - len;
            s_src[j] = A.s_spbase[S0 + j] + A.s_spoff[(u64)(S0 + j) * MAXK + b];
        }
        sp_total += tot;
        __syncthreads();
    }
    if (tid == 0) s_pref[NS] = sp_total;
    const u32 nsrc = ovl + sp_total + (own_ovf ? (u32)B : 0u);
    const u64 hend = db_el < e1 ? db_el : e1;
    const u64 ts = db_el < e1 ? (in_end < e1 ? in_end : e1) : e1;
    const u64 hl = hend - e0;
    const u64 nslots = hl + (e1 - ts);
    if ((u64)nsrc != nslots) {
        if (tid == 0) atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_CONSERVE);
        continue;
    }
    // wait until the bucket owning block d-1 (which holds our head) saved its overhang
    if (tid == 0 && hl > 0 && d >= 1) {
        const u32 x = d - 1;
        u32 lo = 0, hi = b;  // largest o < b with dbl[o] <= x
        while (hi - lo > 1) {
            u32 mid = (lo + hi) >> 1;
            if (dbl[mid] <= x) lo = mid;
            else hi = mid;
        }
        if (lo < b) {
            while (ld_acquire_u32(flag + lo) == 0u) __nanosleep(100);
        }
    }
    __syncthreads();
    const V* spill = reinterpret_cast<const V*>(A.spill);
    const char* ovf = reinterpret_cast<const char*>(A.ovf) + (u64)t * B * TR::S;
    // gather: four sources per thread in flight (each is a stripe lookup in shared memory
    // and one dependent load)
    auto src_of = [&](u32 k) -> V {
        if (k < ovl) return s_ovh[k];
        if (k - ovl < sp_total) {
            const u32 kk = k - ovl;
            u32 lo = 0, hi = NS;  // last j with s_pref[j] <= kk
            while (hi - lo > 1) {
                const u32 mid = (lo + hi) >> 1;
                if (s_pref[mid] <= kk) lo = mid;
                else hi = mid;
            }
            return spill[s_src[lo] + (kk - s_pref[lo])];
        }
        return ovf_get<TR>(ovf, k - ovl - sp_total);
    };
    auto dst_of = [&](u32 k) { return (u64)k < hl ? e0 + k : ts + (k - hl); };
    for (u32 k0 = tid; k0 < nsrc; k0 += 4 * K4_THREADS) {
        V val[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const u32 k = k0 + q * K4_THREADS;
            if (k < nsrc) val[q] = src_of(k);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const u32 k = k0 + q * K4_THREADS;
            if (k < nsrc) mem.st(dst_of(k), val[q]);
        }
    }
    // emit the bucket (PAPER.md:342 for equality buckets)
    if (tid == 0 && A.emit) {
        TaskDesc td;
        const u32 kd = emit_kind<TR>(A, tp, b, e0, e1, &td);
        if (kd < 4u) {
            atomicAdd((unsigned long long*)A.base_elems, (unsigned long long)(e1 - e0));
            const u32 i = atomicAdd(&A.ctr[CTR_BASE0 + kd], 1u);
            if (i < A.qb_cap[kd]) A.q_base[A.qb_off[kd] + i] = td;
            else atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_QUEUE);
        } else if (kd == 4u) {
            const u32 i = atomicAdd(&A.ctr[CTR_NEXT], 1u);
            if (i < A.qn_cap) A.q_next[i] = td;
            else atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_QUEUE);
        } else if (kd == 6u) {
            const u32 i = atomicAdd(&A.ctr[CTR_MED], 1u);
            if (i < A.qm_cap) A.q_med[i] = td;
            else atomicOr(&A.ctr[CTR_ERROR], (u32)ERR_QUEUE);
        }
    }
    }
}

}  // namespace ips4o
