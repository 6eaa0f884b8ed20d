// k_sched.cuh -- the device-side recursion scheduler (§4 preamble: "as long
// as problems with at least beta*n/t elements exist, we partition those problems one after
// another with t threads in parallel; then we assign remaining problems ... which sort them
// sequentially").
//
// The level loop runs on the device, inside one CUDA graph with a while-conditional node
// (ips4o.cu builds it): every iteration is one batch --
//   k_plan   takes the next batch of tasks from the current level's queue (switching to the
//            next level's queue when the current one is exhausted), plans their stripes
//            (the multi-CTA tier) and writes the per-batch fields of LevelDyn;
//   K1..K4   distribute the batch (k_sample, k_classify, k_prepare, k_moves, k_permute_tma,
//            k_cleanup); K4 appends each bucket to the next level's queue (large), to one of
//            the base-case size-class queues (small), or drops it (equality buckets, size <= 1);
//   K5       the base-case kernels sort the batch's leaves (the size-class queues);
//   k_epi    folds the batch's counters into the call's statistics and sets the loop's
//            condition: continue while a level queue holds tasks.
// Nothing in the loop touches host memory, so a sort is fully asynchronous on the caller's
// stream and can itself be captured into a caller's CUDA graph.
#pragma once
#include "common.cuh"

namespace ips4o {

#ifndef IPS4O_LAST_STRIPE_CUT  // a task's last stripe is (1 - this) of the others
#define IPS4O_LAST_STRIPE_CUT 0.75
#endif
#ifndef IPS4O_STRIPES_PER_SM  // stripes per SM of a level (K2 balance vs per-stripe overhead)
#define IPS4O_STRIPES_PER_SM 3
#endif
constexpr u32 MAXT = 512;          // tasks per batch (upper bound of the workspace's tcap)
constexpr u32 MAXS = 512;          // stripes per batch (upper bound of scap)
constexpr u64 MIN_STRIPE = 65536;  // elements
constexpr int PLAN_THREADS = 512;
static_assert(PLAN_THREADS >= (int)MAXT && PLAN_THREADS >= (int)MAXS, "one plan thread per task / stripe");
constexpr u64 MAX_BATCHES = 1ull << 20;  // safety cap of the level loop (ERR_ITER)

// k_init: the call's parameters arrive as kernel arguments (captured by value at launch:
// nothing is staged through host memory).  Resets the scheduler and the statistics and puts
// the whole array into the level queue (n > base capacity) or straight into its base-case
// size class.
__global__ void k_init(LevelArgs A0, void* data, void* vals, u64 n, u64 seed, u32 small_class) {
    if (threadIdx.x != 0) return;
    LevelDyn* D = A0.dyn;
    Sched* Q = A0.sched;
    D->data = data;
    D->vals = vals;
    D->n = n;
    D->q_next = A0.q_lvl1;
    D->seed = seed;
    D->ntasks = 0;
    D->nstripes = 0;
    D->emit = 1;
    D->k4_cta = 0;
    D->moves_gx = 1;
    D->from_splitters = 0;
    D->more = 1;
    for (int i = 0; i < CTR_N; ++i) A0.ctr[i] = 0;
    *A0.spill_ctr = 0;
    *A0.base_elems = 0;
    for (int i = 0; i < DS_N; ++i) A0.dstats[i] = 0;
    Q->qa = A0.q_lvl0;
    Q->qb = A0.q_lvl1;
    Q->ca = 0;
    Q->seed = seed;
    Q->ntot = n;
    if (small_class == NUM_BASE_CLASSES + 1) {
        // a medium problem: one CTA sorts it (the single-CTA tier, k_cta.cuh)
        Q->na = 0;
        Q->level = 0;
        A0.q_med[0] = TaskDesc{0, n, 0u, 0u};
        A0.ctr[CTR_MED] = 1;
    } else if (small_class >= NUM_BASE_CLASSES) {
        A0.q_lvl0[0] = TaskDesc{0, n, 0u, 0u};
        Q->na = 1;
        Q->level = 1;
        A0.dstats[DS_LEVELS] = 1;
    } else {
        Q->na = 0;
        Q->level = 0;
        A0.q_base[A0.qb_off[small_class]] = TaskDesc{0, n, 0u, 0u};
        A0.ctr[CTR_BASE0 + small_class] = 1;
        *A0.base_elems = n;
    }
}

// Debug single step (ips4o_debug_partition_once): one task [0, n) whose classifier K1 builds
// from the nspl splitters in dsplit; nothing is emitted.
__global__ void k_debug_setup(LevelArgs A0, void* data, u64 n, u32 nspl, u32 eq) {
    if (threadIdx.x != 0) return;
    LevelDyn* D = A0.dyn;
    Sched* Q = A0.sched;
    D->data = data;
    D->vals = nullptr;
    D->n = n;
    D->q_next = A0.q_lvl1;
    D->seed = 1;
    D->ntasks = 0;
    D->nstripes = 0;
    D->emit = 0;
    D->from_splitters = 1;
    D->nspl = nspl;
    D->spl_eq = eq;
    for (int i = 0; i < CTR_N; ++i) A0.ctr[i] = 0;
    *A0.spill_ctr = 0;
    *A0.base_elems = 0;
    for (int i = 0; i < DS_N; ++i) A0.dstats[i] = 0;
    Q->qa = A0.q_lvl0;
    Q->qb = A0.q_lvl1;
    Q->na = 1;
    Q->ca = 0;
    Q->level = 1;
    Q->seed = 1;
    Q->ntot = n;
    A0.q_lvl0[0] = TaskDesc{0, n, 0u, 0u};
    A0.dstats[DS_LEVELS] = 1;
}

// Block-wide inclusive scan of one u32 per thread (PLAN_THREADS threads).
__device__ __forceinline__ u32 plan_scan(u32 x, u32* s_w) {
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (u32)o) incl += y;
    }
    if (lane == 31) s_w[w] = incl;
    __syncthreads();
    u32 off = 0;
    for (u32 i = 0; i < w; ++i) off += s_w[i];
    __syncthreads();
    return off + incl;
}
__device__ __forceinline__ u64 plan_sum64(u64 x, u64* s_w) {
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) s_w[w] = x;
    __syncthreads();
    u64 t = 0;
    for (u32 i = 0; i < PLAN_THREADS / 32; ++i) t += s_w[i];
    __syncthreads();
    return t;
}

// k_plan: the next batch of the level loop (one CTA).
//   Level switch: when the current level's queue is exhausted, the next level's queue
//   (filled by K4) becomes current.
//   Batch: the next tasks of the current queue, at most tcap tasks and scap stripes.
//   Stripes: a task of m elements gets ~m/L stripes of whole blocks (L ~ the level's
//   elements / (3 * SMs), at least 2^16), its last stripe a quarter shorter; block grid
//   origin g = the first 16-byte aligned element >= lo (TMA bulk copies need 16 B).  The
//   stripes are handed to the persistent K2 CTAs longest first (LPT).
template <class TR>
__global__ void __launch_bounds__(PLAN_THREADS) k_plan(LevelArgs A0, u32 num_sms) {
    constexpr u32 B = TR::B;
    __shared__ u32 s_go, s_swapped, s_na, s_ca, s_w[PLAN_THREADS / 32];
    __shared__ const TaskDesc* s_qa;
    __shared__ u64 s_w64[PLAN_THREADS / 32];
    __shared__ u32 s_pre[PLAN_THREADS];       // inclusive prefix of stripes per task
    __shared__ u64 s_g[PLAN_THREADS], s_lt[PLAN_THREADS];
    __shared__ u64 s_key[MAXS];               // LPT sort keys
    LevelDyn* D = A0.dyn;
    Sched* Q = A0.sched;
    u32* ctr = A0.ctr;
    const u32 tid = threadIdx.x;
    if (tid == 0) {
        u32 go = 1, swapped = 0;
        if (Q->ca >= Q->na) {
            const u32 nb = min(ctr[CTR_NEXT], A0.qn_cap);
            if (nb == 0) {
                go = 0;
            } else {
                TaskDesc* t = Q->qa;
                Q->qa = Q->qb;
                Q->qb = t;
                Q->na = nb;
                Q->ca = 0;
                Q->level += 1;
                ctr[CTR_NEXT] = 0;
                D->q_next = t;
                A0.dstats[DS_LEVELS] += 1;
                swapped = 1;
            }
        }
        s_go = go;
        s_swapped = swapped;
        s_na = Q->na;
        s_ca = Q->ca;
        s_qa = Q->qa;
    }
    __syncthreads();
    if (!s_go) {
        if (tid == 0) {
            D->ntasks = 0;
            D->nstripes = 0;
        }
        return;
    }
    const TaskDesc* qa = s_qa;
    const u32 na = s_na, ca = s_ca;
    if (s_swapped) {
        u64 sz = 0;
        for (u32 i = tid; i < na; i += PLAN_THREADS) sz += qa[i].hi - qa[i].lo;
        sz = plan_sum64(sz, s_w64);
        if (tid == 0) Q->ntot = sz;
    }
    __syncthreads();
    // candidate tasks of this batch
    u32 cand = min(A0.tcap, na - ca);
    const u64 target = max(1ull, (u64)min(A0.scap, (u32)IPS4O_STRIPES_PER_SM * num_sms));
    u64 L;
    if (A0.wave_elems && Q->level >= 2) {
        // an L2-sized wave: the first tasks whose sizes sum to <= wave_elems (>= 1 task);
        // stripes ~3 per SM over the wave's elements
        const u64 m = tid < cand ? qa[ca + tid].hi - qa[ca + tid].lo : 0ull;
        const u32 mk = (u32)min((m + 1023) >> 10, 0xFFFFFFull);
        const u32 pk = plan_scan(mk, s_w);
        const u32 wk = (u32)min(A0.wave_elems >> 10, 0xFFFFFFFFull);
        const u32 fit = __syncthreads_count(tid < cand && pk <= wk);
        cand = cand ? max(fit, 1u) : 0u;
        const u64 wsum = plan_sum64(tid < cand ? m : 0ull, s_w64);
        L = max((wsum + target - 1) / target, A0.wave_stripe);
    } else {
        // stripe length of the level: ~3 stripes per SM over the level's elements, >= 2^16
        const u64 ntot = Q->ntot;
        L = max((ntot + target - 1) / target, MIN_STRIPE);
    }
    L = (L + B - 1) / B * B;
    // the candidates' stripe counts
    const uintptr_t base = reinterpret_cast<uintptr_t>(D->data);
    u32 ns = 0;
    TaskDesc td = TaskDesc{0, 0, 0u, 0u};
    u64 g = 0, Lt = 0;
    if (tid < cand) {
        td = qa[ca + tid];
        g = td.lo;
        while (((base + g * GridStride<TR>::v) & 15u) != 0 && g < td.hi) ++g;
        const u64 main = td.hi - g;
        u64 nsr = max(1ull, (main + L / 2) / L);
        Lt = main;
        if (nsr > 1) {
            Lt = (u64)ceil((double)main / ((double)nsr - IPS4O_LAST_STRIPE_CUT));
            Lt = (Lt + B - 1) / B * B;
            if ((nsr - 1) * Lt >= main) Lt = ((main + nsr - 1) / nsr + B - 1) / B * B;
        }
        if (Lt == 0) Lt = B;
        nsr = max(1ull, (main + Lt - 1) / Lt);
        ns = (u32)min(nsr, (u64)MAXS + 1);
    }
    const u32 pre = plan_scan(ns, s_w);
    s_pre[tid] = pre;
    s_g[tid] = g;
    s_lt[tid] = Lt;
    // tasks whose stripes fit (the prefix is monotone): T = their number, at least one
    const u32 fits = __syncthreads_count(tid < cand && pre <= A0.scap);
    const u32 T = cand ? max(fits, 1u) : 0u;
    const u32 S = T ? min(s_pre[T - 1], A0.scap) : 0u;
    if (tid == 0 && T && s_pre[T - 1] > A0.scap) atomicOr(&ctr[CTR_ERROR], (u32)ERR_CAPACITY);
    u64 bsz = 0;
    if (tid < T) {
        TaskParam tp;
        memset(&tp, 0, sizeof tp);
        tp.lo = td.lo;
        tp.hi = td.hi;
        tp.g = g;
        tp.nblocks = (u32)((td.hi - g + B - 1) / B);
        tp.part = td.part;
        tp.stripe_begin = pre - ns;
        tp.nstripes = ns;
        const_cast<TaskParam*>(A0.tp)[tid] = tp;
        bsz = td.hi - td.lo;
    }
    // stripes: thread s builds stripe s (its task by binary search over the prefix)
    for (u32 s = tid; s < S; s += PLAN_THREADS) {
        u32 lo = 0, hi = T;  // first task i with pre[i] > s
        while (lo < hi) {
            const u32 mid = (lo + hi) >> 1;
            if (s_pre[mid] > s) hi = mid;
            else lo = mid + 1;
        }
        const u32 i = lo;
        const u32 nsi = s_pre[i] - (i ? s_pre[i - 1] : 0u);
        const u32 j = s - (s_pre[i] - nsi);
        const TaskDesc ti = qa[ca + i];
        const u64 gi = s_g[i], Li = s_lt[i];
        StripeDesc sd;
        sd.begin = j == 0 ? ti.lo : gi + j * Li;
        sd.end = j + 1 == nsi ? ti.hi : gi + (j + 1) * Li;
        sd.task = i;
        const u64 mb = sd.begin > gi ? sd.begin : gi;
        sd.sb = (u32)((mb - gi) / B);
        sd.se = (u32)((sd.end - gi + B - 1) / B);
        sd.first = j == 0;
        const_cast<StripeDesc*>(A0.sd)[s] = sd;
        // LPT order: longest first, ties by index (stable)
        const u64 len = sd.end - sd.begin;
        s_key[s] = ((0xFFFFFFFFFFull - min(len, 0xFFFFFFFFFFull)) << 12) | s;
    }
    for (u32 s = S + tid; s < MAXS; s += PLAN_THREADS) s_key[s] = ~0ull;
    __syncthreads();
    // bitonic sort of the MAXS keys (ascending)
    for (u32 kk = 2; kk <= MAXS; kk <<= 1) {
        for (u32 jj = kk >> 1; jj > 0; jj >>= 1) {
            for (u32 i = tid; i < MAXS; i += PLAN_THREADS) {
                const u32 l = i ^ jj;
                if (l > i) {
                    const u64 a = s_key[i], b = s_key[l];
                    const bool up = (i & kk) == 0;
                    if ((a > b) == up) {
                        s_key[i] = b;
                        s_key[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (u32 s = tid; s < S; s += PLAN_THREADS) const_cast<u32*>(A0.stripe_order)[s] = (u32)(s_key[s] & 0xFFFu);
    // task-done bits of K3 (absent tasks done)
    for (u32 wi = tid; wi < (A0.tcap + 31) / 32; wi += PLAN_THREADS) {
        const u32 lo = wi * 32;
        A0.tdone[wi] = T >= lo + 32 ? 0u : (T <= lo ? ~0u : ~((1u << (T - lo)) - 1u));
    }
    bsz = plan_sum64(bsz, s_w64);
    if (tid == 0) {
        D->ntasks = T;
        D->nstripes = S;
        D->k4_cta = T * (u32)MAXK < 32u * num_sms ? 1u : 0u;
        D->moves_gx = T ? max(1u, (2u * num_sms + T - 1) / T) : 1u;
        Q->seed = mix64(Q->seed);
        D->seed = Q->seed;
        Q->ca = ca + T;
        A0.dstats[DS_DIST_TASKS] += T;
        A0.dstats[DS_DIST_ELEMS] += bsz;
        A0.dstats[DS_BATCHES] += 1;
    }
}

// k_epi: end of a batch -- fold its counters into the statistics, reset them, and decide
// whether the loop continues (a level queue holds tasks; no device error).
__global__ void k_epi(LevelArgs A0, cudaGraphConditionalHandle h, u32 use_handle) {
    if (threadIdx.x != 0) return;
    u32* ctr = A0.ctr;
    u64* st = A0.dstats;
    Sched* Q = A0.sched;
    st[DS_EQ_TASKS] += ctr[CTR_EQ];
    st[DS_ERROR] |= ctr[CTR_ERROR];
    u64 nb = 0;
    for (int c = 0; c < NUM_BASE_CLASSES; ++c) {
        st[DS_BASE_C0 + c] += ctr[CTR_BASE0 + c];
        nb += ctr[CTR_BASE0 + c];
    }
    st[DS_BASE_TASKS] += nb;
    st[DS_FALLBACK] += ctr[CTR_FB];
    st[DS_MED_TASKS] += ctr[CTR_MED];
    st[DS_BLOCK_MOVES] += ctr[CTR_BMOVES];
    st[DS_AMOVES] += ctr[CTR_AMOVES];
    st[DS_BASE_ELEMS] += *A0.base_elems;
    for (int i = 0; i < CTR_N; ++i)
        if (i != CTR_NEXT) ctr[i] = 0;
    *A0.spill_ctr = 0;
    *A0.base_elems = 0;
    st[DS_ITERS] += 1;
    if (st[DS_BATCHES] >= MAX_BATCHES) st[DS_ERROR] |= ERR_ITER;
    const u32 more = (Q->ca < Q->na || ctr[CTR_NEXT] > 0) && st[DS_ERROR] == 0 ? 1u : 0u;
    A0.dyn->more = more;
    if (use_handle) cudaGraphSetConditional(h, more);
}

// Profile stamp (ips4o_profile_enable): globaltimer after the kernel of kind `kind` finished.
__global__ void k_stamp(LevelArgs A0, u32 kind) {
    if (threadIdx.x != 0) return;
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const u32 i = atomicAdd(A0.plog_n, 1u);
    if (i < A0.plog_cap) {
        A0.plog_t[i] = t;
        A0.plog_k[i] = kind;
    }
}

}  // namespace ips4o
