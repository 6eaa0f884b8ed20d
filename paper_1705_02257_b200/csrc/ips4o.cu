// ips4o.cu -- libips4o.so: host planner, kernel launch sequence and the C ABI of
// include/ips4o.h.  The host only plans (stripes per task) and enqueues kernels on the
// caller's stream; every step of the sort runs in the kernels of k_*.cuh.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/ips4o.h"
#include "common.cuh"
#include "k_base.cuh"
#include "k_classify.cuh"
#include "k_classify_rec.cuh"
#include "k_cleanup.cuh"
#include "k_permute.cuh"
#include "k_sample.cuh"

namespace ips4o {

#ifndef IPS4O_LAST_STRIPE_CUT  // a task's last stripe is (1 - this) of the others
#define IPS4O_LAST_STRIPE_CUT 0.75
#endif
#ifndef IPS4O_STRIPES_PER_SM  // stripes per SM of a level (K2 balance vs per-stripe overhead)
#define IPS4O_STRIPES_PER_SM 3
#endif
constexpr u32 MAXT = 512;          // tasks per level batch
constexpr u32 MAXS = 512;          // stripes per level batch
static_assert(MAXS <= (u32)K4_MAXSTRIPES && MAXS <= (u32)K2P_MAXST, "per-task stripe tables in shared memory");
constexpr u32 QCAP = MAXT * MAXK;  // queue capacity (tasks)
constexpr u32 Q_SPEC = 512;        // next-level tasks copied back with a level's counters
constexpr u64 MIN_STRIPE = 65536;  // elements

static std::mutex g_mu;
static char g_errbuf[512];
static ips4o_stats g_stats;

enum KernelKind { KK_SAMPLE = 0, KK_CLASSIFY, KK_PREPARE, KK_MOVES, KK_PERMUTE, KK_CLEANUP, KK_BASE, KK_OTHER };
static const char* kKindNames[IPS4O_NUM_KERNEL_KINDS] = {
    "sample_splitters", "classify_flush", "prepare", "empty_block_moves",
    "block_permute",    "cleanup",        "base_case", "other"};

struct Prof {
    bool on = false;
    struct Rec {
        int kind;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
} g_prof;

struct Workspace {
    int device = -1;
    int num_sms = 0;
    char* dev = nullptr;
    size_t dev_bytes = 0;
    u64 spill_elems = 0;  // capacity in elements (of the current element size)
    int spill_elem_size = 0;
    char* host = nullptr;
    // device carve-up
    TaskParam* tp;
    StripeDesc* sd;
    u32* order;
    u64 *tree, *spl;
    u32 *s_count, *s_fill, *s_spoff, *s_nfull, *prefF, *prefE;
    u64* s_spbase;
    u64* bnd;
    u32 *dblk, *nfb, *mov, *done, *cflag, *tdone, *btot;
    unsigned short* lut;
    u64* wr;
    void* ovf;
    int* ovf_owner;
    TaskDesc *q_next, *q_base;
    u32* ctr;
    u64* spill_ctr;
    u64* dsplit;
    void* spill;
    // pinned host
    TaskParam* h_tp;
    StripeDesc* h_sd;
    u32* h_order;
    u32* h_ctr;
    TaskDesc* h_q;
    cudaStream_t side[4];             // base-case size classes run concurrently
    cudaEvent_t ev_fork, ev_join[4];
    bool side_ready;
    int side_dev;
    u64* h_bnd;
    u32* h_tdone;
    u32 k2_blocks = 0, k3_blocks = 0, k3t_blocks = 0;
    int k2_type = -1;
};
static Workspace g_ws;

static int set_cuda_error(cudaError_t e, const char* what) {
    snprintf(g_errbuf, sizeof g_errbuf, "%s: %s", what, cudaGetErrorString(e));
    return IPS4O_ECUDA;
}
#define CK(x)                                                  \
    do {                                                       \
        cudaError_t e_ = (x);                                  \
        if (e_ != cudaSuccess) return set_cuda_error(e_, #x);  \
    } while (0)

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static size_t fixed_bytes() {
    size_t s = 0;
    auto add = [&](size_t b) { s += align_up(b, 256); };
    add(MAXT * sizeof(TaskParam));
    add(MAXS * sizeof(StripeDesc));
    add(MAXS * 4);
    add((size_t)MAXT * MAXK * 8 * 2);          // tree, spl
    add((size_t)MAXS * MAXK * 4 * 3);          // s_count, s_fill, s_spoff
    add(MAXS * 8 + MAXS * 4 * 3);              // s_spbase, s_nfull, prefF, prefE
    add((size_t)MAXT * (MAXK + 1) * 8);        // bnd
    add((size_t)MAXT * (MAXK + 1) * 4 * 2);    // dblk, mov
    add((size_t)MAXT * MAXK * 4 * 3);          // nfb, cflag, btot
    add((size_t)MAXT * LUT_STRIDE * 2);        // bucket-hint tables
    add((size_t)MAXT * (MAXK / 32) * 4);       // done
    add(MAXT / 32 * 4);                        // tdone
    add((size_t)MAXT * MAXK * 8 * CTL_STRIDE);  // wr control lines
    add((size_t)MAXT * BLOCK_BYTES);           // ovf
    add(MAXT * 4);                             // ovf_owner
    add((size_t)QCAP * sizeof(TaskDesc) * (1 + NUM_BASE_CLASSES));  // queues
    add(CTR_N * 4 + 16);                       // ctr + spill ctr + base-element ctr
    add(MAXK * 8);                             // debug splitters
    return s;
}

static u64 spill_bound_elems(u64 n, int esize) {
    // a stripe spills at most 256 partially filled buffers of < b elements (b*s = 512 B)
    const u64 per_stripe = (u64)MAXK * (BLOCK_BYTES / esize);
    return std::min<u64>(n + 64, (u64)MAXS * per_stripe);
}

static int ensure_ws(u64 n, int esize) {
    int dev;
    CK(cudaGetDevice(&dev));
    if (g_ws.device != dev) {
        if (g_ws.dev) {
            cudaFree(g_ws.dev);
            g_ws.dev = nullptr;
        }
        g_ws.device = dev;
        CK(cudaDeviceGetAttribute(&g_ws.num_sms, cudaDevAttrMultiProcessorCount, dev));
        g_ws.k2_type = -1;
    }
    const u64 need_spill = spill_bound_elems(n, esize);
    const size_t need = fixed_bytes() + align_up(need_spill * esize, 256);
    if (g_ws.dev && g_ws.dev_bytes >= need) {
        g_ws.spill_elems = (g_ws.dev_bytes - fixed_bytes()) / esize;
        g_ws.spill_elem_size = esize;
        return IPS4O_OK;
    }
    if (g_ws.dev) cudaFree(g_ws.dev);
    g_ws.dev = nullptr;
    if (cudaMalloc(&g_ws.dev, need) != cudaSuccess) {
        cudaGetLastError();
        g_ws.dev_bytes = 0;
        snprintf(g_errbuf, sizeof g_errbuf, "workspace allocation of %zu bytes failed", need);
        return IPS4O_ENOMEM;
    }
    g_ws.dev_bytes = need;
    char* p = g_ws.dev;
    auto take = [&](size_t b) {
        char* r = p;
        p += align_up(b, 256);
        return r;
    };
    g_ws.tp = (TaskParam*)take(MAXT * sizeof(TaskParam));
    g_ws.sd = (StripeDesc*)take(MAXS * sizeof(StripeDesc));
    g_ws.order = (u32*)take(MAXS * 4);
    char* tr = take((size_t)MAXT * MAXK * 8 * 2);
    g_ws.tree = (u64*)tr;
    g_ws.spl = (u64*)(tr + (size_t)MAXT * MAXK * 8);
    char* sc = take((size_t)MAXS * MAXK * 4 * 3);
    g_ws.s_count = (u32*)sc;
    g_ws.s_fill = g_ws.s_count + (size_t)MAXS * MAXK;
    g_ws.s_spoff = g_ws.s_fill + (size_t)MAXS * MAXK;
    char* ss = take(MAXS * 8 + MAXS * 4 * 3);
    g_ws.s_spbase = (u64*)ss;
    g_ws.s_nfull = (u32*)(ss + MAXS * 8);
    g_ws.prefF = g_ws.s_nfull + MAXS;
    g_ws.prefE = g_ws.prefF + MAXS;
    g_ws.bnd = (u64*)take((size_t)MAXT * (MAXK + 1) * 8);
    char* dm = take((size_t)MAXT * (MAXK + 1) * 4 * 2);
    g_ws.dblk = (u32*)dm;
    g_ws.mov = g_ws.dblk + (size_t)MAXT * (MAXK + 1);
    char* nr = take((size_t)MAXT * MAXK * 4 * 3);
    g_ws.nfb = (u32*)nr;
    g_ws.cflag = g_ws.nfb + (size_t)MAXT * MAXK;
    g_ws.btot = g_ws.cflag + (size_t)MAXT * MAXK;
    g_ws.lut = (unsigned short*)take((size_t)MAXT * LUT_STRIDE * 2);
    g_ws.done = (u32*)take((size_t)MAXT * (MAXK / 32) * 4);
    g_ws.tdone = (u32*)take(MAXT / 32 * 4);
    g_ws.wr = (u64*)take((size_t)MAXT * MAXK * 8 * CTL_STRIDE);
    g_ws.ovf = take((size_t)MAXT * BLOCK_BYTES);
    g_ws.ovf_owner = (int*)take(MAXT * 4);
    char* q = take((size_t)QCAP * sizeof(TaskDesc) * (1 + NUM_BASE_CLASSES));
    g_ws.q_next = (TaskDesc*)q;
    g_ws.q_base = g_ws.q_next + QCAP;
    char* c = take(CTR_N * 4 + 16);
    g_ws.ctr = (u32*)c;
    g_ws.spill_ctr = (u64*)(c + CTR_N * 4);
    g_ws.dsplit = (u64*)take(MAXK * 8);
    g_ws.spill = p;
    g_ws.spill_elems = (g_ws.dev_bytes - fixed_bytes()) / esize;
    g_ws.spill_elem_size = esize;
    if (!g_ws.host) {
        size_t hb = MAXT * sizeof(TaskParam) + MAXS * sizeof(StripeDesc) + MAXS * 4 + CTR_N * 4 + 64 +
                    (size_t)QCAP * sizeof(TaskDesc) + (MAXK + 1) * 8 + MAXT / 32 * 4 + 4096;
        CK(cudaMallocHost(&g_ws.host, hb));
        char* h = g_ws.host;
        g_ws.h_tp = (TaskParam*)h;
        h += MAXT * sizeof(TaskParam);
        g_ws.h_sd = (StripeDesc*)h;
        h += MAXS * sizeof(StripeDesc);
        g_ws.h_order = (u32*)h;
        h += MAXS * 4;
        g_ws.h_ctr = (u32*)h;
        h += CTR_N * 4 + 64;
        g_ws.h_q = (TaskDesc*)h;
        h += (size_t)QCAP * sizeof(TaskDesc);
        g_ws.h_bnd = (u64*)h;
        h += (MAXK + 1) * 8;
        g_ws.h_tdone = (u32*)h;
    }
    return IPS4O_OK;
}

// ------------------------------------------------------------------ launching

template <class F>
static int launch(int kind, cudaStream_t st, F&& f) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (g_prof.on) {
        a = g_prof.get();
        b = g_prof.get();
        cudaEventRecord(a, st);
    }
    f();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, kKindNames[kind]);
    static int sync_check = -1;  // IPS4O_SYNC_CHECK=1: synchronise after every launch (debugging)
    if (sync_check < 0) {
        const char* v = getenv("IPS4O_SYNC_CHECK");
        sync_check = (v && v[0] == '1') ? 1 : 0;
    }
    if (sync_check) {
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return set_cuda_error(e, kKindNames[kind]);
    }
    if (g_prof.on) {
        cudaEventRecord(b, st);
        g_prof.recs.push_back({kind, a, b});
    }
    g_stats.kernel_launches++;
    return IPS4O_OK;
}
#define LAUNCH(kind, ...)                                         \
    do {                                                          \
        int rc_ = launch(kind, st, [&]() { __VA_ARGS__; });       \
        if (rc_) return rc_;                                      \
    } while (0)

template <class TR, int TH>
static cudaError_t set_base_attr1() {
    return cudaFuncSetAttribute(k_base_merge<TR, TH, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)BaseClass<TR, TH, 16>::smem);
}
// cell base-case configurations of the size classes <= 2048 and <= 4096 (threads,
// elements per thread); the <= 8192 class uses (512, 16)
#ifndef IPS4O_CELL_BIG_NT  // threads of the base-case CTA for leaves of 4097..8192 elements
#define IPS4O_CELL_BIG_NT 512
#endif
#ifndef IPS4O_CELL_SMALL
#define IPS4O_CELL_SMALL 1
#endif
// 8-byte types: 16 elements per thread in small CTAs (more leaves in flight per SM);
// 16-byte types: 8 per thread (register budget)
template <class TR> struct CellCfg {
    static constexpr bool small = IPS4O_CELL_SMALL && TR::S == 8;
    static constexpr int NT0 = small ? 128 : 256, E0 = small ? 16 : 8;
    static constexpr int NT1 = small ? (int)TR::C1MAX / 16 : 512, E1 = small ? 16 : 8;
    static constexpr int NT2 = IPS4O_CELL_BIG_NT, E2 = 8192 / IPS4O_CELL_BIG_NT;  // leaves of <= 8192
};
template <class TR, int NT, int E>
static cudaError_t set_cell_attr() {
    return cudaFuncSetAttribute(k_base_cell<TR, NT, E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)CellBase<TR, NT, E>::smem);
}
template <class TR>
static cudaError_t set_base_attrs() {
    cudaError_t e = set_base_attr1<TR, (TR::CAP >= 16384 ? 1024 : 512)>();
    if (e == cudaSuccess) e = set_cell_attr<TR, CellCfg<TR>::NT0, CellCfg<TR>::E0>();
    if (e == cudaSuccess) e = set_cell_attr<TR, CellCfg<TR>::NT1, CellCfg<TR>::E1>();
    if (e == cudaSuccess) e = set_cell_attr<TR, CellCfg<TR>::NT2, CellCfg<TR>::E2>();
    if constexpr (TR::CAP >= 16384) {
        if (e == cudaSuccess) e = set_cell_attr<TR, 1024, 16>();
    }
    return e;
}

// K2 configurations: (threads, elements per thread).  IPS4O_K2_VARIANT=1 selects the
// 512-thread configuration (tuning experiments); the default is variant 0.
#if IPS4O_BLOCK_BYTES == 512
// 256 buffers of 512 B = 128 KB of shared memory: one CTA per SM
// (640 threads: 20 warps hide more of the barrier and shared-memory latency than 16, at
// 96 registers per thread; two 40 KB stages still fit next to the buffers)
template <class TR> struct K2Cfg0 { static constexpr int NT = 640, E = 16 / TR::S * 4, MINB = 1; };
template <class TR> struct K2Cfg1 { static constexpr int NT = 512, E = 16 / TR::S * 4, MINB = 1; };
#else
// 256 buffers of 256 B = 64 KB: two CTAs per SM
template <class TR> struct K2Cfg0 { static constexpr int NT = 256, E = 16 / TR::S * 4, MINB = 2; };
template <class TR> struct K2Cfg1 { static constexpr int NT = 512, E = 16 / TR::S * 2, MINB = 2; };
#endif
// IPS4O_K3=regs selects the register-buffer permutation for the 8/16-byte types (tuning)
static int k3_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IPS4O_K3");
        v = (e && e[0] == 'r') ? 1 : 0;
    }
    return v;
}
static int k2_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IPS4O_K2_VARIANT");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v;
}
template <class TR, class C>
static cudaError_t k2_setup(int* occ) {
    cudaError_t e = cudaFuncSetAttribute(k_classify<TR, C::NT, C::E, C::MINB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)K2Smem<TR, C::NT, C::E>::total);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k_classify<TR, C::NT, C::E, C::MINB>, C::NT,
                                                         K2Smem<TR, C::NT, C::E>::total);
}

constexpr int K2REC_THREADS = 256;

template <class TR>
static int prepare_kernels(void) {
    if (g_ws.k2_type == TR::TYPE) return IPS4O_OK;
    if constexpr (TR::S == 100) {
        int occ2 = 0, occ3 = 0;
        CK(cudaFuncSetAttribute(k_classify_rec<K2REC_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)K2RecSmem<K2REC_THREADS>::total));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_classify_rec<K2REC_THREADS>, K2REC_THREADS,
                                                         K2RecSmem<K2REC_THREADS>::total));
        CK(cudaFuncSetAttribute(k_base_rec<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RecBase<2>::smem));
        CK(cudaFuncSetAttribute(k_base_rec<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RecBase<4>::smem));
        CK(cudaFuncSetAttribute(k_sample<TR, K1_SAMPLE_BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(padidx(K1_SAMPLE_BIG) * 8 + 16)));
        CK(cudaFuncSetAttribute(k_sample<TR, K1_SAMPLE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(padidx(K1_SAMPLE) * 8 + 16)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_permute<TR>, K3_THREADS, 0));
        int occ3t = 0;
        CK(cudaFuncSetAttribute(k_permute_tma<TR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)K3TSmem<TR>::total));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3t, k_permute_tma<TR>, K3T_THREADS, K3TSmem<TR>::total));
        if (occ2 < 1 || occ3 < 1 || occ3t < 1) {
            snprintf(g_errbuf, sizeof g_errbuf, "occupancy query returned %d/%d/%d", occ2, occ3, occ3t);
            return IPS4O_ECUDA;
        }
        g_ws.k2_blocks = (u32)(occ2 * g_ws.num_sms);
        g_ws.k3_blocks = (u32)(occ3 * g_ws.num_sms);
        g_ws.k3t_blocks = (u32)(occ3t * g_ws.num_sms);
        g_ws.k2_type = TR::TYPE;
        return IPS4O_OK;
    } else {
    CK(set_base_attrs<TR>());
    CK(cudaFuncSetAttribute(k_sample<TR, K1_SAMPLE_BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(padidx(K1_SAMPLE_BIG) * 8 + 16)));
    CK(cudaFuncSetAttribute(k_sample<TR, K1_SAMPLE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(padidx(K1_SAMPLE) * 8 + 16)));
    int occ2 = 0, occ3 = 0;
    if (k2_variant() == 1) CK((k2_setup<TR, K2Cfg1<TR>>(&occ2)));
    else CK((k2_setup<TR, K2Cfg0<TR>>(&occ2)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_permute<TR>, K3_THREADS, 0));
    int occ3t = 0;
    CK(cudaFuncSetAttribute(k_permute_tma<TR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)K3TSmem<TR>::total));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3t, k_permute_tma<TR>, K3T_THREADS, K3TSmem<TR>::total));
    if (occ2 < 1 || occ3 < 1 || occ3t < 1) {
        snprintf(g_errbuf, sizeof g_errbuf, "occupancy query returned %d/%d/%d", occ2, occ3, occ3t);
        return IPS4O_ECUDA;
    }
    g_ws.k2_blocks = (u32)(occ2 * g_ws.num_sms);
    g_ws.k3_blocks = (u32)(occ3 * g_ws.num_sms);
    g_ws.k3t_blocks = (u32)(occ3t * g_ws.num_sms);
    g_ws.k2_type = TR::TYPE;
    return IPS4O_OK;
    }
}

template <class TR>
static LevelArgs level_args(void* data, u32 T, u32 S, int emit, u64 seed) {
    LevelArgs A;
    memset(&A, 0, sizeof A);
    A.data = data;
    A.tp = g_ws.tp;
    A.ntasks = T;
    A.sd = g_ws.sd;
    A.stripe_order = g_ws.order;
    A.nstripes = S;
    A.tree = g_ws.tree;
    A.spl = g_ws.spl;
    A.s_count = g_ws.s_count;
    A.s_fill = g_ws.s_fill;
    A.s_spoff = g_ws.s_spoff;
    A.s_spbase = g_ws.s_spbase;
    A.s_nfull = g_ws.s_nfull;
    A.prefF = g_ws.prefF;
    A.prefE = g_ws.prefE;
    A.spill = g_ws.spill;
    A.spill_cap = g_ws.spill_elems;
    A.bnd = g_ws.bnd;
    A.dblk = g_ws.dblk;
    A.nfb = g_ws.nfb;
    A.btot = g_ws.btot;
    A.lut = g_ws.lut;
    A.mov = g_ws.mov;
    A.wr = g_ws.wr;
    A.done = g_ws.done;
    A.tdone = g_ws.tdone;
    A.cflag = g_ws.cflag;
    A.ovf = g_ws.ovf;
    A.ovf_owner = g_ws.ovf_owner;
    A.q_next = g_ws.q_next;
    A.q_base = g_ws.q_base;
    A.q_cap = QCAP;
    A.ctr = g_ws.ctr;
    A.spill_ctr = g_ws.spill_ctr;
    A.base_elems = g_ws.spill_ctr + 1;
    A.base_cap = TR::CAP;
    A.emit = emit;
    A.seed = seed;
    return A;
}

// Stripe length of a level: about 3 stripes per SM over the level's Ntot elements (at
// least MIN_STRIPE), a whole number of blocks.
template <class TR>
static u64 stripe_len(u64 Ntot) {
    const u64 target = std::max<u64>(1, std::min<u64>(MAXS, (u64)IPS4O_STRIPES_PER_SM * g_ws.num_sms));
    u64 L = std::max<u64>((Ntot + target - 1) / target, MIN_STRIPE);
    return (L + TR::B - 1) / TR::B * TR::B;
}
// number of stripes plan_batch creates for a task of `size` elements (an upper bound: the
// task's aligned main part is at most size)
static u32 stripes_for(u64 size, u64 L) { return (u32)std::max<u64>(1, (size + L / 2) / L); }

// Plan the stripes of a batch of tasks (host) into g_ws.h_tp / h_sd / h_order.
template <class TR>
static void plan_batch(const TaskDesc* tasks, u32 T, uintptr_t base_addr, u64 L, u32* S_out) {
    constexpr int B = TR::B;
    u32 S = 0;
    for (u32 i = 0; i < T; ++i) {
        const u64 lo = tasks[i].lo, hi = tasks[i].hi;
        u64 g = lo;  // block grid origin: the first 16-byte aligned element (TMA block moves)
        while (((base_addr + g * TR::S) & 15u) != 0 && g < hi) ++g;
        TaskParam& tp = g_ws.h_tp[i];
        memset(&tp, 0, sizeof tp);
        tp.lo = lo;
        tp.hi = hi;
        tp.g = g;
        tp.nblocks = (u32)((hi - g + B - 1) / B);
        tp.part = tasks[i].part;
        const u64 main = hi - g;
        u64 ns = std::max<u64>(1, (main + L / 2) / L);
        // the task's last stripe is a quarter of the others: with the stripes handed out
        // longest first, the short ones fill the persistent K2 CTAs' last round
        u64 Lt = ns > 1 ? (u64)std::ceil((double)main / ((double)ns - IPS4O_LAST_STRIPE_CUT)) : main;
        Lt = (Lt + B - 1) / B * B;
        if (ns > 1 && (ns - 1) * Lt >= main) Lt = ((main + ns - 1) / ns + B - 1) / B * B;
        ns = std::max<u64>(1, (main + Lt - 1) / Lt);
        tp.stripe_begin = S;
        tp.nstripes = (u32)ns;
        for (u64 j = 0; j < ns; ++j) {
            StripeDesc& sd = g_ws.h_sd[S];
            sd.begin = j == 0 ? lo : g + j * Lt;
            sd.end = j + 1 == ns ? hi : g + (j + 1) * Lt;
            sd.task = i;
            const u64 mb = std::max(sd.begin, g);
            sd.sb = (u32)((mb - g) / B);
            sd.se = (u32)((sd.end - g + B - 1) / B);
            sd.first = j == 0;
            ++S;
        }
    }
    // longest stripes first (LPT) for the persistent K2 CTAs
    for (u32 j = 0; j < S; ++j) g_ws.h_order[j] = j;
    std::stable_sort(g_ws.h_order, g_ws.h_order + S, [](u32 a, u32 b) {
        return (g_ws.h_sd[a].end - g_ws.h_sd[a].begin) > (g_ws.h_sd[b].end - g_ws.h_sd[b].begin);
    });
    *S_out = S;
}

// One distribution level over T <= MAXT tasks (already planned into h_tp/h_sd).
template <class TR>
static int run_level(void* data, u32 T, u32 S, cudaStream_t st, bool from_splitters, u32 nspl,
                     u32 eq, int emit, u64 seed) {
    CK(cudaMemcpyAsync(g_ws.tp, g_ws.h_tp, T * sizeof(TaskParam), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(g_ws.sd, g_ws.h_sd, S * sizeof(StripeDesc), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(g_ws.order, g_ws.h_order, S * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(g_ws.ctr, 0, CTR_N * 4 + 16, st));
    LevelArgs A = level_args<TR>(data, T, S, emit, seed);
    if (from_splitters) {
        LAUNCH(KK_SAMPLE, (k_tree_from_splitters<<<1, 256, 0, st>>>(A, g_ws.dsplit, nspl, eq)));
    } else {
        u64 maxn = 0;
        for (u32 i = 0; i < T; ++i) maxn = std::max<u64>(maxn, g_ws.h_tp[i].hi - g_ws.h_tp[i].lo);
        if (maxn >= K1_BIG_TASK)
            LAUNCH(KK_SAMPLE, (k_sample<TR, K1_SAMPLE_BIG><<<T, K1Cfg<K1_SAMPLE_BIG>::THREADS, padidx(K1_SAMPLE_BIG) * 8 + 16, st>>>(A)));
        else
            LAUNCH(KK_SAMPLE, (k_sample<TR, K1_SAMPLE><<<T, K1Cfg<K1_SAMPLE>::THREADS, padidx(K1_SAMPLE) * 8 + 16, st>>>(A)));
    }
    const u32 g2 = std::min<u32>(S, g_ws.k2_blocks);
    if constexpr (TR::S == 100) {
        LAUNCH(KK_CLASSIFY, (k_classify_rec<K2REC_THREADS><<<g2, K2REC_THREADS, K2RecSmem<K2REC_THREADS>::total, st>>>(A)));
    } else if (k2_variant() == 1) {
        typedef K2Cfg1<TR> C;
        LAUNCH(KK_CLASSIFY, (k_classify<TR, C::NT, C::E, C::MINB><<<g2, C::NT, K2Smem<TR, C::NT, C::E>::total, st>>>(A)));
    } else {
        typedef K2Cfg0<TR> C;
        LAUNCH(KK_CLASSIFY, (k_classify<TR, C::NT, C::E, C::MINB><<<g2, C::NT, K2Smem<TR, C::NT, C::E>::total, st>>>(A)));
    }
    LAUNCH(KK_PREPARE, (k_prepare<TR><<<T, MAXK, 0, st>>>(A)));
    const u32 gx = std::max<u32>(1, (2 * g_ws.num_sms + T - 1) / T);
    LAUNCH(KK_MOVES, (k_moves<TR><<<dim3(gx, T), 256, 0, st>>>(A)));
    {
        u32 tw[MAXT / 32];
        const u32 nwd = (T + 31) / 32;
        for (u32 i = 0; i < nwd; ++i) {
            const u32 lo = i * 32;
            tw[i] = (T >= lo + 32) ? 0u : ~((1u << (T - lo)) - 1u);  // bits of absent tasks set
        }
        memcpy(g_ws.h_tdone, tw, nwd * 4);
        CK(cudaMemcpyAsync(g_ws.tdone, g_ws.h_tdone, nwd * 4, cudaMemcpyHostToDevice, st));
    }
#ifdef IPS4O_K3_TIMELINE
    {
        static unsigned int zero[4096];
        unsigned long long t0 = 0;
        cudaStreamSynchronize(st);
        cudaMemcpyToSymbol(g_k3_hist, zero, sizeof zero);
        // a timestamp slightly after the launch: the kernel's first events define t0 instead
        LAUNCH(KK_OTHER, (k_timer_start<<<1, 1, 0, st>>>()));
        (void)t0;
    }
#endif
    {
        if (k3_variant() == 0)
            LAUNCH(KK_PERMUTE, (k_permute_tma<TR><<<g_ws.k3t_blocks, K3T_THREADS, K3TSmem<TR>::total, st>>>(A)));
        else
            LAUNCH(KK_PERMUTE, (k_permute<TR><<<g_ws.k3_blocks, K3_THREADS, 0, st>>>(A)));
    }
#ifdef IPS4O_K3_TIMELINE
    {
        static unsigned int h[4096];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_k3_hist, sizeof h);
        unsigned long long tp = 0, tt = 0;
        int last = 0;
        for (int i = 0; i < 2048; ++i) { tp += h[i]; tt += h[2048 + i]; if (h[i] || h[2048 + i]) last = i; }
        fprintf(stderr, "K3 timeline T=%u: placements %llu takes %llu, last bin %d us\n", T, tp, tt, last);
        for (int i = 0; i <= last; i += (last > 40 ? last / 40 : 1)) {
            unsigned long long a = 0, b = 0;
            for (int j = i; j < i + (last > 40 ? last / 40 : 1) && j <= last; ++j) { a += h[j]; b += h[2048 + j]; }
            fprintf(stderr, "  t=%4d us  place %8llu  take %8llu\n", i, a, b);
        }
    }
#endif
    if (T * MAXK >= 32u * g_ws.num_sms) {
        // many buckets: one warp per group of K4_GROUP buckets
        const u32 nw = T * MAXK / K4_GROUP, want = (nw + K4_WARPS - 1) / K4_WARPS;
        LAUNCH(KK_CLEANUP, (k_cleanup<TR><<<std::min<u32>(want, 8u * g_ws.num_sms), K4_THREADS, 0, st>>>(A)));
    } else {
        LAUNCH(KK_CLEANUP, (k_cleanup_cta<TR><<<T * MAXK, K4_THREADS, 0, st>>>(A)));
    }
    CK(cudaMemcpyAsync(g_ws.h_ctr, g_ws.ctr, CTR_N * 4 + 16, cudaMemcpyDeviceToHost, st));
    // the first next-level tasks come back with the counters (one sync fewer when a level
    // emits at most Q_SPEC of them, e.g. the 256 of the top level)
    if (emit) CK(cudaMemcpyAsync(g_ws.h_q, g_ws.q_next, Q_SPEC * sizeof(TaskDesc), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    g_stats.host_syncs++;
    if (g_ws.h_ctr[CTR_ERROR]) {
        snprintf(g_errbuf, sizeof g_errbuf, "device consistency check failed (flags 0x%x)",
                 g_ws.h_ctr[CTR_ERROR]);
        return IPS4O_EINTERNAL;
    }
    g_stats.equality_tasks += g_ws.h_ctr[CTR_EQ];
    {
        u64 be;
        memcpy(&be, (const char*)g_ws.h_ctr + CTR_N * 4 + 8, 8);
        g_stats.base_elements += be;
    }
    return IPS4O_OK;
}

// Base case of one level batch: size classes 0..2 (<= 2K / 4K / 8K elements) by the cell
// kernel, class 3 (<= CAP) and any leaf the cell kernel hands back by the merge sort,
// which reads its task count from the device (the fallback queue is appended to class 3).
#ifndef IPS4O_CELL_OVERSUB  // base-case grid: resident CTAs times this
#define IPS4O_CELL_OVERSUB 8
#endif
#ifndef IPS4O_BASE_STREAMS
#define IPS4O_BASE_STREAMS 1
#endif
static cudaError_t side_streams_ready() {
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    if (g_ws.side_ready && g_ws.side_dev == dev) return cudaSuccess;
    if (g_ws.side_ready) {  // the streams belong to another device: make new ones here
        for (int c = 0; c < 4; ++c) {
            cudaStreamDestroy(g_ws.side[c]);
            cudaEventDestroy(g_ws.ev_join[c]);
        }
        cudaEventDestroy(g_ws.ev_fork);
        g_ws.side_ready = false;
    }
    g_ws.side_dev = dev;
    for (int c = 0; c < 4; ++c) {
        cudaError_t e = cudaStreamCreateWithFlags(&g_ws.side[c], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_ws.ev_join[c], cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventCreateWithFlags(&g_ws.ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) g_ws.side_ready = true;
    return e;
}
template <class TR, int NT, int E>
static int run_cell_class(void* data, u32 count, TaskDesc* d_tasks, cudaStream_t st) {
    if (!count) return IPS4O_OK;
    typedef CellBase<TR, NT, E> CB;
    // resident CTAs x IPS4O_CELL_OVERSUB (persistent loop over the class's leaves)
    static int occ = 0;
    if (!occ) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_base_cell<TR, NT, E>, NT, CB::smem));
        if (occ < 1) occ = 1;
    }
    const u32 grid = std::min<u32>(count, (u32)occ * IPS4O_CELL_OVERSUB * g_ws.num_sms);
    LAUNCH(KK_BASE, (k_base_cell<TR, NT, E><<<grid, NT, CB::smem, st>>>(d_tasks, count, data, g_ws.q_base + 3 * QCAP,
                                                                        g_ws.ctr + CTR_BASE0 + 3, QCAP)));
    g_stats.base_tasks += count;
    return IPS4O_OK;
}

// counts[c] tasks of size class c at d_queues + c*QCAP
template <class TR>
static int run_base(void* data, const u32* counts, TaskDesc* d_queues, cudaStream_t st) {
    if constexpr (TR::S == 100) {
        if (counts[2] || counts[3]) {
            snprintf(g_errbuf, sizeof g_errbuf, "record base task above capacity");
            return IPS4O_EINTERNAL;
        }
        if (counts[0]) {
            const u32 grid = std::min<u32>(counts[0], 4u * g_ws.num_sms);
            LAUNCH(KK_BASE, (k_base_rec<2><<<grid, KREC_THREADS, RecBase<2>::smem, st>>>(d_queues, counts[0], data)));
        }
        if (counts[1]) {
            const u32 grid = std::min<u32>(counts[1], 4u * g_ws.num_sms);
            LAUNCH(KK_BASE, (k_base_rec<4><<<grid, KREC_THREADS, RecBase<4>::smem, st>>>(d_queues + QCAP, counts[1],
                                                                                         data)));
        }
        g_stats.base_tasks += counts[0] + counts[1];
        return IPS4O_OK;
    } else {
        if (!(counts[0] | counts[1] | counts[2] | counts[3])) return IPS4O_OK;
        // the class-3 count lives on the device: the cell kernels append their fallbacks
        memcpy(g_ws.h_ctr + CTR_BASE0 + 3, counts + 3, 4);
        CK(cudaMemcpyAsync(g_ws.ctr + CTR_BASE0 + 3, g_ws.h_ctr + CTR_BASE0 + 3, 4, cudaMemcpyHostToDevice, st));
        // the size classes touch disjoint leaves: each runs on its own side stream, so that
        // one class's tail overlaps the others' work (fork / join through events)
        // (serialised while the per-launch profiling events are on: they time each kernel
        // alone)
        cudaStream_t ss[4] = {st, st, st, st};
        const bool conc = IPS4O_BASE_STREAMS && !g_prof.on;
        if (conc) {
            CK(side_streams_ready());
            CK(cudaEventRecord(g_ws.ev_fork, st));
            for (int c = 0; c < 4; ++c) {
                ss[c] = g_ws.side[c];
                CK(cudaStreamWaitEvent(ss[c], g_ws.ev_fork, 0));
            }
        }
        int rc = run_cell_class<TR, CellCfg<TR>::NT0, CellCfg<TR>::E0>(data, counts[0], d_queues, ss[0]);
        if (!rc) rc = run_cell_class<TR, CellCfg<TR>::NT1, CellCfg<TR>::E1>(data, counts[1], d_queues + QCAP, ss[1]);
        if (!rc) rc = run_cell_class<TR, CellCfg<TR>::NT2, CellCfg<TR>::E2>(data, counts[2], d_queues + 2 * QCAP, ss[2]);
        if (rc) return rc;
#ifdef IPS4O_BASE_PROF
        {
            static unsigned long long h[2][8], z[2][8];
            cudaStreamSynchronize(st);
            cudaMemcpyFromSymbol(h, g_base_prof, sizeof h);
            cudaMemcpyToSymbol(g_base_prof, z, sizeof z);
            static const char* nm[8] = {"wb+top", "load+mm", "range", "rank", "sum", "scan+chk", "scatter", "fix"};
            for (int c = 0; c < 2; ++c) {
                unsigned long long t = 0;
                for (int i = 0; i < 8; ++i) t += h[c][i];
                if (!t) continue;
                fprintf(stderr, "base prof class %s:", c ? "NT>=512" : "NT<512");
                for (int i = 0; i < 8; ++i) fprintf(stderr, " %s %.1f%%", nm[i], 100.0 * h[c][i] / t);
                fprintf(stderr, "\n");
            }
        }
#endif
        // class 3 (8193..16384 elements, 8-byte types) by the cell kernel with 1024 threads;
        // the merge sort then takes only the leaves the cell kernels handed back (appended
        // to the class-3 queue after the level's own class-3 tasks)
        u32 mstart = 0;
        if constexpr (TR::CAP >= 16384) {
            rc = run_cell_class<TR, 1024, 16>(data, counts[3], d_queues + 3 * QCAP, ss[3]);
            if (rc) return rc;
            mstart = counts[3];
        }
        if (conc) {
            for (int c = 0; c < 4; ++c) {
                CK(cudaEventRecord(g_ws.ev_join[c], ss[c]));
                CK(cudaStreamWaitEvent(st, g_ws.ev_join[c], 0));
            }
        }
        constexpr int TH = TR::CAP >= 16384 ? 1024 : 512;
        typedef BaseClass<TR, TH, 16> BC;
        const u32 grid = 2u * g_ws.num_sms;
        LAUNCH(KK_BASE, (k_base_merge<TR, TH, 16><<<grid, TH, BC::smem, st>>>(d_queues + 3 * QCAP, mstart,
                                                                              g_ws.ctr + CTR_BASE0 + 3, data)));
        if (TR::CAP < 16384) g_stats.base_tasks += counts[3];
        return IPS4O_OK;
    }
}

template <class TR>
static int sort_impl(void* data, u64 n, cudaStream_t st) {
    int rc = ensure_ws(n, TR::S);
    if (rc) return rc;
    rc = prepare_kernels<TR>();
    if (rc) return rc;
    g_stats.aux_bytes = fixed_bytes() + align_up(spill_bound_elems(n, TR::S) * TR::S, 256);
    if (n <= (u64)TR::CAP) {
        g_stats.base_elements += n;
        const u32 c = base_class(n, TR::C0MAX, TR::C1MAX);
        g_ws.h_q[0] = TaskDesc{0, n, 0u, 0u};
        CK(cudaMemcpyAsync(g_ws.q_base + (size_t)c * QCAP, g_ws.h_q, sizeof(TaskDesc),
                           cudaMemcpyHostToDevice, st));
        u32 counts[NUM_BASE_CLASSES] = {0, 0, 0, 0};
        counts[c] = 1;
        return run_base<TR>(data, counts, g_ws.q_base, st);
    }
    std::vector<TaskDesc> cur(1, TaskDesc{0, n, 0u, 0u}), next;
    u64 seed = 0x1234567ull;
    while (!cur.empty()) {
        g_stats.levels++;
        next.clear();
        // largest tasks first; batches of <= MAXT tasks and <= MAXS stripes
        std::sort(cur.begin(), cur.end(),
                  [](const TaskDesc& a, const TaskDesc& b) { return a.hi - a.lo > b.hi - b.lo; });
        u64 Ntot = 0;
        for (auto& t : cur) Ntot += t.hi - t.lo;
        const u64 Lst = stripe_len<TR>(Ntot);
        size_t i0 = 0;
        while (i0 < cur.size()) {
            size_t i1 = i0;
            u32 sacc = 0;
            while (i1 < cur.size() && i1 - i0 < MAXT) {
                u32 s = stripes_for(cur[i1].hi - cur[i1].lo, Lst);
                if (sacc + s > MAXS && i1 > i0) break;
                sacc += s;
                ++i1;
            }
            const u32 T = (u32)(i1 - i0);
            u32 S = 0;
            plan_batch<TR>(&cur[i0], T, (uintptr_t)data, Lst, &S);
            if (S > MAXS) {
                snprintf(g_errbuf, sizeof g_errbuf, "stripe planning overflow");
                return IPS4O_EINTERNAL;
            }
            seed = mix64(seed);
            rc = run_level<TR>(data, T, S, st, false, 0, 0, 1, seed);
            if (rc) return rc;
            g_stats.distribution_tasks += T;
            for (u32 q = 0; q < T; ++q) g_stats.distributed_elements += cur[i0 + q].hi - cur[i0 + q].lo;
            const u32 nn = g_ws.h_ctr[CTR_NEXT];
            rc = run_base<TR>(data, g_ws.h_ctr + CTR_BASE0, g_ws.q_base, st);
            if (rc) return rc;
            if (nn > Q_SPEC) {
                CK(cudaMemcpyAsync(g_ws.h_q, g_ws.q_next, nn * sizeof(TaskDesc), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
            }
            if (nn) next.insert(next.end(), g_ws.h_q, g_ws.h_q + nn);
            i0 = i1;
        }
        cur.swap(next);
    }
    return IPS4O_OK;
}

static int type_size(int t) {
    switch (t) {
        case IPS4O_U64: return 8;
        case IPS4O_F64: return 8;
        case IPS4O_PAIR_U64: return 16;
        case IPS4O_REC100_K10: return 100;
        default: return 0;
    }
}

static int check_args(const void* p, u64 n, int type) {
    if (type_size(type) == 0) {
        snprintf(g_errbuf, sizeof g_errbuf, "unknown element type %d", type);
        return IPS4O_EINVAL;
    }
    if (n >= (1ull << 40)) {
        snprintf(g_errbuf, sizeof g_errbuf, "n too large");
        return IPS4O_EINVAL;
    }
    if (n > 0 && !p) {
        snprintf(g_errbuf, sizeof g_errbuf, "null data pointer");
        return IPS4O_EINVAL;
    }
    const uintptr_t a = (uintptr_t)p;
    const int need = type == IPS4O_PAIR_U64 ? 16 : type == IPS4O_REC100_K10 ? 4 : 8;
    if (n > 0 && (a % need)) {
        snprintf(g_errbuf, sizeof g_errbuf, "data pointer not %d-byte aligned", need);
        return IPS4O_EALIGN;
    }
    return IPS4O_OK;
}

template <class TR>
static int splitters_to_keys(const void* h, u32 nspl, std::vector<u64>& out) {
    out.resize(nspl);
    if (TR::TYPE == 1) {
        for (u32 i = 0; i < nspl; ++i) {
            u64 bits;
            memcpy(&bits, (const char*)h + 8 * i, 8);
            out[i] = TF64::key(bits);
        }
    } else {
        memcpy(out.data(), h, 8ull * nspl);
    }
    for (u32 i = 1; i < nspl; ++i)
        if (!(out[i - 1] < out[i])) return IPS4O_EINVAL;
    return IPS4O_OK;
}

template <class TR>
static int debug_classify_impl(const void* d_in, u64 n, const void* h_spl, u32 nspl, int eq,
                               u32* d_out, cudaStream_t st) {
    int rc = ensure_ws(n, TR::S);
    if (rc) return rc;
    std::vector<u64> keys;
    if (splitters_to_keys<TR>(h_spl, nspl, keys)) {
        snprintf(g_errbuf, sizeof g_errbuf, "splitters must be strictly increasing");
        return IPS4O_EINVAL;
    }
    CK(cudaMemcpyAsync(g_ws.dsplit, keys.data(), 8ull * nspl, cudaMemcpyHostToDevice, st));
    LevelArgs A = level_args<TR>(const_cast<void*>(d_in), 1, 0, 0, 0);
    LAUNCH(KK_OTHER, (k_tree_from_splitters<<<1, 256, 0, st>>>(A, g_ws.dsplit, nspl, (u32)eq)));
    if (n) {
        const u32 grid = (u32)std::min<u64>((n + 255) / 256, 4096);
        LAUNCH(KK_OTHER, (k_debug_classify<TR><<<grid, 256, 0, st>>>(d_in, n, g_ws.tree, g_ws.spl,
                                                                      g_ws.tp, d_out)));
    }
    return IPS4O_OK;
}

template <class TR>
static int debug_partition_impl(void* d, u64 n, const void* h_spl, u32 nspl, int eq, u64* h_bnd,
                                u32* K_out, cudaStream_t st) {
    int rc = ensure_ws(n, TR::S);
    if (rc) return rc;
    rc = prepare_kernels<TR>();
    if (rc) return rc;
    std::vector<u64> keys;
    if (splitters_to_keys<TR>(h_spl, nspl, keys)) {
        snprintf(g_errbuf, sizeof g_errbuf, "splitters must be strictly increasing");
        return IPS4O_EINVAL;
    }
    CK(cudaMemcpyAsync(g_ws.dsplit, keys.data(), 8ull * nspl, cudaMemcpyHostToDevice, st));
    TaskDesc td{0, n, 0u, 0u};
    u32 S = 0;
    plan_batch<TR>(&td, 1, (uintptr_t)d, stripe_len<TR>(n), &S);
    rc = run_level<TR>(d, 1, S, st, true, nspl, (u32)eq, 0, 1);
    if (rc) return rc;
    g_stats.levels = 1;
    g_stats.distribution_tasks = 1;
    CK(cudaMemcpyAsync(h_bnd, g_ws.bnd, (MAXK + 1) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    u32 kp = 2;
    while (kp < nspl + 1) kp <<= 1;
    *K_out = eq ? 2 * kp - 1 : kp;
    return IPS4O_OK;
}

}  // namespace ips4o

using namespace ips4o;

extern "C" {

int ips4o_sort(void* d_data, uint64_t n, int elem_type, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = check_args(d_data, n, elem_type);
    if (rc) return rc;
    memset(&g_stats, 0, sizeof g_stats);
    g_stats.n = n;
    g_stats.elem_type = (uint32_t)elem_type;
    if (n <= 1) return IPS4O_OK;
    cudaStream_t st = (cudaStream_t)stream;
    switch (elem_type) {
        case IPS4O_U64: return sort_impl<TU64>(d_data, n, st);
        case IPS4O_F64: return sort_impl<TF64>(d_data, n, st);
        case IPS4O_PAIR_U64: return sort_impl<TPair>(d_data, n, st);
        case IPS4O_REC100_K10: return sort_impl<TRec>(d_data, n, st);
        default: return IPS4O_EINVAL;
    }
}

int ips4o_sort_host(void* h_data, uint64_t n, int elem_type, void* stream) {
    static void* d_stage = nullptr;
    static size_t stage_bytes = 0;
    static int stage_dev = -1;
    const int s = type_size(elem_type);
    if (!s || (n > 0 && !h_data)) return IPS4O_EINVAL;
    if (n <= 1) return IPS4O_OK;
    const size_t bytes = (size_t)n * s;
    cudaStream_t st = (cudaStream_t)stream;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int dev = 0;
        CK(cudaGetDevice(&dev));
        if (d_stage && (stage_bytes < bytes || stage_dev != dev)) {
            cudaFree(d_stage);
            d_stage = nullptr;
        }
        if (!d_stage) {
            if (cudaMalloc(&d_stage, bytes) != cudaSuccess) {
                cudaGetLastError();
                return IPS4O_ENOMEM;
            }
            stage_bytes = bytes;
            stage_dev = dev;
        }
        CK(cudaMemcpyAsync(d_stage, h_data, bytes, cudaMemcpyHostToDevice, st));
    }
    int rc = ips4o_sort(d_stage, n, elem_type, stream);
    if (rc) return rc;
    CK(cudaMemcpyAsync(h_data, d_stage, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return IPS4O_OK;
}

}  // extern "C"

namespace ips4o {
// SoA <-> staging records {key image, value}; f64 keys through the order-preserving map
// (and back: the map is a bijection on the non-NaN, non -0.0 doubles)
__global__ void k_kv_gather(const u64* keys, const u64* vals, ulonglong2* out, u64 n, int f64) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 k = keys[i];
        out[i] = make_ulonglong2(f64 ? TF64::key(k) : k, vals[i]);
    }
}
__global__ void k_kv_scatter(const ulonglong2* in, u64* keys, u64* vals, u64 n, int f64) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const ulonglong2 p = in[i];
        keys[i] = f64 ? ((p.x >> 63) ? (p.x & 0x7FFFFFFFFFFFFFFFull) : ~p.x) : p.x;
        vals[i] = p.y;
    }
}
static void* g_kv_stage = nullptr;
static size_t g_kv_bytes = 0;
static int g_kv_dev = -1;
}  // namespace ips4o

extern "C" {

int ips4o_sort_kv(uint64_t* d_keys, uint64_t* d_vals, uint64_t n, int key_type, void* stream) {
    if (key_type != IPS4O_U64 && key_type != IPS4O_F64) {
        snprintf(g_errbuf, sizeof g_errbuf, "sort_kv: key type must be u64 or f64");
        return IPS4O_EINVAL;
    }
    if (n > 0 && (!d_keys || !d_vals)) {
        snprintf(g_errbuf, sizeof g_errbuf, "sort_kv: null pointer");
        return IPS4O_EINVAL;
    }
    if (n >= (1ull << 40)) return IPS4O_EINVAL;
    if ((((uintptr_t)d_keys) | ((uintptr_t)d_vals)) & 7u) return IPS4O_EALIGN;
    if (n <= 1) return IPS4O_OK;
    cudaStream_t st = (cudaStream_t)stream;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int dev = 0;
        CK(cudaGetDevice(&dev));
        const size_t need = (size_t)n * 16;
        if (g_kv_stage && (g_kv_bytes < need || g_kv_dev != dev)) {
            cudaFree(g_kv_stage);
            g_kv_stage = nullptr;
        }
        if (!g_kv_stage) {
            if (cudaMalloc(&g_kv_stage, need) != cudaSuccess) {
                cudaGetLastError();
                snprintf(g_errbuf, sizeof g_errbuf, "sort_kv: staging allocation of %zu bytes failed", need);
                return IPS4O_ENOMEM;
            }
            g_kv_bytes = need;
            g_kv_dev = dev;
        }
        const u32 grid = (u32)std::min<u64>((n + 255) / 256, 4096);
        k_kv_gather<<<grid, 256, 0, st>>>((const u64*)d_keys, (const u64*)d_vals, (ulonglong2*)g_kv_stage, n, key_type == IPS4O_F64);
        CK(cudaGetLastError());
    }
    int rc = ips4o_sort(g_kv_stage, n, IPS4O_PAIR_U64, stream);
    if (rc) return rc;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        const u32 grid = (u32)std::min<u64>((n + 255) / 256, 4096);
        k_kv_scatter<<<grid, 256, 0, st>>>((const ulonglong2*)g_kv_stage, (u64*)d_keys, (u64*)d_vals, n, key_type == IPS4O_F64);
        CK(cudaGetLastError());
        g_stats.elem_type = (uint32_t)key_type;
    }
    return IPS4O_OK;
}

size_t ips4o_aux_bytes(uint64_t n, int elem_type) {
    const int s = type_size(elem_type);
    if (!s) return 0;
    return fixed_bytes() + align_up(spill_bound_elems(n, s) * s, 256);
}

int ips4o_last_stats(ips4o_stats* out) {
    if (!out) return IPS4O_EINVAL;
    *out = g_stats;
    return IPS4O_OK;
}

const char* ips4o_error_string(int status) {
    switch (status) {
        case IPS4O_OK: return "ok";
        case IPS4O_EINVAL: return g_errbuf[0] ? g_errbuf : "invalid argument";
        case IPS4O_EALIGN: return g_errbuf[0] ? g_errbuf : "misaligned pointer";
        case IPS4O_ENOMEM: return g_errbuf[0] ? g_errbuf : "out of device memory";
        case IPS4O_ECUDA: return g_errbuf[0] ? g_errbuf : "CUDA error";
        case IPS4O_EINTERNAL: return g_errbuf[0] ? g_errbuf : "internal consistency check failed";
        default: return "unknown status";
    }
}

int ips4o_release_workspace(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_kv_stage) cudaFree(g_kv_stage);
    g_kv_stage = nullptr;
    g_kv_bytes = 0;
    if (g_ws.dev) cudaFree(g_ws.dev);
    g_ws.dev = nullptr;
    g_ws.dev_bytes = 0;
    g_ws.device = -1;
    if (g_ws.side_ready) {
        for (int c = 0; c < 4; ++c) {
            cudaStreamDestroy(g_ws.side[c]);
            cudaEventDestroy(g_ws.ev_join[c]);
        }
        cudaEventDestroy(g_ws.ev_fork);
        g_ws.side_ready = false;
    }
    return IPS4O_OK;
}

int ips4o_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_prof.on = on != 0;
    return IPS4O_OK;
}

int ips4o_profile_read(uint64_t* launches, double* ms) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (int k = 0; k < IPS4O_NUM_KERNEL_KINDS; ++k) {
        if (launches) launches[k] = 0;
        if (ms) ms[k] = 0;
    }
    for (auto& r : g_prof.recs) {
        cudaEventSynchronize(r.b);
        float t = 0;
        cudaEventElapsedTime(&t, r.a, r.b);
        if (launches) launches[r.kind]++;
        if (ms) ms[r.kind] += t;
        g_prof.pool.push_back(r.a);
        g_prof.pool.push_back(r.b);
    }
    g_prof.recs.clear();
    return IPS4O_OK;
}

const char* ips4o_kernel_kind_name(int kind) {
    if (kind < 0 || kind >= IPS4O_NUM_KERNEL_KINDS) return "unknown";
    return kKindNames[kind];
}

int ips4o_debug_classify(const void* d_in, uint64_t n, int elem_type, const void* h_splitters,
                         uint32_t nspl, int eq, uint32_t* d_bucket_out, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = check_args(d_in, n, elem_type);
    if (rc) return rc;
    if (!h_splitters || nspl < 1 || nspl > 255 || (eq && nspl > 127) || (n && !d_bucket_out))
        return IPS4O_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    switch (elem_type) {
        case IPS4O_U64: return debug_classify_impl<TU64>(d_in, n, h_splitters, nspl, eq, d_bucket_out, st);
        case IPS4O_F64: return debug_classify_impl<TF64>(d_in, n, h_splitters, nspl, eq, d_bucket_out, st);
        case IPS4O_PAIR_U64:
            return debug_classify_impl<TPair>(d_in, n, h_splitters, nspl, eq, d_bucket_out, st);
        case IPS4O_REC100_K10:
            return debug_classify_impl<TRec>(d_in, n, h_splitters, nspl, eq, d_bucket_out, st);
        default: return IPS4O_EINVAL;
    }
}

int ips4o_debug_partition_once(void* d_data, uint64_t n, int elem_type, const void* h_splitters,
                               uint32_t nspl, int eq, uint64_t* h_bounds_out, uint32_t* K_out,
                               void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = check_args(d_data, n, elem_type);
    if (rc) return rc;
    if (!h_splitters || nspl < 1 || nspl > 255 || (eq && nspl > 127) || n < 64 || !h_bounds_out ||
        !K_out)
        return IPS4O_EINVAL;
    memset(&g_stats, 0, sizeof g_stats);
    g_stats.n = n;
    g_stats.elem_type = (uint32_t)elem_type;
    cudaStream_t st = (cudaStream_t)stream;
    switch (elem_type) {
        case IPS4O_U64:
            return debug_partition_impl<TU64>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st);
        case IPS4O_F64:
            return debug_partition_impl<TF64>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st);
        case IPS4O_PAIR_U64:
            return debug_partition_impl<TPair>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st);
        case IPS4O_REC100_K10:
            return debug_partition_impl<TRec>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st);
        default: return IPS4O_EINVAL;
    }
}

}  // extern "C"
