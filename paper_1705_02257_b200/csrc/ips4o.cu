// ips4o.cu -- libips4o.so: workspace, the CUDA graph of the device-side level loop, and the
// C ABI of include/ips4o.h.  The host only enqueues: one k_init launch (the call's parameters
// as kernel arguments) and one graph launch whose while-loop runs the recursion on the device
// (k_sched.cuh).  Every step of the sort runs in the kernels of k_*.cuh.
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
#include "k_cta.cuh"
#include "k_permute.cuh"
#include "k_sample.cuh"
#include "k_sched.cuh"

namespace ips4o {

static_assert(MAXS <= (u32)K4_MAXSTRIPES && MAXS <= (u32)K2P_MAXST, "per-task stripe tables in shared memory");

static std::mutex g_mu;
static char g_errbuf[512];
static ips4o_stats g_stats;  // host-side fields of the last call (the rest comes from the device)

enum KernelKind { KK_SAMPLE = 0, KK_CLASSIFY, KK_PREPARE, KK_MOVES, KK_PERMUTE, KK_CLEANUP, KK_BASE, KK_OTHER, KK_MEDIUM };
static const char* kKindNames[IPS4O_NUM_KERNEL_KINDS] = {
    "sample_splitters", "classify_flush", "prepare", "empty_block_moves",
    "block_permute",    "cleanup",        "base_case", "other",             "medium_cta"};
constexpr u32 STAMP_BEGIN = 255;
constexpr u32 PLOG_CAP = 1u << 12;

// ------------------------------------------------------------------ workspace

// Capacities of a workspace, derived from n and the element type (every bound is a
// property of the planner, see ips4o_aux_bytes in include/ips4o.h).
struct Caps {
    u32 tcap = 1, scap = 1;      // tasks / stripes per batch
    u32 qb_cap[4] = {1, 1, 1, 1};  // base-case queue per size class
    u32 q_fb = 1;                // fallback queue
    u32 qn = 1;                  // level queue
    u32 qm = 1;                  // medium queue (single-CTA tier)
    u64 spill = 64;              // spilled partial-buffer elements
    int esize = 8;
};

template <class TR>
static Caps caps_for(u64 n) {
    Caps c;
    c.esize = TR::S;
    const u64 CAPB = TR::CAP;
    // a batch's tasks each hold > CAP elements (the debug step: one task)
    c.tcap = (u32)std::min<u64>(MAXT, n / (CAPB + 1) + 1);
    // stripes of a task: <= m/L + 1.5 with L >= MIN_STRIPE (k_plan)
    c.scap = (u32)std::min<u64>(MAXS, 2ull * c.tcap + n / MIN_STRIPE + 8);
    // base tasks of one batch: <= tcap*256 buckets, and <= n / (smallest size of the class)
    const u64 minsz[4] = {2, (u64)TR::C0MAX + 1, (u64)TR::C1MAX + 1, (u64)TR::C2MAX + 1};
    u64 tot = 0;
    for (int k = 0; k < 4; ++k) {
        const u64 q = std::min<u64>((u64)c.tcap * MAXK, n / minsz[k] + 1);
        c.qb_cap[k] = (u32)std::max<u64>(1, q);
        tot += c.qb_cap[k];
    }
    c.q_fb = (u32)tot;
    // next-level tasks hold > CAP elements each
    c.qn = (u32)(n / (CAPB + 1) + 2);
    // medium tasks of one batch (single-CTA tier): > CAP elements each
    c.qm = TR::WIDE ? 1u : (u32)std::min<u64>((u64)c.tcap * MAXK, n / (CAPB + 1) + 2);
    // Spill (the partially filled buffers of every stripe): a stripe spills at most
    // min(its length, K*(b-1)) elements.  Multi-stripe tasks have stripes >= 2^16 elements
    // (one quarter-length last stripe), single-stripe tasks an adaptive K < 4*m/LEAF
    // (PAPER.md:404-407), so the spill never exceeds n/2 (+ one stripe's worth).
    const u64 per_stripe = (u64)MAXK * (TR::B - 1);
    c.spill = std::min<u64>(std::min<u64>(n + 64, n / 2 + per_stripe + 64), (u64)c.scap * per_stripe + 64);
    return c;
}

struct Layout {
    size_t tp, sd, order, tree, s_count, s_small, bnd, dblk, nfb, btot, lut, done, tdone, wr, ovf, ovf_owner,
        qbase, qfb, qlvl, qmed, ctr, dsplit, dyn, sched, dstats, plog, spill, total;
};
static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
static Layout layout_of(const Caps& c) {
    Layout L;
    size_t s = 0;
    auto add = [&](size_t b) {
        const size_t r = s;
        s += align_up(b, 256);
        return r;
    };
    const size_t T = c.tcap, S = c.scap;
    L.tp = add(T * sizeof(TaskParam));
    L.sd = add(S * sizeof(StripeDesc));
    L.order = add(S * 4);
    L.tree = add(T * MAXK * 8 * 2);            // tree, spl
    L.s_count = add(S * MAXK * 4 * 3);         // s_count, s_fill, s_spoff
    L.s_small = add(S * 8 + S * 4 * 3);        // s_spbase, s_nfull, prefF, prefE
    L.bnd = add(T * (MAXK + 1) * 8);
    L.dblk = add(T * (MAXK + 1) * 4 * 2);      // dblk, mov
    L.nfb = add(T * MAXK * 4 * 2);             // nfb, cflag
    L.btot = add(T * MAXK * 8);
    L.lut = add(T * LUT_STRIDE * 2);
    L.done = add(T * (MAXK / 32) * 4);
    L.tdone = add((T + 31) / 32 * 4 + 64);
    L.wr = add(T * MAXK * 8 * CTL_STRIDE);
    L.ovf = add(T * 512);                      // one overflow block per task (<= 512 B)
    L.ovf_owner = add(T * 4);
    size_t qb = 0;
    for (int k = 0; k < 4; ++k) qb += c.qb_cap[k];
    L.qbase = add(qb * sizeof(TaskDesc));
    L.qfb = add((size_t)c.q_fb * sizeof(TaskDesc));
    L.qlvl = add((size_t)c.qn * sizeof(TaskDesc) * 2);
    L.qmed = add((size_t)c.qm * sizeof(TaskDesc));
    L.ctr = add(CTR_N * 4 + 16);
    L.dsplit = add(MAXK * 8);
    L.dyn = add(sizeof(LevelDyn));
    L.sched = add(sizeof(Sched));
    L.dstats = add(DS_N * 8);
    L.plog = add((size_t)PLOG_CAP * 12 + 16);
    L.spill = add((size_t)c.spill * c.esize);
    L.total = s;
    return L;
}

struct GraphCache {
    cudaGraphExec_t exec = nullptr;
    u32 nodes_per_iter = 0;
    bool valid = false;
};

struct Workspace {
    int device = -1;
    int num_sms = 0;
    char* dev = nullptr;
    size_t dev_bytes = 0;
    int type = -1;               // element type the capacities / kernels are set up for
    Caps caps;
    Layout lay;
    u64 gen = 0;                 // bumps on every (re)allocation: cached graphs are rebuilt
    cudaStream_t cap_stream = nullptr;   // graph-building capture stream
    cudaStream_t side[5];        // base-case size classes and the single-CTA tier run as parallel graph branches
    cudaEvent_t ev_fork, ev_join[5];
    cudaEvent_t ev_done;         // recorded after every call: the workspace is free again
    bool have_done = false;
    bool last_captured = false;
    cudaStream_t last_stream = nullptr;
    bool streams_ready = false;
    u32 k2_blocks = 0, k3_blocks = 0, k3t_blocks = 0, k4w_blocks = 0, k4c_blocks = 0;
    u32 cell_grid[5] = {0, 0, 0, 0, 0};
    int kernels_type = -1;
    GraphCache graphs[8][2];     // [type][profile]
    u64 graphs_gen = 0;
    LevelArgs A;                 // static fields (workspace pointers, capacities)
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

static void drop_graphs() {
    for (auto& row : g_ws.graphs)
        for (auto& gc : row) {
            if (gc.exec) cudaGraphExecDestroy(gc.exec);
            gc = GraphCache();
        }
}

static int ensure_streams() {
    if (g_ws.streams_ready) return IPS4O_OK;
    CK(cudaStreamCreateWithFlags(&g_ws.cap_stream, cudaStreamNonBlocking));
    for (int c = 0; c < 5; ++c) {
        CK(cudaStreamCreateWithFlags(&g_ws.side[c], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&g_ws.ev_join[c], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&g_ws.ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g_ws.ev_done, cudaEventDisableTiming));
    g_ws.streams_ready = true;
    return IPS4O_OK;
}

static void release_all() {
    drop_graphs();
    if (g_ws.dev) cudaFree(g_ws.dev);
    g_ws.dev = nullptr;
    g_ws.dev_bytes = 0;
    g_ws.type = -1;
    g_ws.kernels_type = -1;
    if (g_ws.streams_ready) {
        cudaStreamDestroy(g_ws.cap_stream);
        for (int c = 0; c < 5; ++c) {
            cudaStreamDestroy(g_ws.side[c]);
            cudaEventDestroy(g_ws.ev_join[c]);
        }
        cudaEventDestroy(g_ws.ev_fork);
        cudaEventDestroy(g_ws.ev_done);
        g_ws.streams_ready = false;
    }
    g_ws.have_done = false;
    g_ws.device = -1;
}

static bool caps_cover(const Caps& have, const Caps& need) {
    if (have.esize != need.esize || have.tcap < need.tcap || have.scap < need.scap || have.q_fb < need.q_fb ||
        have.qn < need.qn || have.qm < need.qm || have.spill < need.spill)
        return false;
    for (int k = 0; k < 4; ++k)
        if (have.qb_cap[k] < need.qb_cap[k]) return false;
    return true;
}

// Tasks of (base capacity, medium_max] elements go to the single-CTA tier (k_cta.cuh);
// IPS4O_MEDIUM_MAX (environment, read once) sets it, 0 = no tier.  The default is 0: on B200 one
// CTA per subproblem sorts 3-10x slower per SM than the multi-CTA levels plus the multi-CTA-per-SM
// base case (measured), so the tier is an opt-in mode (the strictly in-place driver
// of PAPER.md:381-395).
#ifndef IPS4O_MEDIUM_MAX
#define IPS4O_MEDIUM_MAX 0ull
#endif
static u64 medium_max() {
    static long long v = -1;
    if (v < 0) {
        const char* e = getenv("IPS4O_MEDIUM_MAX");
        v = e ? atoll(e) : (long long)IPS4O_MEDIUM_MAX;
        if (v < 0) v = 0;
    }
    return (u64)v;
}

// Levels >= 2 run in L2-sized waves: a batch holds at most IPS4O_WAVE elements (environment, read
// once; 0 = off), so that a wave's blocks, written by K2 and K3, are still in L2 when K3 and the
// base case read them (§4.7: the last level sorted while the buckets are in
// cache).  IPS4O_WAVE_STRIPE: minimum stripe length inside a wave.
#ifndef IPS4O_WAVE
#define IPS4O_WAVE 0ll
#endif
#ifndef IPS4O_WAVE_STRIPE
#define IPS4O_WAVE_STRIPE 16384ll
#endif
static u64 env_u64(const char* name, long long dflt) {
    const char* e = getenv(name);
    long long v = e ? atoll(e) : dflt;
    return v < 0 ? 0ull : (u64)v;
}
static u64 wave_elems() {
    static u64 v = env_u64("IPS4O_WAVE", IPS4O_WAVE);
    return v;
}
static u64 wave_stripe() {
    static u64 v = env_u64("IPS4O_WAVE_STRIPE", IPS4O_WAVE_STRIPE);
    return v;
}

static void fill_args() {
    char* p = g_ws.dev;
    const Layout& L = g_ws.lay;
    const Caps& c = g_ws.caps;
    LevelArgs A;
    memset(&A, 0, sizeof A);
    const size_t T = c.tcap, S = c.scap;
    A.tp = (const TaskParam*)(p + L.tp);
    A.sd = (const StripeDesc*)(p + L.sd);
    A.stripe_order = (const u32*)(p + L.order);
    A.tree = (u64*)(p + L.tree);
    A.spl = A.tree + T * MAXK;
    A.s_count = (u32*)(p + L.s_count);
    A.s_fill = A.s_count + S * MAXK;
    A.s_spoff = A.s_fill + S * MAXK;
    A.s_spbase = (u64*)(p + L.s_small);
    A.s_nfull = (u32*)(p + L.s_small + S * 8);
    A.prefF = A.s_nfull + S;
    A.prefE = A.prefF + S;
    A.spill = p + L.spill;
    A.spill_cap = c.spill;
    A.bnd = (u64*)(p + L.bnd);
    A.dblk = (u32*)(p + L.dblk);
    A.mov = A.dblk + T * (MAXK + 1);
    A.nfb = (u32*)(p + L.nfb);
    A.cflag = A.nfb + T * MAXK;
    A.btot = (u64*)(p + L.btot);
    A.lut = (unsigned short*)(p + L.lut);
    A.done = (u32*)(p + L.done);
    A.tdone = (u32*)(p + L.tdone);
    A.wr = (u64*)(p + L.wr);
    A.ovf = p + L.ovf;
    A.ovf_owner = (int*)(p + L.ovf_owner);
    A.q_base = (TaskDesc*)(p + L.qbase);
    u32 off = 0;
    for (int k = 0; k < 4; ++k) {
        A.qb_off[k] = off;
        A.qb_cap[k] = c.qb_cap[k];
        off += c.qb_cap[k];
    }
    A.q_fb = (TaskDesc*)(p + L.qfb);
    A.q_cap = c.q_fb;
    A.q_med = (TaskDesc*)(p + L.qmed);
    A.qm_cap = c.qm;
    A.medium_max = medium_max();
    A.wave_elems = wave_elems();
    A.wave_stripe = std::max<u64>(wave_stripe(), 1024);
    A.q_lvl0 = (TaskDesc*)(p + L.qlvl);
    A.q_lvl1 = A.q_lvl0 + c.qn;
    A.qn_cap = c.qn;
    A.tcap = c.tcap;
    A.scap = c.scap;
    A.ctr = (u32*)(p + L.ctr);
    A.spill_ctr = (u64*)(p + L.ctr + CTR_N * 4);
    A.base_elems = A.spill_ctr + 1;
    A.dsplit = (u64*)(p + L.dsplit);
    A.dyn = (LevelDyn*)(p + L.dyn);
    A.sched = (Sched*)(p + L.sched);
    A.dstats = (u64*)(p + L.dstats);
    A.plog_t = (u64*)(p + L.plog);
    A.plog_k = (u32*)(p + L.plog + (size_t)PLOG_CAP * 8);
    A.plog_n = A.plog_k + PLOG_CAP;
    A.plog_cap = PLOG_CAP;
    g_ws.A = A;
}

// The workspace of the current device, grown to cover n elements of type TR.  Waits for the
// previous call's work on its stream before anything is freed.
template <class TR>
static int ensure_ws(u64 n) {
    int dev;
    CK(cudaGetDevice(&dev));
    if (g_ws.device != dev) {
        if (g_ws.device >= 0) release_all();
        g_ws.device = dev;
        CK(cudaDeviceGetAttribute(&g_ws.num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    int rs = ensure_streams();
    if (rs) return rs;
    Caps need = caps_for<TR>(n);
    if (g_ws.dev && g_ws.type == TR::TYPE && caps_cover(g_ws.caps, need)) {
        g_ws.A.base_cap = TR::CAP;
        return IPS4O_OK;
    }
    if (g_ws.dev && g_ws.caps.esize == need.esize) {
        // grow: keep every capacity at least as large as before
        const Caps& h = g_ws.caps;
        need.tcap = std::max(need.tcap, h.tcap);
        need.scap = std::max(need.scap, h.scap);
        for (int k = 0; k < 4; ++k) need.qb_cap[k] = std::max(need.qb_cap[k], h.qb_cap[k]);
        need.q_fb = std::max(need.q_fb, h.q_fb);
        need.qn = std::max(need.qn, h.qn);
        need.qm = std::max(need.qm, h.qm);
        need.spill = std::max(need.spill, h.spill);
    }
    const Layout L = layout_of(need);
    const bool same_layout = g_ws.dev && caps_cover(need, g_ws.caps) && caps_cover(g_ws.caps, need);
    if (g_ws.dev && g_ws.dev_bytes >= L.total) {
        // the allocation is large enough for the new layout: re-carve it
    } else {
        if (g_ws.dev) {
            if (g_ws.have_done) CK(cudaEventSynchronize(g_ws.ev_done));
            drop_graphs();
            cudaFree(g_ws.dev);
            g_ws.dev = nullptr;
            g_ws.dev_bytes = 0;
        }
        if (cudaMalloc(&g_ws.dev, L.total) != cudaSuccess) {
            cudaGetLastError();
            g_ws.dev = nullptr;
            g_ws.type = -1;
            snprintf(g_errbuf, sizeof g_errbuf, "workspace allocation of %zu bytes failed", L.total);
            return IPS4O_ENOMEM;
        }
        g_ws.dev_bytes = L.total;
    }
    g_ws.type = TR::TYPE;
    g_ws.A.base_cap = TR::CAP;
    if (same_layout) return IPS4O_OK;  // (another element type of the same size: same carve-up)
    if (g_ws.have_done) CK(cudaEventSynchronize(g_ws.ev_done));
    g_ws.caps = need;
    g_ws.lay = L;
    g_ws.gen++;
    fill_args();
    g_ws.A.base_cap = TR::CAP;
    CK(cudaMemset(g_ws.A.plog_n, 0, 4));
    return IPS4O_OK;
}

// ------------------------------------------------------------------ kernels and grids

// cell base-case configurations of the size classes (threads, elements per thread)
// 8 elements per thread (16 in the 8-byte types' largest class), the CTA sized to the class.
#ifndef IPS4O_CELL_E  // elements per thread of the 8-byte types' base-case classes 0-2
#define IPS4O_CELL_E 16
#endif
#ifndef IPS4O_CELL_NT3  // threads of the 8-byte types' largest class (0: the base-case capacity / 16); leaves above its tile: merge sort
#define IPS4O_CELL_NT3 0
#endif
template <class TR> struct CellCfg {
    static constexpr int E0 = TR::S == 8 ? IPS4O_CELL_E : 8, NT0 = (int)TR::C0MAX / E0;
    static constexpr int E1 = TR::S == 8 ? IPS4O_CELL_E : 8, NT1 = (int)TR::C1MAX / E1;
    static constexpr int E2 = TR::S == 8 ? IPS4O_CELL_E : 8, NT2 = (int)TR::C2MAX / E2;
    static constexpr int E3 = TR::S == 8 ? 16 : 8, NT3 = (TR::S == 8 && IPS4O_CELL_NT3) ? IPS4O_CELL_NT3 : (int)TR::CAP / E3;
};
template <class TR>
struct MergeCfg {
    static constexpr int TH = TR::CAP >= 16384 ? 1024 : TR::CAP >= 8192 ? 512 : 256;
    typedef BaseClass<TR, TH, 16> BC;
};
template <class TR, int NT, int E>
static cudaError_t cell_setup(u32* grid, int nsm) {
    typedef CellBase<TR, NT, E> CB;
    cudaError_t e = cudaFuncSetAttribute(k_base_cell<TR, NT, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CB::smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_base_cell<TR, NT, E>, NT, CB::smem);
    *grid = (u32)std::max(1, occ) * (u32)nsm;  // resident CTAs (leaves are taken by ticket)
    return e;
}

// K2 configuration: (threads, elements per thread); 256 buffers of 512 B = 128 KB of shared
// memory: one CTA per SM (640 threads: 20 warps hide more of the barrier and shared-memory
// latency than 16, at 96 registers per thread; two 40 KB stages still fit next to the buffers)
#ifndef IPS4O_K2_NT  // K2 threads per CTA (one CTA per SM)
#define IPS4O_K2_NT 640
#endif
#ifndef IPS4O_K2_EMUL  // K2 elements per thread = 16-byte vectors per thread x elements per vector
#define IPS4O_K2_EMUL 4
#endif
#ifndef IPS4O_K2_MINB  // K2 CTAs per SM the launch bounds aim at
#define IPS4O_K2_MINB 1
#endif
template <class TR> struct K2Cfg { static constexpr int NT = IPS4O_K2_NT, E = 16 / TR::S * IPS4O_K2_EMUL, MINB = IPS4O_K2_MINB; };
constexpr int K4_GRID_PER_SM = 8;

// IPS4O_K3=regs selects the register-buffer permutation (tuning experiments)
static int k3_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IPS4O_K3");
        v = (e && e[0] == 'r') ? 1 : 0;
    }
    return v;
}

template <class TR>
static int prepare_kernels(void) {
    if (g_ws.kernels_type == TR::TYPE) return IPS4O_OK;
    const int nsm = g_ws.num_sms;
    int occ2 = 0, occ3 = 0, occ3t = 0;
    CK(cudaFuncSetAttribute(k_sample<TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1_SMEM));
    if constexpr (TR::WIDE) {
        CK(cudaFuncSetAttribute(k_classify_rec<TR, K2RecRpt<TR>::NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)K2RecSmem<TR, K2RecRpt<TR>::NT>::total));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_classify_rec<TR, K2RecRpt<TR>::NT>, K2RecRpt<TR>::NT,
                                                         K2RecSmem<TR, K2RecRpt<TR>::NT>::total));
        if constexpr (TR::S == 100) {
            CK(cudaFuncSetAttribute(k_base_rec<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RecBase<2>::smem));
            CK(cudaFuncSetAttribute(k_base_rec<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RecBase<4>::smem));
            g_ws.cell_grid[0] = g_ws.cell_grid[1] = 4u * nsm;
        } else {
            CK((cell_setup<TR, CellCfg<TR>::NT0, CellCfg<TR>::E0>(&g_ws.cell_grid[0], nsm)));
            CK((cell_setup<TR, CellCfg<TR>::NT1, CellCfg<TR>::E1>(&g_ws.cell_grid[1], nsm)));
            typedef MergeCfg<TR> M;
            CK(cudaFuncSetAttribute(k_base_merge<TR, M::TH, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)M::BC::smem));
            g_ws.cell_grid[4] = 2u * nsm;
        }
    } else {
        typedef K2Cfg<TR> C;
        CK(cudaFuncSetAttribute(k_classify<TR, C::NT, C::E, C::MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)K2Smem<TR, C::NT, C::E, K2_MAIN_STAGES>::total));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_classify<TR, C::NT, C::E, C::MINB>, C::NT,
                                                         K2Smem<TR, C::NT, C::E, K2_MAIN_STAGES>::total));
        CK((cell_setup<TR, CellCfg<TR>::NT0, CellCfg<TR>::E0>(&g_ws.cell_grid[0], nsm)));
        CK((cell_setup<TR, CellCfg<TR>::NT1, CellCfg<TR>::E1>(&g_ws.cell_grid[1], nsm)));
        CK((cell_setup<TR, CellCfg<TR>::NT2, CellCfg<TR>::E2>(&g_ws.cell_grid[2], nsm)));
        if constexpr (TR::CAP > TR::C2MAX) CK((cell_setup<TR, CellCfg<TR>::NT3, CellCfg<TR>::E3>(&g_ws.cell_grid[3], nsm)));
        typedef MergeCfg<TR> M;
        CK(cudaFuncSetAttribute(k_base_merge<TR, M::TH, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)M::BC::smem));
        if constexpr (FbCell2<TR, M::TH, 16>::on)
            CK(cudaFuncSetAttribute(k_base_fb<TR, M::TH, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)FbCell2<TR, M::TH, 16>::smem));
        g_ws.cell_grid[4] = 2u * nsm;
    }
    if constexpr (!TR::KV) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_permute<TR>, K3_THREADS, 0));
    else occ3 = 1;
    CK(cudaFuncSetAttribute(k_permute_tma<TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3TSmem<TR>::total));
    if constexpr (!TR::WIDE)
        CK(cudaFuncSetAttribute(k_cta_sort<TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CtaCfg<TR>::smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3t, k_permute_tma<TR>, K3T_THREADS, K3TSmem<TR>::total));
    if (occ2 < 1 || occ3 < 1 || occ3t < 1) {
        snprintf(g_errbuf, sizeof g_errbuf, "occupancy query returned %d/%d/%d", occ2, occ3, occ3t);
        return IPS4O_ECUDA;
    }
    g_ws.k2_blocks = (u32)(occ2 * nsm);
    g_ws.k3_blocks = (u32)(occ3 * nsm);
    g_ws.k3t_blocks = (u32)(occ3t * nsm);
    g_ws.k4w_blocks = (u32)(K4_GRID_PER_SM * nsm);
    g_ws.k4c_blocks = (u32)(K4_GRID_PER_SM * nsm);
    g_ws.kernels_type = TR::TYPE;
    return IPS4O_OK;
}

// ------------------------------------------------------------------ enqueueing

struct Enq {
    cudaStream_t st;
    bool prof;
    u32 launches = 0;
};
#define LAUNCH(kind, ...)                                                   \
    do {                                                                    \
        __VA_ARGS__;                                                        \
        cudaError_t e_ = cudaGetLastError();                                \
        if (e_ != cudaSuccess) return set_cuda_error(e_, kKindNames[kind]); \
        q.launches++;                                                       \
    } while (0)
#define STAMP(kind)                                                         \
    do {                                                                    \
        if (q.prof) {                                                       \
            k_stamp<<<1, 32, 0, q.st>>>(A, (u32)(kind));                    \
            CK(cudaGetLastError());                                         \
        }                                                                   \
    } while (0)

// K1..K4 of one batch (the grids are fixed: every kernel reads the batch from LevelDyn)
template <class TR>
static int enqueue_level(Enq& q) {
    const LevelArgs& A = g_ws.A;
    const cudaStream_t st = q.st;
    const u32 T = A.tcap;
    LAUNCH(KK_SAMPLE, (k_sample<TR><<<T, K1_THREADS, K1_SMEM, st>>>(A)));
    STAMP(KK_SAMPLE);
    if constexpr (TR::WIDE) {
        LAUNCH(KK_CLASSIFY, (k_classify_rec<TR, K2RecRpt<TR>::NT><<<g_ws.k2_blocks, K2RecRpt<TR>::NT,
                                                                 K2RecSmem<TR, K2RecRpt<TR>::NT>::total, st>>>(A)));
    } else {
        typedef K2Cfg<TR> C;
        LAUNCH(KK_CLASSIFY, (k_classify<TR, C::NT, C::E, C::MINB><<<g_ws.k2_blocks, C::NT, K2Smem<TR, C::NT, C::E, K2_MAIN_STAGES>::total, st>>>(A)));
    }
    STAMP(KK_CLASSIFY);
    LAUNCH(KK_PREPARE, (k_prepare<TR><<<T, MAXK, 0, st>>>(A)));
    STAMP(KK_PREPARE);
    LAUNCH(KK_MOVES, (k_moves<TR><<<2 * g_ws.num_sms, 256, 0, st>>>(A)));
    STAMP(KK_MOVES);
    if constexpr (!TR::KV) {
        if (k3_variant() == 1) {
            LAUNCH(KK_PERMUTE, (k_permute<TR><<<g_ws.k3_blocks, K3_THREADS, 0, st>>>(A)));
            STAMP(KK_PERMUTE);
            goto k3_done;
        }
    }
    LAUNCH(KK_PERMUTE, (k_permute_tma<TR><<<g_ws.k3t_blocks, K3T_THREADS, K3TSmem<TR>::total, st>>>(A)));
k3_done:
    STAMP(KK_PERMUTE);
    LAUNCH(KK_CLEANUP, (k_cleanup<TR><<<g_ws.k4w_blocks, K4_THREADS, 0, st>>>(A)));
    LAUNCH(KK_CLEANUP, (k_cleanup_cta<TR><<<g_ws.k4c_blocks, K4_THREADS, 0, st>>>(A)));
    STAMP(KK_CLEANUP);
    return IPS4O_OK;
}

template <class TR, int NT, int E>
static int enqueue_cell(Enq& q, cudaStream_t s, u32 c) {
    const LevelArgs& A = g_ws.A;
    typedef CellBase<TR, NT, E> CB;
    LAUNCH(KK_BASE, (k_base_cell<TR, NT, E><<<g_ws.cell_grid[c], NT, CB::smem, s>>>(
                         A.q_base + A.qb_off[c], A.ctr + CTR_BASE0 + c, A.qb_cap[c], A.ctr + CTR_TK0 + c, A.dyn,
                         A.q_fb, A.ctr + CTR_FB, A.q_cap)));
    return IPS4O_OK;
}

// The base case of one batch: the size classes touch disjoint leaves, so each runs on its own
// branch of the graph (fork / join through events; serialised in the profiling graph, where
// each kernel is timed alone); then the merge sort takes the leaves the cell kernels handed
// back (fallback queue).
template <class TR>
static int enqueue_base(Enq& q) {
    const LevelArgs& A = g_ws.A;
    const cudaStream_t st = q.st;
    if constexpr (TR::S == 100) {
        LAUNCH(KK_BASE, (k_base_rec<2><<<g_ws.cell_grid[0], KREC_THREADS, RecBase<2>::smem, st>>>(
                             A.q_base + A.qb_off[0], A.ctr + CTR_BASE0 + 0, A.dyn, A.qb_cap[0])));
        STAMP(KK_BASE);
        LAUNCH(KK_BASE, (k_base_rec<4><<<g_ws.cell_grid[1], KREC_THREADS, RecBase<4>::smem, st>>>(
                             A.q_base + A.qb_off[1], A.ctr + CTR_BASE0 + 1, A.dyn, A.qb_cap[1])));
        STAMP(KK_BASE);
        return IPS4O_OK;
    } else if constexpr (TR::WIDE) {
        // quartets: two cell classes (cells on k0, cells ordered by the lexicographic key), then
        // the merge sort for the leaves they hand back (equal or clustered k0)
        int rc = enqueue_cell<TR, CellCfg<TR>::NT0, CellCfg<TR>::E0>(q, st, 0);
        if (rc) return rc;
        STAMP(KK_BASE);
        rc = enqueue_cell<TR, CellCfg<TR>::NT1, CellCfg<TR>::E1>(q, st, 1);
        if (rc) return rc;
        STAMP(KK_BASE);
        typedef MergeCfg<TR> M;
        LAUNCH(KK_BASE, (k_base_merge<TR, M::TH, 16><<<g_ws.cell_grid[4], M::TH, M::BC::smem, st>>>(
                             A.q_fb, 0u, A.ctr + CTR_FB, A.dyn, A.q_cap)));
        STAMP(KK_BASE);
        return IPS4O_OK;
    } else {
        cudaStream_t ss[5] = {st, st, st, st, st};
        const bool conc = !q.prof;
        if (conc) {
            CK(cudaEventRecord(g_ws.ev_fork, st));
            for (int c = 0; c < 5; ++c) {
                ss[c] = g_ws.side[c];
                CK(cudaStreamWaitEvent(ss[c], g_ws.ev_fork, 0));
            }
        }
        // the single-CTA tier: medium tasks, each sorted completely by one CTA (k_cta.cuh)
        if (A.medium_max) {
            const cudaStream_t s4 = ss[4];
            LAUNCH(KK_MEDIUM, (k_cta_sort<TR><<<g_ws.num_sms, CtaCfg<TR>::NT, CtaCfg<TR>::smem, s4>>>(
                                  A, A.q_med, A.ctr + CTR_MED, A.qm_cap, A.ctr + CTR_MTK)));
            if (q.prof) STAMP(KK_MEDIUM);
        }
        int rc = enqueue_cell<TR, CellCfg<TR>::NT0, CellCfg<TR>::E0>(q, ss[0], 0);
        if (rc) return rc;
        STAMP(KK_BASE);
        rc = enqueue_cell<TR, CellCfg<TR>::NT1, CellCfg<TR>::E1>(q, ss[1], 1);
        if (rc) return rc;
        STAMP(KK_BASE);
        rc = enqueue_cell<TR, CellCfg<TR>::NT2, CellCfg<TR>::E2>(q, ss[2], 2);
        if (rc) return rc;
        STAMP(KK_BASE);
        if constexpr (TR::CAP > TR::C2MAX) {
            rc = enqueue_cell<TR, CellCfg<TR>::NT3, CellCfg<TR>::E3>(q, ss[3], 3);
            if (rc) return rc;
            STAMP(KK_BASE);
        }
        if (conc) {
            for (int c = 0; c < 5; ++c) {
                CK(cudaEventRecord(g_ws.ev_join[c], ss[c]));
                CK(cudaStreamWaitEvent(st, g_ws.ev_join[c], 0));
            }
        }
        typedef MergeCfg<TR> M;
        if constexpr (FbCell2<TR, M::TH, 16>::on) {
            LAUNCH(KK_BASE, (k_base_fb<TR, M::TH, 16><<<g_ws.cell_grid[4], M::TH, FbCell2<TR, M::TH, 16>::smem, st>>>(
                                 A.q_fb, 0u, A.ctr + CTR_FB, A.dyn, A.q_cap)));
        } else {
            LAUNCH(KK_BASE, (k_base_merge<TR, M::TH, 16><<<g_ws.cell_grid[4], M::TH, M::BC::smem, st>>>(
                                 A.q_fb, 0u, A.ctr + CTR_FB, A.dyn, A.q_cap)));
        }
        STAMP(KK_BASE);
        return IPS4O_OK;
    }
}

// One iteration of the level loop: plan, K1..K4, base case, epilogue (sets the condition;
// eager mode: no handle, the host reads LevelDyn::more).
template <class TR>
static int enqueue_body(Enq& q, cudaGraphConditionalHandle h, u32 use_handle = 1u) {
    const LevelArgs& A = g_ws.A;
    STAMP(STAMP_BEGIN);
    LAUNCH(KK_OTHER, (k_plan<TR><<<1, PLAN_THREADS, 0, q.st>>>(A, (u32)g_ws.num_sms)));
    STAMP(KK_OTHER);
    int rc = enqueue_level<TR>(q);
    if (rc) return rc;
    rc = enqueue_base<TR>(q);
    if (rc) return rc;
    LAUNCH(KK_OTHER, (k_epi<<<1, 32, 0, q.st>>>(A, h, use_handle)));
    STAMP(KK_OTHER);
    return IPS4O_OK;
}

// Adds the level loop -- a while-conditional node whose body is captured from enqueue_body --
// to graph g after deps.  Returns the node and the body's kernel count.
template <class TR>
static int add_loop_node(cudaGraph_t g, const cudaGraphNode_t* deps, size_t ndeps, bool prof, cudaGraphNode_t* out,
                         u32* nodes) {
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    CK(cudaGraphAddNode(out, g, deps, ndeps, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(g_ws.cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    Enq q{g_ws.cap_stream, prof};
    const int rc = enqueue_body<TR>(q, h);
    cudaGraph_t got = body;
    const cudaError_t e = cudaStreamEndCapture(g_ws.cap_stream, &got);
    if (rc) return rc;
    CK(e);
    *nodes = q.launches;
    return IPS4O_OK;
}

template <class TR>
static int get_graph(bool prof, GraphCache** out) {
    if (g_ws.graphs_gen != g_ws.gen) {
        drop_graphs();
        g_ws.graphs_gen = g_ws.gen;
    }
    GraphCache& gc = g_ws.graphs[TR::TYPE][prof ? 1 : 0];
    if (!gc.valid) {
        cudaGraph_t g;
        CK(cudaGraphCreate(&g, 0));
        cudaGraphNode_t node;
        u32 nodes = 0;
        int rc = add_loop_node<TR>(g, nullptr, 0, prof, &node, &nodes);
        if (rc) {
            cudaGraphDestroy(g);
            return rc;
        }
        cudaError_t e = cudaGraphInstantiate(&gc.exec, g, 0);
        cudaGraphDestroy(g);
        CK(e);
        gc.nodes_per_iter = nodes;
        gc.valid = true;
    }
    *out = &gc;
    return IPS4O_OK;
}

static bool g_prof_on = false;
static u32 g_nodes_per_iter = 0;

// IPS4O_EAGER=1: the same loop driven from the host (one stream sync per iteration to read
// LevelDyn::more) -- for profilers that cannot look inside conditional graphs (ncu).  Not
// the product path: it synchronises.
static bool eager_mode() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IPS4O_EAGER");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}
template <class TR>
static int run_eager(cudaStream_t st) {
    for (u64 it = 0;; ++it) {
        Enq q{st, false};
        int rc = enqueue_body<TR>(q, 0, 0u);
        if (rc) return rc;
        g_nodes_per_iter = q.launches;
        u32 more = 0;
        CK(cudaMemcpyAsync(&more, &g_ws.A.dyn->more, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        g_stats.host_syncs++;
        if (!more || it > MAX_BATCHES) break;
    }
    return IPS4O_OK;
}

template <class TR>
static int sort_impl(void* data, u64 n, cudaStream_t st, void* vals = nullptr) {
    int rc = ensure_ws<TR>(n);
    if (rc) return rc;
    rc = prepare_kernels<TR>();
    if (rc) return rc;
    g_stats.aux_bytes = g_ws.dev_bytes;
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &cst));
    const bool capturing = cst != cudaStreamCaptureStatusNone;
    // every call shares the workspace: a call on another stream first waits for the
    // previous call's work (the event is recorded at the end of every call)
    if (!capturing && g_ws.have_done && !g_ws.last_captured && g_ws.last_stream != st)
        CK(cudaStreamWaitEvent(st, g_ws.ev_done, 0));
    const u32 small = n <= (u64)TR::CAP                     ? base_class<TR>(n)
                      : (!TR::WIDE && n <= g_ws.A.medium_max) ? (u32)NUM_BASE_CLASSES + 1
                                                              : (u32)NUM_BASE_CLASSES;
    k_init<<<1, 32, 0, st>>>(g_ws.A, data, vals, n, 0x1234567ull, small);
    CK(cudaGetLastError());
    g_stats.host_syncs = 0;
    if (!capturing && eager_mode()) {
        rc = run_eager<TR>(st);
        if (rc) return rc;
        CK(cudaEventRecord(g_ws.ev_done, st));
        g_ws.have_done = true;
        g_ws.last_captured = false;
        g_ws.last_stream = st;
    } else if (!capturing) {
        GraphCache* gc = nullptr;
        rc = get_graph<TR>(g_prof_on, &gc);
        if (rc) return rc;
        CK(cudaGraphLaunch(gc->exec, st));
        g_nodes_per_iter = gc->nodes_per_iter;
        CK(cudaEventRecord(g_ws.ev_done, st));
        g_ws.have_done = true;
        g_ws.last_captured = false;
        g_ws.last_stream = st;
    } else {
        // the caller is capturing this stream into a graph: the loop node joins that graph
        cudaGraph_t ug;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        CK(cudaStreamGetCaptureInfo(st, &cst, nullptr, &ug, &deps, &nd));
        cudaGraphNode_t node;
        u32 nodes = 0;
        rc = add_loop_node<TR>(ug, deps, nd, false, &node, &nodes);
        if (rc) return rc;
        CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
        g_nodes_per_iter = nodes;
        g_ws.last_captured = true;
    }
    return IPS4O_OK;
}

static int type_size(int t) {
    switch (t) {
        case IPS4O_U64: return 8;
        case IPS4O_F64: return 8;
        case IPS4O_PAIR_U64: return 16;
        case IPS4O_REC100_K10: return 100;
        case IPS4O_PAIR_F64: return 16;
        case IPS4O_QUARTET_F64: return 32;
        default: return 0;
    }
}

constexpr u64 N_LIMIT = 1ull << 36;  // block indices stay < 2^31 (packed (w, r) words)

static int check_args(const void* p, u64 n, int type) {
    if (type_size(type) == 0) {
        snprintf(g_errbuf, sizeof g_errbuf, "unknown element type %d", type);
        return IPS4O_EINVAL;
    }
    if (n >= N_LIMIT) {
        snprintf(g_errbuf, sizeof g_errbuf, "n too large (limit 2^36)");
        return IPS4O_EINVAL;
    }
    if (n > 0 && !p) {
        snprintf(g_errbuf, sizeof g_errbuf, "null data pointer");
        return IPS4O_EINVAL;
    }
    const uintptr_t a = (uintptr_t)p;
    const int need = (type == IPS4O_PAIR_U64 || type == IPS4O_PAIR_F64 || type == IPS4O_QUARTET_F64) ? 16
                     : type == IPS4O_REC100_K10                                                   ? 4
                                                                                                  : 8;
    if (n > 0 && (a % need)) {
        snprintf(g_errbuf, sizeof g_errbuf, "data pointer not %d-byte aligned", need);
        return IPS4O_EALIGN;
    }
    return IPS4O_OK;
}

template <class TR>
static int splitters_to_keys(const void* h, u32 nspl, std::vector<u64>& out) {
    out.resize(nspl);
    if (TR::F64KEY) {
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

// Debug classification of d_in by the tree descent (flags bit 1 clear) or by K2's
// production bucket-hint table (bit 1 set).
template <class TR>
__global__ void k_debug_classify_lut(const void* vin, u64 n, const u64* spl_g, const unsigned short* lut_g,
                                     const TaskParam* tp, u32* out) {
    __shared__ u64 spl[MAXK];
    __shared__ unsigned short lut[LUT_STRIDE];
    for (u32 i = threadIdx.x; i < (u32)MAXK; i += blockDim.x) spl[i] = spl_g[i];
    for (u32 i = threadIdx.x; i < LUT_STRIDE; i += blockDim.x) lut[i] = lut_g[i];
    __syncthreads();
    const typename TR::V* in = reinterpret_cast<const typename TR::V*>(vin);
    const u64 lut_lo = tp->lut_lo;
    const u32 lut_sh = tp->lut_sh, eq = tp->eq;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    // whole warps iterate together (the classifier uses warp votes)
    for (u64 i0 = (u64)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const u64 i = i0 + threadIdx.x;
        u64 key[1] = {i < n ? TR::key(in[i], 0) : 0ull};
        u32 bk[1];
        // (K2's two variants: the cell from the keys' high words when cells are >= 2^32 wide)
        if (lut_sh >= 32u) k2_bucket_keys_lut<1, false, true>(key, i < n ? 1u : 0u, lut, spl, lut_lo, lut_sh, eq, bk);
        else k2_bucket_keys_lut<1>(key, i < n ? 1u : 0u, lut, spl, lut_lo, lut_sh, eq, bk);
        if (i < n) out[i] = bk[0];
    }
}

template <class TR>
static int debug_classify_impl(const void* d_in, u64 n, const void* h_spl, u32 nspl, int flags, u32* d_out,
                               cudaStream_t st) {
    int rc = ensure_ws<TR>(std::max<u64>(n, 64));
    if (rc) return rc;
    std::vector<u64> keys;
    if (splitters_to_keys<TR>(h_spl, nspl, keys)) {
        snprintf(g_errbuf, sizeof g_errbuf, "splitters must be strictly increasing");
        return IPS4O_EINVAL;
    }
    if (g_ws.have_done) CK(cudaStreamWaitEvent(st, g_ws.ev_done, 0));
    const LevelArgs& A = g_ws.A;
    CK(cudaMemcpyAsync(A.dsplit, keys.data(), 8ull * nspl, cudaMemcpyHostToDevice, st));
    k_tree_from_splitters<<<1, 256, 0, st>>>(A, A.dsplit, nspl, (u32)(flags & 1));
    CK(cudaGetLastError());
    if (n) {
        const u32 grid = (u32)std::min<u64>((n + 255) / 256, 4096);
        if (flags & 2)
            k_debug_classify_lut<TR><<<grid, 256, 0, st>>>(d_in, n, A.spl, A.lut, A.tp, d_out);
        else
            k_debug_classify<TR><<<grid, 256, 0, st>>>(d_in, n, A.tree, A.spl, A.tp, d_out);
        CK(cudaGetLastError());
    }
    // the splitter copy reads host memory: complete before returning
    CK(cudaStreamSynchronize(st));
    return IPS4O_OK;
}

template <class TR>
static int debug_partition_impl(void* d, u64 n, const void* h_spl, u32 nspl, int eq, u64* h_bnd, u32* K_out,
                                cudaStream_t st) {
    int rc = ensure_ws<TR>(n);
    if (rc) return rc;
    rc = prepare_kernels<TR>();
    if (rc) return rc;
    std::vector<u64> keys;
    if (splitters_to_keys<TR>(h_spl, nspl, keys)) {
        snprintf(g_errbuf, sizeof g_errbuf, "splitters must be strictly increasing");
        return IPS4O_EINVAL;
    }
    if (g_ws.have_done) CK(cudaStreamWaitEvent(st, g_ws.ev_done, 0));
    const LevelArgs& A = g_ws.A;
    CK(cudaMemcpyAsync(A.dsplit, keys.data(), 8ull * nspl, cudaMemcpyHostToDevice, st));
    k_debug_setup<<<1, 32, 0, st>>>(A, d, n, nspl, (u32)eq);
    CK(cudaGetLastError());
    k_plan<TR><<<1, PLAN_THREADS, 0, st>>>(A, (u32)g_ws.num_sms);
    CK(cudaGetLastError());
    Enq q{st, false};
    rc = enqueue_level<TR>(q);
    if (rc) return rc;
    k_epi<<<1, 32, 0, st>>>(A, 0, 0u);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h_bnd, A.bnd, (MAXK + 1) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(g_ws.ev_done, st));
    g_ws.have_done = true;
    g_ws.last_captured = false;
    g_ws.last_stream = st;
    CK(cudaStreamSynchronize(st));
    g_nodes_per_iter = q.launches + 3;
    u64 err = 0;
    CK(cudaMemcpy(&err, A.dstats + DS_ERROR, 8, cudaMemcpyDeviceToHost));
    if (err) {
        snprintf(g_errbuf, sizeof g_errbuf, "device consistency check failed (flags 0x%llx)", (unsigned long long)err);
        return IPS4O_EINTERNAL;
    }
    u32 kp = 2;
    while (kp < nspl + 1) kp <<= 1;
    *K_out = eq ? 2 * kp - 1 : kp;
    return IPS4O_OK;
}

// Reads the device statistics of the last call into g_stats (waits for that call).
static int fetch_stats() {
    if (!g_ws.have_done || g_ws.last_captured || !g_ws.dev) return IPS4O_OK;
    CK(cudaEventSynchronize(g_ws.ev_done));
    u64 ds[DS_N];
    CK(cudaMemcpy(ds, g_ws.A.dstats, sizeof ds, cudaMemcpyDeviceToHost));
    g_stats.levels = (uint32_t)ds[DS_LEVELS];
    g_stats.distribution_tasks = ds[DS_DIST_TASKS];
    g_stats.base_tasks = ds[DS_BASE_TASKS];
    g_stats.equality_tasks = ds[DS_EQ_TASKS];
    g_stats.distributed_elements = ds[DS_DIST_ELEMS];
    g_stats.base_elements = ds[DS_BASE_ELEMS];
    g_stats.batches = ds[DS_BATCHES];
    g_stats.device_error = ds[DS_ERROR];
    g_stats.block_moves = ds[DS_BLOCK_MOVES];
    g_stats.empty_block_moves = ds[DS_AMOVES];
    g_stats.base_fallback_tasks = ds[DS_FALLBACK];
    for (int c = 0; c < 4; ++c) g_stats.base_tasks_by_class[c] = ds[DS_BASE_C0 + c];
    g_stats.medium_tasks = ds[DS_MED_TASKS];
    g_stats.medium_partitions = ds[DS_MED_PARTS];
    g_stats.medium_marks = ds[DS_MED_MARKS];
    g_stats.medium_leaves = ds[DS_MED_LEAVES];
    // one k_init, then every iteration of the loop launches the body's kernels
    g_stats.kernel_launches = 1 + ds[DS_ITERS] * g_nodes_per_iter;
    return IPS4O_OK;
}

}  // namespace ips4o

using namespace ips4o;

// ------------------------------------------------------------------ C ABI

namespace ips4o {
static int sort_locked(void* d_data, uint64_t n, int elem_type, cudaStream_t st) {
    int rc = check_args(d_data, n, elem_type);
    if (rc) return rc;
    memset(&g_stats, 0, sizeof g_stats);
    g_stats.n = n;
    g_stats.elem_type = (uint32_t)elem_type;
    if (n <= 1) return IPS4O_OK;
    switch (elem_type) {
        case IPS4O_U64: rc = sort_impl<TU64>(d_data, n, st); break;
        case IPS4O_F64: rc = sort_impl<TF64>(d_data, n, st); break;
        case IPS4O_PAIR_U64: rc = sort_impl<TPair>(d_data, n, st); break;
        case IPS4O_REC100_K10: rc = sort_impl<TRec>(d_data, n, st); break;
        case IPS4O_PAIR_F64: rc = sort_impl<TPairF64>(d_data, n, st); break;
        case IPS4O_QUARTET_F64: rc = sort_impl<TQuad>(d_data, n, st); break;
        default: rc = IPS4O_EINVAL;
    }
    g_stats.has_device_stats = rc == IPS4O_OK ? 1u : 0u;
    return rc;
}

struct Staging {
    void* p = nullptr;
    size_t bytes = 0;
    int dev = -1;
};
static Staging g_stage_host;
static int stage_alloc(Staging& s, size_t bytes) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (s.p && (s.bytes < bytes || s.dev != dev)) {
        if (g_ws.have_done) cudaEventSynchronize(g_ws.ev_done);
        cudaFree(s.p);
        s.p = nullptr;
        s.bytes = 0;
    }
    if (!s.p) {
        if (cudaMalloc(&s.p, bytes) != cudaSuccess) {
            cudaGetLastError();
            snprintf(g_errbuf, sizeof g_errbuf, "staging allocation of %zu bytes failed", bytes);
            return IPS4O_ENOMEM;
        }
        s.bytes = bytes;
        s.dev = dev;
    }
    return IPS4O_OK;
}
static void stage_free(Staging& s) {
    if (s.p) cudaFree(s.p);
    s = Staging();
}
}  // namespace ips4o

extern "C" {

int ips4o_sort(void* d_data, uint64_t n, int elem_type, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return sort_locked(d_data, n, elem_type, (cudaStream_t)stream);
}

int ips4o_sort_host(void* h_data, uint64_t n, int elem_type, void* stream) {
    const int s = type_size(elem_type);
    if (!s || (n > 0 && !h_data)) return IPS4O_EINVAL;
    if (n <= 1) return IPS4O_OK;
    std::lock_guard<std::mutex> lk(g_mu);  // held across copy-in, sort and copy-out
    const size_t bytes = (size_t)n * s;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = stage_alloc(g_stage_host, bytes);
    if (rc) return rc;
    if (g_ws.have_done) CK(cudaStreamWaitEvent(st, g_ws.ev_done, 0));
    CK(cudaMemcpyAsync(g_stage_host.p, h_data, bytes, cudaMemcpyHostToDevice, st));
    rc = sort_locked(g_stage_host.p, n, elem_type, st);
    if (rc) return rc;
    CK(cudaMemcpyAsync(h_data, g_stage_host.p, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    g_stats.staging_bytes = bytes;
    return IPS4O_OK;
}

int ips4o_sort_kv(uint64_t* d_keys, uint64_t* d_vals, uint64_t n, int key_type, void* stream) {
    if (key_type != IPS4O_U64 && key_type != IPS4O_F64) {
        snprintf(g_errbuf, sizeof g_errbuf, "sort_kv: key type must be u64 or f64");
        return IPS4O_EINVAL;
    }
    if (n > 0 && (!d_keys || !d_vals)) {
        snprintf(g_errbuf, sizeof g_errbuf, "sort_kv: null pointer");
        return IPS4O_EINVAL;
    }
    if (n >= N_LIMIT) {
        snprintf(g_errbuf, sizeof g_errbuf, "sort_kv: n too large (limit 2^36)");
        return IPS4O_EINVAL;
    }
    if (n > 0 && ((((uintptr_t)d_keys) | ((uintptr_t)d_vals)) & 15u)) {
        snprintf(g_errbuf, sizeof g_errbuf, "sort_kv: keys and values must be 16-byte aligned");
        return IPS4O_EALIGN;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    memset(&g_stats, 0, sizeof g_stats);
    g_stats.n = n;
    g_stats.elem_type = (uint32_t)key_type;
    if (n <= 1) return IPS4O_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int rc = key_type == IPS4O_F64 ? sort_impl<TKVF64>(d_keys, n, st, d_vals) : sort_impl<TKV>(d_keys, n, st, d_vals);
    g_stats.has_device_stats = rc == IPS4O_OK ? 1u : 0u;
    return rc;
}

size_t ips4o_aux_bytes(uint64_t n, int elem_type) {
    Caps c;
    switch (elem_type) {
        case IPS4O_U64: c = caps_for<TU64>(n); break;
        case IPS4O_F64: c = caps_for<TF64>(n); break;
        case IPS4O_PAIR_U64: c = caps_for<TPair>(n); break;
        case IPS4O_REC100_K10: c = caps_for<TRec>(n); break;
        case IPS4O_PAIR_F64: c = caps_for<TPairF64>(n); break;
        case IPS4O_QUARTET_F64: c = caps_for<TQuad>(n); break;
        default: return 0;
    }
    return layout_of(c).total;
}

int ips4o_last_stats(ips4o_stats* out) {
    if (!out) return IPS4O_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_stats.has_device_stats) {
        int rc = fetch_stats();
        if (rc) return rc;
    }
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
    if (g_ws.have_done) cudaEventSynchronize(g_ws.ev_done);
    stage_free(g_stage_host);
    release_all();
    return IPS4O_OK;
}

int ips4o_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_prof_on = on != 0;
    return IPS4O_OK;
}

// Per kernel kind: stamps recorded by the profiling graph of the last call(s) since the
// previous read.  Each stamp closes one kernel (or one group of kernels of a kind); its
// duration is the globaltimer difference to the stamp before it.
int ips4o_profile_read(uint64_t* launches, double* ms) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (int k = 0; k < IPS4O_NUM_KERNEL_KINDS; ++k) {
        if (launches) launches[k] = 0;
        if (ms) ms[k] = 0;
    }
    if (!g_ws.dev || !g_ws.have_done) return IPS4O_OK;
    CK(cudaEventSynchronize(g_ws.ev_done));
    u32 cnt = 0;
    CK(cudaMemcpy(&cnt, g_ws.A.plog_n, 4, cudaMemcpyDeviceToHost));
    cnt = std::min(cnt, PLOG_CAP);
    std::vector<u64> t(cnt);
    std::vector<u32> k(cnt);
    if (cnt) {
        CK(cudaMemcpy(t.data(), g_ws.A.plog_t, cnt * 8ull, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(k.data(), g_ws.A.plog_k, cnt * 4ull, cudaMemcpyDeviceToHost));
    }
    for (u32 i = 1; i < cnt; ++i) {
        if (k[i] == STAMP_BEGIN || k[i] >= (u32)IPS4O_NUM_KERNEL_KINDS) continue;
        if (launches) launches[k[i]]++;
        if (ms) ms[k[i]] += (double)(t[i] - t[i - 1]) * 1e-6;
    }
    CK(cudaMemset(g_ws.A.plog_n, 0, 4));
    return IPS4O_OK;
}

const char* ips4o_kernel_kind_name(int kind) {
    if (kind < 0 || kind >= IPS4O_NUM_KERNEL_KINDS) return "unknown";
    return kKindNames[kind];
}

int ips4o_debug_classify(const void* d_in, uint64_t n, int elem_type, const void* h_splitters, uint32_t nspl,
                         int flags, uint32_t* d_bucket_out, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = check_args(d_in, n, elem_type);
    if (rc) return rc;
    const int eq = flags & 1;
    if (!h_splitters || nspl < 1 || nspl > 255 || (eq && nspl > 127) || (n && !d_bucket_out) || (flags & ~3))
        return IPS4O_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    switch (elem_type) {
        case IPS4O_U64: return debug_classify_impl<TU64>(d_in, n, h_splitters, nspl, flags, d_bucket_out, st);
        case IPS4O_F64: return debug_classify_impl<TF64>(d_in, n, h_splitters, nspl, flags, d_bucket_out, st);
        case IPS4O_PAIR_U64: return debug_classify_impl<TPair>(d_in, n, h_splitters, nspl, flags, d_bucket_out, st);
        case IPS4O_REC100_K10: return debug_classify_impl<TRec>(d_in, n, h_splitters, nspl, flags, d_bucket_out, st);
        case IPS4O_PAIR_F64: return debug_classify_impl<TPairF64>(d_in, n, h_splitters, nspl, flags, d_bucket_out, st);
        case IPS4O_QUARTET_F64: return debug_classify_impl<TQuad>(d_in, n, h_splitters, nspl, flags, d_bucket_out, st);
        default: return IPS4O_EINVAL;
    }
}

int ips4o_debug_partition_once(void* d_data, uint64_t n, int elem_type, const void* h_splitters, uint32_t nspl,
                               int eq, uint64_t* h_bounds_out, uint32_t* K_out, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = check_args(d_data, n, elem_type);
    if (rc) return rc;
    if (!h_splitters || nspl < 1 || nspl > 255 || (eq && nspl > 127) || n < 64 || !h_bounds_out || !K_out)
        return IPS4O_EINVAL;
    memset(&g_stats, 0, sizeof g_stats);
    g_stats.n = n;
    g_stats.elem_type = (uint32_t)elem_type;
    cudaStream_t st = (cudaStream_t)stream;
    switch (elem_type) {
        case IPS4O_U64: rc = debug_partition_impl<TU64>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st); break;
        case IPS4O_F64: rc = debug_partition_impl<TF64>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st); break;
        case IPS4O_PAIR_U64: rc = debug_partition_impl<TPair>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st); break;
        case IPS4O_REC100_K10: rc = debug_partition_impl<TRec>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st); break;
        case IPS4O_PAIR_F64: rc = debug_partition_impl<TPairF64>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st); break;
        case IPS4O_QUARTET_F64: rc = debug_partition_impl<TQuad>(d_data, n, h_splitters, nspl, eq, (u64*)h_bounds_out, K_out, st); break;
        default: rc = IPS4O_EINVAL;
    }
    g_stats.has_device_stats = rc == IPS4O_OK ? 1u : 0u;
    return rc;
}

}  // extern "C"
