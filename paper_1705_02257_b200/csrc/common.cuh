// common.cuh -- element traits, level descriptors and small device helpers shared by
// the sm_100a kernels of libips4o.so.  (Product code; shares nothing with oracle/.)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ips4o {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr int MAXK = 256;            // buckets per step: k = 256, or 2k'-1 <= 255 with eq
constexpr u32 RBIAS = 0x80000000u;   // bias of the packed read pointer
// Each bucket's permutation control pair: the packed (w, r) word, then its reader count.
// (Spreading the pairs over 256-byte lines -- one L2 slice each -- measured no faster.)
constexpr int CTL_STRIDE = 2;        // u64 words per bucket control pair (16 B)
#ifndef IPS4O_CELL_C1MAX  // largest leaf of base-case class 1 (8-byte types)
#define IPS4O_CELL_C1MAX 4096
#endif
#ifndef IPS4O_CAP8  // base-case capacity of the 8-byte key types (larger buckets are distributed again)
#define IPS4O_CAP8 16384
#endif
#ifndef IPS4O_LEAF8  // target leaf size of the adaptive k for u64 / f64 keys
#define IPS4O_LEAF8 4096
#endif
#ifndef IPS4O_CELL_C2MAX  // largest leaf of base-case class 2 (8/16-byte types)
#define IPS4O_CELL_C2MAX 6144
#endif
#ifndef IPS4O_K2_LUT  // K2 classifies through the bucket-hint table (1) or the splitter tree only (0)
#define IPS4O_K2_LUT 1
#endif
#ifndef IPS4O_K2_WFLUSH  // K2 flushes buffer blocks by TMA bulk stores (0) or warp copies (1, measured slower)
#define IPS4O_K2_WFLUSH 0
#endif
#ifndef IPS4O_K2_STAGES  // two TMA tile stages when the tree copies are not needed
#define IPS4O_K2_STAGES (IPS4O_K2_LUT ? 2 : 1)
#endif
constexpr int K2_STAGES = IPS4O_K2_STAGES;   // tiles staged ahead in K2 (TMA)
#ifndef IPS4O_K2_MAIN_STAGES  // the multi-CTA K2 kernel's stages (the single-CTA tier keeps K2_STAGES)
#define IPS4O_K2_MAIN_STAGES K2_STAGES
#endif
constexpr int K2_MAIN_STAGES = IPS4O_K2_MAIN_STAGES;
// replicated splitter tree in K2: 16 copies (conflict-free lookups) when shared memory
// allows, else 8 (lanes l, l+8 of a half-warp share a copy)
constexpr int TREE_COPIES = K2_STAGES == 1 ? 16 : 8;
constexpr u32 TREE_NODE_BYTES = 8 * TREE_COPIES;
constexpr u32 INV_BUCKET = 0xFFFFu;  // "no element" marker in classification registers
constexpr int K3_THREADS = 256;      // block permutation CTA
#ifndef IPS4O_K3_SLOTS
#define IPS4O_K3_SLOTS 4
#endif
#ifndef IPS4O_K3_ACQUIRE
#define IPS4O_K3_ACQUIRE 0
#endif
constexpr int K3_SLOTS = IPS4O_K3_SLOTS;  // independent chains per warp
#ifndef IPS4O_K3_MINB
#define IPS4O_K3_MINB (IPS4O_K3_SLOTS <= 2 ? 6 : IPS4O_K3_SLOTS <= 4 ? 4 : 2)
#endif
constexpr int K3_MINB = IPS4O_K3_MINB;  // CTAs per SM (register budget 65536 / (256 * MINB))
constexpr int K4_THREADS = 256;      // cleanup CTA
#ifndef IPS4O_BLOCK_BYTES
#define IPS4O_BLOCK_BYTES 512
#endif
constexpr int BLOCK_BYTES = IPS4O_BLOCK_BYTES;  // block b*s in bytes for the 8/16-byte types (records: 400)

// ----------------------------------------------------------------- element traits
// key(): order-preserving unsigned 64-bit image of the sort key.
// less(): the base-case order.  For PAIR it is (key, payload) lexicographic -- a valid
// unstable order that also makes padding with the all-ones element harmless.

// Trait flags: WIDE = elements are moved as 32-bit words by the record-style K2 (k_classify_wide);
// F64KEY = key parts are IEEE doubles compared through the order-preserving image.
struct TU64 {
    typedef u64 V;
    static constexpr int S = 8, B = BLOCK_BYTES / 8, VEC = 2, CAP = IPS4O_CAP8, TYPE = 0, PARTS = 1;
    static constexpr bool WIDE = false, F64KEY = false, KV = false;
    static constexpr u32 LEAF = IPS4O_LEAF8;  // target base-case size of the adaptive k
    static constexpr u32 C0MAX = 2048, C1MAX = IPS4O_CELL_C1MAX, C2MAX = IPS4O_CELL_C2MAX;  // largest leaves of base-case classes 0-2
    __device__ __forceinline__ static u64 key(V v, u32 = 0) { return v; }
    __device__ __forceinline__ static bool less(V a, V b) { return a < b; }
    __host__ __device__ __forceinline__ static V pad() { return ~0ull; }
};

// IEEE doubles without NaN/-0.0: flip all bits of negatives, set the sign bit of
// non-negatives -> unsigned order equals '<' (PAPER.md:452 uses 64-bit floats).
struct TF64 {
    typedef u64 V;
    static constexpr int S = 8, B = BLOCK_BYTES / 8, VEC = 2, CAP = IPS4O_CAP8, TYPE = 1, PARTS = 1;
    static constexpr bool WIDE = false, F64KEY = true, KV = false;
    static constexpr u32 LEAF = IPS4O_LEAF8;
    static constexpr u32 C0MAX = 2048, C1MAX = IPS4O_CELL_C1MAX, C2MAX = IPS4O_CELL_C2MAX;
    __host__ __device__ __forceinline__ static u64 key(V v, u32 = 0) {
        return (v >> 63) ? ~v : (v | 0x8000000000000000ull);
    }
    __device__ __forceinline__ static bool less(V a, V b) { return key(a) < key(b); }
    __host__ __device__ __forceinline__ static V pad() { return 0x7FFFFFFFFFFFFFFFull; }  // key = ~0
};

struct TPair {
    typedef ulonglong2 V;
    static constexpr int S = 16, B = BLOCK_BYTES / 16, VEC = 1, CAP = 8192, TYPE = 2, PARTS = 1;
    static constexpr bool WIDE = false, F64KEY = false, KV = false;
    static constexpr u32 LEAF = 4096;
    static constexpr u32 C0MAX = 2048, C1MAX = 4096, C2MAX = IPS4O_CELL_C2MAX;
    __device__ __forceinline__ static u64 key(V v, u32 = 0) { return v.x; }
    __device__ __forceinline__ static bool less(V a, V b) {
        return a.x < b.x || (a.x == b.x && a.y < b.y);
    }
    __host__ __device__ __forceinline__ static V pad() { return make_ulonglong2(~0ull, ~0ull); }
};

// 100-byte record, 4-byte aligned; key = bytes [0,10) in memcmp order.  The key is
// compared in two 64-bit parts: part 0 = big-endian bytes 0..7, part 1 = big-endian bytes
// 8..9.  A distribution step classifies on one part; an equality bucket of part 0 (equal
// first 8 bytes) is re-partitioned on part 1, and the base case compares both.
struct Rec100 {
    u32 w[25];
};
struct TRec {
    typedef Rec100 V;
    static constexpr int S = 100, B = 4, VEC = 0, CAP = 1024, TYPE = 3, PARTS = 2, RW = 25;
    static constexpr bool WIDE = true, F64KEY = false, KV = false;
    static constexpr u32 LEAF = 512;
    static constexpr u32 C0MAX = 512, C1MAX = 1024, C2MAX = 1024;  // record leaves: base-case classes
    __device__ __forceinline__ static u64 hi_of(u32 w0, u32 w1) {
        return ((u64)__byte_perm(w0, 0, 0x0123) << 32) | (u64)__byte_perm(w1, 0, 0x0123);
    }
    __device__ __forceinline__ static u64 lo_of(u32 w2) { return (u64)__byte_perm(w2, 0, 0x4401); }
    __device__ __forceinline__ static u64 key(const V& v, u32 part) {
        return part ? lo_of(v.w[2]) : hi_of(v.w[0], v.w[1]);
    }
    // key part from the record's words (K2 works on word copies)
    __device__ __forceinline__ static u64 key_w(const u32* w, u32 part) { return part ? lo_of(w[2]) : hi_of(w[0], w[1]); }
};

// The paper's Pair: an f64 key and an f64 value, 16 B, ordered by the key
// (through the order-preserving image; no NaN / -0.0), unstable.
struct TPairF64 {
    typedef ulonglong2 V;
    static constexpr int S = 16, B = BLOCK_BYTES / 16, VEC = 1, CAP = 8192, TYPE = 4, PARTS = 1;
    static constexpr bool WIDE = false, F64KEY = true, KV = false;
    static constexpr u32 LEAF = 4096;
    static constexpr u32 C0MAX = 2048, C1MAX = 4096, C2MAX = IPS4O_CELL_C2MAX;
    __device__ __forceinline__ static u64 key(V v, u32 = 0) { return TF64::key(v.x); }
    __device__ __forceinline__ static bool less(V a, V b) {
        const u64 ka = key(a), kb = key(b);
        return ka < kb || (ka == kb && a.y < b.y);
    }
    __host__ __device__ __forceinline__ static V pad() { return make_ulonglong2(0x7FFFFFFFFFFFFFFFull, ~0ull); }
};

// The paper's Quartet: three f64 keys compared lexicographically and an f64 value
// (PAPER.md:447-449), 32 B.  Like the records, a distribution step classifies on one key
// part (the image of k_part); an equality bucket of part p is re-partitioned on part p+1;
// the base case compares all three.
struct Quad {
    u64 w[4];
};
struct TQuad {
    typedef Quad V;
    static constexpr int S = 32, B = BLOCK_BYTES / 32, VEC = 0, CAP = 4096, TYPE = 5, PARTS = 3, RW = 8;
    static constexpr bool WIDE = true, F64KEY = true, KV = false;
    static constexpr u32 LEAF = 2048;
    static constexpr u32 C0MAX = 2048, C1MAX = 4096, C2MAX = 4096;  // base-case classes (cells on k0)
    __device__ __forceinline__ static u64 key(const V& v, u32 part = 0) { return TF64::key(v.w[part]); }
    __device__ __forceinline__ static u64 key_w(const u32* w, u32 part) {
        return TF64::key(((u64)w[2 * part + 1] << 32) | w[2 * part]);
    }
    __device__ __forceinline__ static bool less(const V& a, const V& b) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const u64 x = TF64::key(a.w[i]), y = TF64::key(b.w[i]);
            if (x != y) return x < y;
        }
        return a.w[3] < b.w[3];
    }
    __host__ __device__ __forceinline__ static V pad() {
        Quad q;
        q.w[0] = q.w[1] = q.w[2] = 0x7FFFFFFFFFFFFFFFull;  // key image ~0 (above every key)
        q.w[3] = ~0ull;
        return q;
    }
};

// Structure-of-arrays key-value elements (ips4o_sort_kv): keys (u64, or f64 through the
// order-preserving image) in one array, u64 values in another, moved together.  In registers,
// shared memory and the spill an element is the pair {key, value}; in global memory a block
// of B elements is a key block (B*8 bytes) in the key array and a value block in the value
// array.  Both arrays must be 16-byte aligned (TMA).
struct TKV {
    typedef ulonglong2 V;
    static constexpr int S = 16, B = BLOCK_BYTES / 16, VEC = 1, CAP = 8192, TYPE = 6, PARTS = 1;
    static constexpr bool WIDE = false, F64KEY = false, KV = true;
    static constexpr u32 LEAF = 4096;
    static constexpr u32 C0MAX = 2048, C1MAX = 4096, C2MAX = IPS4O_CELL_C2MAX;
    __device__ __forceinline__ static u64 key(V v, u32 = 0) { return v.x; }
    __device__ __forceinline__ static bool less(V a, V b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }
    __host__ __device__ __forceinline__ static V pad() { return make_ulonglong2(~0ull, ~0ull); }
};
struct TKVF64 {
    typedef ulonglong2 V;
    static constexpr int S = 16, B = BLOCK_BYTES / 16, VEC = 1, CAP = 8192, TYPE = 7, PARTS = 1;
    static constexpr bool WIDE = false, F64KEY = true, KV = true;
    static constexpr u32 LEAF = 4096;
    static constexpr u32 C0MAX = 2048, C1MAX = 4096, C2MAX = IPS4O_CELL_C2MAX;
    __device__ __forceinline__ static u64 key(V v, u32 = 0) { return TF64::key(v.x); }
    __device__ __forceinline__ static bool less(V a, V b) {
        const u64 ka = key(a), kb = key(b);
        return ka < kb || (ka == kb && a.y < b.y);
    }
    __host__ __device__ __forceinline__ static V pad() { return make_ulonglong2(0x7FFFFFFFFFFFFFFFull, ~0ull); }
};
// bytes per element index in the (first) data array: the block grid's 16-byte alignment
template <class TR> struct GridStride { static constexpr int v = TR::KV ? 8 : TR::S; };

// ------------------------------------------------------------- level descriptors

struct TaskDesc {
    u64 lo, hi;
    u32 part, pad_;   // key part the next distribution step classifies on (records only)
};

// Per task of one distribution level.  Block grid origin g: the first element index
// >= lo whose address is 16-byte aligned (TMA bulk copies need 16 B); block x covers
// elements [g + x*B, g + (x+1)*B).  nblocks = ceil((hi-g)/B) (the last block may
// reach past hi: its writes go to the overflow block).
struct TaskParam {
    u64 lo, hi, g;
    u32 nblocks;
    u32 kprime, logk, eq, K;      // classifier (written by k_sample or the debug path)
    u32 stripe_begin, nstripes;   // this task's stripes in the stripe table (contiguous)
    u32 part;                     // key part (TRec); 0 otherwise
    u32 lut_sh;                   // bucket-hint table: cell of key = (key - lut_lo) >> lut_sh
    u64 lut_lo;                   //   (written with the classifier)
};

// Bucket-hint table of a task (K2's classification, written with the classifier): the key
// range [s_1, inf) is cut into LUT_N cells of 2^lut_sh keys from lut_lo = s_1 (keys below s_1
// use entry LUT_N).  Entry c = A | d << 8: A = #{padded splitters <= the cell's first key},
// d = #{padded splitters inside the cell}.  The leaf a key reaches in the splitter tree is
// A + #{j in 1..d : s_{A+j} <= key} (PAPER.md:137-142 computes the same count).
constexpr u32 LUT_LOG = 12, LUT_N = 1u << LUT_LOG, LUT_STRIDE = LUT_N + 8;  // u16 entries

// A stripe: [begin, end) elements of one task.  Its whole blocks [sb, se) (relative to
// the task's g) receive the flushed blocks at the front.
struct StripeDesc {
    u64 begin, end;
    u32 task, sb, se, first;      // first: 1 if this is the task's first stripe
};

enum {
    CTR_STRIPE = 0,   // K2 stripe ticket
    CTR_NEXT = 1,     // next-level task queue length (accumulates over a level's batches)
    CTR_TICKET = 2,   // cleanup ticket
    CTR_ERROR = 3,    // error bits
    CTR_EQ = 4,       // tasks partitioned with equality buckets
    CTR_BMOVES = 5,   // K3 block writes (swaps and placements)
    CTR_AMOVES = 6,   // Appendix-A empty-block moves
    CTR_FB = 7,       // base-case fallback queue length (leaves the cell kernel hands back)
    CTR_BASE0 = 8,    // base-case queue lengths, one per size class (4)
    CTR_TK0 = 12,     // base-case leaf tickets, one per size class (4)
    CTR_MED = 16,     // medium (single-CTA tier) queue length
    CTR_MTK = 17,     // medium task ticket
    CTR_N = 20
};
constexpr int NUM_BASE_CLASSES = 4;
// base-case size classes (8-byte types): <= 2048, <= 4096, <= 6144, <= 16384 elements; each
// class's CTA tile is sized to its leaves, so that the per-element loops stay mostly full
template <class TR>
__host__ __device__ __forceinline__ u32 base_class(u64 n) {
    return n <= TR::C0MAX ? 0u : n <= TR::C1MAX ? 1u : n <= TR::C2MAX ? 2u : 3u;
}
enum { ERR_SPILL = 1, ERR_CONSERVE = 2, ERR_QUEUE = 4, ERR_CAPACITY = 8, ERR_PROGRESS = 16, ERR_ITER = 32 };

// Per-batch fields written on the device (k_init, k_plan) and read by every level kernel at
// entry: the host never writes them, so nothing is staged through host memory and the
// whole level loop can run inside one CUDA graph (asynchronous on the
// caller's stream, no host synchronisation inside the sort).
struct LevelDyn {
    void* data;           // the array being sorted (element 0 of the call); KV types: the keys
    void* vals;           // KV types: the values (else unused)
    u64 n;
    TaskDesc* q_next;     // next-level queue K4 appends to (ctr[CTR_NEXT] entries)
    u64 seed;             // this batch's sampling seed
    u32 ntasks, nstripes; // this batch
    u32 emit;             // 0: debug single step, no emission
    u32 k4_cta;           // cleanup: one CTA per bucket (few buckets) instead of warp groups
    u32 moves_gx;         // k_moves: CTAs per task
    u32 from_splitters;   // K1 builds task 0's classifier from dsplit (debug partition step)
    u32 nspl, spl_eq;     //   (its splitter count, equality buckets)
    u32 more;             // set by k_epi: tasks remain
    u32 pad_;
};

// Device-side recursion scheduler state (the task queues of the level loop).
struct Sched {
    TaskDesc* qa;         // tasks of the current level (na of them, ca already planned)
    TaskDesc* qb;         // tasks of the next level (ctr[CTR_NEXT] of them)
    u32 na, ca;
    u32 level;
    u32 pad_;
    u64 ntot;             // elements of the current level (stripe length)
    u64 seed;
};

// Device statistics of a call (u64 words), accumulated by k_init / k_plan / k_epi.
enum {
    DS_LEVELS = 0, DS_DIST_TASKS, DS_BASE_TASKS, DS_EQ_TASKS, DS_DIST_ELEMS, DS_BASE_ELEMS,
    DS_BATCHES, DS_ERROR, DS_BLOCK_MOVES, DS_AMOVES, DS_FALLBACK, DS_BASE_C0, DS_BASE_C1, DS_BASE_C2,
    DS_BASE_C3, DS_ITERS, DS_MED_TASKS, DS_MED_PARTS, DS_MED_MARKS, DS_MED_LEAVES, DS_N = 24
};

struct LevelArgs {
    void* data;       // (from dyn)
    void* vals;       // (from dyn) KV types: the value array
    const TaskParam* tp;
    u32 ntasks;       // (from dyn)
    const StripeDesc* sd;
    const u32* stripe_order;
    u32 nstripes;     // (from dyn)
    u64* tree;        // [T][256] BFS tree a[1..k'-1] (index 0 unused)
    u64* spl;         // [T][256] sorted padded splitters s[1..k'-1]
    u32* s_count;     // [S][256] elements per bucket in stripe
    u32* s_fill;      // [S][256] partial buffer fill at the end of the stripe
    u32* s_spoff;     // [S][256] offset of the partial buffer in the stripe's spill
    u64* s_spbase;    // [S] stripe spill base (elements)
    u32* s_nfull;     // [S] full blocks flushed at the stripe front
    u32* prefF;       // [S] full blocks in earlier stripes of the same task
    u32* prefE;       // [S] empty blocks in earlier stripes of the same task
    void* spill;
    u64 spill_cap;    // elements
    u64* bnd;         // [T][257] element-exact bucket starts e_0..e_256
    u32* dblk;        // [T][257] delimiters d_i (block index, rounded up)
    u32* nfb;         // [T][256] full blocks of bucket i
    u64* btot;        // [T][256] bucket sizes: zeroed by K1, each K2 stripe adds its counts
    unsigned short* lut;  // [T][LUT_STRIDE] bucket-hint tables
    u32* mov;         // [T][257] prefix of Appendix-A moves over buckets
    u64* wr;          // [T][256] control lines: word 0 packed (w:32 | r+RBIAS:32) block
                      // pointers, word 1 (low half) the bucket's reader count
    u32* done;        // [T][8]   bucket has no unprocessed block left
    u32* tdone;       // [T/32]   task has no unprocessed block left
    u32* cflag;       // [T][256] cleanup: overhang saved
    void* ovf;        // [T][B]   overflow blocks
    int* ovf_owner;   // [T]
    TaskDesc* q_next; // (from dyn)
    TaskDesc* q_base; // base-case queues by size class: class c at q_base + qb_off[c], qb_cap[c] tasks
    TaskDesc* q_fb;   // [q_cap] base-case fallback queue (clustered leaves -> merge sort)
    TaskDesc* q_med;  // [qm_cap] medium tasks of the batch (single-CTA tier, k_cta.cuh)
    u32 qm_cap;
    u64 medium_max;   // tasks of base_cap < n <= medium_max go to the single-CTA tier (0: none)
    u64 wave_elems;   // levels >= 2: at most this many elements per batch (L2-sized waves; 0: off)
    u64 wave_stripe;  // minimum stripe length of a wave batch (elements)
    TaskDesc* q_lvl0; // [qn_cap] level queue A
    TaskDesc* q_lvl1; // [qn_cap] level queue B
    u32 qb_off[4], qb_cap[4];
    u32 q_cap;        // fallback queue capacity (tasks) = sum of qb_cap
    u32 qn_cap;       // level queue capacity (tasks)
    u32 tcap, scap;   // tasks / stripes per batch this workspace holds
    u32* ctr;         // [CTR_N]
    u64* spill_ctr;
    u64* base_elems;  // sum of sizes of emitted base-case tasks
    u64* dsplit;      // [256] debug splitters (key images)
    u32 base_cap;     // tasks with <= base_cap elements go to the base case
    int emit;         // (from dyn)
    u64 seed;         // (from dyn)
    LevelDyn* dyn;
    Sched* sched;
    u64* dstats;      // [DS_N]
    u64* plog_t;      // profile stamps (globaltimer ns) and kinds; plog_n entries
    u32* plog_k;
    u32* plog_n;
    u32 plog_cap;
};

// Each level kernel starts with this: the per-batch fields come from device memory.
__device__ __forceinline__ LevelArgs with_dyn(const LevelArgs& A0) {
    LevelArgs A = A0;
    const LevelDyn* D = A0.dyn;
    A.data = D->data;
    A.vals = D->vals;
    A.ntasks = D->ntasks;
    A.nstripes = D->nstripes;
    A.emit = (int)D->emit;
    A.seed = D->seed;
    A.q_next = D->q_next;
    return A;
}

// Element access to the sorted array(s): one array of V, or (KV types) a key array and a
// value array addressed with the same element index.
template <class TR, bool KV = TR::KV>
struct Mem {
    typedef typename TR::V V;
    V* d;
    __device__ __forceinline__ Mem(void* data, void*) : d(reinterpret_cast<V*>(data)) {}
    __device__ __forceinline__ V ld(u64 i) const { return d[i]; }
    __device__ __forceinline__ void st(u64 i, const V& x) const { d[i] = x; }
    __device__ __forceinline__ u64 key(u64 i, u32 part) const { return TR::key(d[i], part); }
};
template <class TR>
struct Mem<TR, true> {
    typedef typename TR::V V;
    u64* k;
    u64* v;
    __device__ __forceinline__ Mem(void* keys, void* vals) : k(reinterpret_cast<u64*>(keys)), v(reinterpret_cast<u64*>(vals)) {}
    __device__ __forceinline__ V ld(u64 i) const { return make_ulonglong2(k[i], v[i]); }
    __device__ __forceinline__ void st(u64 i, const V& x) const {
        k[i] = x.x;
        v[i] = x.y;
    }
    __device__ __forceinline__ u64 key(u64 i, u32) const { return TR::key(make_ulonglong2(k[i], 0ull), 0); }
};

// ---------------------------------------------------------------- device helpers

__device__ __forceinline__ u64* ctl_wr(u64* wr, u64 t, u32 b) { return wr + (t * MAXK + b) * CTL_STRIDE; }
__device__ __forceinline__ u32* ctl_readers(u64* wr, u64 t, u32 b) {
    return reinterpret_cast<u32*>(ctl_wr(wr, t, b) + 1);
}

__device__ __forceinline__ u32 lanemask_lt() {
    u32 r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p)
                 : "memory");
    return r;
}
// A block held by one warp in registers (K3 swap buffers, Appendix-A moves): 4 words per
// lane.  8/16-byte types: 512-byte blocks, one 16-byte vector per lane.  Records: 400-byte
// blocks (4 records, 4-byte aligned), lane l holds words l, l+32, l+64, l+96.
struct BlockRegs {
    u32 w[4];
};
template <class TR>
struct BlockIO {
    static constexpr u32 BB = TR::B * TR::S;  // block bytes
    __device__ __forceinline__ static BlockRegs load(const char* blk, u32 lane) {
        BlockRegs r;
        if constexpr (TR::S == 100) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const u32 idx = lane + 32 * i;
                r.w[i] = idx < BB / 4 ? *(volatile const u32*)(blk + 4 * idx) : 0u;
            }
        } else {
            static_assert(BB % 16 == 0 && BB <= 512, "a block is at most one vector per lane");
            r.w[0] = r.w[1] = r.w[2] = r.w[3] = 0u;
            if (16 * lane < BB)
                asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
                             : "l"(blk + 16 * lane)
                             : "memory");
        }
        return r;
    }
    __device__ __forceinline__ static void store(char* blk, u32 lane, const BlockRegs& r) {
        if constexpr (TR::S == 100) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const u32 idx = lane + 32 * i;
                if (idx < BB / 4) *(volatile u32*)(blk + 4 * idx) = r.w[i];
            }
        } else {
            if (16 * lane < BB)
                asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(blk + 16 * lane), "r"(r.w[0]),
                             "r"(r.w[1]), "r"(r.w[2]), "r"(r.w[3])
                             : "memory");
        }
    }
    // key part `part` of the block's first element (warp-collective)
    __device__ __forceinline__ static u64 first_key(const BlockRegs& r, u32 part) {
        if constexpr (TR::S == 100) {
            const u32 w0 = __shfl_sync(0xffffffffu, r.w[0], 0);
            const u32 w1 = __shfl_sync(0xffffffffu, r.w[0], 1);
            const u32 w2 = __shfl_sync(0xffffffffu, r.w[0], 2);
            return part ? TRec::lo_of(w2) : TRec::hi_of(w0, w1);
        } else if constexpr (TR::S == 32) {
            // key part p = words 2p, 2p+1 of element 0: lane p/2, words (2p)%4, (2p)%4+1
            const u32 src = part >> 1, o = (part & 1u) * 2u;
            const u32 w0 = __shfl_sync(0xffffffffu, o ? r.w[2] : r.w[0], src);
            const u32 w1 = __shfl_sync(0xffffffffu, o ? r.w[3] : r.w[1], src);
            u32 ww[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            ww[2 * part] = w0;
            ww[2 * part + 1] = w1;
            return TR::key_w(ww, part);
        } else {
            const u32 w0 = __shfl_sync(0xffffffffu, r.w[0], 0);
            const u32 w1 = __shfl_sync(0xffffffffu, r.w[1], 0);
            typename TR::V v;
            memset(&v, 0, sizeof(v));
            const u64 raw = ((u64)w1 << 32) | w0;
            memcpy(&v, &raw, 8);
            return TR::key(v, part);
        }
    }
};

__device__ __forceinline__ void st_v4(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// TMA bulk copy shared -> global (cp.async.bulk, SASS UBLKCP), bulk-group completion.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, u32 bytes) {
    u32 s = (u32)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s),
                 "r"(bytes)
                 : "memory");
}
// TMA bulk copy global -> shared with mbarrier transaction-count completion
__device__ __forceinline__ void mbar_init(u64* mbar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((u32)__cvta_generic_to_shared(mbar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, u32 bytes, u64* mbar) {
    const u32 mb = (u32)__cvta_generic_to_shared(mbar), sd = (u32)__cvta_generic_to_shared(sdst);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sd), "l"(gsrc), "r"(bytes), "r"(mb)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* mbar, u32 parity) {
    const u32 mb = (u32)__cvta_generic_to_shared(mbar);
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W;\n\t}" ::"r"(mb), "r"(parity)
                 : "memory");
}
// several bulk copies completing on one mbarrier: one arrive with the total byte count, then
// copies without arrive
__device__ __forceinline__ void mbar_expect_tx(u64* mbar, u32 bytes) {
    const u32 mb = (u32)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_tx(void* sdst, const void* gsrc, u32 bytes, u64* mbar) {
    const u32 mb = (u32)__cvta_generic_to_shared(mbar), sd = (u32)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sd), "l"(gsrc), "r"(bytes), "r"(mb)
                 : "memory");
}
// TMA bulk prefetch of [src, src+bytes) into L2 (16-byte aligned, multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, u32 bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy global writes before later async-proxy (TMA) accesses of the same data
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ u32 ld_acquire_u32(const u32* p) {
    u32 v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(u32* p, u32 v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// scoped atomics for the permutation's pointer / reader protocol
__device__ __forceinline__ u64 atom_add_acqrel_u64(u64* p, u64 v) {
    u64 old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_add_release_u32(u32* p, u32 v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ u64 atom_add_release_u64(u64* p, u64 v) {
    u64 old;
    asm volatile("atom.release.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ u64 atom_add_acquire_u64(u64* p, u64 v) {
    u64 old;
    asm volatile("atom.acquire.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ u32 atom_add_acquire_u32(u32* p, u32 v) {
    u32 old;
    asm volatile("atom.acquire.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__host__ __device__ __forceinline__ u64 mix64(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Branchless descent of the implicit search tree: j <- 2j + [a_j <= e]
// (ties go right: s_{i-1} <= e < s_i), then with equality buckets one
// extra comparison against the lower splitter: 2i-1 for {s_i}, 2i else.
__device__ __forceinline__ u32 classify_key(u64 k, const u64* tree, const u64* spl, u32 logk,
                                            u32 kprime, u32 eq) {
    u32 j = 1;
#pragma unroll
    for (int l = 0; l < 8; ++l)
        if ((u32)l < logk) j = 2 * j + (k >= tree[j] ? 1u : 0u);
    u32 i = j - kprime;
    if (eq) {
        u32 ii = i ? i : 1u;
        u32 isq = (i >= 1u && spl[ii] >= k) ? 1u : 0u;
        return 2 * i - isq;
    }
    return i;
}

}  // namespace ips4o
