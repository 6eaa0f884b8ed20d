/*
 * ips4o.h -- C ABI of libips4o.so, a B200-native (sm_100a) in-place samplesort.
 *
 * The operation is the paper's problem statement (Axtmann et al., "In-place
 * Parallel Super Scalar Samplesort (IPS4o)", arXiv 1705.02257; PAPER.md:22,
 * §1): sort A[1..n] in place under a total order on keys, using only
 * sublinear extra memory.  The method is the paper's
 * distribution step -- sampling, branchless classification
 * with equality buckets, block-buffered local
 * classification (§4.1), block permutation with atomic
 * fetch-and-add on per-bucket (w,r) pointers (§4.2), cleanup
 * (§4.3) -- recursed until subproblems fit a base-case sort
 * (PAPER.md:147-153, 403).
 *
 * Element types (all little-endian, contiguous arrays in device memory):
 *   IPS4O_U64        8 B unsigned integer, ascending unsigned order.
 *   IPS4O_F64        8 B IEEE double, ascending '<'.  Inputs must contain no NaN and
 *                    no -0.0 (the order is then total); behaviour is unspecified otherwise.
 *   IPS4O_PAIR_U64   16 B {uint64 key; uint64 payload}; ordered by key only; unstable:
 *                    the payload order inside a run of equal keys is unspecified.
 *   IPS4O_REC100_K10 100 B record; key = bytes [0,10) compared as unsigned bytes
 *                    (memcmp order); payload = bytes [10,100); unstable.
 *   IPS4O_PAIR_F64   16 B {double key; double value}: the paper's Pair;
 *                    ordered by the key (no NaN / -0.0 keys); unstable.
 *   IPS4O_QUARTET_F64 32 B {double k0, k1, k2; double value}: the paper's Quartet
 *                    (PAPER.md:447-449); keys compared lexicographically (no NaN / -0.0);
 *                    unstable.  16-byte aligned.
 *
 * Conventions for every entry point:
 *   - Device pointers are CUDA device memory of the current device; the caller owns it.
 *   - Work is enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *     stream) and the call returns without waiting for it: the recursion is scheduled on
 *     the device (a CUDA-graph while-loop over a device task queue), so
 *     there is no host synchronisation inside a sort.  A sort may be captured into the
 *     caller's CUDA graph (stream capture) once the workspace exists for that element type
 *     and at least that n (call it once outside the capture); the captured graph then refers
 *     to that workspace and must not run concurrently with another sort.
 *   - Calls on different streams are ordered by the library (each call waits for the
 *     previous one's work through an event): they share one workspace.
 *   - Argument errors return synchronously and leave the data untouched.
 *   - Device faults surface as IPS4O_ECUDA from this or a later call (CUDA convention).
 *   - The library owns a lazily grown per-device auxiliary workspace whose size is
 *     reported by ips4o_aux_bytes(); it is O(k * b * CTAs + tasks), never O(n) beyond that.
 *   - Host-side calls are serialised by an internal mutex.
 *   - n < 2^36 (block indices of the permutation stay below 2^31).
 */
#ifndef IPS4O_H
#define IPS4O_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    IPS4O_U64 = 0,
    IPS4O_F64 = 1,
    IPS4O_PAIR_U64 = 2,
    IPS4O_REC100_K10 = 3,
    IPS4O_PAIR_F64 = 4,
    IPS4O_QUARTET_F64 = 5
} ips4o_type;

typedef enum {
    IPS4O_OK = 0,
    IPS4O_EINVAL = -1,   /* null pointer with n > 0, bad type, n >= 2^36, bad splitters */
    IPS4O_EALIGN = -2,   /* data pointer not aligned to 8 B (u64/f64), 16 B (pairs, quartets), 4 B (rec100) */
    IPS4O_ENOMEM = -3,   /* workspace allocation failed */
    IPS4O_ECUDA = -4,    /* CUDA launch/runtime error, see ips4o_error_string */
    IPS4O_EINTERNAL = -5 /* a device-side consistency check failed (conservation, capacity) */
} ips4o_status;

/* Statistics of the most recent ips4o_sort / ips4o_debug_partition_once call.  The
 * device-side fields are read when ips4o_last_stats() is called: it waits for that call's
 * work to finish (the sort itself never waits).  A call captured into a CUDA graph reports
 * only the host-side fields (n, elem_type, aux_bytes, host_syncs). */
typedef struct {
    uint64_t n;                 /* elements sorted */
    uint32_t elem_type;
    uint32_t levels;            /* distribution levels executed (multi-CTA tier) */
    uint64_t distribution_tasks;/* subproblems partitioned by the distribution kernels (multi-CTA tier) */
    uint64_t base_tasks;        /* subproblems finished by the base-case kernels (shared-memory tier) */
    uint64_t equality_tasks;    /* subproblems partitioned with equality buckets */
    uint64_t aux_bytes;         /* device workspace bytes reserved while sorting (see ips4o_aux_bytes) */
    uint64_t kernel_launches;   /* kernels launched by this call (k_init + loop iterations x body kernels) */
    uint64_t host_syncs;        /* host synchronisations inside the sort: always 0 */
    uint64_t distributed_elements; /* sum over distribution steps of the subproblem sizes */
    uint64_t base_elements;     /* sum of the base-case subproblem sizes */
    uint64_t batches;           /* iterations of the device-side level loop that distributed tasks */
    uint64_t base_tasks_by_class[4]; /* base-case leaves per size class (<=2K, <=4K, <=8K, <=16K elements;
                                        records: <=512, <=1024) */
    uint64_t base_fallback_tasks;/* leaves the cell kernel handed to the merge sort (clustered keys) */
    uint64_t block_moves;       /* block writes of the block permutation (swaps and placements) */
    uint64_t empty_block_moves; /* Appendix-A moves */
    uint64_t device_error;      /* sticky device consistency flags (0 = none; nonzero: the output is invalid) */
    uint64_t staging_bytes;     /* device staging of ips4o_sort_host (0 for ips4o_sort, ips4o_sort_kv) */
    uint64_t medium_tasks;      /* subproblems sorted completely by one CTA (single-CTA tier) */
    uint64_t medium_partitions; /* partitioning steps inside the single-CTA tier */
    uint64_t medium_marks;      /* buckets whose maximum was moved to their first position so that
                                   searchNextLargest finds them (strictly in-place driver) */
    uint64_t medium_leaves;     /* leaves sorted in shared memory inside the single-CTA tier */
    uint32_t has_device_stats;  /* 1 if the device-side fields above are valid */
    uint32_t reserved_;
} ips4o_stats;

/* ---------------------------------------------------------------- sorting */

/* Sort d_data[0..n) ascending, in place.  n = 0 and n = 1 are no-ops.
 * Returns IPS4O_OK or a negative ips4o_status. */
int ips4o_sort(void* d_data, uint64_t n, int elem_type, void* stream);

/* Host-buffer convenience entry point (the end-to-end path): copies h_data[0..n) (host
 * memory; pinned memory gives full PCIe/C2C bandwidth) to a library-owned device buffer,
 * sorts it there with ips4o_sort, and copies the result back into h_data.  Returns after
 * the stream has been synchronised.  The device staging buffer is n * elem_size bytes,
 * reused across calls and released by ips4o_release_workspace(). */
int ips4o_sort_host(void* h_data, uint64_t n, int elem_type, void* stream);

/* Key-value sort of structure-of-arrays data, in place: d_keys[0..n)
 * (uint64 if key_type == IPS4O_U64, IEEE double if IPS4O_F64; no NaN / -0.0) are sorted
 * ascending and d_vals[0..n) (uint64) travel with their keys; unstable.  Both arrays are device
 * memory of the current device owned by the caller, 16-byte aligned.  The same distribution
 * steps as ips4o_sort run on the pair of arrays: every block move moves a key block and its
 * value block together, so the only extra memory is the workspace of
 * ips4o_aux_bytes(n, IPS4O_PAIR_U64) (no n-proportional staging).  Asynchronous like
 * ips4o_sort.  Returns IPS4O_OK, IPS4O_EINVAL (bad key_type, null pointer with n > 0,
 * n >= 2^36), IPS4O_EALIGN (pointers not 16-byte aligned), IPS4O_ENOMEM or IPS4O_ECUDA. */
int ips4o_sort_kv(uint64_t* d_keys, uint64_t* d_vals, uint64_t n, int key_type, void* stream);

/* Bytes of the device workspace ips4o_sort(n, elem_type) allocates on a fresh workspace
 * (Theorem 2: O(k b t) buffers with t = stripes, plus the task queues).
 * Every term is a capacity bound of the planner: per-batch task and stripe tables
 * (<= 512 each), base-case queues (<= n / smallest leaf of the class), level queues
 * (<= n / (base capacity + 1)), and the partial-buffer spill (<= n/2 + K*(b-1), in practice
 * K*(b-1) per stripe).  A larger earlier call leaves the workspace at its larger size. */
size_t ips4o_aux_bytes(uint64_t n, int elem_type);

/* Statistics of the last call (host memory). */
int ips4o_last_stats(ips4o_stats* out);

const char* ips4o_error_string(int status);

/* Release the workspace of the current device. */
int ips4o_release_workspace(void);

/* ------------------------------------------------------------- profiling */
/* When enabled, every kernel launch is bracketed by CUDA events on the launch stream.
 * ips4o_profile_read() synchronises the recorded events and returns, per kernel kind,
 * the number of launches and the summed device milliseconds, then clears the record.
 * Kinds: 0 sample/splitters, 1 classify_flush, 2 prepare, 3 empty-block moves,
 * 4 block permutation, 5 cleanup, 6 base case, 7 other, 8 single-CTA tier. */
#define IPS4O_NUM_KERNEL_KINDS 9
int ips4o_profile_enable(int on);
int ips4o_profile_read(uint64_t* launches /*[9]*/, double* ms /*[9]*/);
const char* ips4o_kernel_kind_name(int kind);

/* ------------------------------------------------------- test-only hooks */

/* Classification of d_in[0..n) with GIVEN splitters:
 * h_splitters is HOST memory holding nspl strictly increasing keys in the element
 * type's key format (u64: uint64; f64: double; pair: uint64 key; rec100: the big-endian
 * uint64 of key bytes 0..7, the key part a distribution step classifies on; pair_f64: double
 * key; quartet_f64: double k0).
 * flags bit 0 enables equality buckets; bit 1 selects K2's production classifier (the
 * bucket-hint table, k2_bucket_keys_lut) instead of the tree descent (classify_key).
 * Writes the bucket index of every element to d_bucket_out (device, uint32[n]), using the
 * numbering of SURVEY.md §8(c) O5.  1 <= nspl <= 255 (<= 127 with eq).  Returns after the
 * stream is synchronised. */
int ips4o_debug_classify(const void* d_in, uint64_t n, int elem_type, const void* h_splitters,
                         uint32_t nspl, int flags, uint32_t* d_bucket_out, void* stream);

/* One distribution step (local classification, block permutation, cleanup) over
 * d_data[0..n) with GIVEN splitters (same format as above), without recursion.
 * On return (the stream is synchronised) d_data is partitioned and h_bounds_out
 * (HOST, >= 257 entries) holds the element-exact bucket starts e_0..e_K, *K_out = K.
 * n >= 64. */
int ips4o_debug_partition_once(void* d_data, uint64_t n, int elem_type, const void* h_splitters,
                               uint32_t nspl, int eq, uint64_t* h_bounds_out, uint32_t* K_out,
                               void* stream);

#ifdef __cplusplus
}
#endif
#endif
