/*
 * ips4o_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, sequential CPU samplesort written from the paper
 * (Axtmann, Witt, Ferizovic, Sanders: "In-place Parallel Super Scalar
 * Samplesort (IPS4o)", arXiv 1705.02257; /root/reference/PAPER.md).
 * It is IS4o, the t=1 variant, following
 * SURVEY.md §8(c) steps O1-O9 in the paper's order and notation.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_1705_02257_b200/csrc).
 *
 * Element types (same numbering as the product's C ABI, but declared
 * independently here):
 *   0 u64     8 B, unsigned order
 *   1 f64     8 B, IEEE '<' (inputs carry no NaN and no -0.0)
 *   2 pair    16 B {u64 key; u64 payload}, ordered by key only
 *   3 rec100  100 B, key = bytes [0,10) compared with memcmp
 *   4 pair_f64     16 B {f64 key; f64 payload}, ordered by the key (the paper's Pair,
 *                  PAPER.md:447-448)
 *   5 quartet_f64  32 B {f64 k0, k1, k2; f64 payload}, keys compared lexicographically
 *                  (the paper's Quartet)
 */
#ifndef IPS4O_ORACLE_H
#define IPS4O_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t k_max;   /* maximum buckets per step, power of two >= 4 (paper: 256) */
    uint64_t b;       /* block size in elements (paper: ~2 KiB) */
    uint64_t n0;      /* base-case size (paper: 16) */
    uint64_t seed;    /* sampling generator seed (splitmix64 stream) */
    int32_t  debug;   /* 1: assert the three-zone invariant after every permutation step */
    int32_t  pad_;
} oracle_params;

typedef struct {
    uint64_t partition_steps;   /* one per partition() call */
    uint64_t eq_steps;          /* partition steps that used equality buckets */
    uint64_t overflow_uses;     /* writes redirected to the overflow block */
    uint64_t overhang_uses;     /* cleanup sources taken from a next bucket's head */
    uint64_t block_moves;       /* block writes during block permutation */
    uint64_t skipped_blocks;    /* unprocessed blocks found already in place */
    uint64_t invariant_checks;  /* three-zone invariant evaluations (debug) */
    uint64_t base_cases;        /* insertion sorts */
    uint64_t max_depth;         /* recursion depth reached */
} oracle_stats;

/* error codes */
#define ORACLE_OK 0
#define ORACLE_EINVAL (-1)
#define ORACLE_EINVARIANT (-2)   /* an internal assertion failed (conservation / invariant) */

uint64_t oracle_default_block(int type);      /* b = max(1, 2^floor(11 - log2 s)) */
uint64_t oracle_alpha(uint64_t n);            /* max(1, round(0.2*log2 n)) */
uint64_t oracle_bucket_count(uint64_t n, uint64_t k_max);  /* O2 */
void     oracle_default_params(int type, oracle_params* p);

/* Sort a[0..n) ascending in place (O1-O9).  stats may be NULL. */
int oracle_sort(int type, void* a, uint64_t n, const oracle_params* p, oracle_stats* stats);
/* Sort each of `rows` consecutive arrays of n elements independently. */
int oracle_sort_rows(int type, void* a, uint64_t rows, uint64_t n, const oracle_params* p,
                     oracle_stats* stats);

/* One distribution step (O5-O8) over a[0..n) with GIVEN strictly increasing
 * splitters spl[0..nspl) and equality flag eq, block size b.  Writes the
 * element-exact bucket bounds e_0..e_K to bounds (K+1 entries, K <= 511) and
 * K to *K_out. */
int oracle_partition_with(int type, void* a, uint64_t n, const void* spl, uint32_t nspl,
                          int eq, uint64_t b, int debug, uint64_t* bounds, uint32_t* K_out,
                          oracle_stats* stats);

/* O5 classification of n elements with given splitters (strictly increasing). */
int oracle_classify(int type, const void* spl, uint32_t nspl, int eq, const void* elems,
                    uint64_t n, uint32_t* out);

/* O4 tree layout: breadth-first search tree over the padded splitters.
 * Writes k'-1 elements to tree_out and k' to *kprime. */
int oracle_build_tree(int type, const void* spl, uint32_t nspl, void* tree_out, uint32_t* kprime);

/* O4 splitter pick from an already sorted sample of m = alpha*k - 1 elements:
 * s_i = S[i*alpha - 1], i = 1..k-1, adjacent duplicates removed.
 * Writes the distinct splitters to out, their count to *nout, eq to *eq. */
int oracle_select_splitters(int type, const void* sorted_sample, uint64_t m, uint32_t k,
                            uint32_t alpha, void* out, uint32_t* nout, int* eq);

#ifdef __cplusplus
}
#endif
#endif
