/*
 * ips4o_oracle.c -- TEST INFRASTRUCTURE ONLY (see ips4o_oracle.h).
 *
 * Plain sequential IS4o (IPS4o with t = 1)
 * written from /root/reference/PAPER.md, step by step in the paper's order:
 *
 *   O1 base case            insertion sort below n0          PAPER.md:403, 416 (§4.7)
 *   O2 bucket count, alpha  k <= 256, alpha = 0.2 log n      PAPER.md:413-414 (§4.7)
 *   O3 sampling             swap sample to the front, sort   PAPER.md:135, 162-164 (§3, §4)
 *   O4 splitters + tree     equidistant picks, dedup, BFS    PAPER.md:136-141 (§3), 399-401 (§4.7)
 *   O5 classification       j <- 2j + [a_j <= e], eq test    PAPER.md:137-142 (§3), 341 (§4.4)
 *   O6 local classification buffer blocks, flush to front    PAPER.md:190-207 (§4.1)
 *   O7 block permutation    delimiters, (w_i, r_i), chains   PAPER.md:211-296 (§4.2)
 *   O8 cleanup              heads / tails / buffers / ovf    PAPER.md:308-323 (§4.3)
 *   O9 recursion            non-equality buckets, size > 1
 *
 * Readings where the paper is silent follow SURVEY.md §8(c) S1-S28 and are
 * listed in DESIGN.md "Readings".  No blocking, fusion or reordering beyond
 * what the algorithm states; every element is moved with memcpy and compared
 * through a per-type less() so the code reads the same for all six types.
 * Nothing here is shared with the CUDA path.
 */
#include "ips4o_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ types */

typedef int (*less_fn)(const void*, const void*);

static int less_u64(const void* a, const void* b) {
    uint64_t x, y;
    memcpy(&x, a, 8);
    memcpy(&y, b, 8);
    return x < y;
}
static int less_f64(const void* a, const void* b) {
    double x, y;
    memcpy(&x, a, 8);
    memcpy(&y, b, 8);
    return x < y;
}
static int less_pair(const void* a, const void* b) { return less_u64(a, b); } /* key at offset 0 */
static int less_rec100(const void* a, const void* b) { return memcmp(a, b, 10) < 0; }
/* The paper's Pair: one 64-bit floating point key and one 64-bit value. */
static int less_pair_f64(const void* a, const void* b) { return less_f64(a, b); } /* key at offset 0 */
/* The paper's Quartet: three 64-bit floating point keys compared lexicographically, and one
 * 64-bit value. */
static int less_quartet_f64(const void* a, const void* b) {
    double x[3], y[3];
    memcpy(x, a, 24);
    memcpy(y, b, 24);
    if (x[0] != y[0]) return x[0] < y[0];
    if (x[1] != y[1]) return x[1] < y[1];
    return x[2] < y[2];
}

typedef struct {
    size_t s;
    less_fn less;
} etype;

static int get_type(int type, etype* t) {
    switch (type) {
        case 0: t->s = 8; t->less = less_u64; return 1;
        case 1: t->s = 8; t->less = less_f64; return 1;
        case 2: t->s = 16; t->less = less_pair; return 1;
        case 3: t->s = 100; t->less = less_rec100; return 1;
        case 4: t->s = 16; t->less = less_pair_f64; return 1;
        case 5: t->s = 32; t->less = less_quartet_f64; return 1;
        default: return 0;
    }
}

#define AT(base, i, s) ((unsigned char*)(base) + (size_t)(i) * (s))

typedef struct {
    etype t;
    oracle_params p;
    oracle_stats* st;
    uint64_t rng;
    int failed;
} ctx;

static uint64_t splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static void swap_elems(void* a, void* b, size_t s, unsigned char* tmp) {
    if (a == b) return;
    memcpy(tmp, a, s);
    memcpy(a, b, s);
    memcpy(b, tmp, s);
}

/* ------------------------------------------------------------ parameters */

uint64_t oracle_default_block(int type) {
    etype t;
    if (!get_type(type, &t)) return 0;
    /* b = max(1, 2^floor(11 - log2 s)) */
    double e = floor(11.0 - log2((double)t.s));
    if (e < 0) return 1;
    return (uint64_t)1 << (uint64_t)e;
}

uint64_t oracle_alpha(uint64_t n) {
    /* alpha = 0.2 log n; log2, rounded to nearest, floor 1 (S1) */
    if (n < 2) return 1;
    long a = lround(0.2 * log2((double)n));
    return a < 1 ? 1 : (uint64_t)a;
}

static uint64_t pow2_floor(uint64_t x) {
    uint64_t r = 1;
    if (x == 0) return 0;
    while (r <= x / 2) r <<= 1;
    return r;
}

uint64_t oracle_bucket_count(uint64_t n, uint64_t k_max) {
    /* O2: k = min(k_max, max(4, pow2_floor(n/16))); k >= 4 guarantees progress (S9) */
    uint64_t k = pow2_floor(n / 16);
    if (k < 4) k = 4;
    if (k > k_max) k = k_max;
    return k;
}

void oracle_default_params(int type, oracle_params* p) {
    p->k_max = 256;
    p->b = oracle_default_block(type);
    p->n0 = 16;
    p->seed = 1;
    p->debug = 0;
    p->pad_ = 0;
}

/* ------------------------------------------------------------ O1 base case */

static void insertion_sort(const etype* t, unsigned char* a, uint64_t lo, uint64_t hi,
                           unsigned char* tmp) {
    size_t s = t->s;
    for (uint64_t i = lo + 1; i < hi; i++) {
        memcpy(tmp, AT(a, i, s), s);
        uint64_t j = i;
        while (j > lo && t->less(tmp, AT(a, j - 1, s))) {
            memcpy(AT(a, j, s), AT(a, j - 1, s), s);
            j--;
        }
        memcpy(AT(a, j, s), tmp, s);
    }
}

/* --------------------------------------------------- O4 tree, O5 classify */

typedef struct {
    uint32_t kprime;      /* number of leaves, power of two */
    uint32_t logk;
    int eq;               /* equality buckets on */
    uint32_t K;           /* number of buckets: kprime, or 2*kprime-1 with eq */
    unsigned char* spl;   /* 1-based sorted padded splitters spl[1..kprime-1] (slot 0 unused) */
    unsigned char* tree;  /* 1-based BFS tree a[1..kprime-1] (slot 0 unused) */
} classifier;

static int build_classifier(const etype* t, const void* distinct, uint32_t nd, int eq,
                            classifier* c) {
    size_t s = t->s;
    uint32_t kp = 2;
    /* k' = next power of two >= nd + 1; pad by repeating the largest splitter (S6) */
    while (kp < nd + 1) kp <<= 1;
    c->kprime = kp;
    c->logk = 0;
    while ((1u << c->logk) < kp) c->logk++;
    c->eq = eq;
    c->K = eq ? 2 * kp - 1 : kp;
    c->spl = (unsigned char*)malloc((size_t)kp * s);
    c->tree = (unsigned char*)malloc((size_t)kp * s);
    if (!c->spl || !c->tree) return 0;
    for (uint32_t i = 1; i < kp; i++) {
        uint32_t src = i <= nd ? i - 1 : nd - 1;
        memcpy(AT(c->spl, i, s), AT(distinct, src, s), s);
    }
    /* a_1 = s_{k/2}, a_2 = s_{k/4}, a_3 = s_{3k/4}; children of a_j are a_{2j}, a_{2j+1}
       (PAPER.md:139-141).  Node j at depth l, position p = j - 2^l holds s_{(2p+1) k / 2^(l+1)}. */
    for (uint32_t j = 1; j < kp; j++) {
        uint32_t l = 0;
        while ((2u << l) <= j) l++;
        uint32_t pos = j - (1u << l);
        uint32_t idx = (2 * pos + 1) * (kp >> (l + 1));
        memcpy(AT(c->tree, j, s), AT(c->spl, idx, s), s);
    }
    return 1;
}

static void free_classifier(classifier* c) {
    free(c->spl);
    free(c->tree);
    c->spl = c->tree = NULL;
}

/* O5: bucket i with s_{i-1} <= e < s_i (ties go right, S5); with equality
 * buckets one extra comparison against the lower splitter (S7):
 * index 2i for (s_i, s_{i+1}), 2i-1 for {s_i}. */
static uint32_t classify_one(const etype* t, const classifier* c, const void* e) {
    size_t s = t->s;
    uint32_t j = 1;
    for (uint32_t l = 0; l < c->logk; l++) j = 2 * j + (t->less(e, AT(c->tree, j, s)) ? 0u : 1u);
    uint32_t i = j - c->kprime;
    if (!c->eq) return i;
    if (i >= 1 && !t->less(AT(c->spl, i, s), e)) return 2 * i - 1;
    return 2 * i;
}

static int is_equality_bucket(const classifier* c, uint32_t idx) { return c->eq && (idx & 1u); }

/* ---------------------------------------------- O6-O8: one partition step */

static int64_t ceil_to_block(int64_t x, int64_t lo, int64_t b) {
    return lo + ((x - lo + b - 1) / b) * b;
}

enum { BLK_EMPTY = 0, BLK_FULL = 1 };

/* Debug: the three-zone invariant of PAPER.md:239-243 (Fig. 3) for every bucket:
 * [d_i, w_i) correct, [w_i, r_i] unprocessed (full), [max(w_i, r_i+b), d_{i+1}) empty. */
static int check_invariant(ctx* cx, const classifier* c, const unsigned char* a, int64_t lo,
                           int64_t hi, int64_t b, const int64_t* d, const int64_t* w,
                           const int64_t* r, const unsigned char* state, int64_t nblocks,
                           int ovf_owner, const unsigned char* ovf) {
    size_t s = cx->t.s;
    if (cx->st) cx->st->invariant_checks++;
    for (uint32_t i = 0; i < c->K; i++) {
        if (w[i] < d[i] || w[i] > d[i + 1]) return 0;
        for (int64_t x = d[i]; x < d[i + 1]; x += b) {
            int64_t blk = (x - lo) / b;
            if (blk >= nblocks) return 0;
            if (x < w[i]) {
                /* correct zone: every element of the block belongs to bucket i */
                const unsigned char* src = AT(a, x, s);
                if (state[blk] != BLK_FULL) return 0;
                if (x + b > hi) {
                    if (ovf_owner != (int)i) return 0;
                    src = ovf;
                }
                for (int64_t q = 0; q < b; q++)
                    if (classify_one(&cx->t, c, AT(src, q, s)) != i) return 0;
            } else if (x <= r[i]) {
                if (state[blk] != BLK_FULL) return 0;   /* unprocessed zone */
            } else {
                if (state[blk] != BLK_EMPTY) return 0;  /* empty zone */
            }
        }
    }
    return 1;
}

/* One distribution step over a[lo, hi) with classifier c, block size b.
 * Writes e_0..e_K into bounds.  Returns 0 on an internal assertion failure. */
static int partition_step(ctx* cx, unsigned char* a, int64_t lo, int64_t hi, const classifier* c,
                          int64_t b, int64_t* bounds) {
    const etype* t = &cx->t;
    size_t s = t->s;
    uint32_t K = c->K;
    int64_t n = hi - lo;
    int ok = 1;

    unsigned char* buf = (unsigned char*)malloc((size_t)K * b * s);
    int64_t* fill = (int64_t*)calloc(K, sizeof(int64_t));
    int64_t* count = (int64_t*)calloc(K, sizeof(int64_t));
    int64_t* d = (int64_t*)malloc((K + 1) * sizeof(int64_t));
    int64_t* w = (int64_t*)malloc(K * sizeof(int64_t));
    int64_t* r = (int64_t*)malloc(K * sizeof(int64_t));
    unsigned char* swap1 = (unsigned char*)malloc((size_t)b * s);
    unsigned char* swap2 = (unsigned char*)malloc((size_t)b * s);
    unsigned char* ovf = (unsigned char*)malloc((size_t)b * s);
    unsigned char* tmp = (unsigned char*)malloc((size_t)3 * b * s + s);
    int64_t nblocks = (n + b - 1) / b;
    unsigned char* state = (unsigned char*)calloc((size_t)nblocks + 1, 1);
    if (!buf || !fill || !count || !d || !w || !r || !swap1 || !swap2 || !ovf || !tmp || !state) {
        ok = 0;
        goto out;
    }

    /* ---- O6 local classification: one stripe = [lo, hi).
       Each element goes to its bucket's buffer block; a full buffer is first written
       back to the stripe front.  Counts come as a side effect. */
    int64_t wcur = 0; /* flushed blocks */
    for (int64_t p = 0; p < n; p++) {
        memcpy(tmp, AT(a, lo + p, s), s);
        uint32_t ci = classify_one(t, c, tmp);
        if (fill[ci] == b) {
            /* there is room: at least b more elements were scanned than written back */
            if (lo + (wcur + 1) * b > lo + p) { ok = 0; goto out; }
            memcpy(AT(a, lo + wcur * b, s), AT(buf, (int64_t)ci * b, s), (size_t)b * s);
            state[wcur] = BLK_FULL;
            wcur++;
            fill[ci] = 0;
        }
        memcpy(AT(buf, (int64_t)ci * b + fill[ci], s), tmp, s);
        fill[ci]++;
        count[ci]++;
    }
    int64_t F = wcur;

    /* ---- O7 delimiters: prefix sum -> e_i; d_i = e_i rounded up
       to the next block; d_K marks the end of the last bucket. */
    bounds[0] = lo;
    for (uint32_t i = 0; i < K; i++) bounds[i + 1] = bounds[i] + count[i];
    if (bounds[K] != hi) { ok = 0; goto out; }
    for (uint32_t i = 0; i <= K; i++) d[i] = ceil_to_block(bounds[i], lo, b);
    int64_t full_end = lo + F * b;
    for (uint32_t i = 0; i < K; i++) {
        /* t = 1: full blocks are exactly [lo, lo+F*b), so each bucket already reads
           "full blocks then empty blocks" (App. A).  w_i = d_i;
           r_i = last full block in [d_i, d_{i+1}), or d_i - 1 block. */
        w[i] = d[i];
        int64_t last = (d[i + 1] < full_end ? d[i + 1] : full_end) - b;
        r[i] = last >= d[i] ? last : d[i] - b;
    }

    /* ---- O7 block permutation, sequential: primary bucket p,
       two swap buffers, skip blocks already in place. */
    int ovf_owner = -1;
    unsigned char* cur = swap1;
    unsigned char* other = swap2;
    if (cx->p.debug &&
        !check_invariant(cx, c, a, lo, hi, b, d, w, r, state, nblocks, ovf_owner, ovf)) {
        ok = 0;
        goto out;
    }
    for (uint32_t pb = 0; pb < K; pb++) {
        for (;;) {
            while (w[pb] <= r[pb] && classify_one(t, c, AT(a, w[pb], s)) == pb) {
                w[pb] += b;
                if (cx->st) cx->st->skipped_blocks++;
            }
            if (w[pb] > r[pb]) break;
            /* read an unprocessed block from the primary bucket into a swap buffer */
            memcpy(cur, AT(a, r[pb], s), (size_t)b * s);
            state[(r[pb] - lo) / b] = BLK_EMPTY;
            r[pb] -= b;
            for (;;) {
                uint32_t dest = classify_one(t, c, cur); /* first element decides */
                while (w[dest] <= r[dest] && classify_one(t, c, AT(a, w[dest], s)) == dest) {
                    w[dest] += b;
                    if (cx->st) cx->st->skipped_blocks++;
                }
                if (w[dest] >= d[dest + 1]) { ok = 0; goto out; } /* capacity */
                if (w[dest] <= r[dest]) {
                    /* case 1: w_dest points to an unprocessed block -> swap */
                    memcpy(other, AT(a, w[dest], s), (size_t)b * s);
                    memcpy(AT(a, w[dest], s), cur, (size_t)b * s);
                    unsigned char* x = cur;
                    cur = other;
                    other = x;
                    w[dest] += b;
                    if (cx->st) cx->st->block_moves++;
                } else {
                    /* case 2: w_dest points to an empty block -> write, then refill.
                       A block reaching past the array end goes to the overflow block
                       (PAPER.md:220-221). */
                    if (w[dest] + b > hi) {
                        if (ovf_owner >= 0) { ok = 0; goto out; }
                        memcpy(ovf, cur, (size_t)b * s);
                        ovf_owner = (int)dest;
                        if (cx->st) cx->st->overflow_uses++;
                    } else {
                        memcpy(AT(a, w[dest], s), cur, (size_t)b * s);
                    }
                    state[(w[dest] - lo) / b] = BLK_FULL;
                    w[dest] += b;
                    if (cx->st) cx->st->block_moves++;
                    break;
                }
            }
            if (cx->p.debug &&
                !check_invariant(cx, c, a, lo, hi, b, d, w, r, state, nblocks, ovf_owner, ovf)) {
                ok = 0;
                goto out;
            }
        }
    }

    /* ---- O8 cleanup, buckets left to right.  Empty slots of bucket i:
       its head [e_i, min(d_i, e_{i+1})) and [min(w_i, e_{i+1}), e_{i+1}).  Sources: the
       overhang of its last block into the next bucket's head (S15), its partially filled
       buffer, and the overflow block if it owns it.  Left-to-right order reads every
       overhang before the next bucket's head is written. */
    int64_t D = d[K];
    for (uint32_t i = 0; i < K; i++) {
        int own_ovf = (ovf_owner == (int)i);
        int64_t in_end = own_ovf ? D - b : w[i]; /* end of blocks written inside the array */
        int64_t e0 = bounds[i], e1 = bounds[i + 1];
        int64_t nsrc = 0;
        if (in_end > d[i] && in_end > e1) {
            memcpy(AT(tmp, nsrc, s), AT(a, e1, s), (size_t)(in_end - e1) * s);
            nsrc += in_end - e1;
            if (cx->st) cx->st->overhang_uses++;
        }
        memcpy(AT(tmp, nsrc, s), AT(buf, (int64_t)i * b, s), (size_t)fill[i] * s);
        nsrc += fill[i];
        if (own_ovf) {
            memcpy(AT(tmp, nsrc, s), ovf, (size_t)b * s);
            nsrc += b;
        }
        int64_t head_end = d[i] < e1 ? d[i] : e1;
        int64_t tail_start = d[i] < e1 ? (in_end < e1 ? in_end : e1) : e1;
        int64_t nslots = (head_end - e0) + (e1 - tail_start);
        if (nslots != nsrc) { ok = 0; goto out; } /* conservation */
        int64_t q = 0;
        if (head_end > e0) {
            memcpy(AT(a, e0, s), AT(tmp, q, s), (size_t)(head_end - e0) * s);
            q += head_end - e0;
        }
        if (e1 > tail_start) memcpy(AT(a, tail_start, s), AT(tmp, q, s), (size_t)(e1 - tail_start) * s);
    }

out:
    free(buf); free(fill); free(count); free(d); free(w); free(r);
    free(swap1); free(swap2); free(ovf); free(tmp); free(state);
    return ok;
}

/* ------------------------------------------------ O2-O4: choose splitters */

static int choose_classifier(ctx* cx, unsigned char* a, int64_t lo, int64_t hi, classifier* c) {
    const etype* t = &cx->t;
    size_t s = t->s;
    int64_t n = hi - lo;
    uint64_t k = oracle_bucket_count((uint64_t)n, cx->p.k_max);   /* O2 */
    uint64_t alpha = oracle_alpha((uint64_t)n);
    int64_t m = (int64_t)(alpha * k - 1);
    if (m > n) return 0; /* O1 guards this (S21) */
    unsigned char tmp[128];
    /* O3: swap m random elements to the front (partial Fisher-Yates), sort them
       (PAPER.md:135, 162-164). */
    for (int64_t j = 0; j < m; j++) {
        uint64_t rnd = splitmix_next(&cx->rng);
        int64_t pick = j + (int64_t)(rnd % (uint64_t)(n - j));
        swap_elems(AT(a, lo + j, s), AT(a, lo + pick, s), s, tmp);
    }
    insertion_sort(t, a, (uint64_t)lo, (uint64_t)(lo + m), tmp);
    /* O4: s_i = S[i*alpha - 1], i = 1..k-1; drop adjacent duplicates;
       equality buckets iff any dropped, or a single distinct splitter (S9). */
    unsigned char* distinct = (unsigned char*)malloc((size_t)k * s);
    if (!distinct) return 0;
    uint32_t nd = 0;
    int removed = 0;
    for (uint64_t i = 1; i < k; i++) {
        const unsigned char* x = AT(a, lo + (int64_t)(i * alpha) - 1, s);
        if (nd > 0 && !t->less(AT(distinct, nd - 1, s), x)) {
            removed = 1;
            continue;
        }
        memcpy(AT(distinct, nd, s), x, s);
        nd++;
    }
    int eq = removed || nd == 1;
    int ok = build_classifier(t, distinct, nd, eq, c);
    free(distinct);
    return ok;
}

/* ------------------------------------------------------ O9: the recursion */

typedef struct {
    int64_t lo, hi;
    uint64_t depth;
} task;

static int sort_range(ctx* cx, unsigned char* a, int64_t lo0, int64_t hi0) {
    const etype* t = &cx->t;
    unsigned char tmp[128];
    size_t cap = 64, top = 0;
    task* stack = (task*)malloc(cap * sizeof(task));
    int64_t* bounds = (int64_t*)malloc(512 * sizeof(int64_t));
    if (!stack || !bounds) { free(stack); free(bounds); return 0; }
    stack[top++] = (task){lo0, hi0, 0};
    int ok = 1;
    uint64_t floor3 = cx->p.n0 > 3 ? cx->p.n0 : 3;
    while (top > 0 && ok) {
        task tk = stack[--top];
        int64_t n = tk.hi - tk.lo;
        if (cx->st && tk.depth > cx->st->max_depth) cx->st->max_depth = tk.depth;
        if ((uint64_t)n <= floor3) {                 /* O1 */
            insertion_sort(t, a, (uint64_t)tk.lo, (uint64_t)tk.hi, tmp);
            if (cx->st) cx->st->base_cases++;
            continue;
        }
        classifier c;
        memset(&c, 0, sizeof c);
        if (!choose_classifier(cx, a, tk.lo, tk.hi, &c)) { ok = 0; free_classifier(&c); break; }
        if (cx->st) {
            cx->st->partition_steps++;
            if (c.eq) cx->st->eq_steps++;
        }
        if (!partition_step(cx, a, tk.lo, tk.hi, &c, (int64_t)cx->p.b, bounds)) {
            ok = 0;
            free_classifier(&c);
            break;
        }
        for (uint32_t i = 0; i < c.K; i++) {          /* O9 */
            if (is_equality_bucket(&c, i)) continue;  /* never recursed */
            if (bounds[i + 1] - bounds[i] <= 1) continue;
            if (top == cap) {
                cap *= 2;
                task* ns = (task*)realloc(stack, cap * sizeof(task));
                if (!ns) { ok = 0; break; }
                stack = ns;
            }
            stack[top++] = (task){bounds[i], bounds[i + 1], tk.depth + 1};
        }
        free_classifier(&c);
    }
    free(stack);
    free(bounds);
    return ok;
}

static int valid_params(const oracle_params* p) {
    if (!p) return 0;
    if (p->k_max < 4 || (p->k_max & (p->k_max - 1)) || p->k_max > 256) return 0;
    if (p->b < 1 || p->n0 < 1) return 0;
    return 1;
}

int oracle_sort(int type, void* a, uint64_t n, const oracle_params* p, oracle_stats* stats) {
    ctx cx;
    memset(&cx, 0, sizeof cx);
    if (!get_type(type, &cx.t) || !valid_params(p) || (n > 0 && !a)) return ORACLE_EINVAL;
    cx.p = *p;
    cx.st = stats;
    cx.rng = p->seed;
    if (n <= 1) return ORACLE_OK;
    return sort_range(&cx, (unsigned char*)a, 0, (int64_t)n) ? ORACLE_OK : ORACLE_EINVARIANT;
}

int oracle_sort_rows(int type, void* a, uint64_t rows, uint64_t n, const oracle_params* p,
                     oracle_stats* stats) {
    etype t;
    if (!get_type(type, &t)) return ORACLE_EINVAL;
    for (uint64_t r = 0; r < rows; r++) {
        int rc = oracle_sort(type, AT(a, r * n, t.s), n, p, stats);
        if (rc) return rc;
    }
    return ORACLE_OK;
}

static int strictly_increasing(const etype* t, const void* spl, uint32_t nspl) {
    for (uint32_t i = 1; i < nspl; i++)
        if (!t->less(AT(spl, i - 1, t->s), AT(spl, i, t->s))) return 0;
    return 1;
}

int oracle_partition_with(int type, void* a, uint64_t n, const void* spl, uint32_t nspl,
                          int eq, uint64_t b, int debug, uint64_t* bounds, uint32_t* K_out,
                          oracle_stats* stats) {
    ctx cx;
    memset(&cx, 0, sizeof cx);
    if (!get_type(type, &cx.t) || nspl < 1 || nspl > 255 || b < 1 || !spl || !bounds)
        return ORACLE_EINVAL;
    if (eq && nspl > 255) return ORACLE_EINVAL;
    if (!strictly_increasing(&cx.t, spl, nspl)) return ORACLE_EINVAL;
    oracle_default_params(type, &cx.p);
    cx.p.b = b;
    cx.p.debug = debug;
    cx.st = stats;
    classifier c;
    memset(&c, 0, sizeof c);
    if (!build_classifier(&cx.t, spl, nspl, eq, &c)) { free_classifier(&c); return ORACLE_EINVAL; }
    int64_t* bd = (int64_t*)malloc((c.K + 1) * sizeof(int64_t));
    int ok = bd != NULL;
    if (ok && n > 0) ok = partition_step(&cx, (unsigned char*)a, 0, (int64_t)n, &c, (int64_t)b, bd);
    if (ok && n == 0)
        for (uint32_t i = 0; i <= c.K; i++) bd[i] = 0;
    if (ok) {
        for (uint32_t i = 0; i <= c.K; i++) bounds[i] = (uint64_t)bd[i];
        if (K_out) *K_out = c.K;
        if (stats) stats->partition_steps++;
    }
    free(bd);
    free_classifier(&c);
    return ok ? ORACLE_OK : ORACLE_EINVARIANT;
}

int oracle_classify(int type, const void* spl, uint32_t nspl, int eq, const void* elems,
                    uint64_t n, uint32_t* out) {
    etype t;
    if (!get_type(type, &t) || nspl < 1 || nspl > 255 || !spl) return ORACLE_EINVAL;
    if (!strictly_increasing(&t, spl, nspl)) return ORACLE_EINVAL;
    classifier c;
    memset(&c, 0, sizeof c);
    if (!build_classifier(&t, spl, nspl, eq, &c)) { free_classifier(&c); return ORACLE_EINVAL; }
    for (uint64_t i = 0; i < n; i++) out[i] = classify_one(&t, &c, AT(elems, i, t.s));
    free_classifier(&c);
    return ORACLE_OK;
}

int oracle_build_tree(int type, const void* spl, uint32_t nspl, void* tree_out, uint32_t* kprime) {
    etype t;
    if (!get_type(type, &t) || nspl < 1 || nspl > 255 || !spl) return ORACLE_EINVAL;
    classifier c;
    memset(&c, 0, sizeof c);
    if (!build_classifier(&t, spl, nspl, 0, &c)) { free_classifier(&c); return ORACLE_EINVAL; }
    memcpy(tree_out, AT(c.tree, 1, t.s), (size_t)(c.kprime - 1) * t.s);
    if (kprime) *kprime = c.kprime;
    free_classifier(&c);
    return ORACLE_OK;
}

int oracle_select_splitters(int type, const void* sorted_sample, uint64_t m, uint32_t k,
                            uint32_t alpha, void* out, uint32_t* nout, int* eq) {
    etype t;
    if (!get_type(type, &t) || k < 2 || alpha < 1 || (uint64_t)alpha * k - 1 > m) return ORACLE_EINVAL;
    uint32_t nd = 0;
    int removed = 0;
    for (uint32_t i = 1; i < k; i++) {
        const unsigned char* x = AT(sorted_sample, (uint64_t)i * alpha - 1, t.s);
        if (nd > 0 && !t.less(AT(out, nd - 1, t.s), x)) {
            removed = 1;
            continue;
        }
        memcpy(AT(out, nd, t.s), x, t.s);
        nd++;
    }
    *nout = nd;
    *eq = removed || nd == 1;
    return ORACLE_OK;
}
