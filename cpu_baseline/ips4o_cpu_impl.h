/* ips4o_cpu_impl.h -- body of the multi-core CPU IPS4o baseline, instantiated once per
 * element layout by ips4o_cpu.c (ELEM_S = element bytes, KEY_T / KEY_OF / KEY_LT / KEY_EQ
 * define the key).  The paper's parallel algorithm (§4):
 *
 *   partition(task, t threads):
 *     sampling     (one thread)  alpha*k-1 random elements, k-1 equidistant splitters,
 *                                duplicates removed -> equality buckets (PAPER.md:134-142,
 *                                162-164, 336-342, 399-401)
 *     local classification (t)   thread i classifies its stripe of whole blocks into k
 *                                buffers of b elements, flushing full buffers to the front
 *                                of its stripe
 *     prefix sums, empty-block movement (one thread)  bucket starts e_i, delimiters d_i,
 *                                full blocks compacted to the front of each bucket's
 *                                block range (App. A 578-590)
 *     block permutation (t)      atomic fetch-and-add on packed (w, r) pointers per
 *                                bucket, two swap buffers per thread, readers counted at
 *                                the crossing
 *     cleanup (t)                partial blocks and overhangs at the bucket boundaries
 *
 *   driver: tasks with >= n/t elements are partitioned by all threads one after another;
 *   the rest are assigned to threads (largest first) and sorted sequentially by the same
 *   partition with one thread (beta = 1).  Base case: insertion sort
 *   below n0 = 16 elements.
 *
 * This is a reported CPU baseline: it is not the oracle and shares
 * no code with the oracle or the CUDA path.
 */

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, CAT(_, SUFFIX))

typedef struct {
    unsigned char* a;     /* the array */
    size_t lo, hi;        /* task */
    int t;                /* threads */
    /* classifier */
    KEY_T tree[512];      /* a[1..kp-1] */
    KEY_T spl[512];       /* sorted padded splitters s[1..kp-1] */
    unsigned logk, kp, K, eq;
    /* per bucket */
    size_t bstart[2 * MAXKB + 2];   /* element-exact starts e_i, e_K = hi */
    size_t dl[2 * MAXKB + 2];       /* delimiters d_i (element index, block aligned from lo) */
    size_t nfb[2 * MAXKB + 1];      /* full blocks in [d_i, d_{i+1}) */
    uint64_t wr[2 * MAXKB + 1];     /* packed (w:32 | r+2^31:32) block indices from lo */
    unsigned readers[2 * MAXKB + 1];
    size_t wfin[2 * MAXKB + 1];
    /* per thread */
    size_t cnt[MAXT][2 * MAXKB + 1];
    size_t fill[MAXT][2 * MAXKB + 1];
    size_t sbeg[MAXT + 1];          /* stripe starts (block aligned from lo) */
    size_t nfull[MAXT];             /* full blocks flushed by thread i */
    unsigned char* tbuf[MAXT];      /* per thread: K buffers of B elements + 2 swap blocks */
    unsigned char ovf[ELEM_S * BLK];/* overflow block */
    int ovf_owner;
    unsigned char* ovh;             /* per bucket overhang save area: K * B elements */
    size_t ovh_len[2 * MAXKB + 1];
    uint64_t seed;
} FN(Part);

#define EL(p, i) ((p) + (size_t)(i) * ELEM_S)

static inline void FN(ecpy)(unsigned char* d, const unsigned char* s) { memcpy(d, s, ELEM_S); }

static void FN(insertion)(unsigned char* a, size_t lo, size_t hi) {
    unsigned char x[ELEM_S];
    for (size_t i = lo + 1; i < hi; ++i) {
        memcpy(x, EL(a, i), ELEM_S);
        const KEY_T kx = KEY_OF(x);
        size_t j = i;
        while (j > lo && KEY_LT(kx, KEY_OF(EL(a, j - 1)))) {
            memcpy(EL(a, j), EL(a, j - 1), ELEM_S);
            --j;
        }
        memcpy(EL(a, j), x, ELEM_S);
    }
}

/* Branchless descent: j <- 2j + [a_j <= key]; ties go right
 * (s_{i-1} <= e < s_i); equality buckets: one extra comparison with the lower splitter. */
static inline unsigned FN(classify)(const FN(Part) * P, KEY_T k) {
    unsigned j = 1;
    for (unsigned l = 0; l < P->logk; ++l) j = 2 * j + (unsigned)!KEY_LT(k, P->tree[j]);
    unsigned i = j - P->kp;
    if (P->eq) {
        const unsigned isq = (i >= 1) && !KEY_LT(P->spl[i], k);
        i = 2 * i - isq;
    }
    return i;
}

static inline uint64_t FN(rnd)(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static int FN(keycmp)(const void* x, const void* y) {
    const KEY_T a = *(const KEY_T*)x, b = *(const KEY_T*)y;
    return KEY_LT(a, b) ? -1 : KEY_LT(b, a) ? 1 : 0;
}

/* Sampling and the classifier (one thread). */
static void FN(sample)(FN(Part) * P) {
    const size_t n = P->hi - P->lo;
    unsigned k = 4;
    while (k < MAXKB && (size_t)k * 16 * 2 <= n) k *= 2;  /* k = min(256, max(4, pow2_floor(n/16))) */
    unsigned alpha = (unsigned)llround(0.2 * log2((double)n));
    if (alpha < 1) alpha = 1;
    size_t m = (size_t)alpha * k - 1;
    if (m > n) m = n;
    KEY_T* s = (KEY_T*)malloc(sizeof(KEY_T) * m);
    for (size_t i = 0; i < m; ++i) s[i] = KEY_OF(EL(P->a, P->lo + FN(rnd)(&P->seed) % n));
    qsort(s, m, sizeof(KEY_T), FN(keycmp));
    KEY_T d[MAXKB];
    unsigned nd = 0, dup = 0;
    for (unsigned i = 1; i < k; ++i) {
        size_t idx = (size_t)i * alpha - 1;
        if (idx >= m) idx = m - 1;
        if (nd && KEY_EQ(d[nd - 1], s[idx])) dup = 1;
        else d[nd++] = s[idx];
    }
    free(s);
    if (nd == 1) dup = 1;
    unsigned kp = 2;
    while (kp < nd + 1) kp <<= 1;
    unsigned logk = 0;
    while ((1u << logk) < kp) ++logk;
    for (unsigned i = 1; i < kp; ++i) P->spl[i] = d[(i <= nd ? i : nd) - 1];
    for (unsigned j = 1; j < kp; ++j) {
        const unsigned l = 31 - (unsigned)__builtin_clz(j), pos = j - (1u << l);
        const unsigned idx = (2 * pos + 1) * (kp >> (l + 1));
        P->tree[j] = d[(idx <= nd ? idx : nd) - 1];
    }
    P->kp = kp;
    P->logk = logk;
    P->eq = dup;
    P->K = dup ? 2 * kp - 1 : kp;
}

/* Local classification of thread i's stripe. */
static void FN(classify_stripe)(FN(Part) * P, int i) {
    const unsigned K = P->K;
    unsigned char* buf = P->tbuf[i];
    size_t* cnt = P->cnt[i];
    size_t* fl = P->fill[i];
    memset(cnt, 0, sizeof(size_t) * K);
    memset(fl, 0, sizeof(size_t) * K);
    const size_t b0 = P->sbeg[i], b1 = P->sbeg[i + 1];
    const size_t e0 = P->lo + b0 * BLK;
    size_t e1 = P->lo + b1 * BLK;
    if (e1 > P->hi) e1 = P->hi;
    size_t wp = e0;  /* write position (behind the read frontier) */
    for (size_t x = e0; x < e1; ++x) {
        const unsigned char* e = EL(P->a, x);
        const unsigned bk = FN(classify)(P, KEY_OF(e));
        unsigned char* slot = buf + ((size_t)bk * BLK + fl[bk]) * ELEM_S;
        memcpy(slot, e, ELEM_S);
        cnt[bk]++;
        if (++fl[bk] == BLK) {
            memcpy(EL(P->a, wp), buf + (size_t)bk * BLK * ELEM_S, (size_t)BLK * ELEM_S);
            wp += BLK;
            fl[bk] = 0;
        }
    }
    P->nfull[i] = (wp - e0) / BLK;
}

static inline int FN(block_belongs)(const FN(Part) * P, size_t blk, unsigned bucket) {
    return FN(classify)(P, KEY_OF(EL(P->a, P->lo + blk * BLK))) == bucket;
}

/* Block blk (from lo) holds a flushed full block after local classification: it lies in the
 * front part of its stripe. */
static inline int FN(is_full)(const FN(Part) * P, size_t blk) {
    int lo = 0, hi = P->t;  /* last stripe i with sbeg[i] <= blk */
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (P->sbeg[mid] <= blk) lo = mid;
        else hi = mid;
    }
    return blk - P->sbeg[lo] < P->nfull[lo];
}

/* Prefix sums, delimiters, empty-block movement (one thread; App. A). */
static void FN(prepare)(FN(Part) * P) {
    const unsigned K = P->K;
    const int t = P->t;
    const size_t n = P->hi - P->lo;
    const size_t nblocks = (n + BLK - 1) / BLK;
    size_t e = P->lo;
    for (unsigned j = 0; j < K; ++j) {
        P->bstart[j] = e;
        size_t s = 0;
        for (int i = 0; i < t; ++i) s += P->cnt[i][j];
        e += s;
    }
    P->bstart[K] = P->hi;
    for (unsigned j = 0; j <= K; ++j) {
        size_t d = (P->bstart[j] - P->lo + BLK - 1) / BLK;
        if (d > nblocks) d = nblocks;
        P->dl[j] = d;
    }
    P->dl[K] = nblocks;
    for (unsigned j = 0; j < K; ++j) {
        size_t nf = 0;
        for (size_t x = P->dl[j]; x < P->dl[j + 1]; ++x) nf += FN(is_full)(P, x);
        /* compact the bucket's full blocks to the front of [d_j, d_j + nf): the holes and
         * the sources lie in disjoint ranges, so the stripe layout still tells them apart */
        size_t hole = P->dl[j], src = P->dl[j] + nf;
        for (;;) {
            while (hole < P->dl[j] + nf && FN(is_full)(P, hole)) ++hole;
            if (hole >= P->dl[j] + nf) break;
            while (src < P->dl[j + 1] && !FN(is_full)(P, src)) ++src;
            memcpy(EL(P->a, P->lo + hole * BLK), EL(P->a, P->lo + src * BLK), (size_t)BLK * ELEM_S);
            ++hole;
            ++src;
        }
        P->nfb[j] = nf;
        const uint64_t w = P->dl[j], r = P->dl[j] + nf - 1 + 0x80000000ull;
        P->wr[j] = (w << 32) | (uint32_t)r;
        P->readers[j] = 0;
    }
    P->ovf_owner = -1;
}

/* Block permutation by one thread: take a block from the primary bucket
 * (r--), classify it, claim w_dest++ and swap with an unprocessed block or write into an
 * empty one (waiting for readers at the crossing); skip blocks already in place. */
static void FN(permute)(FN(Part) * P, int i) {
    const unsigned K = P->K;
    const size_t n = P->hi - P->lo;
    unsigned char* sw0 = P->tbuf[i] + (size_t)K * BLK * ELEM_S;
    unsigned char* sw1 = sw0 + (size_t)BLK * ELEM_S;
    unsigned p = (unsigned)((size_t)i * K / (size_t)P->t);
    for (unsigned c = 0; c < K; ++c, p = (p + 1) % K) {
        for (;;) {
            /* take: announce as reader, then r <- r-1 */
            __atomic_fetch_add(&P->readers[p], 1u, __ATOMIC_ACQ_REL);
            const uint64_t old = __atomic_fetch_add(&P->wr[p], ~0ull, __ATOMIC_ACQ_REL);
            const int64_t ow = (int64_t)(old >> 32), orr = (int64_t)((uint32_t)old) - 0x80000000ll;
            if (orr < ow) {
                __atomic_fetch_sub(&P->readers[p], 1u, __ATOMIC_RELEASE);
                break;
            }
            memcpy(sw0, EL(P->a, P->lo + (size_t)orr * BLK), (size_t)BLK * ELEM_S);
            __atomic_fetch_sub(&P->readers[p], 1u, __ATOMIC_RELEASE);
            unsigned char* cur = sw0;
            unsigned char* other = sw1;
            for (;;) {
                const unsigned dest = FN(classify)(P, KEY_OF(cur));
                const uint64_t o2 = __atomic_fetch_add(&P->wr[dest], 1ull << 32, __ATOMIC_ACQ_REL);
                const int64_t w = (int64_t)(o2 >> 32), r = (int64_t)((uint32_t)o2) - 0x80000000ll;
                if (w <= r) {
                    /* unprocessed block at w: already in place -> skip; else swap */
                    unsigned char* tgt = EL(P->a, P->lo + (size_t)w * BLK);
                    if (FN(classify)(P, KEY_OF(tgt)) == dest) continue;
                    memcpy(other, tgt, (size_t)BLK * ELEM_S);
                    memcpy(tgt, cur, (size_t)BLK * ELEM_S);
                    unsigned char* tmp = cur;
                    cur = other;
                    other = tmp;
                } else {
                    /* empty block at w: wait for readers of dest, then write (past the end:
                     * the overflow block) */
                    while (__atomic_load_n(&P->readers[dest], __ATOMIC_ACQUIRE) != 0) {
                    }
                    if (((size_t)w + 1) * BLK > n) {
                        memcpy(P->ovf, cur, (size_t)BLK * ELEM_S);
                        P->ovf_owner = (int)dest;
                    } else {
                        memcpy(EL(P->a, P->lo + (size_t)w * BLK), cur, (size_t)BLK * ELEM_S);
                    }
                    break;
                }
            }
        }
    }
}

/* Cleanup, part 1: save each bucket's overhang into the next bucket's head. */
static void FN(save_overhang)(FN(Part) * P, unsigned j) {
    const size_t n = P->hi - P->lo;
    const size_t w = (size_t)(P->wr[j] >> 32);
    const size_t nblocks = (n + BLK - 1) / BLK;
    const size_t dj = P->dl[j];
    const size_t e1 = P->bstart[j + 1];
    size_t in_end = P->lo + w * BLK;
    if (P->ovf_owner == (int)j) in_end = P->lo + (nblocks - 1) * BLK;  /* the shadowed block is empty */
    P->wfin[j] = in_end;
    size_t len = 0;
    if (w > dj && in_end > e1) {
        len = in_end - e1;
        memcpy(P->ovh + (size_t)j * BLK * ELEM_S, EL(P->a, e1), len * ELEM_S);
    }
    P->ovh_len[j] = len;
}

/* Cleanup, part 2: fill bucket j's empty slots (its head before the first
 * block and the tail after its last written block) from its overhang, every thread's partial
 * buffer and the overflow block. */
static void FN(fill_bucket)(FN(Part) * P, unsigned j) {
    const size_t e0 = P->bstart[j], e1 = P->bstart[j + 1];
    const size_t dj = P->lo + P->dl[j] * BLK;
    const size_t in_end = P->wfin[j];
    const size_t hend = dj < e1 ? dj : e1;
    size_t ts = e1;
    if (dj < e1) ts = in_end > dj ? (in_end < e1 ? in_end : e1) : dj;
    size_t pos = e0;
    #define PUT(src)                                   \
        do {                                           \
            if (pos == hend) pos = ts;                 \
            memcpy(EL(P->a, pos), (src), ELEM_S);      \
            ++pos;                                     \
        } while (0)
    for (size_t q = 0; q < P->ovh_len[j]; ++q) PUT(P->ovh + ((size_t)j * BLK + q) * ELEM_S);
    for (int i = 0; i < P->t; ++i) {
        const unsigned char* b = P->tbuf[i] + (size_t)j * BLK * ELEM_S;
        for (size_t q = 0; q < P->fill[i][j]; ++q) PUT(b + q * ELEM_S);
    }
    if (P->ovf_owner == (int)j)
        for (size_t q = 0; q < BLK; ++q) PUT(P->ovf + q * ELEM_S);
    #undef PUT
}

static void FN(barrier)(int t) {
    if (t > 1) {
#pragma omp barrier
    }
}

/* One partitioning step of [lo, hi) by t threads (t == omp team size when t > 1). */
static void FN(partition_team)(FN(Part) * P, int tid) {
    const int t = P->t;
    if (tid == 0) {
        FN(sample)(P);
        const size_t n = P->hi - P->lo, nblocks = (n + BLK - 1) / BLK;
        for (int i = 0; i <= t; ++i) P->sbeg[i] = nblocks * (size_t)i / (size_t)t;
    }
    FN(barrier)(t);
    FN(classify_stripe)(P, tid);
    FN(barrier)(t);
    if (tid == 0) FN(prepare)(P);
    FN(barrier)(t);
    FN(permute)(P, tid);
    FN(barrier)(t);
    for (unsigned j = (unsigned)tid; j < P->K; j += (unsigned)t) FN(save_overhang)(P, j);
    FN(barrier)(t);
    for (unsigned j = (unsigned)tid; j < P->K; j += (unsigned)t) FN(fill_bucket)(P, j);
    FN(barrier)(t);
}

typedef struct {
    size_t lo, hi;
} FN(Task);

static int FN(task_cmp)(const void* x, const void* y) {
    const FN(Task)* a = (const FN(Task)*)x;
    const FN(Task)* b = (const FN(Task)*)y;
    const size_t na = a->hi - a->lo, nb = b->hi - b->lo;
    return na > nb ? -1 : na < nb ? 1 : 0;
}

static FN(Part) * FN(part_new)(unsigned char* a, int t) {
    FN(Part)* P = (FN(Part)*)calloc(1, sizeof(FN(Part)));
    P->a = a;
    P->t = t;
    for (int i = 0; i < t; ++i) P->tbuf[i] = (unsigned char*)malloc((size_t)(2 * MAXKB + 2) * BLK * ELEM_S);
    P->ovh = (unsigned char*)malloc((size_t)(2 * MAXKB + 1) * BLK * ELEM_S);
    return P;
}
static void FN(part_free)(FN(Part) * P) {
    for (int i = 0; i < P->t; ++i) free(P->tbuf[i]);
    free(P->ovh);
    free(P);
}

/* children of the last partition: non-equality buckets of more than one element */
static void FN(emit)(const FN(Part) * P, FN(Task) * *v, size_t* nv, size_t* cap, int* bad) {
    for (unsigned j = 0; j < P->K; ++j) {
        const size_t b = P->bstart[j], e = P->bstart[j + 1];
        if (e - b <= 1 || (P->eq && (j & 1u))) continue;
        if (e - b == P->hi - P->lo) {
            *bad = 1;  /* no progress: cannot happen with k >= 4 */
            continue;
        }
        if (*nv == *cap) {
            *cap = *cap ? 2 * *cap : 1024;
            *v = (FN(Task)*)realloc(*v, *cap * sizeof(FN(Task)));
        }
        (*v)[(*nv)++] = (FN(Task)){b, e};
    }
}

static int FN(keyonly_cmp)(const void* x, const void* y) {
    const KEY_T a = KEY_OF((const unsigned char*)x), b = KEY_OF((const unsigned char*)y);
    return KEY_LT(a, b) ? -1 : KEY_LT(b, a) ? 1 : 0;
}

/* sequential IS4o of one subproblem (partition with one thread, explicit task stack) */
static void FN(seq_sort)(FN(Part) * P, size_t lo, size_t hi, uint64_t seed) {
    FN(Task)* st = NULL;
    size_t ns = 0, cap = 0;
    int bad = 0;
    FN(Task) root = {lo, hi};
    if (cap == 0) {
        cap = 1024;
        st = (FN(Task)*)malloc(cap * sizeof(FN(Task)));
    }
    st[ns++] = root;
    while (ns) {
        const FN(Task) tk = st[--ns];
        if (tk.hi - tk.lo <= 16) {
            FN(insertion)(P->a, tk.lo, tk.hi);
            continue;
        }
        P->lo = tk.lo;
        P->hi = tk.hi;
        P->seed = seed ^ (tk.lo * 0x9E3779B97F4A7C15ull);
        FN(partition_team)(P, 0);
        bad = 0;
        FN(emit)(P, &st, &ns, &cap, &bad);
        if (bad) qsort(EL(P->a, tk.lo), tk.hi - tk.lo, ELEM_S, FN(keyonly_cmp));
    }
    free(st);
}

/* The driver: problems of >= n/t elements are partitioned by all t
 * threads one after another; the others are assigned to threads, largest first to the least
 * loaded thread, and sorted sequentially. */
static void FN(sort)(unsigned char* a, size_t n, int t, uint64_t seed) {
    if (n <= 16) {
        FN(insertion)(a, 0, n);
        return;
    }
    if (t < 1) t = 1;
    if (t > MAXT) t = MAXT;
    FN(Task)* big = NULL;
    FN(Task)* small = NULL;
    size_t nbig = 0, capbig = 0, nsmall = 0, capsmall = 0;
    const size_t thr = n / (size_t)t;
    if (t > 1 && n >= thr && n > 1u << 16) {
        big = (FN(Task)*)malloc(sizeof(FN(Task)) * 16);
        capbig = 16;
        big[nbig++] = (FN(Task)){0, n};
        FN(Part)* P = FN(part_new)(a, t);
        while (nbig) {
            const FN(Task) tk = big[--nbig];
            P->lo = tk.lo;
            P->hi = tk.hi;
            P->seed = seed ^ (tk.lo * 0x9E3779B97F4A7C15ull);
#pragma omp parallel num_threads(t)
            FN(partition_team)(P, omp_get_thread_num());
            FN(Task)* ch = NULL;
            size_t nch = 0, capch = 0;
            int bad = 0;
            FN(emit)(P, &ch, &nch, &capch, &bad);
            if (bad) qsort(EL(a, tk.lo), tk.hi - tk.lo, ELEM_S, FN(keyonly_cmp));
            for (size_t c = 0; c < nch; ++c) {
                FN(Task)** v = (ch[c].hi - ch[c].lo >= thr && ch[c].hi - ch[c].lo > 1u << 16) ? &big : &small;
                size_t* nv = v == &big ? &nbig : &nsmall;
                size_t* cp = v == &big ? &capbig : &capsmall;
                if (*nv == *cp) {
                    *cp = *cp ? 2 * *cp : 1024;
                    *v = (FN(Task)*)realloc(*v, *cp * sizeof(FN(Task)));
                }
                (*v)[(*nv)++] = ch[c];
            }
            free(ch);
        }
        FN(part_free)(P);
    } else {
        small = (FN(Task)*)malloc(sizeof(FN(Task)));
        small[nsmall++] = (FN(Task)){0, n};
    }
    /* the remaining problems: largest first, each to the least loaded thread */
    qsort(small, nsmall, sizeof(FN(Task)), FN(task_cmp));
    int* owner = (int*)malloc(sizeof(int) * (nsmall ? nsmall : 1));
    size_t load[MAXT] = {0};
    for (size_t i = 0; i < nsmall; ++i) {
        int best = 0;
        for (int q = 1; q < t; ++q)
            if (load[q] < load[best]) best = q;
        owner[i] = best;
        load[best] += small[i].hi - small[i].lo;
    }
#pragma omp parallel num_threads(t)
    {
        const int me = omp_get_thread_num();
        FN(Part)* Q = FN(part_new)(a, 1);
        for (size_t i = 0; i < nsmall; ++i)
            if (owner[i] == me) FN(seq_sort)(Q, small[i].lo, small[i].hi, seed + i);
        FN(part_free)(Q);
    }
    free(owner);
    free(small);
    free(big);
}

#undef EL
#undef FN
#undef CAT
#undef CAT2
