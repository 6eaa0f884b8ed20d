/* ips4o_cpu.c -- multi-core CPU IPS4o ("parallel CPU IPS4o baseline, t
 * host threads, OpenMP-style").  A reported baseline for bench.py,
 * not the oracle (oracle/ is the sequential checker) and not the product path.
 *
 *   int ips4o_cpu_sort(void* a, uint64_t n, int elem_type, int threads);
 *     elem_type 0 u64, 1 f64 (no NaN / -0.0), 2 pair16 {u64 key, u64 payload}, 3 rec100
 *     (10-byte memcmp key); sorts a[0..n) in place in host memory; returns 0, or -1 for a
 *     bad type.
 *
 * Block size b = max(1, 2^floor(11 - log2 s)) elements (about 2 KiB),
 * k <= 256 buckets, alpha = 0.2 log n, n0 = 16.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXKB 256
#define MAXT 64

static inline uint64_t ld64(const unsigned char* p) {
    uint64_t x;
    memcpy(&x, p, 8);
    return x;
}

/* ---- u64 (also f64 through the order-preserving image) */
#define ELEM_S 8
#define BLK 256
#define SUFFIX u64
#define KEY_T uint64_t
#define KEY_OF(p) ld64((const unsigned char*)(p))
#define KEY_LT(a, b) ((a) < (b))
#define KEY_EQ(a, b) ((a) == (b))
#include "ips4o_cpu_impl.h"
#undef ELEM_S
#undef BLK
#undef SUFFIX

/* ---- pair16: key = the first u64 */
#define ELEM_S 16
#define BLK 128
#define SUFFIX pair
#include "ips4o_cpu_impl.h"
#undef ELEM_S
#undef BLK
#undef SUFFIX
#undef KEY_T
#undef KEY_OF
#undef KEY_LT
#undef KEY_EQ

/* ---- rec100: key = bytes [0,10) in memcmp order = (big-endian u64 of bytes 0..7, u16 of 8..9) */
typedef struct {
    uint64_t hi;
    uint32_t lo;
} reckey;
static inline reckey rec_key(const unsigned char* p) {
    reckey k;
    k.hi = __builtin_bswap64(ld64(p));
    k.lo = ((uint32_t)p[8] << 8) | p[9];
    return k;
}
#define ELEM_S 100
#define BLK 16
#define SUFFIX rec
#define KEY_T reckey
#define KEY_OF(p) rec_key((const unsigned char*)(p))
#define KEY_LT(a, b) ((a).hi < (b).hi || ((a).hi == (b).hi && (a).lo < (b).lo))
#define KEY_EQ(a, b) ((a).hi == (b).hi && (a).lo == (b).lo)
#include "ips4o_cpu_impl.h"

static void f64_to_key(uint64_t* a, uint64_t n, int t) {
#pragma omp parallel for num_threads(t) schedule(static)
    for (uint64_t i = 0; i < n; ++i) a[i] = (a[i] >> 63) ? ~a[i] : (a[i] | 0x8000000000000000ull);
}
static void key_to_f64(uint64_t* a, uint64_t n, int t) {
#pragma omp parallel for num_threads(t) schedule(static)
    for (uint64_t i = 0; i < n; ++i) a[i] = (a[i] >> 63) ? (a[i] & 0x7FFFFFFFFFFFFFFFull) : ~a[i];
}

int ips4o_cpu_sort(void* a, uint64_t n, int elem_type, int threads) {
    if (threads < 1) threads = omp_get_max_threads();
    const uint64_t seed = 0x5EED5EEDull;
    switch (elem_type) {
        case 0: sort_u64((unsigned char*)a, n, threads, seed); return 0;
        case 1:
            f64_to_key((uint64_t*)a, n, threads);
            sort_u64((unsigned char*)a, n, threads, seed);
            key_to_f64((uint64_t*)a, n, threads);
            return 0;
        case 2: sort_pair((unsigned char*)a, n, threads, seed); return 0;
        case 3: sort_rec((unsigned char*)a, n, threads, seed); return 0;
        default: return -1;
    }
}

int ips4o_cpu_max_threads(void) { return omp_get_max_threads(); }
