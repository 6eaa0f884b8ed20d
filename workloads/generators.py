"""Counter-based seeded generators for the synthetic workloads.

Stand-ins for the paper's inputs (§5 "nine input
distributions" and the Pair/100Bytes data types) with the exact recipes of
BASELINE.json's configs and SURVEY.md §8(d) "Generators".  The suites the
paper draws from (shun2012brief, edelkamp2016blockquicksort) are not
reproduced; these are our own definitions of the same shapes.

Base stream:
    u(seed, i) = splitmix64_finalizer(((seed << 32) + i + 1) * GAMMA  mod 2^64)

Element layouts (numpy):
    ELEM_U64     uint64[n]
    ELEM_F64     float64[n]           (no NaN, no -0.0 by construction)
    ELEM_PAIR    uint64[n, 2]         (column 0 = key, column 1 = payload)
    ELEM_REC100  uint8[n, 100]        (bytes [0,10) = key, memcmp order)

Nothing here sorts, classifies or partitions: these functions only produce
inputs.  Both the oracle side and the CUDA side consume them.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "ELEM_U64", "ELEM_F64", "ELEM_PAIR", "ELEM_REC100", "ELEM_PAIR_F64", "ELEM_QUARTET_F64", "ELEM_SIZE",
    "ELEM_NAMES", "pair_f64", "quartet_f64", "quartet_f64_dup",
    "u_stream", "u64_uniform", "f64_uniform", "f64_exponential", "root_dup",
    "two_dup", "eight_dup", "almost_sorted", "reverse_sorted", "sorted_seq", "zeros", "ones",
    "pair16", "rec100", "make", "DISTRIBUTIONS", "CONFIGS",
]

ELEM_U64, ELEM_F64, ELEM_PAIR, ELEM_REC100, ELEM_PAIR_F64, ELEM_QUARTET_F64 = 0, 1, 2, 3, 4, 5
ELEM_SIZE = {ELEM_U64: 8, ELEM_F64: 8, ELEM_PAIR: 16, ELEM_REC100: 100, ELEM_PAIR_F64: 16, ELEM_QUARTET_F64: 32}
ELEM_NAMES = {ELEM_U64: "u64", ELEM_F64: "f64", ELEM_PAIR: "pair16", ELEM_REC100: "rec100",
              ELEM_PAIR_F64: "pair_f64", ELEM_QUARTET_F64: "quartet_f64"}

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_CHUNK = 1 << 23


def _finalize(z: np.ndarray) -> np.ndarray:
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


def u_stream(seed: int, start: int, count: int) -> np.ndarray:
    """u(seed, i) for i in [start, start+count), uint64."""
    out = np.empty(count, dtype=np.uint64)
    base = (np.uint64((seed << 32) & 0xFFFFFFFFFFFFFFFF))
    with np.errstate(over="ignore"):
        for c0 in range(0, count, _CHUNK):
            c1 = min(count, c0 + _CHUNK)
            z = np.arange(start + c0 + 1, start + c1 + 1, dtype=np.uint64)
            z += base
            z *= _GAMMA
            out[c0:c1] = _finalize(z)
    return out


def u64_uniform(n: int, seed: int) -> np.ndarray:
    """Config 1 / headline: A[i] = u(seed, i), i.i.d. uniform over [0, 2^64)."""
    return u_stream(seed, 0, n)


def f64_uniform(n: int, seed: int) -> np.ndarray:
    """Config 2a: A[i] = (u(seed,i) >> 11) * 2^-53, uniform in [0, 1)."""
    u = u_stream(seed, 0, n)
    u >>= np.uint64(11)
    out = u.astype(np.float64)
    out *= 2.0 ** -53
    return out


def f64_exponential(n: int, seed: int) -> np.ndarray:
    """Config 2b: A[i] = -log1p(-U_i), exponential(lambda=1)."""
    out = f64_uniform(n, seed)
    np.negative(out, out=out)
    np.log1p(out, out=out)
    np.negative(out, out=out)
    out += 0.0  # turns any -0.0 into +0.0 (U=0 gives -log1p(-0) = -0.0 -> +0.0)
    return out


def root_dup(n: int, seed: int = 0) -> np.ndarray:
    """RootDup: A[i] = i mod floor(sqrt n) (PAPER.md:445, 0-based i)."""
    r = math.isqrt(n) if n > 0 else 1
    return (np.arange(n, dtype=np.uint64) % np.uint64(max(r, 1))).astype(np.uint64)


def _pow_dup(n: int, power: int) -> np.ndarray:
    # (i^power + n/2) mod n with wrapping u64 arithmetic; exact for n = 2^e.
    out = np.empty(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for c0 in range(0, n, _CHUNK):
            c1 = min(n, c0 + _CHUNK)
            i = np.arange(c0, c1, dtype=np.uint64)
            p = i.copy()
            for _ in range(power - 1):
                p *= i
            p += np.uint64(n // 2)
            if n & (n - 1) == 0:
                p &= np.uint64(n - 1)
            else:
                p %= np.uint64(n)
            out[c0:c1] = p
    return out


def two_dup(n: int, seed: int = 0) -> np.ndarray:
    """TwoDup: A[i] = (i^2 + n/2) mod n."""
    return _pow_dup(n, 2)


def eight_dup(n: int, seed: int = 0) -> np.ndarray:
    """EightDup: A[i] = (i^8 + n/2) mod n."""
    return _pow_dup(n, 8)


def almost_sorted(n: int, seed: int) -> np.ndarray:
    """AlmostSorted: A[i] = i, then floor(sqrt n) sequential seeded swaps."""
    a = np.arange(n, dtype=np.uint64)
    if n == 0:
        return a
    s = math.isqrt(n)
    u = u_stream(seed, 0, 2 * s)
    idx = (u % np.uint64(n)).astype(np.int64)
    for j in range(s):
        x, y = idx[2 * j], idx[2 * j + 1]
        a[x], a[y] = a[y], a[x]
    return a


def reverse_sorted(n: int, seed: int = 0) -> np.ndarray:
    """ReverseSorted: A[i] = n-1-i."""
    return np.arange(n - 1, -1, -1, dtype=np.uint64) if n else np.zeros(0, np.uint64)


def sorted_seq(n: int, seed: int = 0) -> np.ndarray:
    return np.arange(n, dtype=np.uint64)


def zeros(n: int, seed: int = 0) -> np.ndarray:
    """all-zero (BASELINE config 3's stand-in for the paper's Ones)."""
    return np.zeros(n, dtype=np.uint64)


def ones(n: int, seed: int = 0) -> np.ndarray:
    return np.ones(n, dtype=np.uint64)


def pair16(n: int, seed: int) -> np.ndarray:
    """Config 4: key = u(seed,i) >> 32 (uniform [0,2^32)), payload = i. uint64[n,2]."""
    out = np.empty((n, 2), dtype=np.uint64)
    out[:, 0] = u_stream(seed, 0, n) >> np.uint64(32)
    out[:, 1] = np.arange(n, dtype=np.uint64)
    return out


def rec100(n: int, seed: int) -> np.ndarray:
    """Config 5: record i = 13 LE words u(seed+1000, 13i+w), truncated to 100 bytes."""
    out = np.empty((n, 100), dtype=np.uint8)
    step = max(1, _CHUNK // 13)
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        w = u_stream(seed + 1000, 13 * r0, 13 * (r1 - r0)).reshape(r1 - r0, 13)
        out[r0:r1] = w.view(np.uint8).reshape(r1 - r0, 104)[:, :100]
    return out


def pair_f64(n: int, seed: int) -> np.ndarray:
    """The paper's Pair: f64 key uniform [0,1) = (u(seed,i) >> 11) * 2^-53,
    f64 payload = i (exact below 2^53).  float64[n,2]."""
    out = np.empty((n, 2), dtype=np.float64)
    out[:, 0] = f64_uniform(n, seed)
    out[:, 1] = np.arange(n, dtype=np.float64)
    return out


def _f64_stream(seed: int, start: int, n: int) -> np.ndarray:
    return (u_stream(seed, start, n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def quartet_f64(n: int, seed: int) -> np.ndarray:
    """The paper's Quartet: three f64 keys, each uniform [0,1) from its own
    stretch of the seed's stream (k_j = f64 rule at index j*n + i), compared
    lexicographically; f64 payload = i.  float64[n,4]."""
    out = np.empty((n, 4), dtype=np.float64)
    for j in range(3):
        out[:, j] = _f64_stream(seed + 2000, j * n, n)
    out[:, 3] = np.arange(n, dtype=np.float64)
    return out


def quartet_f64_dup(n: int, seed: int) -> np.ndarray:
    """Quartet with duplicate-heavy leading keys (test input for the lexicographic order):
    k0 in 64 values, k1 in 16 values (both in [-0.5, 0.5), nonzero), k2 uniform [0,1)."""
    out = quartet_f64(n, seed)
    out[:, 0] = np.floor(out[:, 0] * 64.0) / 64.0 - 0.4921875
    out[:, 1] = np.floor(out[:, 1] * 16.0) / 16.0 - 0.46875
    return out


DISTRIBUTIONS = {
    "uniform": (ELEM_U64, u64_uniform),
    "f64_uniform": (ELEM_F64, f64_uniform),
    "f64_exponential": (ELEM_F64, f64_exponential),
    "rootdup": (ELEM_U64, root_dup),
    "twodup": (ELEM_U64, two_dup),
    "eightdup": (ELEM_U64, eight_dup),
    "almostsorted": (ELEM_U64, almost_sorted),
    "reversesorted": (ELEM_U64, reverse_sorted),
    "sorted": (ELEM_U64, sorted_seq),
    "zeros": (ELEM_U64, zeros),
    "ones": (ELEM_U64, ones),
    "pair16": (ELEM_PAIR, pair16),
    "rec100": (ELEM_REC100, rec100),
    "pair_f64": (ELEM_PAIR_F64, pair_f64),
    "quartet_f64": (ELEM_QUARTET_F64, quartet_f64),
    "quartet_f64_dup": (ELEM_QUARTET_F64, quartet_f64_dup),
}

# BASELINE.json configs (name -> (distribution, log2 n)); "H" is the headline.
CONFIGS = {
    "H_u64_2p28": [("uniform", 28)],
    "C1_u64_2p20": [("uniform", 20)],
    "C2_f64_2p28": [("f64_uniform", 28), ("f64_exponential", 28)],
    "C3_dup_2p27": [("rootdup", 27), ("twodup", 27), ("eightdup", 27),
                    ("almostsorted", 27), ("reversesorted", 27), ("zeros", 27)],
    "C4_pair16_2p27": [("pair16", 27)],
    "C5_rec100_2p24": [("rec100", 24)],
}


def make(dist: str, n: int, seed: int = 1):
    """(elem_type, array) for a named distribution."""
    et, fn = DISTRIBUTIONS[dist]
    return et, fn(n, seed)
