"""The multi-core CPU IPS4o baseline (cpu_baseline/) against the oracle
(-m "not gpu"): every element type, several thread counts, sizes that reach the parallel
partition (> 2^16 elements), the sequential subproblems, overflow/overhang paths (sizes
that are not multiples of the block), equality buckets and degenerate inputs."""
import numpy as np
import pytest

import cpu_baseline as C
import oracle
import workloads as W

CASES = [("uniform", 0), ("uniform", 1), ("uniform", 17), ("uniform", 1000), ("uniform", 70_001),
         ("uniform", 300_007), ("f64_exponential", 200_003), ("rootdup", 1 << 18), ("twodup", 1 << 18),
         ("eightdup", 1 << 18), ("almostsorted", 1 << 18), ("reversesorted", 1 << 18), ("zeros", 100_000),
         ("ones", 1 << 17), ("sorted", 1 << 18), ("pair16", 250_001), ("rec100", 40_009)]


def _check(et, a, got, exp):
    if et in (W.ELEM_U64, W.ELEM_F64):
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    elif et == W.ELEM_PAIR:
        assert np.array_equal(got[:, 0], exp[:, 0])
        pay = got[:, 1]
        assert np.array_equal(np.sort(pay), np.arange(a.shape[0], dtype=np.uint64))
        assert np.array_equal(a[pay.astype(np.int64), 0], got[:, 0])
    else:
        assert np.array_equal(got[:, :10], exp[:, :10])
        assert np.array_equal(np.sort(got.view("S100").ravel()), np.sort(a.view("S100").ravel()))


@pytest.mark.parametrize("dist,n", CASES, ids=[f"{d}-{n}" for d, n in CASES])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_cpu_ips4o_vs_oracle(dist, n, threads):
    et, a = W.make(dist, n, 2) if n else (W.ELEM_U64, np.zeros(0, np.uint64))
    got = a.copy()
    C.sort_inplace(got, threads)
    _check(et, a, got, oracle.sort(a))
