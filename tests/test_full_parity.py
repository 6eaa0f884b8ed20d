"""Element-by-element oracle parity at the full BASELINE.json sizes (-m gpu).

Every config of BASELINE.json (and the north star's headline H) is sorted on the GPU in the
launch configuration bench.py times (one ips4o_sort of the whole array, default stream of
the binding) and compared with oracle.sort -- the paper's sequential IS4o --
on the same seeded input:
  * u64 / f64: the output array equals the oracle's, bit for bit;
  * Pair16 (C4): the key column equals the oracle's; the payloads are a permutation of
    0..n-1 and every output record carries the key of its original index
    (in[payload].key == out.key), which pins the record multiset exactly;
  * Rec100 (C5): the key bytes equal the oracle's; every record whose key is unique is
    equal (all 100 bytes) to the oracle's record at the same position, and the records of
    equal-key runs form the same multiset (the sort is unstable).
Sizes between the small parity cases and the headline (2^23..2^25) reach the 8192-key
sample of K1 and multi-stripe level-2 tasks.

The oracle needs ~35 s for 2^28 elements on one host core, so the oracle results are
computed in a small thread pool (the C oracle releases the GIL) a few configs ahead of the
test that consumes them.
"""
import concurrent.futures as cf
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_1705_02257_b200 as ips4o  # noqa: E402
import workloads as W  # noqa: E402
from gpu_util import check_equal_to_oracle, to_dev, to_host  # noqa: E402

# (distribution, log2 n, seed)
FULL = [
    ("uniform", 28, 1),            # H (headline)
    ("uniform", 20, 1),            # C1
    ("f64_uniform", 28, 1),        # C2a
    ("f64_exponential", 28, 1),    # C2b
    ("rootdup", 27, 1), ("twodup", 27, 1), ("eightdup", 27, 1),   # C3
    ("almostsorted", 27, 1), ("reversesorted", 27, 1), ("zeros", 27, 1),
    ("sorted", 27, 1), ("ones", 27, 1),                          # f3: Sorted, Ones
    ("pair16", 27, 1),             # C4
    ("rec100", 24, 1),             # C5
    ("uniform", 23, 2), ("uniform", 24, 3), ("uniform", 25, 2),  # K1 8192-key sample, 2-stripe level-2 tasks
    ("f64_exponential", 25, 3),
    ("pair_f64", 27, 1),           # f3: the paper's Pair (f64 key + payload)
    ("quartet_f64", 26, 1),        # f3: the paper's Quartet (three f64 keys + payload)
    ("quartet_f64_dup", 24, 1),    #     with duplicate-heavy leading keys
]
IDS = [f"{d}-2^{e}-s{s}" for d, e, s in FULL]
LOOKAHEAD = 2
WORKERS = max(1, min(3, (os.cpu_count() or 2) - 1))


class _OracleAhead:
    """Oracle results for FULL, computed a few configs ahead of their test."""

    def __init__(self):
        self.pool = cf.ThreadPoolExecutor(max_workers=WORKERS)
        self.fut = {}
        self.lock = threading.Lock()

    @staticmethod
    def _job(dist, e, seed):
        _, a = W.make(dist, 1 << e, seed)
        return oracle.sort(a)

    def _submit(self, i):
        if 0 <= i < len(FULL) and i not in self.fut:
            self.fut[i] = self.pool.submit(self._job, *FULL[i])

    def get(self, i):
        with self.lock:
            for j in range(i, i + LOOKAHEAD + 1):
                self._submit(j)
            f = self.fut[i]
        r = f.result()
        with self.lock:
            del self.fut[i]
        return r


@pytest.fixture(scope="module")
def ahead():
    ips4o.lib()
    torch.cuda.set_device(0)
    o = _OracleAhead()
    yield o
    o.pool.shutdown(wait=True, cancel_futures=True)


def _check_pair(inp, got, exp):
    assert np.array_equal(got[:, 0], exp[:, 0]), "Pair16 key sequence differs from the oracle"
    pay = got[:, 1]
    n = inp.shape[0]
    assert np.array_equal(np.sort(pay), np.arange(n, dtype=np.uint64)), "payloads are not a permutation"
    assert np.array_equal(inp[pay.astype(np.int64), 0], got[:, 0]), "a record lost its key"


def _check_rec(got, exp):
    assert np.array_equal(got[:, :10], exp[:, :10]), "Rec100 key sequence differs from the oracle"
    key = np.ascontiguousarray(got[:, :10]).view("S10").ravel()
    same_prev = np.zeros(key.shape[0], bool)
    same_prev[1:] = key[1:] == key[:-1]
    dup = same_prev.copy()
    dup[:-1] |= same_prev[1:]
    uniq = ~dup
    assert np.array_equal(got[uniq], exp[uniq]), "a record with a unique key differs from the oracle's"
    if dup.any():
        g = np.sort(np.ascontiguousarray(got[dup]).view("S100").ravel())
        e = np.sort(np.ascontiguousarray(exp[dup]).view("S100").ravel())
        assert np.array_equal(g, e), "records of equal-key runs differ from the oracle's multiset"


def test_full_size_sort_kv_vs_oracle():
    """ips4o_sort_kv at the C4 size (2^27): u64 keys uniform in [0, 2^32) (duplicates), values =
    index; keys vs the oracle's key sort, every (key, value) pair preserved."""
    n = 1 << 27
    a = W.pair16(n, 2)
    keys = np.ascontiguousarray(a[:, 0])
    exp = oracle.sort(keys)
    dk = to_dev(keys, W.ELEM_U64)
    dv = torch.from_numpy(np.ascontiguousarray(a[:, 1]).view(np.int64)).cuda()
    ips4o.sort_kv_(dk, dv)
    torch.cuda.synchronize()
    assert ips4o.ips4o_last_stats()["device_error"] == 0
    gk = to_host(dk, W.ELEM_U64)
    gv = dv.cpu().numpy().view(np.uint64)
    assert np.array_equal(gk, exp)
    assert np.array_equal(np.sort(gv), np.arange(n, dtype=np.uint64))
    assert np.array_equal(keys[gv.astype(np.int64)], gk)


@pytest.mark.parametrize("i", range(len(FULL)), ids=IDS)
def test_full_size_vs_oracle(ahead, i):
    dist, e, seed = FULL[i]
    et, a = W.make(dist, 1 << e, seed)
    t = to_dev(a, et)
    ips4o.sort_(t)
    torch.cuda.synchronize()
    st = ips4o.ips4o_last_stats()
    assert st["device_error"] == 0, st
    got = to_host(t, et)
    del t
    exp = ahead.get(i)
    if et in (W.ELEM_U64, W.ELEM_F64):
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64)), f"{dist} 2^{e}: differs from the oracle"
    elif et == W.ELEM_PAIR:
        _check_pair(a, got, exp)
    elif et == W.ELEM_REC100:
        _check_rec(got, exp)
    else:
        check_equal_to_oracle(et, a, got, exp)
