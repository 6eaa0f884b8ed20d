"""Randomised stress run of the sort on the GPU (robustness evidence, not a unit test):
random sizes, distributions, element types and misaligned starts; every output is checked
for sortedness and an unchanged multiset digest.

    python tools/stress.py --iters 200 --seed 7 --max-log2 24
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import workloads as W  # noqa: E402
import paper_1705_02257_b200 as ips4o  # noqa: E402
from gpu_util import to_dev, digest, keys_nondecreasing  # noqa: E402

DISTS = ["uniform", "f64_uniform", "f64_exponential", "rootdup", "twodup", "eightdup", "almostsorted",
         "reversesorted", "sorted", "zeros", "ones", "pair16", "rec100", "pair_f64", "quartet_f64", "quartet_f64_dup"]
WIDE_F64 = (W.ELEM_PAIR_F64, W.ELEM_QUARTET_F64)


def host_check(before: np.ndarray, after: np.ndarray, et: int) -> bool:
    """pair_f64 / quartet_f64 (float64 rows): keys non-decreasing in the type's order (Pair:
    column 0; Quartet: columns 0-2 lexicographically) and the rows a permutation of the input."""
    nk = 1 if et == W.ELEM_PAIR_F64 else 3
    k = after[:, :nk]
    if len(k) > 1:
        lt = np.zeros(len(k) - 1, bool)
        eq = np.ones(len(k) - 1, bool)
        for c in range(nk):
            lt |= eq & (k[1:, c] > k[:-1, c])
            eq &= k[1:, c] == k[:-1, c]
        if not (lt | eq).all():
            return False
    def canon(a):
        return a[np.lexsort(a.T[::-1])]
    return np.array_equal(canon(before), canon(after))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--max-log2", type=int, default=24)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t0 = time.time()
    bad = 0
    for it in range(a.iters):
        dist = DISTS[int(rng.integers(len(DISTS)))]
        top = a.max_log2 - (4 if dist == "rec100" else 2 if dist.startswith(("pair_f64", "quartet")) else 0)
        n = int(2 ** rng.uniform(0, top))
        off = int(rng.integers(0, 3))           # elements before the sorted range
        et, arr = W.make(dist, n + off, int(rng.integers(1, 1 << 30)))
        t = to_dev(arr, et)
        sub = t[off:]
        if et in WIDE_F64:
            before = sub.cpu().numpy().copy()
            head = t[:off].clone()
            ips4o.sort_(sub)
            torch.cuda.synchronize()
            ok = host_check(before, sub.cpu().numpy(), et) and bool((t[:off] == head).all().item())
        else:
            before = digest(sub)
            head = t[:off].clone()
            ips4o.sort_(sub)
            torch.cuda.synchronize()
            ok = keys_nondecreasing(sub, et) and digest(sub) == before and bool((t[:off] == head).all().item())
        if not ok:
            bad += 1
            print(f"FAIL iter {it}: dist={dist} n={n} off={off}", flush=True)
    print(f"stress: {a.iters} sorts, {bad} failures, {time.time() - t0:.1f} s", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
