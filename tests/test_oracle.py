"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/ips4o_oracle.c) is checked here against things other than
itself: numpy.sort (sorting has a unique key sequence), brute force over all
permutations / all {0,1,2}^n inputs, the linear-scan definition of a bucket
(PAPER.md:137), the SPEC.md worked examples (tests/golden/spec_examples.json),
invariants (sortedness, permutation, idempotence, multiset conservation per
bucket) and special cases (all-equal => one partition step).
The tiny-parameter runs (k_max=4, b in {1,2,3}, n0 in {1,2}, debug=1) force
sampling, block flushes, the overflow block, overhangs and equality buckets
on inputs small enough to enumerate, and assert the three-zone invariant
 after every permutation step.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ----------------------------------------------------------------- brute force

def _perm_rows(n):
    return np.array(list(itertools.permutations(range(n))), dtype=np.uint64).reshape(-1, n)


@pytest.mark.parametrize("b", [1, 2, 3])
@pytest.mark.parametrize("n0", [1, 2])
def test_all_permutations_up_to_7(b, n0):
    p = oracle.params(W.ELEM_U64, k_max=4, b=b, n0=n0, debug=True)
    st = oracle.Stats()
    for n in range(0, 8):
        rows = _perm_rows(n) if n > 0 else np.zeros((1, 0), np.uint64)
        if n == 0:
            continue
        out = oracle.sort_rows(W.ELEM_U64, rows, p, st)
        assert np.array_equal(out, np.sort(rows, axis=1)), (n, b, n0)
    assert st.partition_steps > 0 and st.invariant_checks > 0


def test_all_permutations_8():
    rows = _perm_rows(8)
    for b, n0 in [(1, 1), (3, 2)]:
        p = oracle.params(W.ELEM_U64, k_max=4, b=b, n0=n0, debug=True)
        out = oracle.sort_rows(W.ELEM_U64, rows, p)
        assert np.array_equal(out, np.sort(rows, axis=1))


@pytest.mark.parametrize("b", [1, 2, 3])
@pytest.mark.parametrize("n0", [1, 2])
def test_all_ternary_sequences_up_to_8(b, n0):
    """All {0,1,2}^n: duplicates -> equality buckets, tiny buckets, overhangs."""
    p = oracle.params(W.ELEM_U64, k_max=4, b=b, n0=n0, debug=True)
    st = oracle.Stats()
    for n in range(1, 9):
        rows = np.array(list(itertools.product(range(3), repeat=n)), dtype=np.uint64)
        out = oracle.sort_rows(W.ELEM_U64, rows, p, st)
        assert np.array_equal(out, np.sort(rows, axis=1)), (n, b, n0)
    assert st.eq_steps > 0
    if b == 3:   # with b in {1,2} and n <= 8 no block straddles a boundary / the end
        assert st.overhang_uses > 0
        assert st.overflow_uses > 0


def _insertion_sort(xs):
    xs = list(xs)
    for i in range(1, len(xs)):
        v, j = xs[i], i
        while j > 0 and v < xs[j - 1]:
            xs[j] = xs[j - 1]
            j -= 1
        xs[j] = v
    return xs


def test_random_small_vs_insertion_sort():
    rng = np.random.default_rng(7)
    for _ in range(2000):
        n = int(rng.integers(0, 17))
        a = rng.integers(0, int(rng.choice([2, 5, 1 << 20])), size=n).astype(np.uint64)
        p = oracle.params(W.ELEM_U64, k_max=4, b=int(rng.integers(1, 4)), n0=int(rng.integers(1, 3)), debug=True)
        assert list(oracle.sort(a, p)) == _insertion_sort(a)


def test_random_matrix_with_block_machinery():
    """SURVEY §8(c) O-text validation matrix: n < 3000, k_max up to 256, b up to 32."""
    rng = np.random.default_rng(11)
    tot = oracle.Stats()
    for it in range(300):
        n = int(rng.integers(0, 3000))
        kind = it % 6
        if kind == 0:
            a = rng.integers(0, 1 << 62, size=n, dtype=np.uint64)
        elif kind == 1:
            a = rng.integers(0, 5, size=n).astype(np.uint64)
        elif kind == 2:
            a = rng.integers(0, 50, size=n).astype(np.uint64)
        elif kind == 3:
            a = np.arange(n, dtype=np.uint64)
        elif kind == 4:
            a = np.arange(n, dtype=np.uint64)[::-1].copy()
        else:
            a = np.full(n, 9, dtype=np.uint64)
        p = oracle.params(W.ELEM_U64, k_max=int(rng.choice([4, 8, 16, 256])),
                          b=int(rng.integers(1, 33)), n0=int(rng.choice([1, 2, 16])),
                          seed=int(rng.integers(1, 1 << 30)), debug=n < 600)
        st = oracle.Stats()
        out = oracle.sort(a, p, st)
        assert np.array_equal(out, np.sort(a)), (it, n)
        for f in ("overflow_uses", "overhang_uses", "eq_steps", "invariant_checks"):
            setattr(tot, f, getattr(tot, f) + getattr(st, f))
    assert tot.overflow_uses > 0 and tot.overhang_uses > 0 and tot.eq_steps > 0
    assert tot.invariant_checks > 0


# ------------------------------------------------- element types, full sizes

def _check_types(et, a, out):
    if et == W.ELEM_PAIR:
        n = a.shape[0]
        assert np.array_equal(out[:, 0], np.sort(a[:, 0]))
        pay = out[:, 1].astype(np.int64)
        assert np.array_equal(np.sort(pay), np.arange(n))            # payloads are a permutation
        assert np.array_equal(a[pay, 0], out[:, 0])                  # and travel with their keys
    elif et == W.ELEM_REC100:
        kin = np.sort(a[:, :10].copy().view("S10").ravel())
        kout = out[:, :10].copy().view("S10").ravel()
        assert np.array_equal(kin, kout)                             # key sequence bit-exact
        ri = np.sort(a.view("S100").ravel())
        ro = np.sort(out.view("S100").ravel())
        assert np.array_equal(ri, ro)                                # record multiset equal
    else:
        assert np.array_equal(out.view(np.uint64), np.sort(a).view(np.uint64))


@pytest.mark.parametrize("dist", ["uniform", "f64_uniform", "f64_exponential", "rootdup", "twodup",
                                  "eightdup", "almostsorted", "reversesorted", "zeros", "pair16", "rec100"])
def test_distributions_default_params(dist):
    n = 1 << 16 if dist != "rec100" else 1 << 14
    for seed in (1, 2, 3):
        et, a = W.make(dist, n, seed)
        p = oracle.default_params(et)
        p.seed = seed
        out = oracle.sort(a, p)
        _check_types(et, a, out)


def test_config1_full_size_u64():
    """BASELINE config 1 (2^20 uniform u64) at full size against numpy.sort."""
    a = W.u64_uniform(1 << 20, 1)
    assert np.array_equal(oracle.sort(a), np.sort(a))


@pytest.mark.parametrize("et", [W.ELEM_U64, W.ELEM_F64, W.ELEM_PAIR, W.ELEM_REC100])
def test_types_small_blocks_debug(et):
    n = 5000
    a = {W.ELEM_U64: W.u64_uniform, W.ELEM_F64: W.f64_exponential,
         W.ELEM_PAIR: W.pair16, W.ELEM_REC100: W.rec100}[et](n, 5)
    if et == W.ELEM_PAIR:
        a[:, 0] >>= np.uint64(24)   # many duplicate keys -> equality buckets with payloads
    p = oracle.params(et, k_max=16, b=7, n0=4, debug=True)
    st = oracle.Stats()
    out = oracle.sort(a, p, st)
    _check_types(et, a, out)
    assert st.invariant_checks > 0


# --------------------------------------------------------------- degenerate

@pytest.mark.parametrize("n", [0, 1, 2, 3, 255, 256, 257, 511, 4095, 4096, 4097, 65535, 65537])
def test_degenerate_sizes_and_shapes(n):
    b = oracle.default_block(W.ELEM_U64)
    for a in (np.zeros(n, np.uint64), np.arange(n, dtype=np.uint64),
              np.arange(n, dtype=np.uint64)[::-1].copy(),
              (np.arange(n, dtype=np.uint64) % np.uint64(2)),
              W.u64_uniform(n, 3)):
        out = oracle.sort(a)
        assert np.array_equal(out, np.sort(a))
        assert np.array_equal(oracle.sort(out), out)    # idempotence
    assert b == 256


def test_max_key_values():
    a = np.array([np.iinfo(np.uint64).max, 0, np.iinfo(np.uint64).max, 1] * 1000, dtype=np.uint64)
    assert np.array_equal(oracle.sort(a), np.sort(a))


def test_all_equal_is_one_partition_step():
    """Equality buckets make an all-equal input 'easy': 1 step."""
    st = oracle.Stats()
    a = np.zeros(100_000, dtype=np.uint64)
    out = oracle.sort(a, stats=st)
    assert np.array_equal(out, a)
    assert st.partition_steps == 1 and st.eq_steps == 1


def test_eightdup_enables_equality_buckets_at_level_one():
    st = oracle.Stats()
    a = W.eight_dup(1 << 20)
    oracle.sort(a, stats=st)
    assert st.eq_steps >= 1


# ------------------------------------------------------ classifier pins

def _linear_scan(spl_padded, eq, e):
    """Definition: i with s_{i-1} <= e < s_i; equality bucket via e == s_i
    (PAPER.md:341).  spl_padded = s_1..s_{k'-1} (largest repeated, S6)."""
    i = sum(1 for s in spl_padded if s <= e)
    if not eq:
        return i
    if i >= 1 and spl_padded[i - 1] == e:
        return 2 * i - 1
    return 2 * i


def _pad(spl):
    kp = 2
    while kp < len(spl) + 1:
        kp *= 2
    return list(spl) + [spl[-1]] * (kp - 1 - len(spl))


def test_classify_exhaustive_small_k():
    rng = np.random.default_rng(3)
    dom = np.arange(64, dtype=np.uint64)
    for _ in range(400):
        nspl = int(rng.integers(1, 8))
        spl = np.sort(rng.choice(64, size=nspl, replace=False)).astype(np.uint64)
        for eq in (False, True):
            got = oracle.classify(spl, eq, dom)
            exp = [_linear_scan(_pad([int(x) for x in spl]), eq, int(e)) for e in dom]
            assert list(got) == exp


def test_classify_k256_random_and_monotone():
    rng = np.random.default_rng(4)
    for eq in (False, True):
        nspl = 255 if not eq else 127
        spl = np.unique(rng.integers(0, 1 << 40, size=nspl * 2, dtype=np.uint64))[:nspl]
        e = np.concatenate([rng.integers(0, 1 << 40, size=20000, dtype=np.uint64), spl])
        got = oracle.classify(spl, eq, e)
        sp = _pad([int(x) for x in spl])
        exp = [_linear_scan(sp, eq, int(x)) for x in e]
        assert list(got) == exp
        order = np.argsort(e, kind="stable")
        assert np.all(np.diff(got[order].astype(np.int64)) >= 0)   # monotone in e


def test_classify_spec_examples():
    g = GOLD["classify_10_20_30"]
    spl = np.array(g["splitters"], dtype=np.uint64)
    for e, eq, exp in g["cases"]:
        assert oracle.classify(spl, eq, np.array([e], np.uint64))[0] == exp
    # equality on, e = 20 lands in the equality bucket of splitter s_2 = 20 (index 2*2-1)
    assert oracle.classify(spl, True, np.array([20], np.uint64))[0] == 3


def test_classify_f64_and_rec100_orders():
    spl = np.array([-1.5, 0.25, 3.0], dtype=np.float64)
    e = np.array([-2.0, -1.5, 0.0, 0.25, 2.9, 3.0, 1e300], dtype=np.float64)
    assert list(oracle.classify(spl, False, e)) == [0, 1, 1, 2, 2, 3, 3]
    recs = np.zeros((3, 100), np.uint8)
    recs[0, :10] = list(b"\x00" * 9 + b"\x05")
    recs[1, :10] = list(b"\x00" * 9 + b"\xff")
    recs[2, :10] = list(b"\x01" + b"\x00" * 9)
    spl_r = recs[1:2].copy()
    assert list(oracle.classify(spl_r, False, recs)) == [0, 1, 1]


@pytest.mark.parametrize("name", ["tree_k8", "tree_k4", "tree_k2"])
def test_tree_layout_spec(name):
    g = GOLD[name]
    tree, kp = oracle.build_tree(np.array(g["splitters"], np.uint64))
    assert list(tree) == g["tree"]


def test_tree_inorder_is_splitters():
    rng = np.random.default_rng(5)
    for nspl in (1, 3, 7, 15, 31, 63, 127, 255):
        spl = np.sort(rng.choice(1 << 30, size=nspl, replace=False)).astype(np.uint64)
        tree, kp = oracle.build_tree(spl)
        out = []

        def rec(j):
            if j >= kp:
                return
            rec(2 * j)
            out.append(int(tree[j - 1]))
            rec(2 * j + 1)
        rec(1)
        assert out == [int(x) for x in spl]


@pytest.mark.parametrize("name", ["pick_1_15", "pick_all_7", "pick_dups"])
def test_select_splitters_spec(name):
    g = GOLD[name]
    spl, eq = oracle.select_splitters(np.array(g["sample"], np.uint64), g["k"], g["alpha"])
    assert list(spl) == g["splitters"] and eq == g["eq"]


def test_parameter_formulas():
    g = GOLD["default_config"]
    assert oracle.alpha(1 << 20) == g["alpha_2p20"]
    assert oracle.default_block(W.ELEM_U64) == g["b_s8"]
    assert oracle.default_block(W.ELEM_REC100) == g["b_s100"]
    assert oracle.default_block(W.ELEM_PAIR) == 128
    # alpha at the config sizes
    assert [oracle.alpha(1 << e) for e in (24, 27, 28)] == [5, 5, 6]
    assert oracle.bucket_count(1 << 28) == 256 and oracle.bucket_count(100) == 4


# --------------------------------------------------- one level: partition_with

def _check_partition(a, out, bounds, spl, eq):
    K = len(bounds) - 1
    assert bounds[0] == 0 and bounds[-1] == a.shape[0]
    cls_in = oracle.classify(spl, eq, a)
    # e_i is the prefix sum of the bucket histogram: a closed form
    hist = np.bincount(cls_in.astype(np.int64), minlength=K)
    assert np.array_equal(np.diff(bounds), hist[:K])
    cls_out = oracle.classify(spl, eq, out)
    for i in range(K):
        seg = cls_out[bounds[i]:bounds[i + 1]]
        assert np.all(seg == i)                      # every element of [e_i, e_{i+1}) is in bucket i
    assert np.array_equal(np.sort(out), np.sort(a))  # multiset conserved


def test_partition_with_random():
    rng = np.random.default_rng(8)
    for it in range(150):
        n = int(rng.integers(0, 4000))
        a = rng.integers(0, int(rng.choice([7, 100, 1 << 40])), size=n).astype(np.uint64)
        eq = bool(it % 2)
        nspl = int(rng.integers(1, 128 if eq else 256))
        cand = np.unique(rng.integers(0, int(a.max()) + 2 if n else 10, size=nspl).astype(np.uint64))
        b = int(rng.integers(1, 40))
        out, bounds = oracle.partition_with(a, cand, eq, b, debug=n < 1500)
        _check_partition(a, out, bounds, cand, eq)


def test_partition_delimiter_example_bounds():
    """b=4, counts {5,7,4} -> e=[0,5,12,16]."""
    g = GOLD["delimiters"]
    a = np.array([0] * 5 + [1] * 7 + [2] * 4, dtype=np.uint64)
    rng = np.random.default_rng(1)
    rng.shuffle(a)
    out, bounds = oracle.partition_with(a, np.array([1, 2, 3], np.uint64), False, g["b"], debug=True)
    assert list(bounds[:4]) == g["e"]   # k'=4: the fourth bucket [3, inf) is empty
    assert bounds[4] == 16


# ------------------------------------------------------------ generators

def test_generator_examples():
    assert list(W.root_dup(16)) == GOLD["rootdup_16"]["values"]
    assert list(W.two_dup(8)) == GOLD["twodup_8"]["values"]


def test_generators_deterministic_and_clean():
    for d in W.DISTRIBUTIONS:
        _, a1 = W.make(d, 4096, 2)
        _, a2 = W.make(d, 4096, 2)
        assert np.array_equal(a1, a2)
    for f in (W.f64_uniform, W.f64_exponential):
        x = f(1 << 20, 1)
        assert not np.isnan(x).any()
        assert not np.any((x == 0) & np.signbit(x))
        assert x.min() >= 0
    u = W.u_stream(1, 0, 4)
    assert u[0] != W.u_stream(0, 1, 1)[0]   # seeds do not alias at shifted indices
    assert len(np.unique(W.eight_dup(1 << 20))) < (1 << 20)


# ------------------------------- the paper's Pair and Quartet (f64 keys)

def _check_f64_records(et, a, out):
    """Pair (key, payload) / Quartet (k0, k1, k2, payload): the key sequence equals the
    lexicographic sort of the input's keys (numpy.lexsort, a library routine: the key sequence
    is unique), and the payloads (original indices) are a permutation that carries each
    record's keys."""
    nk = 1 if et == W.ELEM_PAIR_F64 else 3
    keys = a[:, :nk]
    order = np.lexsort(tuple(keys[:, j] for j in reversed(range(nk))))
    assert np.array_equal(out[:, :nk].view(np.uint64), keys[order].view(np.uint64))
    pay = out[:, nk].astype(np.int64)
    assert np.array_equal(np.sort(pay), np.arange(a.shape[0]))
    assert np.array_equal(a[pay, :nk].view(np.uint64), out[:, :nk].view(np.uint64))


@pytest.mark.parametrize("dist", ["pair_f64", "quartet_f64", "quartet_f64_dup"])
def test_f64_record_types_default_params(dist):
    for seed in (1, 2, 3):
        et, a = W.make(dist, 1 << 15, seed)
        _check_f64_records(et, a, oracle.sort(a))


@pytest.mark.parametrize("dist", ["pair_f64", "quartet_f64_dup"])
def test_f64_record_types_small_blocks_debug(dist):
    """Block machinery (k_max=8, b=3, n0=2) with the three-zone invariant asserted."""
    rng = np.random.default_rng(11)
    for it in range(60):
        n = int(rng.integers(2, 400))
        et, a = W.make(dist, n, it)
        if et == W.ELEM_PAIR_F64:
            a[:, 0] = np.floor(a[:, 0] * 7) - 3.0 + 0.5        # 7 distinct nonzero keys
        p = oracle.params(et, k_max=8, b=3, n0=2, debug=True)
        st = oracle.Stats()
        _check_f64_records(et, a, oracle.sort(a, p, st))


def test_quartet_brute_force_permutations():
    """All orderings of 6 quartets with ties in k0 and k1 (brute force, lexicographic)."""
    base = np.array([[0.5, 0.25, 0.75, 0], [0.5, 0.25, 0.5, 1], [0.5, -0.5, 0.9, 2],
                     [-1.0, 3.0, 0.1, 3], [0.5, 0.25, 0.75, 4], [2.0, -7.0, 0.3, 5]])
    exp_keys = sorted(tuple(r[:3]) for r in base)
    for perm in itertools.permutations(range(6)):
        a = np.ascontiguousarray(base[list(perm)])
        p = oracle.params(W.ELEM_QUARTET_F64, k_max=4, b=1, n0=1, debug=True)
        out = oracle.sort(a, p)
        assert [tuple(r[:3]) for r in out] == exp_keys


def test_quartet_classify_linear_scan():
    """Classification of quartets: the number of splitters <= e under the lexicographic order
    (ties right) and equality buckets, by a linear scan over
    Python tuples."""
    rng = np.random.default_rng(5)
    for eq in (False, True):
        for it in range(20):
            _, pool = W.make("quartet_f64_dup", 400, it)
            tup = sorted({tuple(r[:3]) for r in pool})
            nspl = int(rng.integers(1, 30 if eq else 60))
            pick = sorted(rng.choice(len(tup), size=min(nspl, len(tup)), replace=False))
            spl = np.array([list(tup[i]) + [0.0] for i in pick])
            _, el = W.make("quartet_f64_dup", 500, 100 + it)
            el[:50] = spl[rng.integers(0, len(spl), 50)]
            got = oracle.classify(spl, eq, el)
            st = [tuple(r[:3]) for r in spl]
            kp = 2
            while kp < len(st) + 1:
                kp *= 2
            st = st + [st[-1]] * (kp - 1 - len(st))   # padded with the largest splitter
            for e, g in zip(el, got):
                k = tuple(e[:3])
                i = sum(1 for s in st if s <= k)
                if eq:
                    i = 2 * i - (1 if i >= 1 and st[i - 1] == k else 0)
                assert g == i
