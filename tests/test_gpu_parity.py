"""CUDA path vs the oracle (-m gpu).  Everything calls through the C ABI of libips4o.so.

Layers (SURVEY.md §4 "build test layers"):
  (ii)  classification (T1) vs oracle.classify, exhaustive small domains + random k=256;
  (iii) one distribution step (T2) vs oracle.partition_with: identical e_i, per-bucket
        multisets, every element of [e_i, e_{i+1}) in bucket i;
  (iv)  whole sorts bit-exact vs oracle.sort on every distribution and type, sizes that
        span several tiles / stripes / levels with ragged tails, degenerate inputs;
  (v)   full BASELINE sizes: tests/test_full_parity.py (element-wise oracle parity);
  (vi)  asynchrony: back-to-back sorts without synchronisation, two streams, CUDA-graph
        capture and replay; measured auxiliary memory.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_1705_02257_b200 as ips4o  # noqa: E402
import workloads as W  # noqa: E402
from gpu_util import check_equal_to_oracle, to_dev, to_host  # noqa: E402

TYPES = [W.ELEM_U64, W.ELEM_F64, W.ELEM_PAIR, W.ELEM_REC100]
CAP = {W.ELEM_U64: 16384, W.ELEM_F64: 16384, W.ELEM_PAIR: 8192, W.ELEM_REC100: 1024}


@pytest.fixture(scope="module", autouse=True)
def _lib():
    ips4o.lib()
    torch.cuda.set_device(0)


def _gen(et, n, seed, kind="uniform"):
    rng = np.random.default_rng(seed)
    if et == W.ELEM_U64:
        if kind == "uniform":
            return W.u64_uniform(n, seed)
        if kind == "few":
            return rng.integers(0, 7, size=n).astype(np.uint64)
        if kind == "max":
            return np.where(rng.random(n) < 0.5, np.uint64(2**64 - 1), np.uint64(0)).astype(np.uint64)
    if et == W.ELEM_F64:
        if kind == "uniform":
            return W.f64_exponential(n, seed)
        if kind == "few":
            return rng.integers(0, 7, size=n).astype(np.float64) - 3.0
        if kind == "max":
            x = rng.standard_normal(n) * 1e300
            x[x == 0] = 1.0
            return x
    if et == W.ELEM_PAIR:
        a = W.pair16(n, seed)
        if kind == "few":
            a[:, 0] = rng.integers(0, 7, size=n).astype(np.uint64)
        if kind == "max":
            a[:, 0] = np.where(rng.random(n) < 0.5, np.uint64(2**64 - 1), np.uint64(0))
        return a
    if et == W.ELEM_REC100:
        a = W.rec100(n, seed)
        if kind == "few":   # 3 values of key bytes 0..7, 5 of bytes 8..9: equality buckets on part 0
            a[:, :8] = (rng.integers(0, 3, size=n)[:, None] * np.array([1, 7, 0, 0, 0, 0, 0, 9])).astype(np.uint8)
            a[:, 8:10] = rng.integers(0, 5, size=(n, 1)).astype(np.uint8)
        if kind == "max":
            a[:, :10] = np.where(rng.random(n)[:, None] < 0.5, 255, 0).astype(np.uint8)
        return a
    raise ValueError


def _sort_gpu(a, et):
    t = to_dev(a, et)
    ips4o.sort_(t)
    torch.cuda.synchronize()
    return to_host(t, et)


# ------------------------------------------------------------- (ii) classification

def _spl_keys(spl, et):
    return spl.astype(np.float64) if et == W.ELEM_F64 else spl.astype(np.uint64)


def _oracle_spl(spl, et):
    """The oracle takes splitters as elements of the sorted type (pairs: key, payload 0;
    records: key bytes 0..7 = the big-endian u64 splitter, bytes 8..9 = 0, so that the
    oracle's 10-byte comparison and the GPU's part-0 comparison agree, ties going right)."""
    if et == W.ELEM_PAIR:
        return np.stack([spl.astype(np.uint64), np.zeros(spl.shape[0], np.uint64)], axis=1)
    if et == W.ELEM_REC100:
        r = np.zeros((spl.shape[0], 100), np.uint8)
        r[:, :8] = spl.astype(">u8").view(np.uint8).reshape(-1, 8)
        return r
    return spl


def _keys_of(a, et):
    if et == W.ELEM_PAIR:
        return a[:, 0]
    if et == W.ELEM_REC100:
        return np.ascontiguousarray(a[:, :8]).view(">u8").ravel().astype(np.uint64)
    return a


def _classify_gpu(el, et, spl, eq, lut):
    d_in = to_dev(el, et)
    out = torch.empty(el.shape[0], dtype=torch.int32, device="cuda")
    buf, ptr, ns = ips4o.splitters_buffer(_spl_keys(spl, et), et)
    ips4o.ips4o_debug_classify(d_in.data_ptr(), el.shape[0], et, ptr, ns, eq, out.data_ptr(),
                               torch.cuda.current_stream().cuda_stream, lut=lut)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32)


def _as_elems(elems, et, seed):
    """Elements of type et whose (classification) key is `elems`.  Records: key bytes 0..7 =
    the big-endian key, bytes 8..9 = 0, so that the oracle's 10-byte order and the GPU's
    part-0 order agree (also for equality with a splitter)."""
    if et == W.ELEM_PAIR:
        return np.stack([elems.astype(np.uint64), np.arange(elems.shape[0], dtype=np.uint64)], axis=1)
    if et == W.ELEM_REC100:
        el = W.rec100(elems.shape[0], seed)
        el[:, :8] = elems.astype(">u8").view(np.uint8).reshape(-1, 8)
        el[:, 8:10] = 0
        return el
    return elems


@pytest.mark.parametrize("et", TYPES)
@pytest.mark.parametrize("eq", [False, True])
@pytest.mark.parametrize("lut", [False, True], ids=["tree", "lut"])
def test_classify_vs_oracle(et, eq, lut):
    """Both GPU classifiers -- the tree descent (classify_key, used by K3) and K2's
    bucket-hint table -- against the oracle's linear-scan-pinned classify."""
    rng = np.random.default_rng(100 + et)
    for trial in range(20):
        nspl = int(rng.integers(1, 128 if eq else 256)) if trial % 3 else int(rng.integers(1, 8))
        if et == W.ELEM_F64:
            spl = np.unique(rng.standard_normal(nspl * 2))[:nspl]
            x = np.concatenate([rng.standard_normal(5000), spl, -spl])
            x[x == 0] = 0.5
            elems = x
        elif trial % 3 == 0:
            spl = np.unique(rng.choice(64, size=nspl, replace=False)).astype(np.uint64)
            elems = np.arange(64, dtype=np.uint64)
        else:
            spl = np.unique(rng.integers(0, 1 << 40, size=nspl * 2, dtype=np.uint64))[:nspl]
            elems = np.concatenate([rng.integers(0, 1 << 40, size=5000, dtype=np.uint64), spl])
        el = _as_elems(elems, et, trial)
        exp = oracle.classify(_oracle_spl(spl, et), eq, el)
        got = _classify_gpu(el, et, spl, eq, lut)
        assert np.array_equal(got, exp), (et, eq, lut, trial)


def _adversarial_cases(rng, et):
    """Splitter sets that stress the bucket-hint table (4096 cells over [s_1, s_k'-1]):
    several splitters in one cell (binary search inside the cell), keys equal to splitters,
    keys below s_1, keys at / past the last cell, the extremes of the key domain."""
    top = (1 << 64) - 1
    cases = []
    # 200 splitters packed into [0, 1000] plus a few far away: one cell holds them all
    a = np.sort(rng.choice(1000, size=200, replace=False)).astype(np.uint64)
    b = np.array([1 << 60, (1 << 60) + 5, top - 3], dtype=np.uint64)
    cases.append(np.concatenate([a, b]))
    # dense runs of consecutive values around several centres
    c = np.unique(np.concatenate([np.arange(k, k + 40, dtype=np.uint64) for k in (10, 1 << 33, 1 << 62)]))
    cases.append(c[:255])
    # powers of two (one splitter per binade: cells of very different populations)
    cases.append(np.array([1 << i for i in range(0, 64, 1)], dtype=np.uint64))
    # a single splitter; two adjacent splitters; the largest keys
    cases.append(np.array([12345], dtype=np.uint64))
    cases.append(np.array([7, 8], dtype=np.uint64))
    cases.append(np.array([top - 2, top - 1, top], dtype=np.uint64))
    # the table origin s_1 rounded down to the cell width pushes the last splitter past
    # the last cell (the cells double: K1's re-rounding), with cells >= 2^32 wide (K2's
    # high-word path) and < 2^32 wide
    for w in (52, 30):
        s1 = (1 << (w - 12)) * 3 // 2 + 12345
        cases.append(np.array([s1, s1 + (1 << (w - 1)), s1 + (1 << w) - 1], dtype=np.uint64))
    out = []
    for spl in cases:
        near = np.concatenate([spl, spl - np.uint64(1), spl + np.uint64(1), np.array([0, 1, top, top - 1], np.uint64)])
        rnd = rng.integers(0, 1 << 63, size=4000, dtype=np.uint64) * np.uint64(2)
        small = rng.integers(0, 2000, size=2000).astype(np.uint64)
        out.append((spl, np.concatenate([near, rnd, small])))
    return out


@pytest.mark.parametrize("et", [W.ELEM_U64, W.ELEM_PAIR, W.ELEM_REC100])
@pytest.mark.parametrize("eq", [False, True])
def test_classify_lut_adversarial(et, eq):
    rng = np.random.default_rng(7 + et + 10 * eq)
    for spl, elems in _adversarial_cases(rng, et):
        if eq:
            spl = spl[:127]
        el = _as_elems(elems, et, 3)
        exp = oracle.classify(_oracle_spl(spl, et), eq, el)
        for lut in (False, True):
            got = _classify_gpu(el, et, spl, eq, lut)
            assert np.array_equal(got, exp), (et, eq, lut, spl[:4])


@pytest.mark.parametrize("eq", [False, True])
def test_classify_lut_f64_signs(eq):
    """f64 keys through the order-preserving image: negative and positive values, splitters
    clustered near 0, huge magnitudes."""
    rng = np.random.default_rng(31 + eq)
    spl = np.unique(np.concatenate([rng.standard_normal(40) * 1e-300, rng.standard_normal(40) * 1e300,
                                    [-1.5, -1.0, 1.0, 1.5]]))[: (127 if eq else 255)]
    x = np.concatenate([spl, -spl, np.nextafter(spl, np.inf), np.nextafter(spl, -np.inf),
                        rng.standard_normal(3000), rng.standard_normal(3000) * 1e300, [1e-320, -1e-320]])
    x = x[np.isfinite(x) & (x != 0)]
    exp = oracle.classify(spl, eq, x)
    for lut in (False, True):
        assert np.array_equal(_classify_gpu(x, W.ELEM_F64, spl, eq, lut), exp), lut


# ------------------------------------------------------------ (iii) one step

def _partition_case(et, n, nspl, eq, seed, offset=0, kind="uniform"):
    rng = np.random.default_rng(seed)
    a = _gen(et, n + offset, seed, kind)
    if et == W.ELEM_REC100 and eq:
        # a record step classifies on key bytes 0..7; with key bytes 8..9 zero its equality
        # buckets are the oracle's (10-byte equality with the splitter)
        a[:, 8:10] = 0
    keys = _keys_of(a, et)
    pool = np.unique(keys[offset:])
    nspl = min(nspl, pool.shape[0])
    spl = np.sort(rng.choice(pool, size=nspl, replace=False))
    # oracle on the sub-array [offset, offset+n)
    sub = np.ascontiguousarray(a[offset:])
    o_out, o_bounds = oracle.partition_with(sub, _oracle_spl(spl, et), eq, 16)
    d = to_dev(a, et)
    esz = W.ELEM_SIZE[et]
    buf, ptr, ns = ips4o.splitters_buffer(_spl_keys(spl, et), et)
    bounds, K = ips4o.ips4o_debug_partition_once(d.data_ptr() + offset * esz, n, et, ptr, ns, eq,
                                                 torch.cuda.current_stream().cuda_stream)
    got = to_host(d, et)
    assert np.array_equal(np.array(bounds), o_bounds), "bucket bounds e_i differ from the oracle"
    assert (got[:offset] == a[:offset]).all()       # nothing outside the range was touched
    g = got[offset:]
    cls = oracle.classify(_oracle_spl(spl, et), eq, g)
    for i in range(K):
        seg = cls[bounds[i]:bounds[i + 1]]
        assert (seg == i).all(), f"bucket {i} holds foreign elements"
    # per-bucket multisets equal to the oracle's
    for i in range(K):
        gs, os_ = g[bounds[i]:bounds[i + 1]], o_out[bounds[i]:bounds[i + 1]]
        if et == W.ELEM_PAIR:
            gs = np.sort(gs.view([("k", "<u8"), ("v", "<u8")]).ravel(), order=["k", "v"])
            os_ = np.sort(os_.view([("k", "<u8"), ("v", "<u8")]).ravel(), order=["k", "v"])
        elif et == W.ELEM_REC100:
            gs = np.sort(np.ascontiguousarray(gs).view("S100").ravel())
            os_ = np.sort(np.ascontiguousarray(os_).view("S100").ravel())
        else:
            gs, os_ = np.sort(gs), np.sort(os_)
        assert np.array_equal(gs, os_)


@pytest.mark.parametrize("et", TYPES)
def test_partition_once_vs_oracle(et):
    cases = [(64, 3, False), (1000, 7, False), (4099, 255, False), (100_003, 255, False),
             (300_001, 100, True), (2_000_003, 255, False), (1_500_017, 127, True)]
    for i, (n, nspl, eq) in enumerate(cases):
        if et == W.ELEM_REC100 and n > 2_000_000:
            n = 1_000_003
        _partition_case(et, n, nspl, eq, seed=7 + i, kind="few" if (eq and et == W.ELEM_REC100) else "uniform")


@pytest.mark.parametrize("et", [W.ELEM_U64, W.ELEM_F64])
def test_partition_once_misaligned_start(et):
    """Data starting at an 8-byte (not 16-byte) boundary: head element + shifted block grid."""
    for i, n in enumerate([777, 65_537, 1_000_001]):
        _partition_case(et, n, 255, False, seed=50 + i, offset=1)
        _partition_case(et, n, 63, True, seed=60 + i, offset=1, kind="few")


def test_partition_once_duplicates_and_skew():
    _partition_case(W.ELEM_U64, 500_000, 3, True, seed=3, kind="few")
    _partition_case(W.ELEM_U64, 500_000, 1, False, seed=4, kind="few")
    _partition_case(W.ELEM_U64, 200_000, 1, True, seed=5, kind="max")


# ------------------------------------------------------------ (iv) whole sorts

# (single-task sizes at every base-case class boundary: 2048/4096/8192/16384 elements,
# 512/1024 records)
SIZES = [0, 1, 2, 3, 17, 1000, 2048, 2049, 4096, 4097, 8192, 8193, 12_345, 16383, 16384, 16385, 40_000,
         131_073, 1_000_003, 3_000_017]
SIZES_REC = [0, 1, 2, 3, 17, 512, 513, 1023, 1024, 1025, 5000, 70_001, 300_007]


@pytest.mark.parametrize("et", TYPES)
def test_sort_sizes_vs_oracle(et):
    for i, n in enumerate(SIZES_REC if et == W.ELEM_REC100 else SIZES):
        a = _gen(et, n, 1000 + i)
        got = _sort_gpu(a, et)
        exp = oracle.sort(a)
        check_equal_to_oracle(et, a, got, exp)


@pytest.mark.parametrize("et", TYPES)
@pytest.mark.parametrize("kind", ["few", "max"])
def test_sort_duplicates_vs_oracle(et, kind):
    for n in ((5000, 70_001, 400_000) if et == W.ELEM_REC100 else (5000, 70_001, 2_000_000)):
        a = _gen(et, n, 77, kind)
        check_equal_to_oracle(et, a, _sort_gpu(a, et), oracle.sort(a))


@pytest.mark.parametrize("et", [W.ELEM_U64, W.ELEM_F64])
@pytest.mark.parametrize("span", [3000, 6000, 15000, 40000, 1 << 40])
def test_fallback_leaves_vs_oracle(et, span):
    """Leaves the cell kernels hand back: one heavy key value plus scattered others.  span < the
    class tile: one key value per cell; class tile <= span < 16384: the fallback's second chance in
    the largest cell tile; beyond: the merge sort.  Single leaves (n <= the base-case capacity)
    and a two-level sort whose buckets are such leaves."""
    rng = np.random.default_rng(span % 9973)
    for n in (1500, 3000, 5000, 12000, 300_000):
        nleaf = max(1, n // 3000)
        parts = []
        for q in range(nleaf):
            m = n // nleaf
            base = np.uint64(q) * np.uint64(min(span, 1 << 41) * 2)
            heavy = base + np.uint64(rng.integers(0, span))
            others = base + rng.integers(0, span, size=m - 2 * m // 3).astype(np.uint64)
            parts.append(np.concatenate([np.full(2 * m // 3, heavy, np.uint64), others]))
        k = np.concatenate(parts)
        rng.shuffle(k)
        a = k if et == W.ELEM_U64 else (k.astype(np.float64) - 1.0e6)
        got = _sort_gpu(a, et)
        check_equal_to_oracle(et, a, got, oracle.sort(a))


@pytest.mark.parametrize("dist", ["rootdup", "twodup", "eightdup", "almostsorted", "reversesorted",
                                  "sorted", "zeros", "ones", "uniform", "f64_uniform", "f64_exponential",
                                  "pair16", "rec100", "pair_f64", "quartet_f64", "quartet_f64_dup"])
def test_distributions_vs_oracle(dist):
    for seed in (1, 2, 3):
        et, a = W.make(dist, (1 << 18) if dist == "rec100" else (1 << 21), seed)
        check_equal_to_oracle(et, a, _sort_gpu(a, et), oracle.sort(a))


@pytest.mark.parametrize("dist", ["pair_f64", "quartet_f64", "quartet_f64_dup"])
def test_f64_record_types_sizes_vs_oracle(dist):
    """The paper's Pair and Quartet: sizes at every base-case boundary
    (quartets: 4096 = capacity of the merge-sort base case), several levels, a ragged tail;
    the duplicate-heavy quartets exercise equality buckets on key parts 0 and 1."""
    for i, n in enumerate([2, 3, 17, 2048, 2049, 4096, 4097, 8192, 8193, 70_001, 1_000_003]):
        et, a = W.make(dist, n, 300 + i)
        check_equal_to_oracle(et, a, _sort_gpu(a, et), oracle.sort(a))
        assert ips4o.ips4o_last_stats()["device_error"] == 0


def test_config1_full_size_vs_oracle():
    """BASELINE config 1 (2^20 uniform u64) at full size, seeds 1-3."""
    for seed in (1, 2, 3):
        a = W.u64_uniform(1 << 20, seed)
        got = _sort_gpu(a, W.ELEM_U64)
        assert np.array_equal(got, oracle.sort(a))


def test_misaligned_whole_sort():
    a = W.u64_uniform((1 << 20) + 3, 9)
    t = to_dev(a, W.ELEM_U64)
    sub = t[1:]
    ips4o.ips4o_sort(sub.data_ptr(), sub.shape[0], W.ELEM_U64, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = to_host(t, W.ELEM_U64)
    assert got[0] == a[0]
    assert np.array_equal(got[1:], oracle.sort(a[1:]))


def test_equality_buckets_all_zero_one_step():
    """All-equal input is an easy instance: one distribution step."""
    a = np.zeros(1 << 22, dtype=np.uint64)
    got = _sort_gpu(a, W.ELEM_U64)
    assert (got == 0).all()
    st = ips4o.ips4o_last_stats()
    assert st["distribution_tasks"] == 1 and st["equality_tasks"] == 1 and st["base_tasks"] == 0


@pytest.mark.parametrize("et,e", [(W.ELEM_U64, 20), (W.ELEM_U64, 24), (W.ELEM_PAIR, 22), (W.ELEM_REC100, 20)])
def test_aux_memory_measured(et, e):
    """Auxiliary device memory, measured: the device-memory delta (cudaMemGetInfo) of the
    first sort after ips4o_release_workspace is the workspace ips4o_aux_bytes(n) reports
    (plus the instantiated level-loop graph, whose size the driver decides, allowed
    <= 4 MiB), and stays a small fraction of the input (Theorem 2)."""
    n = 1 << e
    _, a = W.make({W.ELEM_U64: "uniform", W.ELEM_PAIR: "pair16", W.ELEM_REC100: "rec100"}[et], n, 4)
    t = to_dev(a, et)
    torch.cuda.synchronize()
    ips4o.ips4o_release_workspace()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    ips4o.sort_(t)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    st = ips4o.ips4o_last_stats()
    aux = ips4o.ips4o_aux_bytes(n, et)
    assert st["aux_bytes"] == aux
    delta = free0 - free1
    assert delta <= aux + (4 << 20) + (2 << 20), (delta, aux)   # + graph + allocation granularity
    input_bytes = n * W.ELEM_SIZE[et]
    assert aux < input_bytes, (aux, input_bytes)                # < 1x the input even at 2^20
    assert st["device_error"] == 0
    check_equal_to_oracle(et, a, to_host(t, et), oracle.sort(a))


def test_aux_bytes_headline_fraction():
    """The headline config's workspace is a few percent of its 2 GiB input."""
    assert ips4o.ips4o_aux_bytes(1 << 28, W.ELEM_U64) < 0.05 * (8 << 28)


def test_stats_levels_and_syncs():
    n = 1 << 24
    a = W.u64_uniform(n, 4)
    _sort_gpu(a, W.ELEM_U64)
    st = ips4o.ips4o_last_stats()
    assert st["levels"] == 2 and st["host_syncs"] == 0 and st["device_error"] == 0
    assert st["base_elements"] == n and sum(st["base_tasks_by_class"]) == st["base_tasks"]
    assert st["block_moves"] > 0 and st["batches"] >= 2


# ------------------------------------------------- asynchrony, streams, graph capture

def test_back_to_back_without_sync():
    """Several sorts (different sizes, small and large) enqueued back to back on a stream
    kept busy by other work, with no synchronisation in between: every call's parameters
    travel as kernel arguments, so none can see another call's (staging slots)."""
    s = torch.cuda.Stream()
    arrays = [W.u64_uniform(n, 20 + i) for i, n in enumerate([3000, 70_001, 500, 1 << 20, 9000, 2, 300_000])]
    devs = [to_dev(a, W.ELEM_U64) for a in arrays]
    torch.cuda.synchronize()
    big = torch.empty(1 << 27, dtype=torch.int64, device="cuda")
    with torch.cuda.stream(s):
        for _ in range(3):
            big.add_(1)          # keep the stream busy before the sorts are reached
        for t in devs:
            ips4o.ips4o_sort(t.data_ptr(), t.shape[0], W.ELEM_U64, s.cuda_stream)
    torch.cuda.synchronize()
    for a, t in zip(arrays, devs):
        assert np.array_equal(to_host(t, W.ELEM_U64), oracle.sort(a))


def test_two_streams_share_the_workspace():
    """Sorts alternating between two streams: the library orders them (workspace event)."""
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    arrays = [W.u64_uniform(n, 40 + i) for i, n in enumerate([1 << 20, 12_345, 1 << 19, 4000, 1 << 20])]
    devs = [to_dev(a, W.ELEM_U64) for a in arrays]
    torch.cuda.synchronize()
    for i, t in enumerate(devs):
        s = s1 if i % 2 == 0 else s2
        ips4o.ips4o_sort(t.data_ptr(), t.shape[0], W.ELEM_U64, s.cuda_stream)
    torch.cuda.synchronize()
    for a, t in zip(arrays, devs):
        assert np.array_equal(to_host(t, W.ELEM_U64), oracle.sort(a))


@pytest.mark.parametrize("et,n", [(W.ELEM_U64, 1 << 22), (W.ELEM_U64, 5000), (W.ELEM_PAIR, 1 << 20),
                                  (W.ELEM_F64, (1 << 21) + 3)])
def test_graph_capture_replay(et, n):
    """ips4o_sort captured into a caller's CUDA graph (no host sync inside the sort), replayed
    on restored inputs: every replay matches the oracle bit for bit."""
    _, a = W.make({W.ELEM_U64: "uniform", W.ELEM_PAIR: "pair16", W.ELEM_F64: "f64_exponential"}[et], n, 6)
    exp = oracle.sort(a)
    pristine = to_dev(a, et)
    work = pristine.clone()
    ips4o.sort_(work)            # warm: the workspace exists for this type and n
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    work.copy_(pristine)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        ips4o.ips4o_sort(work.data_ptr(), n, et, torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        work.copy_(pristine)
        g.replay()
        torch.cuda.synchronize()
        check_equal_to_oracle(et, a, to_host(work, et), exp)



@pytest.mark.parametrize("key_type", [W.ELEM_U64, W.ELEM_F64])
def test_sort_kv_vs_oracle(key_type):
    """Structure-of-arrays key-value sort, in place: keys bit-exact vs the oracle's key sort,
    every (key, value) pair preserved, no staging memory (the pair of arrays is distributed
    directly: key blocks and value blocks move together)."""
    for n in (1, 2, 17, 1000, 8192, 8193, 70_001, 1_000_003, (1 << 22) + 5):
        rng = np.random.default_rng(n)
        if key_type == W.ELEM_U64:
            k = W.u64_uniform(n, 5) >> np.uint64(40)   # duplicates
        else:
            k = W.f64_exponential(n, 5) * np.where(rng.random(n) < 0.5, -1.0, 1.0)
        v = rng.integers(0, 2**63, size=n, dtype=np.int64).astype(np.uint64)
        dk = to_dev(k, key_type)
        dv = torch.from_numpy(v.view(np.int64)).cuda()
        ips4o.sort_kv_(dk, dv)
        torch.cuda.synchronize()
        gk = to_host(dk, key_type)
        gv = dv.cpu().numpy().view(np.uint64)
        assert np.array_equal(gk.view(np.uint64), oracle.sort(k).view(np.uint64))
        st = ips4o.ips4o_last_stats()
        assert st["staging_bytes"] == 0 and st["device_error"] == 0
        kb = k.view(np.uint64) if key_type == W.ELEM_F64 else k
        gkb = gk.view(np.uint64) if key_type == W.ELEM_F64 else gk
        a = np.sort(np.stack([kb, v], 1).view([("k", "<u8"), ("v", "<u8")]).ravel(), order=["k", "v"])
        b = np.sort(np.stack([gkb, gv], 1).view([("k", "<u8"), ("v", "<u8")]).ravel(), order=["k", "v"])
        assert np.array_equal(a, b)


def test_sort_kv_alignment_and_types():
    k = torch.zeros(1001, dtype=torch.uint64, device="cuda")
    v = torch.zeros(1001, dtype=torch.int64, device="cuda")
    with pytest.raises(ips4o.Ips4oError):
        ips4o.ips4o_sort_kv(k.data_ptr() + 8, v.data_ptr(), 1000, W.ELEM_U64)   # keys not 16-byte aligned
    with pytest.raises(ips4o.Ips4oError):
        ips4o.sort_kv_(k.view(torch.int64), v)                                  # int64 keys: rejected


def test_sort_host_entry_point():
    a = W.u64_uniform(1 << 20, 11)
    h = a.copy()
    ips4o.ips4o_sort_host(h.ctypes.data, h.shape[0], W.ELEM_U64, 0)
    assert np.array_equal(h, oracle.sort(a))


def test_type_switching_and_reuse():
    for et in (W.ELEM_PAIR, W.ELEM_U64, W.ELEM_REC100, W.ELEM_F64, W.ELEM_PAIR):
        a = _gen(et, 200_001, 5)
        check_equal_to_oracle(et, a, _sort_gpu(a, et), oracle.sort(a))


# (v) full BASELINE sizes: tests/test_full_parity.py (element-wise oracle parity)


# ------------------------------------------------------------ the single-CTA tier

def _tier_run(medium_max, specs):
    import json as _json
    import os as _os
    import subprocess as _sp
    import sys as _sys
    env = dict(_os.environ, IPS4O_MEDIUM_MAX=str(medium_max))
    here = _os.path.dirname(_os.path.abspath(__file__))
    out = _sp.run([_sys.executable, _os.path.join(here, "tier_check.py"), *specs], env=env, capture_output=True,
                  text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return _json.loads(out.stdout.strip().splitlines()[-1])


def test_single_cta_tier_vs_oracle():
    """Every task of <= 2^30 elements sorted by one CTA with the strictly in-place driver
    (k_cta.cuh): all distributions and the 8/16-byte types, sizes from one
    partition to several levels inside the CTA (recursion through searchNextLargest with
    bucket-maximum marking on skewed inputs)."""
    specs = [f"{d}:{n}:{s}" for d, n, s in [
        ("uniform", 20_000, 1), ("uniform", 70_001, 2), ("uniform", 1 << 20, 3), ("uniform", (1 << 22) + 7, 1),
        ("f64_exponential", 300_007, 2), ("rootdup", 1 << 21, 1), ("twodup", 1 << 21, 2), ("eightdup", 1 << 21, 3),
        ("almostsorted", 1 << 20, 1), ("reversesorted", 1 << 20, 1), ("zeros", 1 << 20, 1), ("ones", 100_000, 1),
        ("sorted", 1 << 20, 2), ("pair16", 500_001, 1), ("pair_f64", 300_001, 2)]]
    res = _tier_run(1 << 30, specs)
    for r in res:
        assert r["ok"] and r["err"] == 0, r
    assert all(r["medium_tasks"] >= 1 for r in res if not r["spec"].startswith(("zeros", "ones")))
    assert sum(r["medium_marks"] for r in res) > 0     # the marking path ran (recursion inside a CTA)
