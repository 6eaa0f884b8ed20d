"""CPU oracle for IPS4o -- TEST INFRASTRUCTURE ONLY.

A plain sequential IS4o (t = 1) written in C from the paper (see
ips4o_oracle.c / ips4o_oracle.h for the step-by-step citations).  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this package; the product path
(paper_1705_02257_b200) never does, and shares no code with it.

Parity status per function:
  oracle_sort            pinned: numpy.sort (unique result), brute force over all
                         permutations / {0,1,2}^n, insertion sort, invariants
  oracle_partition_with  pinned: per-bucket membership against the linear-scan
                         definition, multiset conservation, SPEC delimiter example
  oracle_classify        pinned: linear-scan definition s_{i-1} <= e < s_i, exhaustive
                         for k' <= 8 over a 64-value domain
  oracle_build_tree      pinned: SPEC.md:141-143 worked example, in-order = splitters
  oracle_select_splitters pinned: SPEC.md:132-134 worked examples
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ips4o_oracle.c")
_LIB = os.path.join(_HERE, "libips4o_oracle.so")

ELEM_U64, ELEM_F64, ELEM_PAIR, ELEM_REC100, ELEM_PAIR_F64, ELEM_QUARTET_F64 = 0, 1, 2, 3, 4, 5
_SIZES = {0: 8, 1: 8, 2: 16, 3: 100, 4: 16, 5: 32}


class Params(ctypes.Structure):
    _fields_ = [("k_max", ctypes.c_uint64), ("b", ctypes.c_uint64), ("n0", ctypes.c_uint64),
                ("seed", ctypes.c_uint64), ("debug", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "partition_steps", "eq_steps", "overflow_uses", "overhang_uses", "block_moves",
        "skipped_blocks", "invariant_checks", "base_cases", "max_depth")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ips4o_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        L.oracle_default_block.argtypes = [i32]; L.oracle_default_block.restype = u64
        L.oracle_alpha.argtypes = [u64]; L.oracle_alpha.restype = u64
        L.oracle_bucket_count.argtypes = [u64, u64]; L.oracle_bucket_count.restype = u64
        L.oracle_default_params.argtypes = [i32, ctypes.POINTER(Params)]
        L.oracle_sort.argtypes = [i32, vp, u64, ctypes.POINTER(Params), ctypes.POINTER(Stats)]
        L.oracle_sort_rows.argtypes = [i32, vp, u64, u64, ctypes.POINTER(Params), ctypes.POINTER(Stats)]
        L.oracle_partition_with.argtypes = [i32, vp, u64, vp, u32, i32, u64, i32,
                                            ctypes.POINTER(u64), ctypes.POINTER(u32), ctypes.POINTER(Stats)]
        L.oracle_classify.argtypes = [i32, vp, u32, i32, vp, u64, ctypes.POINTER(u32)]
        L.oracle_build_tree.argtypes = [i32, vp, u32, vp, ctypes.POINTER(u32)]
        L.oracle_select_splitters.argtypes = [i32, vp, u64, u32, u32, vp, ctypes.POINTER(u32),
                                              ctypes.POINTER(ctypes.c_int)]
        for f in ("oracle_sort", "oracle_sort_rows", "oracle_partition_with", "oracle_classify",
                  "oracle_build_tree", "oracle_select_splitters"):
            getattr(L, f).restype = i32
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def type_of(a: np.ndarray) -> int:
    if a.dtype == np.float64 and a.ndim == 1:
        return ELEM_F64
    if a.dtype == np.uint64 and a.ndim == 1:
        return ELEM_U64
    if a.dtype == np.uint64 and a.ndim == 2 and a.shape[1] == 2:
        return ELEM_PAIR
    if a.dtype == np.uint8 and a.ndim == 2 and a.shape[1] == 100:
        return ELEM_REC100
    if a.dtype == np.float64 and a.ndim == 2 and a.shape[1] == 2:
        return ELEM_PAIR_F64
    if a.dtype == np.float64 and a.ndim == 2 and a.shape[1] == 4:
        return ELEM_QUARTET_F64
    raise TypeError(f"unsupported array {a.dtype} {a.shape}")


def default_params(et: int) -> Params:
    p = Params()
    lib().oracle_default_params(et, ctypes.byref(p))
    return p


def params(et: int, k_max=None, b=None, n0=None, seed=None, debug=None) -> Params:
    p = default_params(et)
    if k_max is not None: p.k_max = k_max
    if b is not None: p.b = b
    if n0 is not None: p.n0 = n0
    if seed is not None: p.seed = seed
    if debug is not None: p.debug = int(debug)
    return p


def sort(a: np.ndarray, p: Params | None = None, stats: Stats | None = None) -> np.ndarray:
    """Sort a copy of `a` with the oracle; returns the copy."""
    out = np.ascontiguousarray(a).copy()
    et = type_of(out)
    p = p or default_params(et)
    rc = lib().oracle_sort(et, _ptr(out), out.shape[0], ctypes.byref(p),
                           ctypes.byref(stats) if stats is not None else None)
    if rc != 0:
        raise RuntimeError(f"oracle_sort failed rc={rc}")
    return out


def sort_inplace(a: np.ndarray, p: Params | None = None, stats: Stats | None = None) -> None:
    et = type_of(a)
    p = p or default_params(et)
    rc = lib().oracle_sort(et, _ptr(a), a.shape[0], ctypes.byref(p),
                           ctypes.byref(stats) if stats is not None else None)
    if rc != 0:
        raise RuntimeError(f"oracle_sort failed rc={rc}")


def sort_rows(et: int, rows: np.ndarray, p: Params, stats: Stats | None = None) -> np.ndarray:
    """rows: shape (R, n) for 8-byte types. Sorts each row independently."""
    out = np.ascontiguousarray(rows).copy()
    R, n = out.shape[0], out.shape[1]
    rc = lib().oracle_sort_rows(et, _ptr(out), R, n, ctypes.byref(p),
                                ctypes.byref(stats) if stats is not None else None)
    if rc != 0:
        raise RuntimeError(f"oracle_sort_rows failed rc={rc}")
    return out


def partition_with(a: np.ndarray, splitters: np.ndarray, eq: bool, b: int, debug: bool = False,
                   stats: Stats | None = None):
    """One distribution step with given splitters. Returns (partitioned copy, bounds[K+1])."""
    out = np.ascontiguousarray(a).copy()
    et = type_of(out)
    spl = np.ascontiguousarray(splitters)
    bounds = (ctypes.c_uint64 * 512)()
    K = ctypes.c_uint32(0)
    rc = lib().oracle_partition_with(et, _ptr(out), out.shape[0], _ptr(spl), spl.shape[0],
                                     int(eq), b, int(debug), bounds, ctypes.byref(K),
                                     ctypes.byref(stats) if stats is not None else None)
    if rc != 0:
        raise RuntimeError(f"oracle_partition_with failed rc={rc}")
    return out, np.array(bounds[:K.value + 1], dtype=np.int64)


def classify(splitters: np.ndarray, eq: bool, elems: np.ndarray) -> np.ndarray:
    et = type_of(np.ascontiguousarray(elems))
    spl = np.ascontiguousarray(splitters)
    el = np.ascontiguousarray(elems)
    out = np.zeros(el.shape[0], dtype=np.uint32)
    rc = lib().oracle_classify(et, _ptr(spl), spl.shape[0], int(eq), _ptr(el), el.shape[0],
                               out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    if rc != 0:
        raise RuntimeError(f"oracle_classify failed rc={rc}")
    return out


def build_tree(splitters: np.ndarray):
    spl = np.ascontiguousarray(splitters)
    et = type_of(spl)
    kp = ctypes.c_uint32(0)
    tree = np.zeros((256,) + spl.shape[1:], dtype=spl.dtype)
    rc = lib().oracle_build_tree(et, _ptr(spl), spl.shape[0], _ptr(tree), ctypes.byref(kp))
    if rc != 0:
        raise RuntimeError("oracle_build_tree failed")
    return tree[:kp.value - 1], kp.value


def select_splitters(sorted_sample: np.ndarray, k: int, alpha: int):
    s = np.ascontiguousarray(sorted_sample)
    et = type_of(s)
    out = np.zeros((k,) + s.shape[1:], dtype=s.dtype)
    nout = ctypes.c_uint32(0)
    eq = ctypes.c_int(0)
    rc = lib().oracle_select_splitters(et, _ptr(s), s.shape[0], k, alpha, _ptr(out),
                                       ctypes.byref(nout), ctypes.byref(eq))
    if rc != 0:
        raise RuntimeError("oracle_select_splitters failed")
    return out[:nout.value], bool(eq.value)


def default_block(et: int) -> int:
    return int(lib().oracle_default_block(et))


def alpha(n: int) -> int:
    return int(lib().oracle_alpha(n))


def bucket_count(n: int, k_max: int = 256) -> int:
    return int(lib().oracle_bucket_count(n, k_max))
