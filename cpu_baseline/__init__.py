"""Multi-core CPU IPS4o baseline (OpenMP).

A reported host baseline for bench.py, not the oracle and not the product path: the paper's
parallel algorithm (t threads partition large problems together with atomic block
permutation; smaller problems are sorted sequentially by one thread each) in C with OpenMP.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, "ips4o_cpu.c"), os.path.join(_HERE, "ips4o_cpu_impl.h")]
_LIB = os.path.join(_HERE, "libips4o_cpu.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(s) for s in _SRC):
        subprocess.check_call(["gcc", "-O3", "-std=gnu11", "-fopenmp", "-Wall", "-shared", "-fPIC",
                               "-o", _LIB, _SRC[0], "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.ips4o_cpu_sort.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int]
        L.ips4o_cpu_sort.restype = ctypes.c_int
        L.ips4o_cpu_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def type_of(a: np.ndarray) -> int:
    if a.dtype == np.uint64 and a.ndim == 1:
        return 0
    if a.dtype == np.float64 and a.ndim == 1:
        return 1
    if a.dtype == np.uint64 and a.ndim == 2 and a.shape[1] == 2:
        return 2
    if a.dtype == np.uint8 and a.ndim == 2 and a.shape[1] == 100:
        return 3
    raise TypeError(f"unsupported array {a.dtype} {a.shape}")


def sort_inplace(a: np.ndarray, threads: int = 0) -> None:
    assert a.flags.c_contiguous
    rc = lib().ips4o_cpu_sort(a.ctypes.data_as(ctypes.c_void_p), a.shape[0], type_of(a), threads)
    if rc:
        raise RuntimeError(f"ips4o_cpu_sort failed: {rc}")


def max_threads() -> int:
    return int(lib().ips4o_cpu_max_threads())
