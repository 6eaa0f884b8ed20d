"""Thin ctypes binding of libips4o.so (include/ips4o.h): argument marshalling only.

Every step of the sort runs in the sm_100a kernels of csrc/.  PyTorch is used only for
device memory and streams.  There is no CPU fallback: if libips4o.so is missing or the
device is not a CUDA GPU, the calls raise.

    import paper_1705_02257_b200 as ips4o
    ips4o.sort_(t)                  # t: CUDA tensor; sorted in place on the current stream
    ips4o.ips4o_sort(ptr, n, type, stream)   # raw C ABI
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# IPS4O_LIB may name an alternative build (tuning experiments, e.g. libips4o_bb256.so)
LIB_PATH = os.environ.get("IPS4O_LIB") or os.path.join(_HERE, "libips4o.so")

IPS4O_U64, IPS4O_F64, IPS4O_PAIR_U64, IPS4O_REC100_K10, IPS4O_PAIR_F64, IPS4O_QUARTET_F64 = 0, 1, 2, 3, 4, 5
ELEM_SIZE = {0: 8, 1: 8, 2: 16, 3: 100, 4: 16, 5: 32}
NUM_KERNEL_KINDS = 9

# every symbol include/ips4o.h declares
EXPORTS = (
    "ips4o_sort", "ips4o_sort_host", "ips4o_sort_kv", "ips4o_aux_bytes", "ips4o_last_stats", "ips4o_error_string",
    "ips4o_release_workspace", "ips4o_profile_enable", "ips4o_profile_read",
    "ips4o_kernel_kind_name", "ips4o_debug_classify", "ips4o_debug_partition_once",
)


class Ips4oError(RuntimeError):
    pass


class Stats(ctypes.Structure):
    """ips4o_stats of include/ips4o.h (same field order)."""
    _fields_ = [("n", ctypes.c_uint64), ("elem_type", ctypes.c_uint32), ("levels", ctypes.c_uint32),
                ("distribution_tasks", ctypes.c_uint64), ("base_tasks", ctypes.c_uint64),
                ("equality_tasks", ctypes.c_uint64), ("aux_bytes", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64), ("host_syncs", ctypes.c_uint64),
                ("distributed_elements", ctypes.c_uint64), ("base_elements", ctypes.c_uint64),
                ("batches", ctypes.c_uint64), ("base_tasks_by_class", ctypes.c_uint64 * 4),
                ("base_fallback_tasks", ctypes.c_uint64), ("block_moves", ctypes.c_uint64),
                ("empty_block_moves", ctypes.c_uint64), ("device_error", ctypes.c_uint64),
                ("staging_bytes", ctypes.c_uint64), ("medium_tasks", ctypes.c_uint64),
                ("medium_partitions", ctypes.c_uint64), ("medium_marks", ctypes.c_uint64),
                ("medium_leaves", ctypes.c_uint64), ("has_device_stats", ctypes.c_uint32),
                ("reserved_", ctypes.c_uint32)]

    def as_dict(self):
        d = {}
        for n, _ in self._fields_:
            v = getattr(self, n)
            d[n] = [int(x) for x in v] if n == "base_tasks_by_class" else int(v)
        return d


_lib = None


def build(force: bool = False) -> str:
    from . import builder as _b
    return _b.build(force=force)


def lib():
    """Load libips4o.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise Ips4oError(f"{LIB_PATH} is missing: run `python -m paper_1705_02257_b200.builder` "
                             "or __graft_entry__.build() first")
        L = ctypes.CDLL(LIB_PATH)
        vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        L.ips4o_sort.argtypes = [vp, u64, i32, vp]
        L.ips4o_sort_host.argtypes = [vp, u64, i32, vp]
        L.ips4o_sort_kv.argtypes = [vp, vp, u64, i32, vp]
        L.ips4o_aux_bytes.argtypes = [u64, i32]
        L.ips4o_aux_bytes.restype = ctypes.c_size_t
        L.ips4o_last_stats.argtypes = [ctypes.POINTER(Stats)]
        L.ips4o_error_string.argtypes = [i32]
        L.ips4o_error_string.restype = ctypes.c_char_p
        L.ips4o_release_workspace.argtypes = []
        L.ips4o_profile_enable.argtypes = [i32]
        L.ips4o_profile_read.argtypes = [ctypes.POINTER(u64), ctypes.POINTER(ctypes.c_double)]
        L.ips4o_kernel_kind_name.argtypes = [i32]
        L.ips4o_kernel_kind_name.restype = ctypes.c_char_p
        L.ips4o_debug_classify.argtypes = [vp, u64, i32, vp, u32, i32, vp, vp]
        L.ips4o_debug_partition_once.argtypes = [vp, u64, i32, vp, u32, i32,
                                                 ctypes.POINTER(u64), ctypes.POINTER(u32), vp]
        for f in ("ips4o_sort", "ips4o_sort_host", "ips4o_sort_kv", "ips4o_last_stats", "ips4o_release_workspace",
                  "ips4o_profile_enable", "ips4o_profile_read", "ips4o_debug_classify",
                  "ips4o_debug_partition_once"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().ips4o_error_string(rc).decode()
        raise Ips4oError(f"{what} failed: status {rc}: {msg}")


# ------------------------------------------------------------------ C ABI, same names

def ips4o_sort(d_ptr: int, n: int, elem_type: int, stream: int = 0) -> None:
    _check(lib().ips4o_sort(ctypes.c_void_p(d_ptr), n, elem_type, ctypes.c_void_p(stream)), "ips4o_sort")


def ips4o_sort_kv(keys_ptr: int, vals_ptr: int, n: int, key_type: int, stream: int = 0) -> None:
    _check(lib().ips4o_sort_kv(ctypes.c_void_p(keys_ptr), ctypes.c_void_p(vals_ptr), n, key_type,
                               ctypes.c_void_p(stream)), "ips4o_sort_kv")


def sort_kv_(keys, vals):
    """Sort CUDA tensors keys (torch.uint64 or torch.float64) and vals (any 8-byte dtype) by
    key, in place in their own storage (both 16-byte aligned); unstable (include/ips4o.h)."""
    import torch
    if not (keys.is_cuda and vals.is_cuda) or keys.shape != vals.shape or keys.dim() != 1:
        raise Ips4oError("sort_kv_ expects two 1-D CUDA tensors of the same length")
    if keys.device != vals.device:
        raise Ips4oError("sort_kv_ expects keys and vals on the same device")
    if not (keys.is_contiguous() and vals.is_contiguous()) or vals.element_size() != 8:
        raise Ips4oError("sort_kv_ expects contiguous tensors and 8-byte values")
    if keys.dtype == torch.float64:
        kt = IPS4O_F64
    elif keys.dtype == torch.uint64:
        kt = IPS4O_U64
    else:
        raise Ips4oError("sort_kv_ keys must be torch.uint64 or torch.float64 (int64 keys would sort as unsigned)")
    with torch.cuda.device(keys.device):
        ips4o_sort_kv(keys.data_ptr(), vals.data_ptr(), keys.shape[0], kt,
                      torch.cuda.current_stream(keys.device).cuda_stream)


def ips4o_sort_host(h_ptr: int, n: int, elem_type: int, stream: int = 0) -> None:
    _check(lib().ips4o_sort_host(ctypes.c_void_p(h_ptr), n, elem_type, ctypes.c_void_p(stream)),
           "ips4o_sort_host")


def ips4o_aux_bytes(n: int, elem_type: int) -> int:
    return int(lib().ips4o_aux_bytes(n, elem_type))


def ips4o_last_stats() -> dict:
    s = Stats()
    _check(lib().ips4o_last_stats(ctypes.byref(s)), "ips4o_last_stats")
    return s.as_dict()


def ips4o_release_workspace() -> None:
    _check(lib().ips4o_release_workspace(), "ips4o_release_workspace")


def ips4o_profile_enable(on: bool) -> None:
    _check(lib().ips4o_profile_enable(int(on)), "ips4o_profile_enable")


def ips4o_profile_read() -> dict:
    la = (ctypes.c_uint64 * NUM_KERNEL_KINDS)()
    ms = (ctypes.c_double * NUM_KERNEL_KINDS)()
    _check(lib().ips4o_profile_read(la, ms), "ips4o_profile_read")
    return {lib().ips4o_kernel_kind_name(k).decode(): (int(la[k]), float(ms[k]))
            for k in range(NUM_KERNEL_KINDS)}


def ips4o_debug_classify(d_in: int, n: int, elem_type: int, h_splitters, nspl: int, eq: bool,
                         d_out: int, stream: int = 0, lut: bool = False) -> None:
    """flags = eq | lut << 1: lut selects K2's production classifier (bucket-hint table)."""
    flags = int(bool(eq)) | (int(bool(lut)) << 1)
    _check(lib().ips4o_debug_classify(ctypes.c_void_p(d_in), n, elem_type, h_splitters, nspl, flags,
                                      ctypes.c_void_p(d_out), ctypes.c_void_p(stream)),
           "ips4o_debug_classify")


def ips4o_debug_partition_once(d_ptr: int, n: int, elem_type: int, h_splitters, nspl: int, eq: bool,
                               stream: int = 0):
    bounds = (ctypes.c_uint64 * 257)()
    K = ctypes.c_uint32(0)
    _check(lib().ips4o_debug_partition_once(ctypes.c_void_p(d_ptr), n, elem_type, h_splitters, nspl,
                                            int(eq), bounds, ctypes.byref(K), ctypes.c_void_p(stream)),
           "ips4o_debug_partition_once")
    return [int(x) for x in bounds[:K.value + 1]], int(K.value)


# ------------------------------------------------------------------ torch helpers

def elem_type_of(t) -> int:
    import torch
    if t.dtype == torch.uint64 and t.dim() == 1:
        return IPS4O_U64
    if t.dtype == torch.float64 and t.dim() == 1:
        return IPS4O_F64
    if t.dtype == torch.uint64 and t.dim() == 2 and t.shape[1] == 2:
        return IPS4O_PAIR_U64
    if t.dtype == torch.uint8 and t.dim() == 2 and t.shape[1] == 100:
        return IPS4O_REC100_K10
    if t.dtype == torch.float64 and t.dim() == 2 and t.shape[1] == 2:
        return IPS4O_PAIR_F64
    if t.dtype == torch.float64 and t.dim() == 2 and t.shape[1] == 4:
        return IPS4O_QUARTET_F64
    raise TypeError(f"unsupported tensor {t.dtype} {tuple(t.shape)}")


def sort_(t):
    """Sort a contiguous CUDA tensor in place on the current stream (no copies, no CPU path)."""
    import torch
    if not t.is_cuda:
        raise Ips4oError("sort_ expects a CUDA tensor (there is no CPU fallback)")
    if not t.is_contiguous():
        raise Ips4oError("sort_ expects a contiguous tensor")
    et = elem_type_of(t)
    stream = torch.cuda.current_stream(t.device).cuda_stream
    with torch.cuda.device(t.device):
        ips4o_sort(t.data_ptr(), t.shape[0], et, stream)
    return t


def splitters_buffer(splitters, elem_type: int):
    """Host buffer for the debug hooks: keys in the element type's key format."""
    import numpy as np
    a = np.ascontiguousarray(splitters)
    if elem_type == IPS4O_F64:
        a = a.astype(np.float64)
    elif elem_type in (IPS4O_U64, IPS4O_PAIR_U64):
        a = a.astype(np.uint64)
    elif elem_type in (IPS4O_PAIR_F64, IPS4O_QUARTET_F64):
        a = a.astype(np.float64)
    return a, a.ctypes.data_as(ctypes.c_void_p), a.shape[0]
