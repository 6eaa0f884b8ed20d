"""Helpers for the -m gpu tests: numpy <-> CUDA tensors of the four element layouts, and an
order-independent multiset digest (test plumbing, not part of the product)."""
import numpy as np
import torch

import workloads as W


def to_dev(a: np.ndarray, et: int) -> torch.Tensor:
    if et == W.ELEM_F64:
        return torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if et in (W.ELEM_U64, W.ELEM_PAIR):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda().view(torch.uint64)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def to_host(t: torch.Tensor, et: int) -> np.ndarray:
    if et == W.ELEM_F64:
        return t.cpu().numpy()
    if et in (W.ELEM_U64, W.ELEM_PAIR):
        return t.view(torch.int64).cpu().numpy().view(np.uint64)
    return t.cpu().numpy()


def words_i64(t: torch.Tensor) -> torch.Tensor:
    """Rows of 64-bit words (int64 view) of a device tensor of any element layout."""
    if t.dtype == torch.uint8:
        n = t.shape[0]
        pad = torch.zeros((n, 104), dtype=torch.uint8, device=t.device)
        pad[:, :100] = t
        return pad.view(torch.int64).view(n, 13)
    return t.view(torch.int64).reshape(t.shape[0], -1)


def _i64(x: int) -> int:
    return ((x + (1 << 63)) % (1 << 64)) - (1 << 63)


def digest(t: torch.Tensor):
    """Order-independent multiset digest: (sum of h(row), sum of h(row)^2) mod 2^64 with a
    row hash built from wrapping int64 arithmetic."""
    w = words_i64(t)
    h = torch.zeros(w.shape[0], dtype=torch.int64, device=t.device)
    for c in range(w.shape[1]):
        x = w[:, c] + _i64((c + 1) * 0x9E3779B97F4A7C15)
        x = x ^ (x >> 31)
        x = x * -4658895280553007687
        x = x ^ (x >> 29)
        h = (h * 1000003) ^ x
    h = h * -7723592293110705685
    h = h ^ (h >> 32)
    return int(h.sum().item()), int((h * h).sum().item())


def keys_nondecreasing(t: torch.Tensor, et: int) -> bool:
    if et == W.ELEM_F64:
        k = t
        return bool((k[1:] >= k[:-1]).all().item())
    if et == W.ELEM_U64:
        k = t.view(torch.int64) ^ (-(1 << 63))     # unsigned order -> signed order
        return bool((k[1:] >= k[:-1]).all().item())
    if et == W.ELEM_PAIR:
        k = t.view(torch.int64)[:, 0] ^ (-(1 << 63))
        return bool((k[1:] >= k[:-1]).all().item())
    # rec100: key = bytes [0,10): big-endian u64 of bytes 0..7, then u16 of bytes 8..9
    b = t[:, :10].to(torch.int64)
    hi = torch.zeros(t.shape[0], dtype=torch.int64, device=t.device)
    for i in range(8):
        hi = (hi << 8) | b[:, i]
    hi = hi ^ (-(1 << 63))
    lo = (b[:, 8] << 8) | b[:, 9]
    ok_hi = hi[1:] >= hi[:-1]
    eq_hi = hi[1:] == hi[:-1]
    ok = ok_hi & (~eq_hi | (lo[1:] >= lo[:-1]))
    return bool(ok.all().item())


def check_equal_to_oracle(et, inp, got, exp):
    """Keys bit-exact vs the oracle; records: key sequence bit-exact + whole-record multiset."""
    if et in (W.ELEM_U64, W.ELEM_F64):
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    elif et == W.ELEM_PAIR:
        assert np.array_equal(got[:, 0], exp[:, 0])
        ri = np.sort(inp.view([("k", "<u8"), ("v", "<u8")]).ravel(), order=["k", "v"])
        ro = np.sort(got.view([("k", "<u8"), ("v", "<u8")]).ravel(), order=["k", "v"])
        assert np.array_equal(ri, ro)
    elif et in (W.ELEM_PAIR_F64, W.ELEM_QUARTET_F64):
        # keys (1 or 3 doubles) bit-exact; the f64 payload is the original index: a permutation
        # carrying its record's keys
        nk = 1 if et == W.ELEM_PAIR_F64 else 3
        assert np.array_equal(got[:, :nk].view(np.uint64), exp[:, :nk].view(np.uint64))
        pay = got[:, nk].astype(np.int64)
        assert np.array_equal(np.sort(pay), np.arange(inp.shape[0]))
        assert np.array_equal(inp[pay, :nk].view(np.uint64), got[:, :nk].view(np.uint64))
    else:
        assert np.array_equal(got[:, :10], exp[:, :10])
        assert np.array_equal(np.sort(inp.view("S100").ravel()), np.sort(got.view("S100").ravel()))
