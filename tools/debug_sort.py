"""Debug helper (tools only): sort one input, report stats and the first mismatching ranges."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle
import paper_1705_02257_b200 as ips4o
import workloads as W
from gpu_util import to_dev, to_host

def run(dist, n, prof=False, seed=1):
    et, a = W.make(dist, n, seed)
    ips4o.ips4o_profile_enable(prof)
    t = to_dev(a, et)
    ips4o.sort_(t)
    torch.cuda.synchronize()
    st = ips4o.ips4o_last_stats()
    got = to_host(t, et)
    exp = oracle.sort(a)
    k = got if et != W.ELEM_PAIR else got[:, 0]
    ke = exp if et != W.ELEM_PAIR else exp[:, 0]
    bad = np.nonzero(k != ke)[0] if et != W.ELEM_REC100 else np.nonzero((got[:, :10] != exp[:, :10]).any(1))[0]
    print(dist, n, "prof" if prof else "", "mismatches", bad.size, "first", bad[:5], "last", bad[-5:] if bad.size else "")
    print({kk: v for kk, v in st.items() if kk not in ("reserved_",)})
    if bad.size:
        srt = np.all(k[1:] >= k[:-1]) if et != W.ELEM_REC100 else None
        print("output sorted:", srt, " multiset equal:", np.array_equal(np.sort(k), ke) if et != W.ELEM_REC100 else None)

if __name__ == "__main__":
    torch.cuda.set_device(0)
    for spec in sys.argv[1:]:
        d, e = spec.split(":")[:2]
        prof = spec.endswith(":p")
        run(d, int(e), prof)
