"""Debug helper: sort one workload of one size on cuda:0 and compare with numpy (child process)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_02257_b200 as ips4o  # noqa: E402
import workloads as W  # noqa: E402
from gpu_util import to_dev, to_host  # noqa: E402


def main():
    dist, n, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 1
    et, a = W.make(dist, n, seed)
    t = to_dev(a, et)
    t0 = time.time()
    ips4o.sort_(t)
    torch.cuda.synchronize()
    dt = time.time() - t0
    got = to_host(t, et)
    if et == W.ELEM_REC100:
        ok = np.array_equal(np.sort(np.ascontiguousarray(a).view("S100").ravel()),
                            np.ascontiguousarray(got).view("S100").ravel()) or \
            np.array_equal(np.sort(np.ascontiguousarray(a[:, :10]).view("S10").ravel()),
                           np.ascontiguousarray(got[:, :10]).view("S10").ravel())
    elif et == W.ELEM_PAIR:
        ok = np.array_equal(np.sort(a[:, 0]), got[:, 0])
    else:
        ok = np.array_equal(np.sort(a), got)
    print(dist, n, "OK" if ok else "MISMATCH", f"{dt*1e3:.1f} ms", ips4o.ips4o_last_stats(), flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
