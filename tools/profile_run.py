"""Run a fixed number of sorts of one bench workload (for ncu / sanitizer captures)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1705_02257_b200 as ips4o  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="H")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--sorts", type=int, default=2)
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    et, arr, desc = bench.make_input(a.config, a.n)
    pristine = bench.host_to_device(arr, et)
    work = pristine.clone()
    for i in range(a.sorts):
        work.copy_(pristine)
        ips4o.ips4o_sort(work.data_ptr(), arr.shape[0], et, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from gpu_util import digest, keys_nondecreasing
    ok = keys_nondecreasing(work, et) and digest(work) == digest(pristine)
    print("ok" if ok else "MISMATCH", ips4o.ips4o_last_stats())
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
