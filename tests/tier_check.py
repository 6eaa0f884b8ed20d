"""Helper for test_gpu_parity.test_single_cta_tier_*: run in a subprocess so that
IPS4O_MEDIUM_MAX (read once per process) routes every task of the given sizes through the
single-CTA tier; compares with the oracle and prints one JSON line."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
sys.path.insert(0, __file__.rsplit("/", 1)[0])
import oracle  # noqa: E402
import paper_1705_02257_b200 as ips4o  # noqa: E402
import workloads as W  # noqa: E402
from gpu_util import check_equal_to_oracle, to_dev, to_host  # noqa: E402

res = []
torch.cuda.set_device(0)
for spec in sys.argv[1:]:
    dist, n, seed = spec.split(":")
    et, a = W.make(dist, int(n), int(seed))
    t = to_dev(a, et)
    ips4o.sort_(t)
    torch.cuda.synchronize()
    st = ips4o.ips4o_last_stats()
    got = to_host(t, et)
    ok = True
    try:
        check_equal_to_oracle(et, a, got, oracle.sort(a))
    except AssertionError:
        ok = False
    res.append({"spec": spec, "ok": ok, "medium_tasks": st["medium_tasks"], "medium_partitions": st["medium_partitions"],
                "medium_marks": st["medium_marks"], "medium_leaves": st["medium_leaves"], "err": st["device_error"]})
print(json.dumps(res))
