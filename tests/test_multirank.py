"""The N > 1 host path of bench.py on CPU (gloo, world size 2): replicas only -- each rank
times its own sorts, the job's step time is the max over ranks, the value counts every
rank's elements.  No GPU needed."""
import os
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        ws_, r_, _ = bench.dist_env()
        steps = [1.0 + rank, 2.0 + rank, 3.0 + rank]  # rank 1 is the slow one
        ms = bench.replica_ms(steps, "cpu")
        q.put((rank, ws_, r_, ms, bench.replica_value(1 << 20, ws, ms)))
    finally:
        dist.destroy_process_group()


def test_replicas_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ws, r, ms, val in res:
        assert ws == 2 and r == rank
        assert ms == pytest.approx(3.0)  # slowest rank: (2 + 3 + 4) / 3
        assert val == pytest.approx(2 * (1 << 20) / 3e-3 / 1e9)
