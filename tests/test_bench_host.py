"""CPU: bench.py's host-side plumbing that the driver's N > 1 runs depend on — input blocks
(every rank count sees the same global bytes), the reference arm's config equality, and the
distributed helpers (gather_objects, the quiet store wait used while rank 0 runs the CPU
baseline) in two gloo processes."""
import os
import socket
import sys
import time
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_axpy_input_shards_concatenate_to_the_global_input():
    n = 5 * bench.INPUT_BLOCK + 12345
    gx, gy = bench.axpy_inputs(0, n)
    for world in (2, 3, 8):
        per = -(-n // world)
        xs, ys = [], []
        for r in range(world):
            lo, hi = min(n, r * per), min(n, (r + 1) * per)
            x, y = bench.axpy_inputs(lo, hi)
            xs.append(x)
            ys.append(y)
        assert np.array_equal(np.concatenate(xs), gx) and np.array_equal(np.concatenate(ys), gy)
    assert gx.dtype == np.float32 and 0 <= gx.min() and gx.max() < 10


def test_gemm_rows_are_regenerable_one_by_one():
    a = bench.gemm_rows(7, range(10), 33)
    b = np.vstack([bench.gemm_rows(7, [r], 33) for r in range(10)])
    assert np.array_equal(a, b) and a.shape == (10, 33)


def test_both_arms_print_the_same_config():
    for world in (1, 2, 8):
        c = bench.axpy_config(world, 512, 4)
        assert c == bench.axpy_config(world, 512, 4)
        assert c["n_per_rank"] * world >= bench.N_AXPY and c["workdiv"]["blocks"] * 512 * 4 >= c["n_per_rank"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import bench as B
    d = B.Dist(world, "gloo")
    got = d.gather_objects((rank, rank * rank))
    t0 = time.perf_counter()
    if rank == 0:
        time.sleep(1.0)  # "CPU baseline"
    d.quiet_wait_for_rank0("test-key")
    waited = time.perf_counter() - t0
    mx = d.max(float(rank + 1))
    d.close()
    q.put((rank, got, waited, mx))


def test_dist_helpers_world2_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == [(0, 0), (1, 1)] == res[1][1]
    assert res[1][2] >= 0.9  # rank 1 waited for rank 0's work
    assert res[0][3] == res[1][3] == 2.0
