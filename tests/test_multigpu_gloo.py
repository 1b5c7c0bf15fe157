"""CPU, world_size 2 over gloo: the multi-GPU decomposition (sharding.py — the plan bench.py
and kw_dgemm_rowsharded execute on NVLink) reproduces the single-process result bit for bit.
The per-rank compute is the oracle (test infrastructure); what is under test is the host-side
partitioning: AXPY index ranges, DGEMM row blocks, the panel-major B broadcast from the root."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1602_08477_b200 import sharding as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # ---- AXPY: index shards, no collective on the data path; gather only to check
        n = 100003
        alpha, x, y = O.workload_axpy(n, 42, True)
        lo, hi = S.axpy_range(n, world, rank)
        part = O.axpy(alpha, x[lo:hi], y[lo:hi])
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, part))
        full = np.concatenate([p[2] for p in sorted(parts, key=lambda t: t[0])])
        axpy_ok = np.array_equal(full, O.axpy(alpha, x, y))

        # ---- DGEMM: row blocks + B broadcast from rank 0 in two row slabs (the default k-slab
        # schedule: contiguous rows of B at the Buffer pitch, in place at the root)
        m, nn, k = 300, 521, 77  # odd n: B's pitch is padded to round8(n)
        rng = np.random.default_rng(5)
        a = rng.random((m, k)) * 10
        c = rng.random((m, nn)) * 10
        ldp = S.ceil_div(nn, 8) * 8
        b_root = rng.random((k, nn)) * 10 if rank == 0 else None
        r0, r1 = S.dgemm_rows(m, world, rank)
        scratch = torch.zeros(S.dgemm_panel_scratch(nn, k, 3), dtype=torch.float64)
        assert scratch.numel() == k * ldp
        if rank == 0:
            padded = np.zeros((k, ldp))
            padded[:, :nn] = b_root
            scratch.copy_(torch.from_numpy(padded.reshape(-1)))
        slabs = S.dgemm_kslabs(k, 3)
        assert slabs[0][0] == 0 and slabs[-1][1] == k
        for k0, k1 in slabs:
            dist.broadcast(scratch[k0 * ldp:k1 * ldp], src=0)
        b_full = scratch.numpy().reshape(k, ldp)[:, :nn]
        cl = O.gemm(1.3, 0.7, a[r0:r1], b_full, c[r0:r1], threads=1) if r1 > r0 else c[r0:r1]
        blocks = [None] * world
        dist.all_gather_object(blocks, (r0, cl))
        cfull = np.vstack([blk[1] for blk in sorted(blocks, key=lambda t: t[0]) if blk[1].size])
        b_all = [None]
        if rank == 0:
            b_all = [b_root]
        dist.broadcast_object_list(b_all, src=0)
        gemm_ok = np.array_equal(cfull, O.gemm(1.3, 0.7, a, b_all[0], c, threads=1))
        q.put((rank, bool(axpy_ok), bool(gemm_ok), (lo, hi), (r0, r1)))
    finally:
        dist.destroy_process_group()


def test_decomposition_world2_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] for r in res), "AXPY shards differ from the single-process result"
    assert all(r[2] for r in res), "row-sharded DGEMM differs from the single-process result"
    # shards tile the index space exactly
    assert res[0][3][0] == 0 and res[0][3][1] == res[1][3][0] and res[1][3][1] == 100003
    assert res[0][4] == (0, 256) and res[1][4] == (256, 300)


@pytest.mark.parametrize("n,world", [(1 << 28, 8), (1 << 28, 3), (17, 4), (5, 8)])
def test_axpy_ranges_cover_exactly(n, world):
    spans = [S.axpy_range(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and a <= b
    for lo, _ in spans:
        assert lo % 4 == 0 or lo == n


def test_panel_layout_matches_the_c_abi_rule():
    ps = S.dgemm_panels(16384, 16384, 8)
    assert [p.width for p in ps] == [2048] * 8
    assert ps[-1].offset + 16384 * ps[-1].width == 16384 * 16384
    assert S.dgemm_panel_scratch(16384, 16384, 8) == 16384 * 16384  # either schedule
    ps = S.dgemm_panels(1000, 200, 3)
    assert [p.width for p in ps] == [384, 384, 232] and [p.n0 for p in ps] == [0, 384, 768]
    ps = S.dgemm_panels(1001, 200, 3)
    assert [p.width for p in ps] == [384, 384, 233] and [p.ld for p in ps] == [384, 384, 240]
    assert [p.offset for p in ps] == [0, 200 * 384, 2 * 200 * 384]
    assert S.dgemm_panel_scratch(1001, 200, 3) == 200 * 1008  # k-slab schedule: k x round8(n)
    assert [p.width for p in S.dgemm_panels(100, 5, 4)] == [100]  # one tile: a single panel


def test_kslabs_partition_k():
    assert S.dgemm_kslabs(16384, 8) == [(0, 2048), (2048, 16384)]
    assert S.dgemm_kslabs(77, 3) == [(0, 16), (16, 77)]  # 5 k-tiles of 16: the first slab is one
    assert S.dgemm_kslabs(10, 8) == [(0, 10)]  # a single k-tile: one slab
    assert S.dgemm_kslabs(1000, 1) == [(0, 1000)]


@pytest.mark.parametrize("n,k,panels", [(16384, 16384, 8), (1001, 200, 3), (127, 9, 2), (5000, 33, 7), (100, 5, 4)])
def test_scratch_size_matches_the_c_abi(n, k, panels):
    import ctypes as C
    from paper_1602_08477_b200 import _lib as L
    elems = C.c_size_t()
    assert L.lib().kw_dgemm_rowsharded_scratch(n, k, panels, C.byref(elems)) == 0
    assert elems.value == S.dgemm_panel_scratch(n, k, panels)
