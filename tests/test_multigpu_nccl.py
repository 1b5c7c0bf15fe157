"""Multi-GPU parity over NCCL: one process per visible GPU (2..8), the product path end to end.

Each rank runs the CUDA path through the C-ABI on its own device:
  AXPY   its index shard (sharding.axpy_range) with kw_axpy_f32; the gathered Y must equal the
         oracle's single-process Y bit for bit (no collective, bits identical).
  DGEMM  kw_dgemm_rowsharded — A/C row block per rank, B broadcast from rank 0 by ncclBroadcast
         in column panels; the gathered C must equal the single-GPU kw_dgemm result bit for bit
         (every C element is reduced on one rank in the single-GPU kernel's k order).
gloo carries only the test's own gather of results; the data path's one collective is NCCL.

Needs >= 2 GPUs: skipped (with the reason) on a one-GPU box — the world-1 form of the same
pipeline, broadcast included, is tests/test_dgemm_gpu.py::test_rowsharded_single_rank_pipeline.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


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
    import torch.distributed as dist
    from paper_1602_08477_b200 import _lib as L
    from paper_1602_08477_b200 import kernelweave as kw
    from paper_1602_08477_b200 import sharding as S
    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = L.lib()
    try:
        dev = kw.Device.gpu(rank)
        GPU = kw.BackendKind.GpuCudaRt
        qq = kw.Queue(dev, kw.QueueFlavor.Async)

        # ---- AXPY fp32, reference Workload seeding, ragged n
        n = (1 << 22) + 3
        alpha, x, y = O.workload_axpy(n, 42, True)
        lo, hi = S.axpy_range(n, world, rank)
        ns = hi - lo
        X, Y = kw.Buffer(dev, kw.IndexVec(max(ns, 1)), 4), kw.Buffer(dev, kw.IndexVec(max(ns, 1)), 4)
        if ns:
            X.upload(x[lo:hi])
            Y.upload(y[lo:hi])
            qq.enqueue(kw.createExec(GPU, kw.axpyWorkDiv(GPU, ns, 512, 4), kw.AxpyKernel(),
                                     kw.AxpyArgs(ns, float(alpha), X, Y)))
            qq.wait()
        part = Y.download()[:ns] if ns else np.zeros(0, np.float32)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, part))
        axpy_ok = None
        if rank == 0:
            full = np.concatenate([p[1] for p in sorted(parts, key=lambda t: t[0])])
            axpy_ok = bool(np.array_equal(full, O.axpy(alpha, x, y)))

        # ---- DGEMM row-sharded with the NCCL panel broadcast
        m, nn, k, panels = 1000, 1001, 300, 3
        rng = np.random.default_rng(11)
        a, b, c = rng.random((m, k)) * 10, rng.random((k, nn)) * 10, rng.random((m, nn)) * 10
        r0, r1 = S.dgemm_rows(m, world, rank)
        ml = r1 - r0
        A = kw.Buffer(dev, kw.IndexVec(max(ml, 1), k), 8)
        Cb = kw.Buffer(dev, kw.IndexVec(max(ml, 1), nn), 8)
        if ml:
            A.upload(a[r0:r1])
            Cb.upload(c[r0:r1])
        B = None
        if rank == 0:
            B = kw.Buffer(dev, kw.IndexVec(k, nn), 8)
            B.upload(b)
        elems = C.c_size_t()
        assert lib.kw_dgemm_rowsharded_scratch(nn, k, panels, C.byref(elems)) == 0
        scratch = kw.Buffer(dev, kw.IndexVec(elems.value), 8)
        uid = (C.c_char * 128)()
        if rank == 0:
            assert lib.kw_comm_unique_id(uid) == 0
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        comm = C.c_void_p()
        assert lib.kw_comm_init(C.byref(comm), rank, world, rank, uid) == 0, L.last_error()
        st = lib.kw_dgemm_rowsharded(comm, qq.handle(), ml, nn, k, 1.3, A.data(), A.leadingDim(),
                                     B.data() if B is not None else None, B.leadingDim() if B is not None else 0,
                                     0.7, Cb.data(), Cb.leadingDim(), scratch.data(), panels, 0)
        assert st == 0, L.last_error()
        qq.wait()
        lib.kw_comm_destroy(comm)
        blk = Cb.download()[:ml] if ml else np.zeros((0, nn))
        blocks = [None] * world
        dist.all_gather_object(blocks, (r0, blk))
        gemm_ok = None
        if rank == 0:
            got = np.vstack([t[1] for t in sorted(blocks, key=lambda t: t[0]) if t[1].size])
            A1, B1, C1 = (kw.Buffer(dev, kw.IndexVec(*v.shape), 8) for v in (a, b, c))
            A1.upload(a)
            B1.upload(b)
            C1.upload(c)
            kw.executeTask(GPU, kw.gemmTiledWorkDiv(GPU, m, nn, 128), kw.GemmTiledKernel(),
                           kw.GemmArgs(m, nn, k, 1.3, 0.7, A1, B1, C1))
            gemm_ok = bool(np.array_equal(got, C1.download()))
        q.put((rank, axpy_ok, gemm_ok, None))
    except Exception as ex:  # noqa: BLE001 — reported to the parent
        q.put((rank, None, None, f"{type(ex).__name__}: {ex}"))
        raise
    finally:
        dist.destroy_process_group()


def test_nccl_ranks_reproduce_the_single_gpu_bits():
    import torch.multiprocessing as mp
    from paper_1602_08477_b200 import kernelweave as kw
    world = min(kw.device_count(), 8)
    if world < 2:
        pytest.skip(f"needs >= 2 GPUs, {world} visible (world-1 pipeline: test_rowsharded_single_rank_pipeline)")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=400) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    errs = [r[3] for r in res if r[3]]
    assert not errs, errs
    assert res[0][1] is True, "gathered AXPY shards differ from the oracle"
    assert res[0][2] is True, "gathered row-sharded C differs from the single-GPU kw_dgemm"
    assert all(p.exitcode == 0 for p in procs)
