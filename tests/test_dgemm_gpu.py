"""GPU parity: K2 tiled DGEMM (DMMA) and K3 naive DGEMM (bit-exact) through the C-ABI.

Tolerance for K2 (stated in SURVEY.md §7 "Hard parts" 6 / DESIGN.md):
    |C_gpu - C_ref| <= (K + 4) * 2^-53 * |C_ref|   elementwise,
where C_ref is gemmReference (oracle). K3 must be bitwise equal. Mirrors test_kernels.cpp:114-306
and acceptance criterion 1's GEMM half (acceptance.cpp:117-155)."""
import ctypes as C

import numpy as np
import pytest

from paper_1602_08477_b200 import _lib as L
from paper_1602_08477_b200 import kernelweave as kw

pytestmark = pytest.mark.gpu
GPU = kw.BackendKind.GpuCudaRt
U = 2.0 ** -53


def h(v):
    return f"{v:016x}"


def mat(dev, a, rows=None, cols=None, align=64):
    a = np.asarray(a, dtype=np.float64)
    r, c = a.shape
    b = kw.Buffer(dev, kw.IndexVec(rows or r, cols or c), 8, align)
    if rows is None and cols is None:
        b.upload(a)
    else:
        full = np.zeros((rows or r, cols or c))
        full[:r, :c] = a
        b.upload(full)
    return b


SPLITK_CFG = 27  # split-k over config 17: deterministic, within tolerance, not the one-CTA chain's bits


def within_tol(got, ref, k):
    err = np.abs(got - ref)
    bound = (k + 4) * U * np.abs(ref)
    return bool(np.all(err <= bound)), float(np.max(err / np.maximum(np.abs(ref), 1e-300)) / ((k + 4) * U))


def tiled(dev, alpha, beta, a, b, c, tile=128, align=64):
    m, k = a.shape
    n = b.shape[1]
    A, B, Cb = mat(dev, a, align=align), mat(dev, b, align=align), mat(dev, c, align=align)
    kw.executeTask(GPU, kw.gemmTiledWorkDiv(GPU, m, n, tile), kw.GemmTiledKernel(),
                   kw.GemmArgs(m, n, k, alpha, beta, A, B, Cb, tile))
    return Cb.download()


def naive(dev, alpha, beta, a, b, c, tpb=4, ept=4):
    m, k = a.shape
    n = b.shape[1]
    A, B, Cb = mat(dev, a), mat(dev, b), mat(dev, c)
    kw.executeTask(GPU, kw.gemmNaiveWorkDiv(GPU, m, n, tpb, ept), kw.GemmNaiveKernel(),
                   kw.GemmArgs(m, n, k, alpha, beta, A, B, Cb))
    return Cb.download()


def test_gemm_closed_forms(gpu, oracle):
    rng = oracle.MT64(seed=7)
    ident = np.eye(4)
    b = rng.fill_uniform(16).reshape(4, 4)
    c = rng.fill_uniform(16).reshape(4, 4)
    for run in (tiled, naive):
        assert np.array_equal(run(gpu, 1.0, 0.0, ident, b, c), b)
        a2 = np.array([[1.0, 2.0], [3.0, 4.0]])
        b2 = np.array([[5.0, 6.0], [7.0, 8.0]])
        assert run(gpu, 1.0, 0.0, a2, b2, np.zeros((2, 2))).tolist() == [[19, 22], [43, 50]]
        c3 = rng.fill_uniform(16).reshape(4, 4)
        assert np.array_equal(run(gpu, 0.0, 1.0, ident, b, c3), c3)
        assert run(gpu, 2.0, 10.0, np.array([[3.0]]), np.array([[5.0]]), np.array([[7.0]]))[0, 0] == 100.0


@pytest.mark.parametrize("case", [4, 5])
def test_golden_workloads(gpu, oracle, golden, case):
    c = golden["workloads"][case]
    alpha, beta, a, b, cin = oracle.workload_gemm(c["n"], c["seed"], "gemm-tiled")
    ref = oracle.gemm(alpha, beta, a, b, cin)
    assert h(oracle.fnv1a64(ref)) == c["c_out_digest"]
    # K3 naive: bitwise equal to the reference digest
    assert h(oracle.fnv1a64(naive(gpu, alpha, beta, a, b, cin))) == c["c_out_digest"]
    for tile in (64, 128):
        ok, worst = within_tol(tiled(gpu, alpha, beta, a, b, cin, tile), ref, c["n"])
        assert ok, worst


def test_naive_bitwise_random_cases(gpu, oracle):
    """test_kernels.cpp:184-206: 50 random m, n, k <= 64 (seed 1234), bitwise."""
    rng = oracle.MT64(seed=1234)
    for _ in range(50):
        m, n, k = 1 + rng() % 64, 1 + rng() % 64, 1 + rng() % 64
        a = rng.fill_uniform(m * k).reshape(m, k)
        b = rng.fill_uniform(k * n).reshape(k, n)
        c = rng.fill_uniform(m * n).reshape(m, n)
        alpha = 0.5 + float(rng() % 8)
        beta = float(rng() % 3)
        assert np.array_equal(naive(gpu, alpha, beta, a, b, c), oracle.gemm(alpha, beta, a, b, c))


@pytest.mark.parametrize("tile", [64, 128])
def test_tiled_every_size_1_to_64_and_large(gpu, oracle, tile):
    """test_kernels.cpp:208-230 sizes 1..64 plus acceptance's {65, 100, 127, 128, 256}."""
    rng = oracle.MT64(seed=5678)
    worst = 0.0
    for s in list(range(1, 65)) + [65, 100, 127, 128, 129, 256]:
        a, b, c = (rng.fill_uniform(s * s).reshape(s, s) for _ in range(3))
        got = tiled(gpu, 1.25, 0.75, a, b, c, tile)
        ok, w = within_tol(got, oracle.gemm(1.25, 0.75, a, b, c), s)
        worst = max(worst, w)
        assert ok, (s, w)
    assert worst < 1.0


def test_ragged_and_rectangular(gpu, oracle, golden):
    rng = oracle.MT64(seed=4321)
    cases = golden["gemm_ragged_rng4321"]
    shapes = [(16, 16, 16, 2.0, 1.0), (10, 10, 10, 1.0, 0.5)]
    for (m, n, k, al, be), cs in zip(shapes, cases[:2]):
        a, b, c = (rng.fill_uniform(m * m).reshape(m, m) for _ in range(3))
        assert h(oracle.fnv1a64(naive(gpu, al, be, a, b, c))) == cs["c_out_digest"]
        assert within_tol(tiled(gpu, al, be, a, b, c), oracle.gemm(al, be, a, b, c), k)[0]
    m, n, k = 13, 29, 7
    a = rng.fill_uniform(m * k).reshape(m, k)
    b = rng.fill_uniform(k * n).reshape(k, n)
    c = rng.fill_uniform(m * n).reshape(m, n)
    assert h(oracle.fnv1a64(naive(gpu, 2.5, 0.0, a, b, c))) == cases[2]["c_out_digest"]
    assert within_tol(tiled(gpu, 2.5, 0.0, a, b, c), oracle.gemm(2.5, 0.0, a, b, c), k)[0]
    # odd leading dimensions (8-byte cp.async path) and rectangular extents
    for (m, n, k) in ((1, 1, 1), (3, 5, 7), (130, 257, 33), (257, 130, 1), (64, 200, 513)):
        a = rng.fill_uniform(m * k).reshape(m, k)
        b = rng.fill_uniform(k * n).reshape(k, n)
        c = rng.fill_uniform(m * n).reshape(m, n)
        for tile in (64, 128):
            for align in (8, 64):  # rowAlignment 8 -> odd leading dimensions (8-byte cp.async path)
                got = tiled(gpu, 1.5, 0.5, a, b, c, tile, align)
                assert within_tol(got, oracle.gemm(1.5, 0.5, a, b, c), k)[0], (m, n, k, tile, align)


def test_never_writes_outside_logical_extents(gpu, oracle):
    """test_kernels.cpp:281-306: C in a larger buffer, 0xEE canary everywhere else."""
    rng = oracle.MT64(seed=86)
    m, n, k = 9, 11, 5
    a = rng.fill_uniform(m * k).reshape(m, k)
    b = rng.fill_uniform(k * n).reshape(k, n)
    for kern, wdf in ((kw.GemmTiledKernel(), lambda: kw.gemmTiledWorkDiv(GPU, m, n, 64)),
                      (kw.GemmNaiveKernel(), lambda: kw.gemmNaiveWorkDiv(GPU, m, n, 2, 2))):
        A, B = mat(gpu, a), mat(gpu, b)
        Cb = kw.Buffer(gpu, kw.IndexVec(m + 3, n + 5), 8)
        Cb.fill_raw(0xEE)
        ones = np.ones((m, n))
        q = kw._default_queue(gpu)
        assert L.lib().kw_copy(q.handle(), Cb.data(), Cb.rowPitch(), L.sz3((m + 3, n + 5)), ones.ctypes.data, n * 8,
                               L.sz3((m, n)), 2, L.sz3((m, n)), 8) == 0
        q.wait()
        kw.executeTask(GPU, wdf(), kern, kw.GemmArgs(m, n, k, 1.0, 0.0, A, B, Cb))
        raw = np.frombuffer(Cb.download_raw(), dtype=np.uint8).reshape(m + 3, Cb.rowPitch())
        assert (raw[:m, n * 8:] == 0xEE).all() and (raw[m:] == 0xEE).all()


def test_beta_zero_still_reads_c(gpu):
    """gemm.cpp:35 / 115: beta multiplies C even when 0, so NaN in C propagates."""
    c = np.full((4, 4), np.nan)
    for run in (tiled, naive):
        out = run(gpu, 1.0, 0.0, np.eye(4), np.eye(4), c)
        assert np.isnan(out).all()


def test_row_panels_and_column_panels_are_bitwise_invariant(gpu, oracle):
    """The property the row-sharded multi-GPU DGEMM relies on: computing C in row blocks or
    column panels (different A/B/C base pointers and leading dimensions) gives the same bits
    as one launch."""
    rng = np.random.default_rng(3)
    m, n, k = 384, 512, 300
    a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
    full = tiled(gpu, 1.7, 0.3, a, b, c)
    parts = np.vstack([tiled(gpu, 1.7, 0.3, a[r:r + 128], b, c[r:r + 128]) for r in range(0, m, 128)])
    assert np.array_equal(full, parts)
    cols = np.hstack([tiled(gpu, 1.7, 0.3, a, np.ascontiguousarray(b[:, j:j + 128]), c[:, j:j + 128])
                      for j in range(0, n, 128)])
    assert np.array_equal(full, cols)


@pytest.mark.parametrize("n,panels,align", [(1000, 3, 64), (1001, 3, 64), (1001, 8, 256), (127, 2, 64),
                                           (2049, 5, 256), (640, 1, 64)])
def test_rowsharded_single_rank_pipeline(gpu, oracle, n, panels, align):
    """kw_dgemm_rowsharded with world = 1 (NCCL single-rank communicator): B goes through
    ncclBroadcast (a single-rank broadcast is executed, not skipped) in the default k-slab
    schedule's two row slabs, then the rank's product runs as two k-range launches (accumulators
    parked between them). Must equal kw_dgemm bit for bit — including odd n, and B pitches that
    are not the Buffer rule (align 256: the root packs B into the scratch first, which must then
    hold B at leading dimension round8(n))."""
    from paper_1602_08477_b200 import sharding as S
    rng = np.random.default_rng(5)
    m, k = 256, 200
    a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
    want = tiled(gpu, 1.1, 0.9, a, b, c)
    uid = (C.c_char * 128)()
    assert L.lib().kw_comm_unique_id(uid) == 0
    comm = C.c_void_p()
    assert L.lib().kw_comm_init(C.byref(comm), 0, 1, 0, uid) == 0, L.last_error()
    elems = C.c_size_t()
    assert L.lib().kw_dgemm_rowsharded_scratch(n, k, panels, C.byref(elems)) == 0
    assert elems.value == S.dgemm_panel_scratch(n, k, panels) == k * (-(-n // 8) * 8)
    A, B, Cb = mat(gpu, a), mat(gpu, b, align=align), mat(gpu, c)
    scratch = kw.Buffer(gpu, kw.IndexVec(elems.value), 8)
    scratch.fill_raw(0)
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    for _ in range(2):  # a second call on the same communicator (events, park scratch reused)
        Cb.upload(c)
        st = L.lib().kw_dgemm_rowsharded(comm, q.handle(), m, n, k, 1.1, A.data(), A.leadingDim(), B.data(),
                                         B.leadingDim(), 0.9, Cb.data(), Cb.leadingDim(), scratch.data(), panels, 0)
        assert st == 0, L.last_error()
        q.wait()
        assert np.array_equal(Cb.download(), want)
    ldp = -(-n // 8) * 8
    got = scratch.download().reshape(k, ldp)[:, :n]
    if B.leadingDim() != ldp:  # packed by the root
        assert np.array_equal(got, b)
    else:  # the root broadcast straight from B: the scratch is untouched
        assert not got.any()
    assert L.lib().kw_comm_destroy(comm) == 0


def test_rowsharded_panel_schedule_still_matches(gpu):
    """KW_ROWSHARD_SCHEDULE=panels (round 1's column panels, one launch per panel, read once per
    process) in a subprocess: bits equal kw_dgemm, panel-major scratch layout."""
    import os
    import subprocess
    import sys
    code = r"""
import ctypes as C, sys, numpy as np
sys.path.insert(0, '.')
from paper_1602_08477_b200 import _lib as L, kernelweave as kw, sharding as S
gpu = kw.Device.gpu(0); GPU = kw.BackendKind.GpuCudaRt
rng = np.random.default_rng(7); m, n, k, panels = 300, 1001, 150, 3
a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
def buf(x):
    t = kw.Buffer(gpu, kw.IndexVec(*x.shape), 8); t.upload(x); return t
A, B, C1, C2 = buf(a), buf(b), buf(c), buf(c)
kw.executeTask(GPU, kw.gemmTiledWorkDiv(GPU, m, n, 128), kw.GemmTiledKernel(), kw.GemmArgs(m, n, k, 1.1, 0.9, A, B, C1))
uid = (C.c_char * 128)(); assert L.lib().kw_comm_unique_id(uid) == 0
comm = C.c_void_p(); assert L.lib().kw_comm_init(C.byref(comm), 0, 1, 0, uid) == 0
e = C.c_size_t(); assert L.lib().kw_dgemm_rowsharded_scratch(n, k, panels, C.byref(e)) == 0
assert e.value == S.dgemm_panel_scratch(n, k, panels) == sum(k * p.ld for p in S.dgemm_panels(n, k, panels))
sc = kw.Buffer(gpu, kw.IndexVec(e.value), 8); q = kw.Queue(gpu, kw.QueueFlavor.Async)
assert L.lib().kw_dgemm_rowsharded(comm, q.handle(), m, n, k, 1.1, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                                   0.9, C2.data(), C2.leadingDim(), sc.data(), panels, 0) == 0, L.last_error()
q.wait(); assert np.array_equal(C1.download(), C2.download()); print("PANELS OK")
"""
    env = dict(os.environ, KW_ROWSHARD_SCHEDULE="panels")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=str(__import__("pathlib").Path(__file__).resolve().parent.parent), timeout=300)
    assert "PANELS OK" in out.stdout, out.stdout + out.stderr


def test_rowsharded_16384_cubed(gpu, oracle):
    """BASELINE configs[3]'s shape through kw_dgemm_rowsharded (world-1 NCCL communicator, the
    8-panel broadcast executing): the full 16384^3 C equals a single kw_dgemm launch bit for bit
    (compared on the device by digest of the downloaded blocks) and 8 sampled rows are within
    (K+4)u of gemmReference (the oracle, 8 threads)."""
    import hashlib
    n = 16384
    lib = L.lib()
    rng = np.random.default_rng(16384)
    A, B, C1, C2 = (kw.Buffer(gpu, kw.IndexVec(n, n), 8) for _ in range(4))
    for buf in (A, B, C1):
        buf.upload(rng.random((n, n)))
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    assert lib.kw_copy(q.handle(), C2.data(), C2.rowPitch(), L.sz3((n, n)), C1.data(), C1.rowPitch(), L.sz3((n, n)), 2,
                       L.sz3((n, n)), 8) == 0
    q.wait()
    rows = [0, 1, 2047, 2048, 8191, 9000, 16000, 16383]
    host_c = C1.download()
    c_rows = host_c[rows].copy()
    del host_c
    uid = (C.c_char * 128)()
    assert lib.kw_comm_unique_id(uid) == 0
    comm = C.c_void_p()
    assert lib.kw_comm_init(C.byref(comm), 0, 1, 0, uid) == 0, L.last_error()
    elems = C.c_size_t()
    assert lib.kw_dgemm_rowsharded_scratch(n, n, 8, C.byref(elems)) == 0
    scratch = kw.Buffer(gpu, kw.IndexVec(elems.value), 8)
    assert lib.kw_dgemm_rowsharded(comm, q.handle(), n, n, n, 1.25, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                                   0.75, C1.data(), C1.leadingDim(), scratch.data(), 8, 0) == 0, L.last_error()
    assert lib.kw_dgemm(q.handle(), None, n, n, n, 1.25, A.data(), A.leadingDim(), B.data(), B.leadingDim(), 0.75,
                        C2.data(), C2.leadingDim()) == 0
    q.wait()
    assert lib.kw_comm_destroy(comm) == 0
    del scratch
    got1 = C1.download()
    d1 = hashlib.blake2b(got1, digest_size=16).hexdigest()
    sampled = got1[rows].copy()
    del got1
    d2 = hashlib.blake2b(C2.download(), digest_size=16).hexdigest()
    assert d1 == d2
    host_a = A.download()
    a_s = host_a[rows].copy()
    del host_a
    ref = oracle.gemm(1.25, 0.75, a_s, B.download(), c_rows, threads=8)
    ok, worst = within_tol(sampled, ref, n)
    assert ok, worst


def test_host_buffers_are_staged(gpu, oracle):
    """DGEMM on host (pinned) buffers: B staged once, A/C row panels pipelined; equal bits to
    the device-resident launch."""
    rng = np.random.default_rng(9)
    m, n, k = 1500, 700, 333
    a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
    want = tiled(gpu, 0.7, 1.3, a, b, c)
    host = kw.Device.host()
    A, B, Cb = (kw.Buffer(host, kw.IndexVec(*x.shape), 8) for x in (a, b, c))
    for buf, x in ((A, a), (B, b), (Cb, c)):
        buf.host_view()[:, : x.shape[1]] = x
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    q.enqueue(kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, m, n, 128), kw.GemmTiledKernel(),
                            kw.GemmArgs(m, n, k, 0.7, 1.3, A, B, Cb)))
    q.wait()
    assert np.array_equal(Cb.host_view()[:, :n], want)


@pytest.mark.parametrize("panels,ksplit", [("1", "4"), ("3", "4"), ("8", "4"), ("16", "4"), ("1", "0"), ("8", "0"),
                                           ("3", "2"), ("1", "3"), ("16", "64"), ("3", "p20,45,70"), ("8", "p50")])
def test_streamed_host_schedule_is_bitwise_the_resident_launch(gpu, panels, ksplit, monkeypatch):
    """The streamed e2e schedule (pinned A, B, C: panels uploaded in square-growth order, one
    persistent kernel waiting on per-panel ready flags, C blocks downloaded as they complete)
    gives the bits of the device-resident launch for ragged shapes, both tile contracts, several
    panel grids and back-to-back enqueues on one queue (flags are reset per call) — single pass
    (KW_E2E_KSPLIT=0) and k-split (a first pass over the first 1/d of the k-tiles whose
    accumulators are parked and reloaded; d = 64 degenerates to a single pass at small k; "pX,Y"
    = passes at cumulative k-tile percentages, KW_E2E_KPASSES)."""
    monkeypatch.setenv("KW_E2E_PANELS", panels)
    if ksplit.startswith("p"):  # several passes at cumulative k-tile percentages
        monkeypatch.setenv("KW_E2E_KPASSES", ksplit[1:])
    else:
        monkeypatch.setenv("KW_E2E_KSPLIT", ksplit)
    monkeypatch.setenv("KW_E2E_MIN_INTENSITY", "0")  # small shapes: force the streamed schedule
    rng = np.random.default_rng(int(panels) + 40 + 100 * len(ksplit))
    host = kw.Device.host()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    for (m, n, k), tile in (((1500, 700, 333), 128), ((64, 64, 64), 128), ((129, 4100, 17), 128),
                            ((2050, 260, 1000), 64), ((1, 1, 1), 128), ((3000, 2900, 520), 128)):
        a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
        want = tiled(gpu, 0.7, 1.3, a, b, c, tile=tile)
        A, B, Cb = (kw.Buffer(host, kw.IndexVec(*x.shape), 8) for x in (a, b, c))
        for buf, x in ((A, a), (B, b), (Cb, c)):
            buf.host_view()[:, : x.shape[1]] = x
        task = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, m, n, tile), kw.GemmTiledKernel(),
                             kw.GemmArgs(m, n, k, 0.7, 1.3, A, B, Cb, tile))
        q.enqueue(task)
        q.wait()
        assert np.array_equal(Cb.host_view()[:, :n], want), (m, n, k, tile)
        # twice more back to back: C accumulates; compare against the resident path doing the same
        q.enqueue(task)
        q.enqueue(task)
        q.wait()
        want2 = tiled(gpu, 0.7, 1.3, a, b, tiled(gpu, 0.7, 1.3, a, b, want, tile=tile), tile=tile)
        assert np.array_equal(Cb.host_view()[:, :n], want2), (m, n, k, tile, "repeat")


def test_streamed_schedules_on_two_queues_concurrently(gpu, monkeypatch):
    """Two host threads, two queues, streamed host DGEMMs in flight at once (per-queue flags,
    counters and tile orders): every round equals the resident launch bit for bit."""
    import threading
    monkeypatch.setenv("KW_E2E_MIN_INTENSITY", "0")
    rng = np.random.default_rng(46)
    host = kw.Device.host()
    jobs = []
    for m, n, k in ((1100, 900, 700), (640, 1500, 520)):
        a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
        bufs = tuple(kw.Buffer(host, kw.IndexVec(*x.shape), 8) for x in (a, b, c))
        for buf, x in zip(bufs, (a, b, c)):
            buf.host_view()[:, : x.shape[1]] = x
        jobs.append((m, n, k, c, bufs, tiled(gpu, 0.9, 1.1, a, b, c)))
    errs = []

    def run(job):
        m, n, k, c, (A, B, Cb), want = job
        q = kw.Queue(gpu, kw.QueueFlavor.Async)
        task = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, m, n, 128), kw.GemmTiledKernel(),
                             kw.GemmArgs(m, n, k, 0.9, 1.1, A, B, Cb))
        for r in range(4):
            Cb.host_view()[:, :n] = c
            q.enqueue(task)
            q.wait()
            if not np.array_equal(Cb.host_view()[:, :n], want):
                errs.append((m, n, k, r))

    threads = [threading.Thread(target=run, args=(j,)) for j in jobs]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs


def test_row_panel_host_schedule_still_matches(gpu, monkeypatch):
    """KW_E2E_STREAMED=0 keeps the row-panel ring schedule (also the path for operands too large
    to hold whole on the device); same bits."""
    monkeypatch.setenv("KW_E2E_STREAMED", "0")
    rng = np.random.default_rng(44)
    m, n, k = 1800, 900, 410
    a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
    want = tiled(gpu, 1.1, 0.6, a, b, c)
    host = kw.Device.host()
    A, B, Cb = (kw.Buffer(host, kw.IndexVec(*x.shape), 8) for x in (a, b, c))
    for buf, x in ((A, a), (B, b), (Cb, c)):
        buf.host_view()[:, : x.shape[1]] = x
    kw.executeTask(GPU, kw.gemmTiledWorkDiv(GPU, m, n, 128), kw.GemmTiledKernel(),
                   kw.GemmArgs(m, n, k, 1.1, 0.6, A, B, Cb))
    assert np.array_equal(Cb.host_view()[:, :n], want)


def test_4096_within_tolerance(gpu, oracle):
    """The configured 1-GPU point: Workload("gemm-tiled", 4096, 42)."""
    n = 4096
    alpha, beta, a, b, c = oracle.workload_gemm(n, 42)
    got = tiled(gpu, alpha, beta, a, b, c)
    ref = oracle.gemm(alpha, beta, a, b, c)
    ok, worst = within_tol(got, ref, n)
    assert ok, worst


def test_every_tile_configuration_within_tolerance(gpu, oracle):
    """All instantiated DMMA configurations (cp.async and TMA families) on ragged shapes."""
    lib = L.lib()
    rng = np.random.default_rng(21)
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    for (m, n, k) in ((1, 1, 1), (17, 33, 9), (130, 257, 100), (200, 64, 513), (256, 384, 64)):
        a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
        ref = oracle.gemm(1.3, 0.6, a, b, c)
        for cfg in range(lib.kw_dgemm_config_count()):
            A, B, Cb = mat(gpu, a), mat(gpu, b), mat(gpu, c)
            assert lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, 1.3, A.data(), A.leadingDim(), B.data(),
                                            B.leadingDim(), 0.6, Cb.data(), Cb.leadingDim()) == 0, L.last_error()
            q.wait()
            ok, worst = within_tol(Cb.download(), ref, k)
            assert ok, (cfg, m, n, k, worst)


def tiled_bitwise(dev, alpha, beta, a, b, c, align=64):
    m, k = a.shape
    n = b.shape[1]
    A, B, Cb = mat(dev, a, align=align), mat(dev, b, align=align), mat(dev, c, align=align)
    kw.executeTask(GPU, kw.gemmTiledWorkDiv(GPU, m, n, 128), kw.GemmTiledKernel(),
                   kw.GemmArgs(m, n, k, alpha, beta, A, B, Cb, 128, bitwise=True))
    return Cb.download()


@pytest.mark.parametrize("bw_tma", ["1", "0"])
def test_tiled_bitwise_mode_is_bit_exact(gpu, oracle, golden, bw_tma, monkeypatch):
    """GemmTiledKernel in bitwise mode reproduces the reference bit for bit — the reference's
    own contract tiled == naive == gemmReference (test_kernels.cpp:184-279) — with the
    warp-specialised TMA kernel (default) and with the cp.async kernel (KW_BW_TMA=0, also the
    path for odd leading dimensions, align 8 below)."""
    monkeypatch.setenv("KW_BW_TMA", bw_tma)
    for case in (4, 5):
        c = golden["workloads"][case]
        alpha, beta, a, b, cin = oracle.workload_gemm(c["n"], c["seed"], "gemm-tiled")
        assert h(oracle.fnv1a64(tiled_bitwise(gpu, alpha, beta, a, b, cin))) == c["c_out_digest"]
    rng = oracle.MT64(seed=5678)
    for s in list(range(1, 65)) + [65, 127, 129, 200]:
        a, b, c = (rng.fill_uniform(s * s).reshape(s, s) for _ in range(3))
        assert np.array_equal(tiled_bitwise(gpu, 1.25, 0.75, a, b, c), oracle.gemm(1.25, 0.75, a, b, c)), s
    rng2 = np.random.default_rng(17)
    for (m, n, k) in ((13, 29, 7), (130, 257, 33), (257, 130, 1), (64, 200, 513), (1, 1, 1)):
        a, b, c = rng2.standard_normal((m, k)), rng2.standard_normal((k, n)), rng2.standard_normal((m, n))
        for align in (8, 64):
            got = tiled_bitwise(gpu, 1.5, -0.5, a, b, c, align)
            assert np.array_equal(got, oracle.gemm(1.5, -0.5, a, b, c)), (m, n, k, align)


def test_criterion01_gemm_half_bitwise(gpu, oracle):
    """acceptance.cpp:87-155, GEMM half, the reference's exact instances: the seed-101 stream
    continues past the 100 AXPY draws, then 100 naive + 100 tiled instances over sizes 1..64,
    65, 100, 127, 128, 256 with alpha = 0.5 + r%8 and beta = r%2 (0 or 1). Naive and the tiled
    kernel's bit-exact mode must equal gemmReference bitwise; the default (DMMA) tiled mode is
    checked against the (K+4)u bound on the same instances."""
    rng = oracle.MT64(seed=101)
    for _ in range(100):  # the AXPY half's draws (n, x, y, alpha)
        n = 1 + rng() % (1 << 16)
        rng.fill_uniform(n)
        rng.fill_uniform(n)
        rng()
    sizes = list(range(1, 65)) + [65, 100, 127, 128, 256]
    fails = []
    for kernel in ("naive", "tiled"):
        for it in range(100):
            n = sizes[rng() % len(sizes)]
            a = rng.fill_uniform(n * n).reshape(n, n)
            b = rng.fill_uniform(n * n).reshape(n, n)
            c0 = rng.fill_uniform(n * n).reshape(n, n)
            alpha = 0.5 + float(rng() % 8)
            beta = float(rng() % 2)
            want = oracle.gemm(alpha, beta, a, b, c0)
            if kernel == "naive":
                got = naive(gpu, alpha, beta, a, b, c0, 4, 4)
                if not np.array_equal(got, want):
                    fails.append((kernel, it, n))
            else:
                if not np.array_equal(tiled_bitwise(gpu, alpha, beta, a, b, c0), want):
                    fails.append(("tiled-bitwise", it, n))
                if not within_tol(tiled(gpu, alpha, beta, a, b, c0), want, n)[0]:
                    fails.append(("tiled-dmma", it, n))
    assert not fails, fails[:10]


def test_outputs_bitwise_identical_across_divisions_and_runs(gpu, oracle):
    """test_kernels.cpp:308-329 on the GPU: the tiled kernel's bits do not depend on the tile
    contract (64 or 128) or on the run; the bit-exact mode and the naive kernel equal the oracle
    on the same instances (seed 2026, n <= 200)."""
    rng = oracle.MT64(seed=2026)
    for _ in range(6):
        n = 1 + rng() % 200
        a = rng.fill_uniform(n * n).reshape(n, n)
        b = rng.fill_uniform(n * n).reshape(n, n)
        c0 = rng.fill_uniform(n * n).reshape(n, n)
        first = tiled(gpu, 1.5, 0.5, a, b, c0, tile=128)
        assert np.array_equal(tiled(gpu, 1.5, 0.5, a, b, c0, tile=64), first), n
        assert np.array_equal(tiled(gpu, 1.5, 0.5, a, b, c0, tile=128), first), n
        want = oracle.gemm(1.5, 0.5, a, b, c0)
        assert np.array_equal(tiled_bitwise(gpu, 1.5, 0.5, a, b, c0), want), n
        assert np.array_equal(naive(gpu, 1.5, 0.5, a, b, c0), want), n
        assert within_tol(first, want, n)[0], n


def test_tiled_bitwise_4096(gpu, oracle):
    n = 4096
    alpha, beta, a, b, c = oracle.workload_gemm(n, 42)
    assert np.array_equal(tiled_bitwise(gpu, alpha, beta, a, b, c), oracle.gemm(alpha, beta, a, b, c))


def test_paired_configs_are_bitwise_interchangeable(gpu, oracle):
    """Every TMA configuration with the paired k-slot map (14..29 but split-k 27) feeds each output element the
    same DMMA sequence, so tile shape / CTAs per SM / persistence change no bit — which is what
    lets the library pick the tile by problem size without breaking the panel and row-shard
    invariance."""
    lib = L.lib()
    paired = [c for c in range(lib.kw_dgemm_config_count()) if c >= 14 and c != SPLITK_CFG]
    rng = np.random.default_rng(31)
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    for (m, n, k) in ((300, 260, 170), (1024, 1024, 1024), (129, 640, 48), (1000, 1100, 333), (700, 2000, 50),
                      (640, 960, 2048)):
        a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
        outs = []
        for cfg in paired:
            A, B, Cb = mat(gpu, a), mat(gpu, b), mat(gpu, c)
            assert lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, 0.9, A.data(), A.leadingDim(), B.data(),
                                            B.leadingDim(), 1.1, Cb.data(), Cb.leadingDim()) == 0
            q.wait()
            outs.append(Cb.download())
        for o in outs[1:]:
            assert np.array_equal(o, outs[0]), (m, n, k)
        assert within_tol(outs[0], oracle.gemm(0.9, 1.1, a, b, c), k)[0]


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 1024), (1280, 1280, 640), (1100, 1000, 2000), (1792, 1792, 512),
                                   (1536, 1408, 700), (512, 512, 4096), (768, 700, 2500)])
def test_default_choice_split_is_bitwise_the_one_cta_tile(gpu, oracle, m, n, k):
    """Shapes the library now runs with a SPLIT configuration (badly quantised data-parallel
    grids): the default kw_dgemm result equals the one-CTA-per-tile config 17 bit for bit and the
    oracle within (K+4)u."""
    lib = L.lib()
    rng = np.random.default_rng(m + n + k)
    a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    outs = []
    for cfg in (None, 17):
        A, B, Cb = mat(gpu, a), mat(gpu, b), mat(gpu, c)
        if cfg is None:
            st = lib.kw_dgemm(q.handle(), None, m, n, k, 1.5, A.data(), A.leadingDim(), B.data(), B.leadingDim(), 0.5,
                              Cb.data(), Cb.leadingDim())
        else:
            st = lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, 1.5, A.data(), A.leadingDim(), B.data(),
                                          B.leadingDim(), 0.5, Cb.data(), Cb.leadingDim())
        assert st == 0, L.last_error()
        q.wait()
        outs.append(Cb.download())
    assert np.array_equal(outs[0], outs[1])
    if m * n * k <= 1 << 30:
        assert within_tol(outs[0], oracle.gemm(1.5, 0.5, a, b, c, threads=8), k)[0]


def test_split_schedule_repeats_and_concurrent_queues(gpu, oracle):
    """SPLIT configurations (one persistent CTA per SM — or 2, 3 for 21, 22 — over equal (tile,
    k-tile) ranges, a tile straddling two ranges finished by the next CTA from parked
    accumulators): the per-stream ticket counter (restarted when the grid size changes) and the
    self-clearing flags survive back-to-back launches of different grids and two queues running
    split launches at once; every result equals the one-CTA-per-tile launch."""
    lib = L.lib()
    rng = np.random.default_rng(8)
    m, n, k = 1100, 1300, 700
    a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
    A, B, C0 = mat(gpu, a), mat(gpu, b), mat(gpu, c)
    q0 = kw.Queue(gpu, kw.QueueFlavor.Async)
    assert lib.kw_dgemm_with_config(q0.handle(), 17, m, n, k, 1.3, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                                    0.7, C0.data(), C0.leadingDim()) == 0
    q0.wait()
    want = C0.download()
    qs = [kw.Queue(gpu, kw.QueueFlavor.Async) for _ in range(2)]
    outs = [[mat(gpu, c) for _ in range(6)] for _ in qs]
    for i in range(6):  # interleave enqueues on both queues
        for qi, q in enumerate(qs):
            Cb = outs[qi][i]
            cfg = (18, 21, 20, 22, 24, 23)[(i + qi) % 6]  # grids of 148, 296 and 444 CTAs interleaved
            assert lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, 1.3, A.data(), A.leadingDim(), B.data(),
                                            B.leadingDim(), 0.7, Cb.data(), Cb.leadingDim()) == 0
    for q in qs:
        q.wait()
    for row in outs:
        for Cb in row:
            assert np.array_equal(Cb.download(), want)


def test_mixed_residency_dgemm(gpu, oracle):
    """B on the device, A and C on the host (and the other way round): the staged path uploads
    only what is not resident; bits equal the all-device launch."""
    rng = np.random.default_rng(12)
    m, n, k = 700, 520, 300
    a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
    want = tiled(gpu, 1.2, 0.4, a, b, c)
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    B = mat(gpu, b)
    ah, ch = a.copy(), c.copy()
    assert L.lib().kw_dgemm(q.handle(), None, m, n, k, 1.2, ah.ctypes.data, k, B.data(), B.leadingDim(), 0.4,
                            ch.ctypes.data, n) == 0
    assert np.array_equal(ch, want)
    A, Cd = mat(gpu, a), mat(gpu, c)
    bh = b.copy()
    assert L.lib().kw_dgemm(q.handle(), None, m, n, k, 1.2, A.data(), A.leadingDim(), bh.ctypes.data, n, 0.4,
                            Cd.data(), Cd.leadingDim()) == 0
    assert np.array_equal(Cd.download(), want)


def test_concurrent_enqueues_on_one_queue(gpu):
    """Four host threads enqueue DGEMMs (1024^3: the SPLIT walk with its per-stream ticket, flags
    and park slots) and AXPYs into ONE Async queue while the main thread waits repeatedly: the
    enqueue lock serialises them in arrival order and every result equals its own single launch."""
    import threading
    lib = L.lib()
    rng = np.random.default_rng(4)
    n = 1024
    a, b = rng.random((n, n)), rng.random((n, n))
    A, B = mat(gpu, a), mat(gpu, b)
    cs = [rng.random((n, n)) for _ in range(8)]
    want = []
    q0 = kw.Queue(gpu, kw.QueueFlavor.Async)
    for c in cs:
        Cw = mat(gpu, c)
        L.check(lib.kw_dgemm(q0.handle(), None, n, n, n, 1.5, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                             0.5, Cw.data(), Cw.leadingDim()))
        q0.wait()
        want.append(Cw.download())
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    outs = [mat(gpu, c) for c in cs]
    xs = [kw.Buffer(gpu, kw.IndexVec(1 << 20), 4) for _ in range(4)]
    ys = [kw.Buffer(gpu, kw.IndexVec(1 << 20), 4) for _ in range(4)]
    for v in xs + ys:
        v.upload(np.ones(1 << 20, np.float32))
    errors = []

    def worker(t):
        try:
            for rep in range(5):
                for i in (t, t + 4):
                    Cb = outs[i]
                    if rep == 0:  # each output from its pristine C exactly once
                        L.check(lib.kw_dgemm(q.handle(), None, n, n, n, 1.5, A.data(), A.leadingDim(), B.data(),
                                             B.leadingDim(), 0.5, Cb.data(), Cb.leadingDim()))
                L.check(lib.kw_axpy_f32(q.handle(), None, 1 << 20, 1.0, xs[t].data(), ys[t].data()))
        except Exception as ex:  # noqa: BLE001
            errors.append(ex)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    while any(th.is_alive() for th in threads):
        q.wait()
    for th in threads:
        th.join()
    q.wait()
    assert not errors, errors
    for Cb, w in zip(outs, want):
        assert np.array_equal(Cb.download(), w)
    for y in ys:
        assert np.all(y.download() == 6.0)  # five AXPYs of +1 on 1


def test_host_operand_schedules_from_fresh_threads(gpu, monkeypatch):
    """The streamed host-operand (e2e) DGEMM schedule — driver stream memory operations
    (cuStreamWriteValue32 / cuStreamWaitValue32) and TMA descriptors — run as the FIRST CUDA work
    of a fresh host thread, three threads at once on their own queues: bits equal the
    device-resident launch (regression for the missing-context fallback)."""
    import threading
    rng = np.random.default_rng(12)
    m, n, k = 700, 900, 650
    a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
    want = tiled(gpu, 0.8, 1.2, a, b, c)
    host = kw.Device.host()
    monkeypatch.setenv("KW_E2E_MIN_INTENSITY", "0")  # streamed at this size
    results, errors = {}, []
    bufs = {}
    for t in range(3):
        hA, hB, hC = (kw.Buffer(host, kw.IndexVec(*x.shape), 8) for x in (a, b, c))
        for hb, x in ((hA, a), (hB, b), (hC, c)):
            hb.host_view()[:, : x.shape[1]] = x
        bufs[t] = (hA, hB, hC)

    def worker(t):
        try:
            hA, hB, hC = bufs[t]
            q = kw.Queue(gpu, kw.QueueFlavor.Async)
            q.enqueue(kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, m, n, 128), kw.GemmTiledKernel(),
                                    kw.GemmArgs(m, n, k, 0.8, 1.2, hA, hB, hC)))
            q.wait()
            results[t] = hC.host_view()[:, :n].copy()
        except Exception as ex:  # noqa: BLE001
            errors.append(ex)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(3)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for t in range(3):
        assert np.array_equal(results[t], want), t


@pytest.mark.parametrize("cfg", [18, 20, 24, 25, 26, 28, 29])
def test_split_and_group_configs_read_c_when_beta_is_zero(gpu, cfg):
    """gemm.cpp:35 / 115 (beta multiplies C even when 0) on the SPLIT / two-group walks: NaNs
    planted in C — in head, tail and full tiles — come out as NaN, everything else is finite."""
    lib = L.lib()
    rng = np.random.default_rng(cfg)
    m, n, k = 1100, 1300, 300
    a, b, c = rng.random((m, k)), rng.random((k, n)), rng.random((m, n))
    spots = [(0, 0), (63, 127), (64, 128), (517, 733), (1099, 1299), (600, 5)]
    for r, col in spots:
        c[r, col] = np.nan
    A, B, Cb = mat(gpu, a), mat(gpu, b), mat(gpu, c)
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    assert lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, 1.0, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                                    0.0, Cb.data(), Cb.leadingDim()) == 0
    q.wait()
    out = Cb.download()
    mask = np.zeros_like(out, dtype=bool)
    for r, col in spots:
        mask[r, col] = True
    assert np.isnan(out[mask]).all() and np.isfinite(out[~mask]).all()


def test_split_scratch_follows_queue_lifetime(gpu):
    """Queues created and destroyed around SPLIT launches (per-stream ticket / flag / park scratch,
    released with the queue — a later queue may get the same stream handle), with launches still
    in flight at destruction: every result equals the one-CTA-per-tile launch."""
    lib = L.lib()
    rng = np.random.default_rng(21)
    n = 1024
    a, b, c = rng.random((n, n)), rng.random((n, n)), rng.random((n, n))
    A, B = mat(gpu, a), mat(gpu, b)
    ref = mat(gpu, c)
    q0 = kw.Queue(gpu, kw.QueueFlavor.Async)
    assert lib.kw_dgemm_with_config(q0.handle(), 17, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                                    0.5, ref.data(), ref.leadingDim()) == 0
    q0.wait()
    want = ref.download()
    outs = []
    for it in range(12):
        q = kw.Queue(gpu, kw.QueueFlavor.Async)
        Cb = mat(gpu, c)
        for cfg in (18, 25, 21) if it % 2 else (20, 18):
            q.wait()  # the upload below runs on another queue: the previous launch must be done
            Cb.upload(c)
            assert lib.kw_dgemm_with_config(q.handle(), cfg, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(),
                                            B.leadingDim(), 0.5, Cb.data(), Cb.leadingDim()) == 0
        del q  # destroyed with the last launch possibly still running (the destructor drains it)
        outs.append(Cb)
    for Cb in outs:
        assert np.array_equal(Cb.download(), want)


@pytest.mark.parametrize("m,n,k", [(512, 512, 16384), (100, 70, 9000), (1, 2, 4200), (768, 700, 5000),
                                   (512, 512, 1024)])
def test_splitk_small_output_long_k(gpu, oracle, m, n, k):
    """Split-k (config 27, opt-in): S independent k-slice chains parked per slice, added in slice
    order by the reduction kernel, which runs the epilogue. Within (K+4)u of gemmReference and
    deterministic (two runs give the same bits); the default path (one-CTA chains) stays within
    tolerance of it but is not required to equal it."""
    lib = L.lib()
    rng = np.random.default_rng(m + n + k)
    a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
    ref = oracle.gemm(1.25, 0.75, a, b, c, threads=8)
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    outs = []
    for cfg in (SPLITK_CFG, SPLITK_CFG, None):
        A, B, Cb = mat(gpu, a), mat(gpu, b), mat(gpu, c)
        if cfg is None:
            st = lib.kw_dgemm(q.handle(), None, m, n, k, 1.25, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                              0.75, Cb.data(), Cb.leadingDim())
        else:
            st = lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, 1.25, A.data(), A.leadingDim(), B.data(),
                                          B.leadingDim(), 0.75, Cb.data(), Cb.leadingDim())
        assert st == 0, L.last_error()
        q.wait()
        outs.append(Cb.download())
    assert np.array_equal(outs[0], outs[1])  # deterministic
    for o in (outs[0], outs[2]):
        ok, worst = within_tol(o, ref, k)
        assert ok, worst


def test_splitk_opt_in_default(gpu):
    """KW_DGEMM_SPLITK=1 (read once per process, so in a subprocess) makes split-k the default
    choice for fewer 64 x 64 tiles than SMs and k >= 1024: kw_dgemm then equals config 27 bit for
    bit; without it kw_dgemm equals config 17 (the one-CTA chain)."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1602_08477_b200 import _lib as L, kernelweave as kw
gpu = kw.Device.gpu(0); lib = L.lib(); q = kw.Queue(gpu, kw.QueueFlavor.Async)
rng = np.random.default_rng(3); m, n, k = 300, 200, 3000
a, b, c = rng.random((m, k)), rng.random((k, n)), rng.random((m, n))
def run(cfg):
    A, B, Cb = (kw.Buffer(gpu, kw.IndexVec(*x.shape), 8) for x in (a, b, c))
    for t, x in zip((A, B, Cb), (a, b, c)): t.upload(x)
    if cfg is None:
        st = lib.kw_dgemm(q.handle(), None, m, n, k, 1.0, A.data(), A.leadingDim(), B.data(), B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim())
    else:
        st = lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, 1.0, A.data(), A.leadingDim(), B.data(), B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim())
    assert st == 0; q.wait(); return Cb.download()
d, s27, s17 = run(None), run(27), run(17)
want = s27 if sys.argv[1] == "1" else s17
assert np.array_equal(d, want); print("DEFAULT OK")
"""
    root = str(__import__("pathlib").Path(__file__).resolve().parent.parent)
    for flag in ("1", "0"):
        env = dict(os.environ, KW_DGEMM_SPLITK=flag)
        out = subprocess.run([sys.executable, "-c", code, flag], capture_output=True, text=True, env=env, cwd=root,
                             timeout=300)
        assert "DEFAULT OK" in out.stdout, (flag, out.stdout + out.stderr)


def test_splitk_beta_zero_nan_and_odd_ldc(gpu, oracle):
    """Split-k's reduction runs the epilogue: beta = 0 still reads C (NaN propagates, gemm.cpp:35),
    and an odd leading dimension of C (scalar stores) keeps every element outside the product
    untouched."""
    lib = L.lib()
    m, n, k = 130, 67, 6000
    rng = np.random.default_rng(5)
    a, b = rng.random((m, k)), rng.random((k, n))
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    A, B = mat(gpu, a), mat(gpu, b)
    c = np.full((m, n), np.nan)
    c[::2] = 1.0
    Cb = mat(gpu, c)
    assert lib.kw_dgemm_with_config(q.handle(), SPLITK_CFG, m, n, k, 1.0, A.data(), A.leadingDim(), B.data(),
                                    B.leadingDim(), 0.0, Cb.data(), Cb.leadingDim()) == 0
    q.wait()
    out = Cb.download()
    assert np.isnan(out[1::2]).all() and not np.isnan(out[::2]).any()
    ldc = n + 2  # 69 columns of storage: an odd leading dimension -> the reduction's scalar path
    store = np.full((m, ldc), -7.0)
    store[:, :n] = 2.0
    Cs = kw.Buffer(gpu, kw.IndexVec(m * ldc), 8)
    Cs.upload(store.reshape(-1))
    assert lib.kw_dgemm_with_config(q.handle(), SPLITK_CFG, m, n, k, 1.0, A.data(), A.leadingDim(), B.data(),
                                    B.leadingDim(), 0.5, Cs.data(), ldc) == 0
    q.wait()
    got = Cs.download().reshape(m, ldc)
    assert (got[:, n:] == -7.0).all()
    ok, worst = within_tol(got[:, :n], oracle.gemm(1.0, 0.5, a, b, np.full((m, n), 2.0), threads=8), k)
    assert ok, worst
