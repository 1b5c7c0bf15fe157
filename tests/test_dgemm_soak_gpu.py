"""Randomised cross-path soak of kw_dgemm: for random shapes, scalars and leading dimensions,
every execution path — resident, host-pinned (streamed or row-panel schedule, random panel grid),
pageable host arrays, mixed residency, either tile contract — must give the bits of the resident
launch, which itself must sit within (K+4)u of gemmReference (the oracle) — for these signed
inputs relative to |alpha||A||B| + |beta||C|, since cancellation voids a bound on |C_ref|."""
import ctypes as C

import numpy as np
import pytest

from paper_1602_08477_b200 import _lib as L
from paper_1602_08477_b200 import kernelweave as kw

pytestmark = pytest.mark.gpu
GPU = kw.BackendKind.GpuCudaRt
U = 2.0 ** -53


def dev_mat(gpu, a):
    b = kw.Buffer(gpu, kw.IndexVec(*a.shape), 8)
    b.upload(a)
    return b


def host_mat(a):
    b = kw.Buffer(kw.Device.host(), kw.IndexVec(*a.shape), 8)
    b.host_view()[:, : a.shape[1]] = a
    return b


def test_dgemm_paths_agree_bitwise_on_random_cases(gpu, oracle, monkeypatch):
    rng = np.random.default_rng(20261018)
    lib = L.lib()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    for case in range(120):
        m, n, k = (int(v) for v in rng.integers(1, 1400, size=3))
        alpha = float(rng.choice([1.0, -0.5, 0.75, 2.0]))
        beta = float(rng.choice([0.0, 1.0, -1.25, 0.5]))
        a = rng.standard_normal((m, k))
        b = rng.standard_normal((k, n))
        c = rng.standard_normal((m, n))
        tile = int(rng.choice([64, 128]))
        wd = kw.gemmTiledWorkDiv(GPU, m, n, tile).to_c()
        # resident reference launch
        A, B, Cd = dev_mat(gpu, a), dev_mat(gpu, b), dev_mat(gpu, c)
        L.check(lib.kw_dgemm(q.handle(), C.byref(wd), m, n, k, alpha, A.data(), A.leadingDim(), B.data(),
                             B.leadingDim(), beta, Cd.data(), Cd.leadingDim()))
        q.wait()
        want = Cd.download()
        if case % 8 == 0:  # the oracle on a subset (it is the slow part)
            # signed inputs cancel, so the bound scales with the magnitudes summed, not |C_ref|
            ref = oracle.gemm(alpha, beta, a, b, c)
            scale = abs(alpha) * (np.abs(a) @ np.abs(b)) + abs(beta) * np.abs(c)
            assert np.all(np.abs(want - ref) <= (k + 4) * U * scale), case
        path = case % 4
        monkeypatch.setenv("KW_E2E_MIN_INTENSITY", "0" if rng.random() < 0.5 else "400")
        monkeypatch.setenv("KW_E2E_PANELS", str(int(rng.integers(1, 17))))
        if path == 0:  # all host pinned (streamed or row panels)
            Ah, Bh, Ch = host_mat(a), host_mat(b), host_mat(c)
            L.check(lib.kw_dgemm(q.handle(), C.byref(wd), m, n, k, alpha, Ah.data(), Ah.leadingDim(), Bh.data(),
                                 Bh.leadingDim(), beta, Ch.data(), Ch.leadingDim()))
            q.wait()
            got = Ch.host_view()[:, :n].copy()
        elif path == 1:  # pageable numpy arrays
            ap, bp, cp = a.copy(), b.copy(), c.copy()
            L.check(lib.kw_dgemm(q.handle(), C.byref(wd), m, n, k, alpha, ap.ctypes.data, k, bp.ctypes.data, n,
                                 beta, cp.ctypes.data, n))
            q.wait()
            got = cp
        elif path == 2:  # mixed: B resident, A and C pinned host
            Ah, Ch = host_mat(a), host_mat(c)
            L.check(lib.kw_dgemm(q.handle(), C.byref(wd), m, n, k, alpha, Ah.data(), Ah.leadingDim(), B.data(),
                                 B.leadingDim(), beta, Ch.data(), Ch.leadingDim()))
            q.wait()
            got = Ch.host_view()[:, :n].copy()
        else:  # resident again on a fresh C: run-to-run determinism
            C2 = dev_mat(gpu, c)
            L.check(lib.kw_dgemm(q.handle(), C.byref(wd), m, n, k, alpha, A.data(), A.leadingDim(), B.data(),
                                 B.leadingDim(), beta, C2.data(), C2.leadingDim()))
            q.wait()
            got = C2.download()
        assert np.array_equal(got, want), (case, path, m, n, k, tile)


@pytest.mark.parametrize("schedule", ["default", "streamed-ksplit"])
@pytest.mark.parametrize("m,n,k", [(1, 1, 100000), (100000, 1, 16), (16, 100000, 1), (3, 70000, 9),
                                   (65537, 3, 33), (1, 8192, 8192), (8192, 1, 8192)])
def test_extreme_shapes(gpu, oracle, m, n, k, schedule, monkeypatch):
    """Dot products, GEMV-like and outer-product shapes: resident launch within the
    magnitude-scaled (K+4)u bound of gemmReference, and the pinned-host path equal to it — with
    the default schedule choice and with the streamed two-pass k-split forced."""
    if schedule == "streamed-ksplit":
        monkeypatch.setenv("KW_E2E_MIN_INTENSITY", "0")
        monkeypatch.setenv("KW_E2E_KSPLIT", "2")
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    lib = L.lib()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    a, b, c = rng.standard_normal((m, k)), rng.standard_normal((k, n)), rng.standard_normal((m, n))
    A, B, Cd = dev_mat(gpu, a), dev_mat(gpu, b), dev_mat(gpu, c)
    L.check(lib.kw_dgemm(q.handle(), None, m, n, k, 0.75, A.data(), A.leadingDim(), B.data(), B.leadingDim(), -1.5,
                         Cd.data(), Cd.leadingDim()))
    q.wait()
    got = Cd.download()
    ref = oracle.gemm(0.75, -1.5, a, b, c)
    scale = 0.75 * (np.abs(a) @ np.abs(b)) + 1.5 * np.abs(c)
    assert np.all(np.abs(got - ref) <= (k + 4) * U * scale)
    Ah, Bh, Ch = host_mat(a), host_mat(b), host_mat(c)
    L.check(lib.kw_dgemm(q.handle(), None, m, n, k, 0.75, Ah.data(), Ah.leadingDim(), Bh.data(), Bh.leadingDim(),
                         -1.5, Ch.data(), Ch.leadingDim()))
    q.wait()
    assert np.array_equal(Ch.host_view()[:, :n], got)


def test_split_configs_agree_bitwise_on_random_cases(gpu):
    """SPLIT tile walks (configs 18, 20, 24, 25: equal (tile, k-tile) ranges per SM or per consumer
    group, straddling tiles finished from parked accumulators) and the two-group data-parallel
    config 26 on random shapes large enough to split, random scalars and padded leading
    dimensions: bits equal the one-CTA-per-tile launch (config 17)."""
    rng = np.random.default_rng(77001)
    lib = L.lib()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    for case in range(36):
        m, n = (int(v) for v in rng.integers(700, 2200, size=2))
        k = int(rng.integers(17, 1500))
        alpha = float(rng.choice([1.0, -0.5, 0.75]))
        beta = float(rng.choice([0.0, 1.0, -1.25]))
        a, b, c = rng.standard_normal((m, k)), rng.standard_normal((k, n)), rng.standard_normal((m, n))
        outs = []
        # 24: 128 x 128 split, 25/26: two groups, 28/29: 32 x 32 / 32 x 64 tiles
        for cfg in (17, 18 + 2 * (case % 2), 24 + (case % 3), 28 + (case % 2)):
            A, B, Cd = dev_mat(gpu, a), dev_mat(gpu, b), dev_mat(gpu, c)
            L.check(lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, alpha, A.data(), A.leadingDim(), B.data(),
                                             B.leadingDim(), beta, Cd.data(), Cd.leadingDim()))
            q.wait()
            outs.append(Cd.download())
        assert all(np.array_equal(outs[0], o) for o in outs[1:]), (case, m, n, k)


def test_rowsharded_kslab_random_cases(gpu):
    """The k-slab row-sharded schedule (world-1 NCCL communicator, broadcasts executing) on random
    shapes, slab splits (panels), B pitches (root broadcasting in place or packing) and scalars:
    bits equal kw_dgemm of the same block."""
    rng = np.random.default_rng(55501)
    lib = L.lib()
    uid = (C.c_char * 128)()
    assert lib.kw_comm_unique_id(uid) == 0
    comm = C.c_void_p()
    assert lib.kw_comm_init(C.byref(comm), 0, 1, 0, uid) == 0, L.last_error()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    try:
        for case in range(24):
            m, n = (int(v) for v in rng.integers(1, 1500, size=2))
            k = int(rng.integers(1, 1200))
            panels = int(rng.choice([1, 2, 3, 8, 16]))
            align = int(rng.choice([64, 128, 256]))
            alpha, beta = float(rng.choice([1.0, -0.5])), float(rng.choice([0.0, 1.25]))
            a, b, c = rng.standard_normal((m, k)), rng.standard_normal((k, n)), rng.standard_normal((m, n))
            A = kw.Buffer(gpu, kw.IndexVec(m, k), 8, int(rng.choice([8, 64])))  # 8: odd pitches -> one pass
            A.upload(a)
            Cw, Cr = dev_mat(gpu, c), dev_mat(gpu, c)
            B = kw.Buffer(gpu, kw.IndexVec(k, n), 8, align)
            B.upload(b)
            L.check(lib.kw_dgemm(q.handle(), None, m, n, k, alpha, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                                 beta, Cw.data(), Cw.leadingDim()))
            elems = C.c_size_t()
            L.check(lib.kw_dgemm_rowsharded_scratch(n, k, panels, C.byref(elems)))
            sc = kw.Buffer(gpu, kw.IndexVec(max(1, elems.value)), 8)
            L.check(lib.kw_dgemm_rowsharded(comm, q.handle(), m, n, k, alpha, A.data(), A.leadingDim(), B.data(),
                                            B.leadingDim(), beta, Cr.data(), Cr.leadingDim(), sc.data(), panels, 0))
            q.wait()
            assert np.array_equal(Cw.download(), Cr.download()), (case, m, n, k, panels, align)
    finally:
        lib.kw_comm_destroy(comm)
