"""GPU edge cases: empty and degenerate extents, and index ranges beyond 2^31 elements (64-bit
addressing in the AXPY grid and the DGEMM TMA coordinates / epilogue)."""
import numpy as np
import pytest

from paper_1602_08477_b200 import _lib as L
from paper_1602_08477_b200 import kernelweave as kw

pytestmark = pytest.mark.gpu
GPU = kw.BackendKind.GpuCudaRt
U = 2.0 ** -53


def test_axpy_n0_and_n1(gpu, oracle):
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    x = kw.Buffer(gpu, kw.IndexVec(4), 4)
    y = kw.Buffer(gpu, kw.IndexVec(4), 4)
    x.upload(np.float32([1, 2, 3, 4]))
    y.upload(np.float32([5, 6, 7, 8]))
    assert L.lib().kw_axpy_f32(q.handle(), None, 0, 2.0, x.data(), y.data()) == 0  # n = 0: nothing
    assert y.download().tolist() == [5, 6, 7, 8]
    assert L.lib().kw_axpy_f32(q.handle(), None, 1, 2.0, x.data(), y.data()) == 0
    assert y.download().tolist() == [7, 6, 7, 8]


def test_gemm_degenerate_extents(gpu, oracle):
    """k = 0: C = fl(alpha*0) + fl(beta*C) (reference.cpp:21-24 with an empty dot product);
    m = 0 or n = 0: nothing happens."""
    rng = np.random.default_rng(1)
    c = rng.random((5, 7)) * 10
    for f in ("kw_dgemm", "kw_dgemm_naive", "kw_dgemm_bitwise"):
        q = kw.Queue(gpu, kw.QueueFlavor.Sync)
        Cb = kw.Buffer(gpu, kw.IndexVec(5, 7), 8)
        Cb.upload(c)
        A = kw.Buffer(gpu, kw.IndexVec(5, 1), 8)
        B = kw.Buffer(gpu, kw.IndexVec(1, 7), 8)
        fn = getattr(L.lib(), f)
        assert fn(q.handle(), None, 5, 7, 0, 1.5, A.data(), 1, B.data(), 7, 0.5, Cb.data(), Cb.leadingDim()) == 0, f
        assert np.array_equal(Cb.download(), oracle.gemm(1.5, 0.5, np.zeros((5, 0)), np.zeros((0, 7)), c)), f
        assert fn(q.handle(), None, 0, 7, 3, 1.5, A.data(), 3, B.data(), 7, 0.5, Cb.data(), Cb.leadingDim()) == 0
        assert fn(q.handle(), None, 5, 0, 3, 1.5, A.data(), 3, B.data(), 7, 0.5, Cb.data(), Cb.leadingDim()) == 0
        assert np.array_equal(Cb.download(), oracle.gemm(1.5, 0.5, np.zeros((5, 0)), np.zeros((0, 7)), c))


def test_usage_errors_on_bad_leading_dimensions(gpu):
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    A = kw.Buffer(gpu, kw.IndexVec(8, 8), 8)
    assert L.lib().kw_dgemm(q.handle(), None, 8, 8, 8, 1.0, A.data(), 4, A.data(), 8, 0.0, A.data(), 8) == L.KW_USAGE
    assert "lda" in L.last_error()
    assert L.lib().kw_dgemm(q.handle(), None, 8, 8, 8, 1.0, A.data(), 8, A.data(), 8, 0.0, A.data(), 4) == L.KW_USAGE
    q.wait()  # nothing was enqueued, nothing failed


def test_axpy_beyond_2p31_elements(gpu, oracle):
    """n = 2^31 + 13 fp32 elements (8.6 GB per vector): 64-bit element indexing in the vector
    kernel and its ragged end."""
    n = (1 << 31) + 13
    rng = np.random.default_rng(99)
    xs = rng.random(n, dtype=np.float32) * 10
    ys = rng.random(n, dtype=np.float32) * 10
    alpha = np.float32(3.0625)
    x = kw.Buffer(gpu, kw.IndexVec(n), 4)
    y = kw.Buffer(gpu, kw.IndexVec(n), 4)
    x.upload(xs)
    y.upload(ys)
    kw.executeTask(GPU, kw.axpyWorkDiv(GPU, n, 512, 4), kw.AxpyKernel(), kw.AxpyArgs(n, float(alpha), x, y))
    got = y.download()
    want = ys.copy()
    assert oracle.lib().kw_oracle_axpy_threaded(n, float(alpha), xs.ctypes.data, want.ctypes.data, 1, 16) == 0
    assert np.array_equal(got, want)


def test_dgemm_output_beyond_2p31_elements(gpu, oracle):
    """C of 524288 x 4160 doubles (2.2e9 elements, 17 GB): row offsets exceed 2^31 elements in
    the TMA/epilogue addressing; K = 24 keeps the compute small. Sampled rows vs the oracle."""
    m, n, k = 1 << 19, 4160, 24
    rng = np.random.default_rng(7)
    a = rng.random((m, k)) * 10
    b = rng.random((k, n)) * 10
    A = kw.Buffer(gpu, kw.IndexVec(m, k), 8)
    B = kw.Buffer(gpu, kw.IndexVec(k, n), 8)
    Cb = kw.Buffer(gpu, kw.IndexVec(m, n), 8)
    A.upload(a)
    B.upload(b)
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    assert L.lib().kw_memset(q.handle(), Cb.data(), 0, Cb.storageBytes()) == 0
    kw.executeTask(GPU, kw.gemmTiledWorkDiv(GPU, m, n, 128), kw.GemmTiledKernel(),
                   kw.GemmArgs(m, n, k, 2.0, 0.5, A, B, Cb))
    rows = np.array([0, 1, 4095, 262143, 262144, 400000, m - 129, m - 1])
    host = np.empty((len(rows), n))
    for i, r in enumerate(rows):
        ext = (1, n)
        st = L.lib().kw_copy(q.handle(), host[i:i + 1].ctypes.data, n * 8, L.sz3(ext),
                             Cb.data() + int(r) * Cb.rowPitch(), Cb.rowPitch(), L.sz3(ext), 2, L.sz3(ext), 8)
        assert st == 0
    q.wait()
    want = oracle.gemm(2.0, 0.5, a[rows], b, np.zeros((len(rows), n)))
    assert np.all(np.abs(host - want) <= (k + 4) * U * np.abs(want))
