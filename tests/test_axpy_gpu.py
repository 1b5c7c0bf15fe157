"""GPU parity: K1 AXPY through the C-ABI (via the Python mirror of the reference API) against
the oracle and the reference's golden digests. The bar is bit-exact (no FMA contraction).
Mirrors test_kernels.cpp:73-112, 331-349 and acceptance criterion 1 (acceptance.cpp:87-115)."""
import ctypes as C

import numpy as np
import pytest

from paper_1602_08477_b200 import _lib as L
from paper_1602_08477_b200 import kernelweave as kw

pytestmark = pytest.mark.gpu
GPU = kw.BackendKind.GpuCudaRt


def h(v):
    return f"{v:016x}"


def vec(dev, values, dtype=np.float64):
    a = np.asarray(values, dtype=dtype)
    b = kw.Buffer(dev, kw.IndexVec(a.size), a.itemsize)
    b.upload(a)
    return b


def run_axpy(n, alpha, xb, yb, tpb=256, ept=16, wd=None):
    wd = wd or kw.axpyWorkDiv(GPU, n, tpb, ept)
    kw.executeTask(GPU, wd, kw.AxpyKernel(), kw.AxpyArgs(n, alpha, xb, yb))


def test_axpy_on_tiny_vectors(gpu):
    x = vec(gpu, [1, 2, 3])
    y = vec(gpu, [10, 20, 30])
    run_axpy(3, 2.0, x, y, 2, 1)
    assert y.download().tolist() == [12, 24, 36]
    y2 = vec(gpu, [10, 20, 30])
    run_axpy(3, 0.0, x, y2, 2, 1)
    assert y2.download().tolist() == [10, 20, 30]


def test_axpy_guards_the_tail(gpu, oracle, golden):
    t = golden["axpy_tail_canary"]
    rng = oracle.MT64(seed=t["seed"])
    xs = rng.fill_uniform(t["covered"])
    ys = rng.fill_uniform(t["covered"])
    ys[t["n"]:] = -555.25
    x, y = vec(gpu, xs), vec(gpu, ys)
    wd = kw.WorkDiv(kw.IndexVec(2), kw.IndexVec(16), kw.IndexVec(4))
    assert kw.totalExtent(wd, kw.Level.Grid, kw.Unit.Elems) == kw.IndexVec(t["covered"])
    kw.executeTask(GPU, wd, kw.AxpyKernel(), kw.AxpyArgs(t["n"], t["alpha"], x, y))
    assert y.download().tolist() == t["y_out"]


def test_native_axpy_4099_identical_bits(gpu, oracle, golden):
    c = golden["axpy_native_4099"]
    rng = oracle.MT64(seed=c["seed"])
    xs = rng.fill_uniform(c["n"])
    ys = rng.fill_uniform(c["n"])
    for tpb, ept in ((16, 8), (256, 16), (1, 1), (1024, 2), (33, 7)):
        x, y = vec(gpu, xs), vec(gpu, ys)
        run_axpy(c["n"], c["alpha"], x, y, tpb, ept)
        assert h(oracle.fnv1a64(y.download())) == c["y_out_digest"], (tpb, ept)


@pytest.mark.parametrize("case", range(4))
def test_axpy_golden_workloads(gpu, oracle, golden, case):
    """SURVEY.md §8c digests: fp32 2^20 192cf34f12caa910 etc., bit for bit."""
    c = golden["workloads"][case]
    f32 = c["dtype"] == "f32"
    alpha, xs, ys = oracle.workload_axpy(c["n"], c["seed"], f32)
    x, y = vec(gpu, xs, xs.dtype), vec(gpu, ys, ys.dtype)
    run_axpy(c["n"], float(alpha), x, y)
    out = y.download()
    assert h(oracle.fnv1a64(out)) == c["y_out_digest"]
    assert float(out[0]) == c["first"] and float(out[-1]) == c["last"]


def test_criterion01_random_instances_bitwise(gpu, oracle):
    """acceptance.cpp:87-115: 100 seeded AXPY instances (n <= 2^16), both dtypes, bitwise."""
    rng = oracle.MT64(seed=101)
    fails = 0
    for it in range(100):
        n = 1 + rng() % (1 << 16)
        f32 = it % 2 == 0
        dt = np.float32 if f32 else np.float64
        xs = rng.fill_uniform(n, dt)
        ys = rng.fill_uniform(n, dt)
        alpha = 0.25 + float(rng() % 16)
        want = oracle.axpy(dt(alpha), xs, ys)
        x, y = vec(gpu, xs, dt), vec(gpu, ys, dt)
        run_axpy(n, alpha, x, y, 16, 8)
        fails += not np.array_equal(y.download(), want)
    assert fails == 0


@pytest.mark.parametrize("tpb", [32, 128, 256, 512, 1024])
@pytest.mark.parametrize("ept", [1, 2, 4, 8, 16, 3])
def test_workdiv_sweep_is_bit_exact(gpu, oracle, tpb, ept):
    """Every division of the sweep config gives the same bits (elementwise update)."""
    n = 300007
    alpha, xs, ys = oracle.workload_axpy(n, 9, True)
    want = oracle.axpy(alpha, xs, ys)
    x, y = vec(gpu, xs, np.float32), vec(gpu, ys, np.float32)
    run_axpy(n, float(alpha), x, y, tpb, ept)
    assert np.array_equal(y.download(), want)


def test_partial_coverage_touches_only_covered_elements(gpu, oracle):
    """A division covering fewer than n elements updates exactly the covered prefix
    (axpy.cpp:12-17: threads beyond their range do nothing, nothing else runs)."""
    n = 1000
    alpha, xs, ys = oracle.workload_axpy(n, 3, False)
    x, y = vec(gpu, xs), vec(gpu, ys)
    wd = kw.WorkDiv(kw.IndexVec(3), kw.IndexVec(64), kw.IndexVec(4))  # covers 768
    kw.executeTask(GPU, wd, kw.AxpyKernel(), kw.AxpyArgs(n, alpha, x, y))
    out = y.download()
    assert np.array_equal(out[:768], oracle.axpy(alpha, xs[:768], ys[:768]))
    assert np.array_equal(out[768:], ys[768:])


def test_misaligned_pointers_take_the_scalar_path(gpu, oracle):
    """Offset device pointers (not 16-B aligned) go through the scalar kernel, same bits."""
    n = 4097
    alpha, xs, ys = oracle.workload_axpy(n + 1, 5, True)
    xb, yb = vec(gpu, xs, np.float32), vec(gpu, ys, np.float32)
    q = kw._default_queue(gpu)
    w = L.kw_workdiv()
    assert L.lib().kw_axpy_default_workdiv(n, 4, C.byref(w)) == 0
    st = L.lib().kw_axpy_f32(q.handle(), C.byref(w), n, float(alpha), xb.data() + 4, yb.data() + 4)
    assert st == 0
    q.wait()
    out = yb.download()
    assert np.array_equal(out[1:], oracle.axpy(alpha, xs[1:], ys[1:]))
    assert out[0] == ys[0]


@pytest.mark.parametrize("pinned", [True, False])
def test_host_buffers_stream_through_the_gpu(gpu, oracle, pinned):
    """executeTask on Device.host() buffers (the e2e path): chunked H2D / kernel / D2H
    overlapped on two streams; bits equal the oracle. Pageable numpy memory also works."""
    n = (1 << 24) + 12345
    alpha, xs, ys = oracle.workload_axpy(n, 11, True)
    want = oracle.axpy(alpha, xs, ys)
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    if pinned:
        x = kw.Buffer(kw.Device.host(), kw.IndexVec(n), 4)
        y = kw.Buffer(kw.Device.host(), kw.IndexVec(n), 4)
        x.host_view()[:] = xs
        y.host_view()[:] = ys
        q.enqueue(kw.createExec(GPU, kw.axpyWorkDiv(GPU, n, 256, 16), kw.AxpyKernel(), kw.AxpyArgs(n, alpha, x, y)))
        q.wait()
        got = y.host_view().copy()
    else:
        xp, yp = xs.copy(), ys.copy()
        assert L.lib().kw_axpy_f32(q.handle(), None, n, float(alpha), xp.ctypes.data, yp.ctypes.data) == 0
        q.wait()
        got = yp
    assert np.array_equal(got, want)


def test_full_size_2p28_digest(gpu, oracle):
    """BASELINE config: fp32 n = 2^28 in HBM; the whole 1 GiB output hashes like the oracle's."""
    n = 1 << 28
    alpha, xs, ys = oracle.workload_axpy(n, 42, True)
    want = oracle.axpy(alpha, xs, ys)
    x, y = vec(gpu, xs, np.float32), vec(gpu, ys, np.float32)
    del xs
    run_axpy(n, float(alpha), x, y)
    got = y.download()
    assert oracle.fnv1a64(got) == oracle.fnv1a64(want)


def test_queue_failure_surfaces_as_task_error(gpu):
    """A launch that fails (threadsPerBlock > 1024 is rejected as usage before enqueue; an
    out-of-range grid via the raw C-ABI is a usage error too) — and wait() stays clean."""
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    x = vec(gpu, [1.0] * 8)
    with pytest.raises(kw.UsageError, match="1024"):
        q.enqueue(kw.createExec(GPU, kw.WorkDiv(kw.IndexVec(1), kw.IndexVec(2048), kw.IndexVec(1)), kw.AxpyKernel(),
                                kw.AxpyArgs(8, 1.0, x, x)))
    q.wait()


def test_copy_respects_pitches_and_extents(gpu):
    """buffer.cpp:99-146: 2-D/3-D pitched copies between buffers of different extents touch
    only the copied box (acceptance criterion 7 shape)."""
    src = kw.Buffer(gpu, kw.IndexVec(5, 7), 8)
    data = np.arange(35, dtype=np.float64).reshape(5, 7)
    src.upload(data)
    dst = kw.Buffer(gpu, kw.IndexVec(6, 9), 8)
    dst.fill_raw(0xEE)
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    kw.copyBuffer(q, dst, src, kw.IndexVec(4, 5))
    q.wait()
    raw = np.frombuffer(dst.download_raw(), dtype=np.uint8).reshape(6, dst.rowPitch())
    got = raw[:4, :40].copy().view(np.float64)
    assert np.array_equal(got, data[:4, :5])
    assert (raw[:4, 40:] == 0xEE).all() and (raw[4:] == 0xEE).all()
    s3 = kw.Buffer(gpu, kw.IndexVec(3, 4, 5), 4)
    d3 = kw.Buffer(gpu, kw.IndexVec(4, 6, 7), 4)
    v = np.arange(60, dtype=np.float32).reshape(3, 4, 5)
    s3.upload(v)
    d3.fill_raw(0)
    kw.copyBuffer(q, d3, s3, kw.IndexVec(2, 3, 4))
    q.wait()
    assert np.array_equal(d3.download()[:2, :3, :4], v[:2, :3, :4])
    with pytest.raises(kw.UsageError, match="extent"):
        kw.createCopy(src, dst, kw.IndexVec(6, 9))


def test_aliased_x_and_y(gpu, oracle):
    """AxpyArgs with x == y (y = alpha*y + y) is legal in the reference: each element is read
    before it is written by the same thread."""
    n = 100003
    _, xs, _ = oracle.workload_axpy(n, 13, True)
    y = vec(gpu, xs, np.float32)
    run_axpy(n, 1.75, y, y)
    assert np.array_equal(y.download(), oracle.axpy(np.float32(1.75), xs, xs))


def test_queue_shutdown_rejects_enqueue(gpu):
    """Queue::shutdown (queue.hpp:111-112): outstanding work completes, further enqueues are
    usage errors."""
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    x = vec(gpu, [1.0, 2.0])
    q.enqueue(kw.createExec(GPU, kw.axpyWorkDiv(GPU, 2, 32, 1), kw.AxpyKernel(), kw.AxpyArgs(2, 1.0, x, x)))
    q.shutdown()
    assert x.download().tolist() == [2.0, 4.0]
    with pytest.raises(kw.UsageError, match="shutdown"):
        q.enqueue(kw.createExec(GPU, kw.axpyWorkDiv(GPU, 2, 32, 1), kw.AxpyKernel(), kw.AxpyArgs(2, 1.0, x, x)))


def test_concurrent_enqueues_on_one_queue(gpu, oracle):
    """Queue::enqueue is thread-safe (queue.hpp:89-93): four host threads push host-staged AXPYs
    (which share the queue's staging scratch) onto one queue; every result is exact."""
    import threading
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    n = (1 << 22) + 7
    jobs = []
    for t in range(4):
        alpha, xs, ys = oracle.workload_axpy(n, 100 + t, True)
        jobs.append((alpha, xs, ys.copy(), oracle.axpy(alpha, xs, ys)))
    errs = []

    def worker(job):
        alpha, xs, ys, _ = job
        for _ in range(3):
            st = L.lib().kw_axpy_f32(q.handle(), None, n, float(alpha), xs.ctypes.data, ys.ctypes.data)
            if st != 0:
                errs.append(L.last_error())
        # three applications: compare against three oracle applications below

    threads = [threading.Thread(target=worker, args=(j,)) for j in jobs]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    q.wait()
    assert not errs
    for alpha, xs, ys, once in jobs:
        want = oracle.axpy(alpha, xs, oracle.axpy(alpha, xs, once))
        assert np.array_equal(ys, want)


def test_mixed_host_and_device_operands(gpu, oracle):
    n = (1 << 21) + 3
    alpha, xs, ys = oracle.workload_axpy(n, 21, True)
    want = oracle.axpy(alpha, xs, ys)
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    xd = vec(gpu, xs, np.float32)
    yh = ys.copy()
    assert L.lib().kw_axpy_f32(q.handle(), None, n, float(alpha), xd.data(), yh.ctypes.data) == 0
    assert np.array_equal(yh, want)
    yd = vec(gpu, ys, np.float32)
    assert L.lib().kw_axpy_f32(q.handle(), None, n, float(alpha), xs.ctypes.data, yd.data()) == 0
    assert np.array_equal(yd.download(), want)


def test_zero_copy_host_path_matches_oracle(gpu, oracle):
    """KW_AXPY_ZEROCOPY=1 (read once per process, so in a subprocess): the kernel loads X, Y from
    and stores Y to the mapped pinned host pages directly. Same bits as the oracle for fp32 and
    fp64, ragged n, pinned x with pinned y and with a device y; pageable operands still take the
    staged path."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1602_08477_b200 import _lib as L, kernelweave as kw
gpu = kw.Device.gpu(0); GPU = kw.BackendKind.GpuCudaRt; host = kw.Device.host()
q = kw.Queue(gpu, kw.QueueFlavor.Async)
for dt, esz, n in ((np.float32, 4, (1 << 22) + 5), (np.float64, 8, (1 << 21) + 3)):
    alpha, xs, ys = O.workload_axpy(n, 77, dt == np.float32)
    want = O.axpy(alpha, xs, ys)
    x = kw.Buffer(host, kw.IndexVec(n), esz); y = kw.Buffer(host, kw.IndexVec(n), esz)
    x.host_view()[:n] = xs; y.host_view()[:n] = ys
    q.enqueue(kw.createExec(GPU, kw.axpyWorkDiv(GPU, n, 256, 4), kw.AxpyKernel(), kw.AxpyArgs(n, alpha, x, y)))
    q.wait()
    assert np.array_equal(y.host_view()[:n], want), dt
    yd = kw.Buffer(gpu, kw.IndexVec(n), esz); yd.upload(ys)
    q.enqueue(kw.createExec(GPU, kw.axpyWorkDiv(GPU, n, 256, 4), kw.AxpyKernel(), kw.AxpyArgs(n, alpha, x, yd)))
    q.wait()
    assert np.array_equal(yd.download(), want), dt
    xp, yp = np.ascontiguousarray(xs), ys.copy()
    fn = L.lib().kw_axpy_f32 if esz == 4 else L.lib().kw_axpy_f64
    assert fn(q.handle(), None, n, float(alpha), xp.ctypes.data, yp.ctypes.data) == 0
    q.wait()
    assert np.array_equal(yp, want), dt
print("ZEROCOPY OK")
"""
    env = dict(os.environ, KW_AXPY_ZEROCOPY="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=str(__import__("pathlib").Path(__file__).resolve().parent.parent), timeout=300)
    assert "ZEROCOPY OK" in out.stdout, out.stdout + out.stderr
