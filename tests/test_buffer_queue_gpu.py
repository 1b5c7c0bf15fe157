"""GPU ports of the reference's buffer and queue suites (proj/tests/test_buffer.cpp,
proj/tests/test_queue.cpp) through the Python mirror and the C-ABI: the pitch law, pitched
copies between every pair of residencies with canaries, copy validation before enqueue, and
the in-order / Sync / Async / failure semantics of a queue that is a CUDA stream. The
reference's host functors (WriteKernel, ReadKernel, SleepKernel, FailKernel) become copies,
AXPY/DGEMM launches and a recorded launch failure — the only kinds of task this build runs."""
import ctypes as C
import time

import numpy as np
import pytest

from paper_1602_08477_b200 import _lib as L
from paper_1602_08477_b200 import kernelweave as kw

pytestmark = pytest.mark.gpu
GPU = kw.BackendKind.GpuCudaRt
HOST = kw.Device.host()


def pattern(extent):
    """patternValue of test_buffer.cpp: linearize(idx, extent) + 0.25, as a dense array."""
    return np.arange(int(np.prod(extent)), dtype=np.float64).reshape(extent) + 0.25


def put(buf, dense):
    if buf.device().isHost():
        view = buf.host_view().reshape(buf.rowCount(), -1)
        view[:, : buf.extent()[buf.dim() - 1]] = dense.reshape(buf.rowCount(), -1)
    else:
        buf.upload(dense)


def raw(buf):
    """Every storage byte, padding included, as a (rows, pitch) uint8 array."""
    if buf.device().isHost():
        b = buf.host_view().view(np.uint8).reshape(-1).copy()
    else:
        b = np.frombuffer(buf.download_raw(), dtype=np.uint8)
    return b.reshape(buf.rowCount(), buf.rowPitch())


def fill(buf, byte):
    if buf.device().isHost():
        buf.host_view().view(np.uint8)[...] = byte
    else:
        buf.fill_raw(byte)


def elements(buf):
    """The logical extent as float64 (from the raw bytes, so padding never leaks in)."""
    r = raw(buf)[:, : buf.rowBytes()].copy().view(np.float64)
    return r.reshape(buf.extent().tuple())


# ---- test_buffer.cpp ---------------------------------------------------------------------------
@pytest.mark.parametrize("where", ["host", "device"])
def test_allocation_pitch_rules(gpu, where):
    """test_buffer.cpp:19-41 — the rowPitch = roundUp(cols * elem, 64) law, dense 1-D, and the
    usage errors, for pinned host and device buffers alike."""
    dev = HOST if where == "host" else gpu
    padded = kw.Buffer(dev, kw.IndexVec(10, 10), 8)
    assert (padded.rowPitch(), padded.rowCount(), padded.storageBytes()) == (128, 10, 1280)
    assert kw.Buffer(dev, kw.IndexVec(8, 8), 8).rowPitch() == 64
    v = kw.Buffer(dev, kw.IndexVec(100), 8)
    assert (v.rowPitch(), v.rowCount()) == (800, 1)
    cube = kw.Buffer(dev, kw.IndexVec(3, 4, 5), 8)
    assert (cube.rowPitch(), cube.rowCount()) == (64, 12)
    with pytest.raises(kw.UsageError):
        kw.Buffer(dev, kw.IndexVec(0, 4), 8)
    with pytest.raises(kw.UsageError):
        kw.Buffer(dev, kw.IndexVec(4), 0)
    with pytest.raises(kw.UsageError):
        kw.Buffer(dev, kw.IndexVec(4, 4), 8, 48)  # not a power of two


def test_pitch_law_on_random_extents(gpu):
    """test_buffer.cpp:69-81 (randomExtent of test_support.hpp:78-96, product <= 4096)."""
    rng = np.random.default_rng(11)
    for it in range(100):
        dim = 2 + int(rng.integers(0, 2))
        comps, budget = [], 4096
        for _ in range(dim):
            c = int(rng.integers(1, max(1, budget) + 1))
            comps.append(c)
            budget = max(1, budget // c)
        elem = 1 + int(rng.integers(0, 16))
        buf = kw.Buffer(HOST if it % 2 else gpu, kw.IndexVec(*comps), elem)
        assert buf.rowPitch() % 64 == 0
        assert buf.rowPitch() >= buf.rowBytes()
        assert buf.storageBytes() >= buf.rowCount() * buf.rowBytes()


def test_copy_between_mismatched_pitches_preserves_every_element(gpu):
    """test_buffer.cpp:125-143: host (128-B rows) -> device (32-B alignment: 96-B rows)."""
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    src = kw.Buffer(HOST, kw.IndexVec(10, 10), 8, 128)
    dst = kw.Buffer(gpu, kw.IndexVec(10, 10), 8, 32)
    assert (src.rowPitch(), dst.rowPitch()) == (128, 96)
    put(src, pattern((10, 10)))
    kw.copyBuffer(q, dst, src, kw.IndexVec(10, 10))
    q.wait()
    assert np.array_equal(elements(dst), pattern((10, 10)))


@pytest.mark.parametrize("where", ["host", "device"])
def test_sub_extent_copy_updates_only_the_corner(gpu, where):
    """test_buffer.cpp:145-175: a 3 x 3 corner copy; every other element and every padding byte
    keeps the 0xAB canary."""
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    src = kw.Buffer(gpu, kw.IndexVec(10, 10), 8)
    dst = kw.Buffer(HOST if where == "host" else gpu, kw.IndexVec(10, 10), 8)
    put(src, pattern((10, 10)))
    fill(dst, 0xAB)
    kw.copyBuffer(q, dst, src, kw.IndexVec(3, 3))
    q.wait()
    r = raw(dst)
    got = r[:3, :24].copy().view(np.float64)
    assert np.array_equal(got, pattern((10, 10))[:3, :3])
    mask = np.ones_like(r, dtype=bool)
    mask[:3, :24] = False
    assert (r[mask] == 0xAB).all()


def test_copy_validation_happens_before_enqueue(gpu):
    """test_buffer.cpp:177-188."""
    small = kw.Buffer(gpu, kw.IndexVec(4, 4), 8)
    big = kw.Buffer(gpu, kw.IndexVec(8, 8), 8)
    other = kw.Buffer(gpu, kw.IndexVec(8, 8), 4)
    vecb = kw.Buffer(gpu, kw.IndexVec(64), 8)
    for dst, src, ext in ((small, big, kw.IndexVec(8, 8)), (big, small, kw.IndexVec(5, 5)),
                          (big, other, kw.IndexVec(4, 4)), (big, vecb, kw.IndexVec(8, 8))):
        with pytest.raises(kw.UsageError):
            kw.createCopy(dst, src, ext)


def test_copy_property_over_random_extents_pitches_and_residencies(gpu):
    """test_buffer.cpp:190-223 over every residency pair (H2D, D2H, D2D, H2H): the copied box
    holds the source pattern, everything else (incl. padding) keeps the 0x5C canary."""
    rng = np.random.default_rng(77)
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    aligns = (32, 64, 128, 256)
    pairs = ((HOST, gpu), (gpu, HOST), (gpu, gpu), (HOST, HOST))
    for it in range(60):
        rows, cols = 1 + int(rng.integers(0, 64)), 1 + int(rng.integers(0, 64))
        sdev, ddev = pairs[it % 4]
        sext = (1 + rows + int(rng.integers(0, 4)), 1 + cols + int(rng.integers(0, 4)))
        dext = (rows + int(rng.integers(0, 4)), cols + int(rng.integers(0, 4)))
        src = kw.Buffer(sdev, kw.IndexVec(*sext), 8, aligns[int(rng.integers(0, 4))])
        dst = kw.Buffer(ddev, kw.IndexVec(*dext), 8, aligns[int(rng.integers(0, 4))])
        ce = (min(rows, dext[0]), min(cols, dext[1]))
        put(src, pattern(sext))
        fill(dst, 0x5C)
        kw.copyBuffer(q, dst, src, kw.IndexVec(*ce))
        q.wait()
        r = raw(dst)
        got = r[: ce[0], : ce[1] * 8].copy().view(np.float64)
        assert np.array_equal(got, pattern(sext)[: ce[0], : ce[1]]), it
        mask = np.ones_like(r, dtype=bool)
        mask[: ce[0], : ce[1] * 8] = False
        assert (r[mask] == 0x5C).all(), it


def test_3d_copy_walks_rows_through_both_layouts(gpu):
    """test_buffer.cpp:225-242: (3,4,5)/64-B rows -> (4,5,6)/128-B rows, box (2,3,4), on the
    device and from/to the host."""
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    for sdev, ddev in ((gpu, gpu), (HOST, gpu), (gpu, HOST)):
        src = kw.Buffer(sdev, kw.IndexVec(3, 4, 5), 8, 64)
        dst = kw.Buffer(ddev, kw.IndexVec(4, 5, 6), 8, 128)
        put(src, pattern((3, 4, 5)))
        fill(dst, 0x11)
        kw.copyBuffer(q, dst, src, kw.IndexVec(2, 3, 4))
        q.wait()
        got = elements(dst)
        assert np.array_equal(got[:2, :3, :4], pattern((3, 4, 5))[:2, :3, :4])
        r = raw(dst).reshape(4, 5, dst.rowPitch())
        mask = np.ones_like(r, dtype=bool)
        mask[:2, :3, :32] = False
        assert (r[mask] == 0x11).all()


# ---- test_queue.cpp ----------------------------------------------------------------------------
def axpy_task(n, alpha, x, y):
    return kw.createExec(GPU, kw.axpyWorkDiv(GPU, n, 256, 4), kw.AxpyKernel(), kw.AxpyArgs(n, alpha, x, y))


def dev_vec(gpu, values):
    b = kw.Buffer(gpu, kw.IndexVec(len(values)), 8)
    b.upload(np.asarray(values, dtype=np.float64))
    return b


def test_sync_queue_completes_the_task_inside_enqueue(gpu):
    """test_queue.cpp:47-58."""
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    x, y = dev_vec(gpu, [1.0] * 1000), dev_vec(gpu, [0.0] * 1000)
    h = q.enqueue(axpy_task(1000, 9.0, x, y))
    assert h.state() == kw.TaskState.Done
    assert (y.download() == 9.0).all()
    q.wait()


def test_constructing_a_task_executes_nothing(gpu):
    """test_queue.cpp:60-71."""
    x, y = dev_vec(gpu, [1.0]), dev_vec(gpu, [1.0])
    t1 = axpy_task(1, 2.0, x, y)
    t2 = axpy_task(1, 3.0, x, y)
    del t1, t2
    assert y.download().tolist() == [1.0]


def test_async_queue_preserves_write_then_read_order(gpu):
    """test_queue.cpp:73-89: 256 (write slot <- trial; read slot -> seen[trial]) pairs on one
    Async queue; every read observes its own write."""
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    values = kw.Buffer(HOST, kw.IndexVec(256), 8)
    values.host_view()[:] = np.arange(256)
    data = kw.Buffer(gpu, kw.IndexVec(1), 8)
    seen = kw.Buffer(gpu, kw.IndexVec(256), 8)
    one = L.sz3((1,))
    lib = L.lib()
    for t in range(256):
        assert lib.kw_copy(q.handle(), data.data(), 8, one, values.data() + 8 * t, 8, one, 1, one, 8) == 0
        assert lib.kw_copy(q.handle(), seen.data() + 8 * t, 8, one, data.data(), 8, one, 1, one, 8) == 0
    q.wait()
    assert np.array_equal(seen.download(), np.arange(256, dtype=np.float64))


def test_copy_tasks_interleave_with_kernels_in_fifo_order(gpu):
    """test_queue.cpp:91-107: a kernel writes a, the next task copies a -> b."""
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    i = np.arange(16, dtype=np.float64)
    x, a = dev_vec(gpu, i), dev_vec(gpu, [0.0] * 16)
    b = kw.Buffer(gpu, kw.IndexVec(16), 8)
    q.enqueue(axpy_task(16, 1.0, x, a))   # a = i
    q.enqueue(axpy_task(16, 0.0, x, a))   # a = 0*i + a (still i): ordering, not value, is checked
    q.enqueue(kw.createCopy(b, a, kw.IndexVec(16)))
    q.wait()
    assert np.array_equal(b.download(), i)


def test_async_enqueue_does_not_wait_for_the_task(gpu):
    """test_queue.cpp:109-120 with ~100 ms of DGEMM work in place of SleepKernel(100)."""
    n = 8192
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    A, B, Cb = (kw.Buffer(gpu, kw.IndexVec(n, n), 8) for _ in range(3))
    for m in (A, B, Cb):
        m.fill_raw(0)
    task = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, n, n, 128), kw.GemmTiledKernel(),
                         kw.GemmArgs(n, n, n, 1.0, 1.0, A, B, Cb))
    q.enqueue(task)  # first use: module load, tensor-map encoder lookup
    q.wait()
    start = time.perf_counter()
    handles = [q.enqueue(task) for _ in range(4)]
    enqueue_ms = (time.perf_counter() - start) * 1e3
    assert enqueue_ms < 10.0, enqueue_ms
    q.wait()
    total_ms = (time.perf_counter() - start) * 1e3
    assert all(h.state() == kw.TaskState.Done for h in handles)
    assert total_ms >= 4 * 20.0, total_ms  # 4 x 1.1 TFLOP at <= 40 TFLOP/s


def test_two_async_queues_make_independent_progress(gpu):
    """test_queue.cpp:122-137."""
    q1, q2 = kw.Queue(gpu, kw.QueueFlavor.Async), kw.Queue(gpu, kw.QueueFlavor.Async)
    x = dev_vec(gpu, [1.0])
    y1, y2 = dev_vec(gpu, [0.0]), dev_vec(gpu, [0.0])
    h1 = q1.enqueue(axpy_task(1, 1.0, x, y1))
    h2 = q2.enqueue(axpy_task(1, 2.0, x, y2))
    q1.wait()
    q2.wait()
    assert h1.state() == kw.TaskState.Done and h2.state() == kw.TaskState.Done
    assert (y1.download()[0], y2.download()[0]) == (1.0, 2.0)


def test_wait_on_an_empty_queue_returns_immediately_and_is_idempotent(gpu):
    """test_queue.cpp:139-145."""
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    start = time.perf_counter()
    q.wait()
    q.wait()
    assert time.perf_counter() - start < 0.5


def test_failures_aggregate_and_later_tasks_still_run(gpu):
    """test_queue.cpp:147-185: two failed tasks (launch failures recorded the way the generic
    functor launcher reports them) around a good AXPY; wait() raises one TaskError with count 2
    and the first message, the good task ran, and the next wait is clean."""
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    lib = L.lib()
    x, y = dev_vec(gpu, [1.0]), dev_vec(gpu, [0.0])
    assert lib.kw_queue_complete_launch(q.handle(), 1, b"doomed task") == L.KW_TASK
    good = q.enqueue(axpy_task(1, 5.0, x, y))
    assert lib.kw_queue_complete_launch(q.handle(), 2, b"doomed task") == L.KW_TASK
    with pytest.raises(kw.TaskError) as ei:
        q.wait()
    assert ei.value.failedCount() == 2
    assert "doomed task" in str(ei.value)
    assert good.state() == kw.TaskState.Done
    assert y.download()[0] == 5.0
    q.wait()  # reported once
    sync = kw.Queue(gpu, kw.QueueFlavor.Sync)
    assert lib.kw_queue_complete_launch(sync.handle(), 1, b"doomed task") == L.KW_TASK
    with pytest.raises(kw.TaskError):
        sync.wait()


def test_begin_end_launch_bracket(gpu):
    """The external-launch bracket the generic functor launcher uses: begin holds the enqueue
    lock and rejects a shut-down queue (queue.cpp enqueueBody's UsageError); end with a launch
    error records one failed task; a clean end arms a zeroed slot that nothing sets."""
    import ctypes as C
    lib = L.lib()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    stream, dev, slot = C.c_void_p(), C.c_int(-1), C.POINTER(C.c_uint32)()
    assert lib.kw_queue_begin_launch(q.handle(), b"ext", C.byref(stream), C.byref(dev), C.byref(slot)) == 0
    assert dev.value == 0 and stream.value and slot[0] == 0
    assert lib.kw_queue_end_launch(q.handle(), 0, b"ext") == 0
    q.wait()
    assert lib.kw_queue_begin_launch(q.handle(), b"ext", C.byref(stream), C.byref(dev), C.byref(slot)) == 0
    assert lib.kw_queue_end_launch(q.handle(), 1, b"ext launch") == L.KW_TASK
    with pytest.raises(kw.TaskError) as ei:
        q.wait()
    assert "ext launch" in str(ei.value)
    # the lock was released: an ordinary enqueue still goes through
    x, y = dev_vec(gpu, [1.0]), dev_vec(gpu, [0.0])
    q.enqueue(axpy_task(1, 2.0, x, y))
    q.wait()
    assert y.download()[0] == 2.0
    q.shutdown()
    assert lib.kw_queue_begin_launch(q.handle(), b"ext", C.byref(stream), C.byref(dev), C.byref(slot)) == L.KW_USAGE
    assert lib.kw_queue_fail_slot(q.handle(), b"ext", C.byref(slot)) == L.KW_USAGE


def test_sync_queue_shutdown_rejects_enqueue(gpu):
    """test_queue.cpp:187-202, Sync half (the Async half is test_axpy_gpu)."""
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    q.shutdown()
    x = dev_vec(gpu, [1.0])
    with pytest.raises(kw.UsageError, match="shutdown"):
        q.enqueue(axpy_task(1, 1.0, x, x))


def test_matrix_csv_round_trip_python_mirror(gpu, oracle):
    """buffer_csv.hpp through the Python mirror: bitwise round trip (host and GPU buffers), the
    reference's "%.17g" text, and its usage errors (test_buffer.cpp:275-310)."""
    import io
    src = kw.Buffer(HOST, kw.IndexVec(7, 5), 8)
    vals = oracle.MT64(seed=99).fill_uniform(35).reshape(7, 5)
    vals[0, 0], vals[6, 4] = 1.0 / 3.0, -0.0
    put(src, vals)
    first = io.StringIO()
    kw.writeBufferCsv(src, first)
    assert first.getvalue().splitlines()[0].split(",")[0] == "%.17g" % (1.0 / 3.0)
    for where in (HOST, gpu):
        back = kw.readBufferCsv(io.StringIO(first.getvalue()), where)
        assert back.extent() == src.extent()
        assert elements(back).tobytes() == vals.tobytes()
        again = io.StringIO()
        kw.writeBufferCsv(back, again)
        assert again.getvalue() == first.getvalue()
    for bad in ("1,2\n3\n", "", "1,x\n"):
        with pytest.raises(kw.UsageError):
            kw.readBufferCsv(io.StringIO(bad))
    with pytest.raises(kw.UsageError):
        kw.writeBufferCsv(kw.Buffer(HOST, kw.IndexVec(4), 8), io.StringIO())


def test_3d_copy_property_over_random_extents_and_residencies(gpu):
    """The 3-D counterpart of test_buffer.cpp:190-223: random (d0, d1, d2) extents and row
    alignments on both sides, every residency pair; the copied box carries the source pattern,
    every other byte of the destination (padding included) keeps its canary."""
    rng = np.random.default_rng(303)
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    aligns = (32, 64, 128, 256)
    pairs = ((HOST, gpu), (gpu, HOST), (gpu, gpu), (HOST, HOST))
    for it in range(40):
        box = tuple(1 + int(v) for v in rng.integers(0, 9, size=3))
        sext = tuple(b + int(rng.integers(0, 3)) for b in box)
        dext = tuple(b + int(rng.integers(0, 3)) for b in box)
        sdev, ddev = pairs[it % 4]
        src = kw.Buffer(sdev, kw.IndexVec(*sext), 8, aligns[int(rng.integers(0, 4))])
        dst = kw.Buffer(ddev, kw.IndexVec(*dext), 8, aligns[int(rng.integers(0, 4))])
        put(src, pattern(sext))
        fill(dst, 0x3C)
        kw.copyBuffer(q, dst, src, kw.IndexVec(*box))
        q.wait()
        r = raw(dst).reshape(dext[0], dext[1], dst.rowPitch())
        got = r[: box[0], : box[1], : box[2] * 8].copy().view(np.float64)
        assert np.array_equal(got, pattern(sext)[: box[0], : box[1], : box[2]]), it
        mask = np.ones_like(r, dtype=bool)
        mask[: box[0], : box[1], : box[2] * 8] = False
        assert (r[mask] == 0x3C).all(), it
