"""The remaining C-ABI entry points on a GPU (tests/test_abi.py checks that every declared symbol
is exported; this checks each one does what include/kw_b200.h says): version and device queries,
pointer classification, queue flavor, the DGEMM configuration table, the L2 flush and the NCCL
broadcast (world size 1)."""
import ctypes as C

import numpy as np
import pytest

from paper_1602_08477_b200 import _lib as L
from paper_1602_08477_b200 import kernelweave as kw

pytestmark = pytest.mark.gpu


def test_version_and_device_queries(gpu):
    lib = L.lib()
    assert lib.kw_version().decode().strip()
    n = C.c_int()
    L.check(lib.kw_device_count(C.byref(n)))
    assert n.value >= 1
    props = L.kw_device_props()
    L.check(lib.kw_device_props_get(0, C.byref(props)))
    assert (props.cc_major, props.cc_minor) == (10, 0)  # sm_100a: this build's only target
    assert props.sm_count == 148 and b"B200" in props.name
    L.check(lib.kw_device_synchronize(0))
    assert lib.kw_device_props_get(n.value + 3, C.byref(props)) == L.KW_USAGE
    assert lib.kw_device_synchronize(n.value + 3) == L.KW_USAGE
    # a failed query leaves nothing behind for the next task to trip over
    q = kw.Queue(gpu, kw.QueueFlavor.Sync)
    L.check(lib.kw_l2_flush(q.handle()))


def test_pointer_kinds_and_queue_flavor(gpu):
    lib = L.lib()
    dev = kw.Buffer(gpu, kw.IndexVec(16), 8)
    pinned = kw.Buffer(kw.Device.host(), kw.IndexVec(16), 8)
    pageable = np.zeros(16)
    for ptr, want in ((dev.data(), L.KW_MEM_DEVICE), (pinned.data(), L.KW_MEM_PINNED),
                      (pageable.ctypes.data, L.KW_MEM_PAGEABLE)):
        kind, d = C.c_int(), C.c_int()
        L.check(lib.kw_pointer_kind(ptr, C.byref(kind), C.byref(d)))
        assert kind.value == want
    for flavor in (kw.QueueFlavor.Sync, kw.QueueFlavor.Async):
        q = kw.Queue(gpu, flavor)
        f = C.c_int()
        L.check(lib.kw_queue_flavor(q.handle(), C.byref(f)))
        assert f.value == flavor.value


def test_dgemm_configuration_table(gpu):
    lib = L.lib()
    count = lib.kw_dgemm_config_count()
    assert count >= 2
    for cfg in range(count):
        info = (C.c_int * 5)()
        L.check(lib.kw_dgemm_config_info(cfg, info))
        bm, bn, bk, threads, stages = list(info)
        assert bm in (32, 64, 128) and bn in (32, 64, 128) and bk in (16, 32) and threads % 32 == 0 and stages >= 2
    info = (C.c_int * 5)()
    assert lib.kw_dgemm_config_info(count, info) == L.KW_USAGE


def test_l2_flush_and_world1_broadcast(gpu):
    lib = L.lib()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    L.check(lib.kw_l2_flush(q.handle()))
    q.wait()
    uid = (C.c_char * 128)()
    L.check(lib.kw_comm_unique_id(uid))
    comm = C.c_void_p()
    L.check(lib.kw_comm_init(C.byref(comm), 0, 1, 0, uid))
    try:
        buf = kw.Buffer(gpu, kw.IndexVec(1000), 8)
        vals = np.arange(1000, dtype=np.float64)
        buf.upload(vals)
        L.check(lib.kw_comm_broadcast(comm, q.handle(), buf.data(), 8000, 0))
        q.wait()
        assert np.array_equal(buf.download(), vals)  # the root's own data is unchanged
        assert lib.kw_comm_broadcast(comm, q.handle(), buf.data(), 8000, 1) == L.KW_USAGE  # no rank 1
        # row-sharded DGEMM usage errors come back before anything is enqueued: host operands,
        # missing root B, root out of range, zero panels
        m = n = k = 64
        dA, dB, dC = (kw.Buffer(gpu, kw.IndexVec(m, m), 8) for _ in range(3))
        hB = kw.Buffer(kw.Device.host(), kw.IndexVec(m, m), 8)
        sc = kw.Buffer(gpu, kw.IndexVec(m * m), 8)
        args = lambda A, B, Cm, scr, panels=2, root=0: lib.kw_dgemm_rowsharded(  # noqa: E731
            comm, q.handle(), m, n, k, 1.0, A.data(), A.leadingDim(), B.data() if B else None,
            B.leadingDim() if B else 0, 0.0, Cm.data(), Cm.leadingDim(), scr.data(), panels, root)
        assert args(dA, hB, dC, sc) == L.KW_USAGE
        assert "device memory" in L.last_error()
        assert args(dA, None, dC, sc) == L.KW_USAGE
        assert args(dA, dB, dC, sc, root=1) == L.KW_USAGE
        assert args(dA, dB, dC, sc, panels=0) == L.KW_USAGE
        q.wait()  # nothing was enqueued, nothing failed
        assert args(dA, dB, dC, sc) == 0
        q.wait()
    finally:
        L.check(lib.kw_comm_destroy(comm))


def test_failed_calls_leave_no_residue(gpu):
    """Usage errors and failed CUDA calls are reported by the call that made them and never
    resurface in a later, valid task (queue.hpp:86-93: one failure, reported once)."""
    lib = L.lib()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    x = kw.Buffer(gpu, kw.IndexVec(1024), 8)
    y = kw.Buffer(gpu, kw.IndexVec(1024), 8)
    x.upload(np.ones(1024))
    y.upload(np.zeros(1024))
    ptr, pitch = C.c_void_p(), C.c_size_t()
    bad = [
        lambda: lib.kw_buffer_alloc(4096, 1, L.sz3((8,)), 8, 64, C.byref(ptr), C.byref(pitch)),
        lambda: lib.kw_buffer_alloc(0, 1, L.sz3((1 << 62,)), 8, 64, C.byref(ptr), C.byref(pitch)),  # too big
        lambda: lib.kw_axpy_f64(q.handle(), C.byref(kw.WorkDiv(kw.IndexVec(1), kw.IndexVec(2048),
                                                                kw.IndexVec(1)).to_c()), 1024, 1.0,
                                x.data(), y.data()),
        lambda: lib.kw_dgemm(q.handle(), None, 4, 4, 8, 1.0, x.data(), 4, x.data(), 4, 1.0, y.data(), 4),  # lda<k
        lambda: lib.kw_copy(q.handle(), y.data(), 8, L.sz3((1024,)), x.data(), 8, L.sz3((1024,)), 1,
                            L.sz3((2048,)), 8),  # extent beyond both buffers
        lambda: lib.kw_device_synchronize(-1),
        lambda: lib.kw_queue_create(99, 0, C.byref(ptr)),
    ]
    for i, call in enumerate(bad):
        assert call() != L.KW_OK, i
    # a valid task on the same queue, then wait(): clean
    L.check(lib.kw_axpy_f64(q.handle(), None, 1024, 2.0, x.data(), y.data()))
    q.wait()
    assert (y.download() == 2.0).all()
    q2 = kw.Queue(gpu, kw.QueueFlavor.Sync)
    L.check(lib.kw_axpy_f64(q2.handle(), None, 1024, 1.0, x.data(), y.data()))
    q2.wait()
    assert (y.download() == 3.0).all()


def test_task_markers_and_timed_events(gpu):
    """kw_task_marker (what TaskHandles use) completes like kw_event_record but carries no
    timestamp: kw_event_elapsed_ms accepts two recorded events and rejects a marker."""
    lib = L.lib()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    x = kw.Buffer(gpu, kw.IndexVec(1 << 20), 4)
    y = kw.Buffer(gpu, kw.IndexVec(1 << 20), 4)
    x.upload(np.ones(1 << 20, np.float32))
    y.upload(np.ones(1 << 20, np.float32))
    e0, mk, e1 = C.c_void_p(), C.c_void_p(), C.c_void_p()
    L.check(lib.kw_event_record(q.handle(), C.byref(e0)))
    L.check(lib.kw_axpy_f32(q.handle(), None, 1 << 20, 2.0, x.data(), y.data()))
    L.check(lib.kw_task_marker(q.handle(), C.byref(mk)))
    L.check(lib.kw_event_record(q.handle(), C.byref(e1)))
    L.check(lib.kw_queue_wait(q.handle()))
    state = C.c_int()
    L.check(lib.kw_event_state(mk, C.byref(state)))
    assert state.value == L.KW_TASK_DONE
    ms = C.c_float()
    L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
    assert ms.value >= 0.0
    assert lib.kw_event_elapsed_ms(e0, mk, C.byref(ms)) == L.KW_USAGE
    for ev in (e0, mk, e1):
        L.check(lib.kw_event_destroy(ev))
    assert np.array_equal(y.download(), np.full(1 << 20, 3.0, np.float32))


def test_queue_report_on_sync_queues(gpu):
    """kw_queue_report (what executeTask uses): OK after successful Sync tasks, TaskError (once)
    after a failed one, KW_USAGE on an Async queue."""
    lib = L.lib()
    sq = kw.Queue(gpu, kw.QueueFlavor.Sync)
    x = kw.Buffer(gpu, kw.IndexVec(1024), 8)
    y = kw.Buffer(gpu, kw.IndexVec(1024), 8)
    x.upload(np.ones(1024))
    y.upload(np.ones(1024))
    L.check(lib.kw_axpy_f64(sq.handle(), None, 1024, 2.0, x.data(), y.data()))
    assert lib.kw_queue_report(sq.handle()) == L.KW_OK
    assert np.array_equal(y.download(), np.full(1024, 3.0))
    # a task failure on the Sync queue (an illegal division) is reported, then cleared
    bad = kw.WorkDiv(kw.IndexVec(1), kw.IndexVec(2048), kw.IndexVec(1)).to_c()
    st = lib.kw_axpy_f64(sq.handle(), C.byref(bad), 1024, 2.0, x.data(), y.data())
    if st == L.KW_TASK:
        assert lib.kw_queue_report(sq.handle()) == L.KW_TASK
    assert lib.kw_queue_report(sq.handle()) == L.KW_OK
    aq = kw.Queue(gpu, kw.QueueFlavor.Async)
    assert lib.kw_queue_report(aq.handle()) == L.KW_USAGE
