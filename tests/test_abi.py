"""CPU: the C-ABI library loads, exports every entry point include/kw_b200.h declares, and its
pure host-side services (work-division arithmetic, argument validation) behave like the
reference's — no compute call is made without a GPU."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1602_08477_b200 import _lib as L
from paper_1602_08477_b200 import kernelweave as kw

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "kw_b200.h").read_text()
    return sorted(set(re.findall(r"KW_EXPORT\s+[\w\s\*]+?\b(kw_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("kw_axpy_f32", "kw_axpy_f64", "kw_dgemm", "kw_dgemm_naive", "kw_buffer_alloc", "kw_copy",
                 "kw_queue_create", "kw_queue_wait", "kw_dgemm_rowsharded", "kw_comm_init"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # and the ctypes signature table covers them all (what the harness binds)
    assert set(declared_symbols()) == set(L.SIGNATURES)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(L.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def wd(dim, b, t, e):
    w = L.kw_workdiv()
    w.dim = dim
    w.blocks, w.threads, w.elems = L.sz3(b), L.sz3(t), L.sz3(e)
    return w


def test_total_extent_matches_reference_table():
    # work_div.cpp:65-94 / test_work_div.cpp:23-45
    w = wd(2, (3, 5), (4, 2), (2, 7))
    out = L.size3()
    expect = {(0, 0): (3, 5), (0, 1): (12, 10), (0, 2): (24, 70), (1, 1): (4, 2), (1, 2): (8, 14), (2, 2): (2, 7)}
    for (o, u), v in expect.items():
        assert L.lib().kw_total_extent(C.byref(w), o, u, out) == 0
        assert tuple(out[:2]) == v
    for bad in ((1, 0), (2, 0), (2, 1)):
        assert L.lib().kw_total_extent(C.byref(w), *bad, out) == L.KW_USAGE
        assert "unsupported" in L.last_error()


def test_divide_for_gpu_is_thread_level_shape():
    out = L.kw_workdiv()
    assert L.lib().kw_divide_for_gpu(1, L.sz3((4096,)), L.sz3((16,)), L.sz3((4,)), C.byref(out)) == 0
    assert (out.blocks[0], out.threads[0], out.elems[0]) == (64, 16, 4)
    assert L.lib().kw_divide_for_gpu(1, L.sz3((100,)), L.sz3((16,)), L.sz3((4,)), C.byref(out)) == 0
    assert out.blocks[0] == 2
    assert L.lib().kw_divide_for_gpu(1, L.sz3((0,)), L.sz3((16,)), L.sz3((4,)), C.byref(out)) == L.KW_USAGE
    # same answer as the Python mirror's divideForBackend(GpuCudaRt)
    w = kw.divideForBackend(kw.IndexVec(1000, 77), kw.BackendKind.GpuCudaRt, kw.IndexVec(8, 32), kw.IndexVec(2, 3))
    assert L.lib().kw_divide_for_gpu(2, L.sz3((1000, 77)), L.sz3((8, 32)), L.sz3((2, 3)), C.byref(out)) == 0
    assert kw.WorkDiv.from_c(out) == w


def test_default_workdivs():
    out = L.kw_workdiv()
    assert L.lib().kw_axpy_default_workdiv(1 << 28, 4, C.byref(out)) == 0
    assert out.threads[0] * out.elems[0] * out.blocks[0] >= 1 << 28
    assert L.lib().kw_axpy_default_workdiv(10, 3, C.byref(out)) == L.KW_USAGE
    assert L.lib().kw_dgemm_default_workdiv(4096, 1000, 128, C.byref(out)) == 0
    assert (out.blocks[0], out.blocks[1]) == (32, 8)
    assert L.lib().kw_dgemm_default_workdiv(10, 10, 48, C.byref(out)) == L.KW_USAGE


def test_usage_errors_before_anything_is_enqueued():
    q = C.c_void_p()
    # a queue on a device that does not exist is a usage error (no GPU here, or index 999)
    assert L.lib().kw_queue_create(999, 0, C.byref(q)) == L.KW_USAGE
    assert L.lib().kw_axpy_f32(None, None, 10, 1.0, None, None) == L.KW_USAGE
    assert "null queue" in L.last_error()
    ptr, pitch = C.c_void_p(), C.c_size_t()
    assert L.lib().kw_buffer_alloc(0, 2, L.sz3((4, 0)), 8, 64, C.byref(ptr), C.byref(pitch)) == L.KW_USAGE
    assert "positive" in L.last_error()
    assert L.lib().kw_buffer_alloc(0, 2, L.sz3((4, 4)), 8, 48, C.byref(ptr), C.byref(pitch)) == L.KW_USAGE
    assert "power of two" in L.last_error()


def test_no_cpu_backend_in_this_build():
    with pytest.raises(kw.UsageError, match="no CPU fallback"):
        kw.createExec(kw.BackendKind.BlocksParallel, kw.axpyWorkDiv(kw.BackendKind.BlocksParallel, 8, 1, 1),
                      kw.AxpyKernel(), kw.AxpyArgs())
