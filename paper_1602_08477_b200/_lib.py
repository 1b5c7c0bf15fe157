"""ctypes binding of the C-ABI in include/kw_b200.h (libkw_b200.so, built in-tree for sm_100a).

This is the boundary every Python caller (tests, bench, smoke) goes through. There is no CPU
fallback: if the shared library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libkw_b200.so"
if os.environ.get("KW_LIB_PATH"):  # A/B measurements against another build of the same library
    LIB_PATH = Path(os.environ["KW_LIB_PATH"])

KW_OK, KW_USAGE, KW_RESOURCE, KW_TASK = 0, 1, 2, 3
KW_QUEUE_SYNC, KW_QUEUE_ASYNC = 0, 1
KW_TASK_PENDING, KW_TASK_RUNNING, KW_TASK_DONE, KW_TASK_FAILED = 0, 1, 2, 3
KW_MEM_PAGEABLE, KW_MEM_PINNED, KW_MEM_DEVICE = 0, 1, 2

size_t = C.c_size_t
size3 = C.c_size_t * 3


class kw_workdiv(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("blocks", size3), ("threads", size3), ("elems", size3)]


class kw_device_props(C.Structure):
    _fields_ = [("name", C.c_char * 96), ("sm_count", C.c_int), ("cc_major", C.c_int), ("cc_minor", C.c_int),
                ("l2_bytes", size_t), ("global_mem_bytes", size_t), ("smem_per_block_optin", size_t),
                ("sm_clock_khz", C.c_int), ("mem_clock_khz", C.c_int), ("mem_bus_width_bits", C.c_int)]


vp = C.c_void_p
st = C.c_int
# name -> (restype, argtypes); the list is also the export contract checked by the CPU tests.
SIGNATURES = {
    "kw_last_error": (C.c_char_p, []),
    "kw_version": (C.c_char_p, []),
    "kw_device_count": (st, [C.POINTER(C.c_int)]),
    "kw_device_props_get": (st, [C.c_int, C.POINTER(kw_device_props)]),
    "kw_device_synchronize": (st, [C.c_int]),
    "kw_buffer_alloc": (st, [C.c_int, C.c_uint32, size3, size_t, size_t, C.POINTER(vp), C.POINTER(size_t)]),
    "kw_buffer_free": (st, [C.c_int, vp]),
    "kw_pointer_kind": (st, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "kw_memset": (st, [vp, vp, C.c_int, size_t]),
    "kw_queue_create": (st, [C.c_int, C.c_int, C.POINTER(vp)]),
    "kw_queue_destroy": (st, [vp]),
    "kw_queue_wait": (st, [vp]),
    "kw_queue_report": (st, [vp]),
    "kw_queue_device": (st, [vp, C.POINTER(C.c_int)]),
    "kw_queue_flavor": (st, [vp, C.POINTER(C.c_int)]),
    "kw_queue_stream": (st, [vp, C.POINTER(vp)]),
    "kw_queue_shutdown": (st, [vp]),
    "kw_queue_complete_launch": (st, [vp, C.c_int, C.c_char_p]),
    "kw_queue_begin_launch": (st, [vp, C.c_char_p, C.POINTER(vp), C.POINTER(C.c_int),
                                   C.POINTER(C.POINTER(C.c_uint32))]),
    "kw_queue_end_launch": (st, [vp, C.c_int, C.c_char_p]),
    "kw_queue_fail_slot": (st, [vp, C.c_char_p, C.POINTER(C.POINTER(C.c_uint32))]),
    "kw_event_record": (st, [vp, C.POINTER(vp)]),
    "kw_task_marker": (st, [vp, C.POINTER(vp)]),
    "kw_event_state": (st, [vp, C.POINTER(C.c_int)]),
    "kw_event_destroy": (st, [vp]),
    "kw_event_elapsed_ms": (st, [vp, vp, C.POINTER(C.c_float)]),
    "kw_copy": (st, [vp, vp, size_t, size3, vp, size_t, size3, C.c_uint32, size3, size_t]),
    "kw_total_extent": (st, [C.POINTER(kw_workdiv), C.c_int, C.c_int, size3]),
    "kw_divide_for_gpu": (st, [C.c_uint32, size3, size3, size3, C.POINTER(kw_workdiv)]),
    "kw_axpy_default_workdiv": (st, [size_t, C.c_int, C.POINTER(kw_workdiv)]),
    "kw_dgemm_default_workdiv": (st, [size_t, size_t, size_t, C.POINTER(kw_workdiv)]),
    "kw_axpy_f32": (st, [vp, C.POINTER(kw_workdiv), size_t, C.c_float, vp, vp]),
    "kw_axpy_f64": (st, [vp, C.POINTER(kw_workdiv), size_t, C.c_double, vp, vp]),
    "kw_dgemm": (st, [vp, C.POINTER(kw_workdiv), size_t, size_t, size_t, C.c_double, vp, size_t, vp, size_t,
                      C.c_double, vp, size_t]),
    "kw_dgemm_bitwise": (st, [vp, C.POINTER(kw_workdiv), size_t, size_t, size_t, C.c_double, vp, size_t, vp,
                              size_t, C.c_double, vp, size_t]),
    "kw_dgemm_config_count": (C.c_int, []),
    "kw_dgemm_config_info": (st, [C.c_int, C.c_int * 5]),
    "kw_dgemm_with_config": (st, [vp, C.c_int, size_t, size_t, size_t, C.c_double, vp, size_t, vp, size_t,
                                  C.c_double, vp, size_t]),
    "kw_dgemm_naive": (st, [vp, C.POINTER(kw_workdiv), size_t, size_t, size_t, C.c_double, vp, size_t, vp,
                            size_t, C.c_double, vp, size_t]),
    "kw_comm_unique_id": (st, [C.c_char * 128]),
    "kw_comm_init": (st, [C.POINTER(vp), C.c_int, C.c_int, C.c_int, C.c_char * 128]),
    "kw_comm_destroy": (st, [vp]),
    "kw_comm_broadcast": (st, [vp, vp, vp, size_t, C.c_int]),
    "kw_dgemm_rowsharded": (st, [vp, vp, size_t, size_t, size_t, C.c_double, vp, size_t, vp, size_t, C.c_double,
                                 vp, size_t, vp, C.c_int, C.c_int]),
    "kw_dgemm_rowsharded_scratch": (st, [size_t, size_t, C.c_int, C.POINTER(size_t)]),
    "kw_l2_flush": (st, [vp]),
    "kw_dgemm_split_trace": (st, [vp]),
    "kw_dgemm_split_plan": (st, [C.c_longlong, C.c_longlong, C.c_longlong, C.c_longlong, C.c_longlong,
                                 C.POINTER(C.c_int)]),
    "kw_launch_count": (C.c_uint64, []),
    "kw_axpy_kernel_name": (st, [C.POINTER(kw_workdiv), C.c_int, vp, vp, C.c_char_p, size_t]),
    "kw_device_pci_bus_id": (st, [C.c_int, C.c_char_p, C.c_int]),
}


class KwError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


_lib = None


def lib() -> C.CDLL:
    """Loads libkw_b200.so once. Raises (never falls back) when the extension is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        # Prefer the NCCL torch ships (so torch.distributed and kw_comm share one libnccl.so.2).
        if "KW_NCCL_LIBRARY" not in os.environ:
            import importlib.util
            spec = importlib.util.find_spec("nvidia.nccl")
            if spec and spec.submodule_search_locations:
                cand = Path(list(spec.submodule_search_locations)[0]) / "lib" / "libnccl.so.2"
                if cand.exists():
                    os.environ["KW_NCCL_LIBRARY"] = str(cand)
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    return (lib().kw_last_error() or b"").decode(errors="replace")


def check(status: int) -> None:
    if status != KW_OK:
        raise KwError(status, last_error())


def sz3(vals) -> size3:
    v = list(vals) + [1] * (3 - len(vals))
    return size3(*v)
