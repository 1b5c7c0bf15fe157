"""ctypes wrapper of the oracle (TEST INFRASTRUCTURE ONLY).

Loads oracle/liboracle.so (the C restatement, kw_oracle.c) and, when present,
oracle/_ref/libkwref.so (the reference's own sources + ref_shim.cpp). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this
module; the product path (paper_1602_08477_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libkwref.so"
REFERENCE_ROOT = Path("/root/reference/proj")

sz = C.c_size_t
vp = C.c_void_p
dp = C.POINTER(C.c_double)


def build(ref: bool = True) -> None:
    """Compiles liboracle.so, and _ref/libkwref.so when the reference sources exist."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if ref and REFERENCE_ROOT.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


_o = None
_r = None


def lib() -> C.CDLL:
    global _o
    if _o is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        o = C.CDLL(str(ORACLE_SO))
        o.kw_oracle_mt_state_size.restype = sz
        o.kw_mt_seed_u64.argtypes = [vp, C.c_uint64]
        o.kw_mt_seed_seq.argtypes = [vp, C.POINTER(C.c_uint64), sz]
        o.kw_mt_next.argtypes = [vp]
        o.kw_mt_next.restype = C.c_uint64
        o.kw_seed_seq_generate.argtypes = [C.POINTER(C.c_uint32), sz, C.POINTER(C.c_uint32), sz]
        o.kw_fnv1a64.argtypes = [vp, sz, C.c_uint64]
        o.kw_fnv1a64.restype = C.c_uint64
        o.kw_kernel_tag.argtypes = [C.c_char_p]
        o.kw_kernel_tag.restype = C.c_uint64
        o.kw_fill_uniform_f64.argtypes = [vp, vp, sz, C.c_double, C.c_double]
        o.kw_fill_uniform_f32.argtypes = [vp, vp, sz, C.c_float, C.c_float]
        o.kw_workload_init.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_char_p, dp, dp]
        o.kw_oracle_axpy_f64.argtypes = [sz, C.c_double, vp, vp]
        o.kw_oracle_axpy_f32.argtypes = [sz, C.c_float, vp, vp]
        o.kw_oracle_gemm_reference.argtypes = [sz, sz, sz, C.c_double, C.c_double, vp, sz, vp, sz, vp, sz]
        o.kw_oracle_gemm_fast.argtypes = [sz, sz, sz, C.c_double, C.c_double, vp, sz, vp, sz, vp, sz, C.c_int]
        o.kw_oracle_gemm_fast.restype = C.c_int
        o.kw_oracle_axpy_threaded.argtypes = [sz, C.c_double, vp, vp, C.c_int, C.c_int]
        o.kw_oracle_axpy_threaded.restype = C.c_int
        o.kw_workload_axpy_f32.argtypes = [C.c_uint64, C.c_uint64, vp, vp, C.POINTER(C.c_float)]
        o.kw_workload_axpy_f64.argtypes = [C.c_uint64, C.c_uint64, vp, vp, dp]
        o.kw_workload_gemm.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, vp, vp, vp, dp, dp]
        _o = o
    return _o


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    """The reference's own code (oracle/_ref). Raises if it was not built."""
    global _r
    if _r is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref, needs /root/reference)")
        r = C.CDLL(str(REF_SO))
        r.kwref_last_error.restype = C.c_char_p
        r.kwref_axpy_reference_f64.argtypes = [sz, C.c_double, vp, vp]
        r.kwref_gemm_reference.argtypes = [sz, sz, sz, C.c_double, C.c_double, vp, sz, vp, sz, vp, sz]
        r.kwref_axpy_kernel.argtypes = [C.c_int, C.c_int, sz, C.c_double, vp, vp, sz, sz, dp]
        r.kwref_axpy_kernel.restype = C.c_int
        r.kwref_axpy_session_new.argtypes = [C.c_int, C.c_int, sz, C.c_double, vp, vp, sz, sz]
        r.kwref_axpy_session_new.restype = vp
        r.kwref_axpy_session_run.argtypes = [vp, dp]
        r.kwref_axpy_session_read.argtypes = [vp, vp]
        r.kwref_axpy_session_free.argtypes = [vp]
        r.kwref_gemm_kernel.argtypes = [C.c_int, C.c_int, sz, sz, sz, C.c_double, C.c_double, vp, sz, vp, sz, vp,
                                        sz, sz, sz, sz, dp]
        r.kwref_gemm_kernel.restype = C.c_int
        r.kwref_workload.argtypes = [C.c_char_p, sz, C.c_uint64, C.c_int, dp, dp, vp, vp, vp]
        r.kwref_workload.restype = C.c_int
        r.kwref_mt_seed_seq_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, vp, sz]
        r.kwref_run_bench.argtypes = [C.c_char_p, C.c_char_p, sz, C.c_int, C.c_uint64, sz, sz, sz, C.c_int, dp,
                                      C.POINTER(C.c_int)]
        r.kwref_run_bench.restype = C.c_int
        r.kwref_csv_roundtrip.argtypes = [C.c_char_p]
        r.kwref_csv_roundtrip.restype = C.c_long
        r.kwref_buffer_csv_roundtrip.argtypes = [C.c_char_p]
        r.kwref_buffer_csv_roundtrip.restype = C.c_long
        _r = r
    return _r


# ---- convenience -------------------------------------------------------------------------------
def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def fnv1a64(data) -> int:
    a = np.ascontiguousarray(data)
    return int(lib().kw_fnv1a64(_p(a), a.nbytes, 1469598103934665603))


class MT64:
    """std::mt19937_64 restated in C (kw_oracle.c)."""

    def __init__(self, seed=None, seeds=None):
        self._buf = C.create_string_buffer(lib().kw_oracle_mt_state_size())
        if seeds is not None:
            arr = (C.c_uint64 * len(seeds))(*[int(s) & 0xFFFFFFFFFFFFFFFF for s in seeds])
            lib().kw_mt_seed_seq(self._buf, arr, len(seeds))
        else:
            lib().kw_mt_seed_u64(self._buf, int(seed) & 0xFFFFFFFFFFFFFFFF)

    def __call__(self) -> int:
        return int(lib().kw_mt_next(self._buf))

    def fill_uniform(self, count: int, dtype=np.float64, lo=0.0, hi=10.0) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        if dtype == np.float32:
            lib().kw_fill_uniform_f32(self._buf, _p(out), count, lo, hi)
        else:
            lib().kw_fill_uniform_f64(self._buf, _p(out), count, lo, hi)
        return out

    def state(self):
        return self._buf


def workload_axpy(n: int, seed: int = 42, f32: bool = True):
    """(alpha, x, y) exactly as Workload("axpy", n, seed) draws them (runner.cpp:56-73)."""
    dt = np.float32 if f32 else np.float64
    x = np.empty(n, dtype=dt)
    y = np.empty(n, dtype=dt)
    if f32:
        a = C.c_float()
        lib().kw_workload_axpy_f32(seed, n, _p(x), _p(y), C.byref(a))
    else:
        a = C.c_double()
        lib().kw_workload_axpy_f64(seed, n, _p(x), _p(y), C.byref(a))
    return (np.float32(a.value) if f32 else a.value), x, y


def workload_gemm(n: int, seed: int = 42, kernel: str = "gemm-tiled"):
    """(alpha, beta, A, B, C) of Workload(kernel, n, seed) (runner.cpp:75-85)."""
    a = np.empty((n, n))
    b = np.empty((n, n))
    c = np.empty((n, n))
    al, be = C.c_double(), C.c_double()
    lib().kw_workload_gemm(seed, n, kernel.encode(), _p(a), _p(b), _p(c), C.byref(al), C.byref(be))
    return al.value, be.value, a, b, c


def axpy(alpha, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """axpyReference on a copy of y (fp32 restatement for float32 inputs)."""
    out = np.array(y, copy=True)
    if out.dtype == np.float32:
        lib().kw_oracle_axpy_f32(out.size, float(alpha), _p(np.ascontiguousarray(x)), _p(out))
    else:
        lib().kw_oracle_axpy_f64(out.size, float(alpha), _p(np.ascontiguousarray(x)), _p(out))
    return out


def gemm(alpha, beta, a: np.ndarray, b: np.ndarray, c: np.ndarray, threads: int = 0, literal: bool = False):
    """gemmReference on a copy of c; `literal` runs the r,c,p loop verbatim, otherwise the
    bitwise-identical cache-friendly threaded order."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.array(c, dtype=np.float64, copy=True, order="C")
    m, k = a.shape
    n = b.shape[1]
    if literal:
        lib().kw_oracle_gemm_reference(m, n, k, alpha, beta, _p(a), k, _p(b), n, _p(out), n)
    else:
        lib().kw_oracle_gemm_fast(m, n, k, alpha, beta, _p(a), k, _p(b), n, _p(out), n, threads or os.cpu_count())
    return out
