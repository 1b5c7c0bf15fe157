"""Generates tests/golden/golden.json from the REFERENCE's own code (oracle/_ref/libkwref.so,
compiled from /root/reference/proj sources). Runs in the dev container only (needs the
reference); the committed JSON is what travels. TEST INFRASTRUCTURE ONLY.

Contents (all values produced by reference code paths):
  * raw std::mt19937_64 draws for the bench seeding (pins the generator restatement);
  * the bench Workload's alpha/beta and FNV-1a-64 digests of inputs and oracle outputs for
    AXPY fp64 / fp32 (fp32 = restated functor on the reference runtime) at n = 2^20, 1000003,
    and DGEMM at n = 64, 256;
  * the reference test suite's known-answer cases (test_kernels.cpp) evaluated by the
    reference library: tail canary, n = 4099 native-vs-kernel, ragged/rectangular GEMMs.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle import oracle as O  # noqa: E402

OUT = HERE.parent / "tests" / "golden" / "golden.json"


def hx(v: int) -> str:
    return f"{v:016x}"


def ref_workload(kernel: str, n: int, seed: int, f32: bool):
    r = O.ref()
    al, be = C.c_double(), C.c_double()
    if kernel == "axpy":
        dt = np.float32 if f32 else np.float64
        x, y = np.empty(n, dt), np.empty(n, dt)
        assert r.kwref_workload(kernel.encode(), n, seed, int(f32), C.byref(al), C.byref(be), x.ctypes.data,
                                y.ctypes.data, None) == 0
        return al.value, be.value, x, y
    a, b, c = (np.empty((n, n)) for _ in range(3))
    assert r.kwref_workload(kernel.encode(), n, seed, 0, C.byref(al), C.byref(be), a.ctypes.data, b.ctypes.data,
                            c.ctypes.data) == 0
    return al.value, be.value, a, b, c


def ref_axpy_kernel(alpha, x, y, f32, backend=1, tpb=16, ept=8):
    out = y.copy()
    sec = C.c_double()
    assert O.ref().kwref_axpy_kernel(backend, int(f32), x.size, float(alpha), x.ctypes.data, out.ctypes.data, tpb,
                                     ept, C.byref(sec)) == 0
    return out


def ref_gemm(alpha, beta, a, b, c, tiled=1, backend=0, tile=16):
    out = np.array(c, copy=True)
    m, k = a.shape
    n = b.shape[1]
    sec = C.c_double()
    assert O.ref().kwref_gemm_kernel(backend, tiled, m, n, k, alpha, beta, np.ascontiguousarray(a).ctypes.data, k,
                                     np.ascontiguousarray(b).ctypes.data, n, out.ctypes.data, n, tile, 4, 4,
                                     C.byref(sec)) == 0, O.ref().kwref_last_error()
    return out


def main() -> None:
    r = O.ref()
    g: dict = {"generator": "oracle/gen_golden.py (reference: /root/reference/proj via oracle/_ref)"}

    draws = np.empty(16, dtype=np.uint64)
    tag = int(O.lib().kw_kernel_tag(b"axpy"))
    r.kwref_mt_seed_seq_draws(42, 1 << 20, tag, draws.ctypes.data, 16)
    g["mt19937_64_seed_seq_42_2p20_axpy"] = [hx(int(v)) for v in draws]
    g["kernel_tag"] = {k: hx(int(O.lib().kw_kernel_tag(k.encode()))) for k in ("axpy", "gemm-naive", "gemm-tiled")}

    cases = []
    for n in (1 << 20, 1000003):
        for f32 in (True, False):
            al, _, x, y = ref_workload("axpy", n, 42, f32)
            if f32:
                yo = ref_axpy_kernel(np.float32(al), x, y, True)
            else:
                yo = y.copy()
                r.kwref_axpy_reference_f64(n, al, x.ctypes.data, yo.ctypes.data)
            cases.append({"kernel": "axpy", "dtype": "f32" if f32 else "f64", "n": n, "seed": 42,
                          "alpha": float(np.float32(al)) if f32 else al, "x_digest": hx(O.fnv1a64(x)),
                          "y_in_digest": hx(O.fnv1a64(y)), "y_out_digest": hx(O.fnv1a64(yo)),
                          "first": float(yo[0]), "last": float(yo[-1])})
    for n in (64, 256):
        al, be, a, b, c = ref_workload("gemm-tiled", n, 42, False)
        co = ref_gemm(al, be, a, b, c, tiled=1, backend=1, tile=16)
        lit = c.copy()
        r.kwref_gemm_reference(n, n, n, al, be, a.ctypes.data, n, b.ctypes.data, n, lit.ctypes.data, n)
        assert (co == lit).all()
        cases.append({"kernel": "gemm-tiled", "dtype": "f64", "n": n, "seed": 42, "alpha": al, "beta": be,
                      "a_digest": hx(O.fnv1a64(a)), "b_digest": hx(O.fnv1a64(b)), "c_in_digest": hx(O.fnv1a64(c)),
                      "c_out_digest": hx(O.fnv1a64(co)), "c00": float(co[0, 0]), "c_last": float(co[-1, -1])})
    g["workloads"] = cases

    # test_kernels.cpp:88-112 tail canary: rng(42), X, Y of 128, n = 100, alpha 1.5, WorkDiv(2,16,4).
    rng = O.MT64(seed=42)
    x = rng.fill_uniform(128)
    y = rng.fill_uniform(128)
    y[100:] = -555.25
    yo = y.copy()
    r.kwref_axpy_reference_f64(100, 1.5, x.ctypes.data, yo.ctypes.data)
    g["axpy_tail_canary"] = {"seed": 42, "n": 100, "covered": 128, "alpha": 1.5, "y_out": yo.tolist()}

    # test_kernels.cpp:331-349: rng(55), n = 4099, alpha 3.25.
    rng = O.MT64(seed=55)
    x = rng.fill_uniform(4099)
    y = rng.fill_uniform(4099)
    yo = y.copy()
    r.kwref_axpy_reference_f64(4099, 3.25, x.ctypes.data, yo.ctypes.data)
    yk = ref_axpy_kernel(3.25, x, y, False, backend=2, tpb=16, ept=8)
    assert (yk == yo).all()
    g["axpy_native_4099"] = {"seed": 55, "n": 4099, "alpha": 3.25, "y_out_digest": hx(O.fnv1a64(yo))}

    # test_kernels.cpp:232-279 ragged cases (rng 4321) evaluated by the reference's tiled kernel.
    rng = O.MT64(seed=4321)
    rag = []
    s = 16
    mats = [rng.fill_uniform(s * s).reshape(s, s) for _ in range(3)]
    rag.append({"m": s, "n": s, "k": s, "alpha": 2.0, "beta": 1.0,
                "c_out_digest": hx(O.fnv1a64(ref_gemm(2.0, 1.0, *mats, tiled=1, tile=s)))})
    s = 10
    mats = [rng.fill_uniform(s * s).reshape(s, s) for _ in range(3)]
    rag.append({"m": s, "n": s, "k": s, "alpha": 1.0, "beta": 0.5,
                "c_out_digest": hx(O.fnv1a64(ref_gemm(1.0, 0.5, *mats, tiled=1, tile=4)))})
    m, n, k = 13, 29, 7
    a = rng.fill_uniform(m * k).reshape(m, k)
    b = rng.fill_uniform(k * n).reshape(k, n)
    c = rng.fill_uniform(m * n).reshape(m, n)
    rag.append({"m": m, "n": n, "k": k, "alpha": 2.5, "beta": 0.0,
                "c_out_digest": hx(O.fnv1a64(ref_gemm(2.5, 0.0, a, b, c, tiled=1, tile=8)))})
    g["gemm_ragged_rng4321"] = rag

    OUT.parent.mkdir(parents=True, exist_ok=True)
    OUT.write_text(json.dumps(g, indent=1) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
