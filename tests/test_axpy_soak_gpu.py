"""Randomised AXPY soak through the C-ABI: random lengths, dtypes, pointer offsets (alignment),
residencies (device, pinned host, pageable host, mixed) and work divisions — including divisions
that cover only a prefix — must equal axpyReference (the oracle) bit for bit on the covered
prefix and leave every other element untouched (axpy.cpp:10-23)."""
import ctypes as C

import numpy as np
import pytest

from paper_1602_08477_b200 import _lib as L
from paper_1602_08477_b200 import kernelweave as kw

pytestmark = pytest.mark.gpu
GPU = kw.BackendKind.GpuCudaRt


def test_axpy_random_cases_bitwise(gpu, oracle):
    rng = np.random.default_rng(1018)
    lib = L.lib()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    for case in range(150):
        f32 = bool(case % 2)
        dt = np.float32 if f32 else np.float64
        es = 4 if f32 else 8
        n = int(rng.integers(1, 1 << int(rng.integers(1, 23))))
        off_x, off_y = (int(v) for v in rng.integers(0, 4, size=2))  # element offsets: misalignment
        x = rng.standard_normal(n + off_x).astype(dt)
        y = rng.standard_normal(n + off_y).astype(dt)
        alpha = dt(rng.standard_normal())
        tpb = int(rng.choice([32, 96, 128, 256, 512, 1024]))
        ept = int(rng.choice([1, 2, 3, 4, 8, 16]))
        blocks = -(-n // (tpb * ept))
        if rng.random() < 0.25:  # a division that covers only a prefix
            blocks = max(1, blocks - int(rng.integers(1, max(2, blocks))))
        covered = min(n, blocks * tpb * ept)
        wd = kw.WorkDiv(kw.IndexVec(blocks), kw.IndexVec(tpb), kw.IndexVec(ept)).to_c()
        want = y[off_y:].copy()
        want[:covered] = oracle.axpy(alpha, x[off_x:off_x + covered], y[off_y:off_y + covered])
        residency = case % 4  # 0 device, 1 pinned host, 2 pageable host, 3 x device + y pageable
        bufs = []

        def place(arr, where):
            if where == "device":
                b = kw.Buffer(gpu, kw.IndexVec(arr.size), es)
                b.upload(arr)
            elif where == "pinned":
                b = kw.Buffer(kw.Device.host(), kw.IndexVec(arr.size), es)
                b.host_view()[:] = arr
            else:
                return arr, arr.ctypes.data
            bufs.append(b)
            return b, b.data()

        wx, wy = (("device", "device"), ("pinned", "pinned"), ("pageable", "pageable"),
                  ("device", "pageable"))[residency]
        xb, xp = place(x, wx)
        yb, yp = place(y, wy)
        fn = lib.kw_axpy_f32 if f32 else lib.kw_axpy_f64
        L.check(fn(q.handle(), C.byref(wd), n, float(alpha), xp + off_x * es, yp + off_y * es))
        q.wait()
        if wy == "device":
            got = yb.download()[off_y:]
        elif wy == "pinned":
            got = yb.host_view()[off_y:].copy()
        else:
            got = y[off_y:]
        assert got.tobytes() == want.tobytes(), (case, n, f32, off_x, off_y, tpb, ept, blocks, wx, wy)
