"""Rectangular DGEMM shapes: the library's own tile choice (kw_dgemm) vs cuBLAS DGEMM (torch.matmul
fp64) on the same box, and every resident configuration the pick chooses between (16, 17, 18,
20, 25), to find shapes where the pick is far from the best. Median TFLOP/s of back-to-back
launches, 3 rounds. python tools/dgemm_rect.py [m,n,k ...]"""
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402

SHAPES = [(8192, 8192, 256), (8192, 8192, 1024), (256, 8192, 8192), (8192, 256, 8192), (2048, 8192, 2048),
          (8192, 2048, 2048), (1024, 4096, 4096), (4096, 1024, 4096), (512, 512, 16384), (3000, 5000, 700),
          (16384, 1024, 1024), (1024, 16384, 1024)]
CFGS = (-1, 16, 17, 18, 20, 25, 27, 28, 29)


def timed(lib, q, go, flops, reps):
    go()
    q.wait()
    e0, e1 = C.c_void_p(), C.c_void_p()
    lib.kw_event_record(q.handle(), C.byref(e0))
    for _ in range(reps):
        go()
    lib.kw_event_record(q.handle(), C.byref(e1))
    ms = C.c_float()
    L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
    return flops * reps / (ms.value / 1e3) / 1e12


def cublas(m, n, k, reps):
    import torch
    a = torch.rand(m, k, dtype=torch.float64, device="cuda:0")
    b = torch.rand(k, n, dtype=torch.float64, device="cuda:0")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    return 2 * m * n * k * reps / (e0.elapsed_time(e1) / 1e3) / 1e12


def main():
    shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]] or SHAPES
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    rng = np.random.default_rng(0)
    for (m, n, k) in shapes:
        A = kw.Buffer(dev, kw.IndexVec(m, k), 8)
        B = kw.Buffer(dev, kw.IndexVec(k, n), 8)
        Cb = kw.Buffer(dev, kw.IndexVec(m, n), 8)
        A.upload(rng.random((m, k)))
        B.upload(rng.random((k, n)))
        Cb.upload(rng.random((m, n)))
        flops = 2 * m * n * k
        reps = max(5, int(1.5e12 / flops))
        res = {c: [] for c in CFGS}
        for _ in range(3):
            for cfg in CFGS:
                if cfg < 0:
                    go = lambda: L.check(lib.kw_dgemm(q.handle(), None, m, n, k, 1.0, A.data(), A.leadingDim(),  # noqa: E731
                                                      B.data(), B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim()))
                else:
                    go = lambda: L.check(lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, 1.0, A.data(),  # noqa: E731
                                                                  A.leadingDim(), B.data(), B.leadingDim(), 1.0,
                                                                  Cb.data(), Cb.leadingDim()))
                res[cfg].append(timed(lib, q, go, flops, reps))
        med = {c: round(statistics.median(v), 2) for c, v in res.items()}
        best = max((v, c) for c, v in med.items() if c >= 0)
        print(json.dumps({"m": m, "n": n, "k": k, "library": med[-1], "cublas": round(cublas(m, n, k, reps), 2),
                          "best_cfg": best[1], "best": best[0], "cfgs": {str(c): med[c] for c in CFGS if c >= 0}}))
        del A, B, Cb


if __name__ == "__main__":
    main()
