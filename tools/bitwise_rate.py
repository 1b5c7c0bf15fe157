"""TFLOP/s of the bit-exact DGEMM mode (kw_dgemm_bitwise, default division) at the given sizes:
median of 3 timed groups of back-to-back launches. python tools/bitwise_rate.py [n ...]"""
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    for n in [int(v) for v in sys.argv[1:]] or [4096, 8192]:
        A, B, Cb = (kw.Buffer(dev, kw.IndexVec(n, n), 8) for _ in range(3))
        for b in (A, B, Cb):
            b.upload(np.random.default_rng(n).random((n, n)))

        def go():
            L.check(lib.kw_dgemm_bitwise(q.handle(), None, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(),
                                         B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim()))
        go()
        q.wait()
        reps = max(2, int(1e12 / (2 * n ** 3)))
        rates = []
        for _ in range(3):
            e0, e1 = C.c_void_p(), C.c_void_p()
            lib.kw_event_record(q.handle(), C.byref(e0))
            for _ in range(reps):
                go()
            lib.kw_event_record(q.handle(), C.byref(e1))
            q.wait()
            ms = C.c_float()
            L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
            rates.append(2 * n ** 3 * reps / (ms.value / 1e3) / 1e12)
        print(json.dumps({"n": n, "bitwise_tflops": round(statistics.median(rates), 3)}))


if __name__ == "__main__":
    main()
