"""Interleaved A/B timing of DGEMM tile configurations (noise control for sub-1 % decisions):
rounds x configs, each point = median TFLOP/s of `reps` back-to-back launches; prints the
median over rounds per config."""
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
    n = int(sys.argv[1])
    cfgs = [int(c) for c in sys.argv[2].split(",")]  # -1 = kw_dgemm's own tile choice
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    rng = np.random.default_rng(0)
    A, B, Cb = (kw.Buffer(dev, kw.IndexVec(n, n), 8) for _ in range(3))
    for b in (A, B, Cb):
        b.upload(rng.random((n, n)))
    reps = max(3, int(1.5e12 / (2 * n ** 3)))
    res = {c: [] for c in cfgs}
    for _ in range(rounds):
        for cfg in cfgs:
            if cfg < 0:  # the library's own choice (kw_dgemm, default division)
                go = lambda: L.check(lib.kw_dgemm(q.handle(), None, n, n, n, 1.0, A.data(), A.leadingDim(),  # noqa: E731
                                                  B.data(), B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim()))
            else:
                go = lambda: L.check(lib.kw_dgemm_with_config(q.handle(), cfg, n, n, n, 1.0, A.data(),  # noqa: E731
                                                              A.leadingDim(), B.data(), B.leadingDim(), 1.0,
                                                              Cb.data(), Cb.leadingDim()))
            go()
            q.wait()
            e0, e1 = C.c_void_p(), C.c_void_p()
            lib.kw_event_record(q.handle(), C.byref(e0))
            for _ in range(reps):
                go()
            lib.kw_event_record(q.handle(), C.byref(e1))
            ms = C.c_float()
            L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
            res[cfg].append(2 * n ** 3 * reps / (ms.value / 1e3) / 1e12)
    for cfg in cfgs:
        print(json.dumps({"n": n, "cfg": cfg, "median_tflops": round(statistics.median(res[cfg]), 3),
                          "min": round(min(res[cfg]), 3), "max": round(max(res[cfg]), 3)}))


if __name__ == "__main__":
    main()
