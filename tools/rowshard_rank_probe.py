"""One rank's compute schedule of the row-sharded 16384^3 DGEMM, on one GPU: a world-size-1
communicator (no broadcast, no cross-rank waits) with the m_local a rank gets at P ranks, timed
against one kw_dgemm launch of the same shape. Shows the per-panel launch tail cost.
Usage: python tools/rowshard_rank_probe.py [panels] [rounds]"""
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
    panels = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    n = 16384
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    uid = (C.c_char * 128)()
    L.check(lib.kw_comm_unique_id(uid))
    comm = C.c_void_p()
    L.check(lib.kw_comm_init(C.byref(comm), 0, 1, 0, uid))
    B = kw.Buffer(dev, kw.IndexVec(n, n), 8)
    B.fill_raw(0)
    pan = kw.Buffer(dev, kw.IndexVec(n * n), 8)
    for P in (8, 4, 2, 1):
        m = n // P
        A, Cb = kw.Buffer(dev, kw.IndexVec(m, n), 8), kw.Buffer(dev, kw.IndexVec(m, n), 8)
        A.upload(np.random.default_rng(P).random((m, n)))
        Cb.fill_raw(0)

        def sharded():
            L.check(lib.kw_dgemm_rowsharded(comm, q.handle(), m, n, n, 1.0, A.data(), A.leadingDim(), B.data(),
                                            B.leadingDim(), 0.5, Cb.data(), Cb.leadingDim(), pan.data(), panels, 0))

        def single():
            L.check(lib.kw_dgemm(q.handle(), None, m, n, n, 1.0, A.data(), A.leadingDim(), B.data(),
                                 B.leadingDim(), 0.5, Cb.data(), Cb.leadingDim()))

        res = {"sharded": [], "single": []}
        for _ in range(rounds):
            for name, go in (("sharded", sharded), ("single", single)):
                go()
                q.wait()
                e0, e1 = C.c_void_p(), C.c_void_p()
                lib.kw_event_record(q.handle(), C.byref(e0))
                go()
                lib.kw_event_record(q.handle(), C.byref(e1))
                q.wait()
                ms = C.c_float()
                L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
                res[name].append(2 * m * n * n / (ms.value / 1e3) / 1e12)
        print(json.dumps({"ranks": P, "m_local": m, "panels": panels,
                          "rowsharded_tflops": round(statistics.median(res["sharded"]), 2),
                          "single_launch_tflops": round(statistics.median(res["single"]), 2)}))
    lib.kw_comm_destroy(comm)


if __name__ == "__main__":
    main()
