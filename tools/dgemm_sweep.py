"""DGEMM tile-configuration sweep (BASELINE.json configs[4]) on one GPU: every instantiated
DMMA configuration at the given sizes, CUDA-event timed; cuBLAS (torch.matmul fp64) as the
library ceiling for context. Prints one JSON line per (config, size)."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    sizes = [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "4096,8192").split(",")]
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    for n in sizes:
        rng = np.random.default_rng(0)
        bufs = []
        for _ in range(3):
            b = kw.Buffer(dev, kw.IndexVec(n, n), 8)
            b.upload(rng.random((n, n)))
            bufs.append(b)
        A, B, Cb = bufs
        reps = max(3, int(2e12 / (2 * n ** 3)))
        for cfg in range(lib.kw_dgemm_config_count()):
            info = (C.c_int * 5)()
            lib.kw_dgemm_config_info(cfg, info)

            def go():
                L.check(lib.kw_dgemm_with_config(q.handle(), cfg, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(),
                                                 B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim()))
            go(); go()
            q.wait()
            e0, e1 = C.c_void_p(), C.c_void_p()
            lib.kw_event_record(q.handle(), C.byref(e0))
            for _ in range(reps):
                go()
            lib.kw_event_record(q.handle(), C.byref(e1))
            ms = C.c_float()
            L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
            tf = 2 * n ** 3 * reps / (ms.value / 1e3) / 1e12
            print(json.dumps({"n": n, "cfg": cfg, "BM": info[0], "BN": info[1], "BK": info[2], "threads": info[3],
                              "stages": info[4], "tflops": round(tf, 3)}), flush=True)
        # bit-exact tiled mode (kw_dgemm_bitwise)
        def gob():
            L.check(lib.kw_dgemm_bitwise(q.handle(), None, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(),
                                         B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim()))
        gob()
        q.wait()
        e0, e1 = C.c_void_p(), C.c_void_p()
        lib.kw_event_record(q.handle(), C.byref(e0))
        rb = max(2, reps // 2)
        for _ in range(rb):
            gob()
        lib.kw_event_record(q.handle(), C.byref(e1))
        ms = C.c_float()
        L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
        print(json.dumps({"n": n, "cfg": "bitwise", "tflops": round(2 * n ** 3 * rb / (ms.value / 1e3) / 1e12, 3)}),
              flush=True)
        try:
            import torch
            a = torch.rand(n, n, dtype=torch.float64, device="cuda")
            b = torch.rand(n, n, dtype=torch.float64, device="cuda")
            for _ in range(2):
                a @ b
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            for _ in range(reps):
                a @ b
            e.record()
            torch.cuda.synchronize()
            print(json.dumps({"n": n, "cfg": "cublas", "tflops": round(2 * n ** 3 * reps / (s.elapsed_time(e) / 1e3) / 1e12, 3)}))
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"n": n, "cfg": "cublas", "error": str(ex)}))


if __name__ == "__main__":
    main()
