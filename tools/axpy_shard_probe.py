"""AXPY per-GPU throughput at the shard sizes of the strong-scaling run (n = 2^28 / P for
P = 1, 2, 4, 8): 400 back-to-back launches with the default division, CUDA-event timed, the way
bench.py times one rank. Every shard is > L2 (126 MB) so each launch streams from HBM.
Usage: python tools/axpy_shard_probe.py [tpb,ept ...]
KW_PROBE_ALT=1 alternates two disjoint (X, Y) pairs launch by launch, so no step can find the
previous step's operands in L2 (separates a tail effect from cross-launch L2 retention)."""
import os
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    divs = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [None]
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    full = 1 << 28
    x, y = kw.Buffer(dev, kw.IndexVec(full), 4), kw.Buffer(dev, kw.IndexVec(full), 4)
    x.fill_raw(0x3F)
    y.fill_raw(0x3F)
    pairs = [(x, y)]
    if os.environ.get("KW_PROBE_ALT") == "1":
        x2, y2 = kw.Buffer(dev, kw.IndexVec(full), 4), kw.Buffer(dev, kw.IndexVec(full), 4)
        x2.fill_raw(0x3F)
        y2.fill_raw(0x3F)
        pairs.append((x2, y2))
    for P in (1, 2, 4, 8):
        n = full // P
        for d in divs:
            wd = None if d is None else C.byref(kw.axpyWorkDiv(kw.BackendKind.GpuCudaRt, n, d[0], d[1]).to_c())
            for _ in range(5):
                L.check(lib.kw_axpy_f32(q.handle(), wd, n, 1.0000001, x.data(), y.data()))
            q.wait()
            e0, e1 = C.c_void_p(), C.c_void_p()
            reps = 400
            lib.kw_event_record(q.handle(), C.byref(e0))
            for i in range(reps):
                xs, ys = pairs[i % len(pairs)]
                L.check(lib.kw_axpy_f32(q.handle(), wd, n, 1.0000001, xs.data(), ys.data()))
            lib.kw_event_record(q.handle(), C.byref(e1))
            q.wait()
            ms = C.c_float()
            L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
            us = ms.value * 1e3 / reps
            print(json.dumps({"P": P, "n": n, "div": d or "default", "us_per_launch": round(us, 2),
                              "GBps": round(12 * n / (us * 1e-6) / 1e9, 1)}))


if __name__ == "__main__":
    main()
