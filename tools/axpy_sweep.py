"""AXPY work-division sweep (BASELINE.json configs[4]): threads-per-block x elems-per-thread
at fp32 n = 2^28 on one GPU, CUDA-event timed (20 launches after 3 warm-ups). One JSON line per
point; every point is bit-exact by construction (test_workdiv_sweep_is_bit_exact)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    n = 1 << 28
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    x, y = kw.Buffer(dev, kw.IndexVec(n), 4), kw.Buffer(dev, kw.IndexVec(n), 4)
    x.fill_raw(0x3F)
    y.fill_raw(0x3F)
    tpbs = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "64,128,256,512,1024").split(",")]
    epts = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "4,8,16,32,64").split(",")]
    for tpb in tpbs:
        for ept in epts:
            wd = kw.axpyWorkDiv(kw.BackendKind.GpuCudaRt, n, tpb, ept).to_c()
            for _ in range(3):
                L.check(lib.kw_axpy_f32(q.handle(), C.byref(wd), n, 1.0000001, x.data(), y.data()))
            q.wait()
            e0, e1 = C.c_void_p(), C.c_void_p()
            lib.kw_event_record(q.handle(), C.byref(e0))
            reps = 20
            for _ in range(reps):
                L.check(lib.kw_axpy_f32(q.handle(), C.byref(wd), n, 1.0000001, x.data(), y.data()))
            lib.kw_event_record(q.handle(), C.byref(e1))
            ms = C.c_float()
            L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
            print(json.dumps({"tpb": tpb, "ept": ept, "blocks": wd.blocks[0],
                              "gbs": round(12 * n * reps / (ms.value / 1e3) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
