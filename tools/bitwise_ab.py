"""Interleaved A/B of bit-exact tiled DGEMM variants: python tools/bitwise_ab.py n variants rounds.
The library reads no variant switch today — profiles/dgemm_bitwise_variants_r01.txt came from a
temporary KW_BW_VARIANT hook in launch_bitwise (BwCfg<8,1,BK,STAGES> instantiations), removed
once k-tile 32 x 2 stages was adopted; re-add such a hook to compare new variants. Also checks
that every variant's output is bitwise equal to the first's."""
import ctypes as C
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    n = int(sys.argv[1])
    variants = [v for v in sys.argv[2].split(",")]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    rng = np.random.default_rng(0)
    A, B, Cb = (kw.Buffer(dev, kw.IndexVec(n, n), 8) for _ in range(3))
    for b in (A, B, Cb):
        b.upload(rng.random((n, n)))
    res = {v: [] for v in variants}
    outs = {}
    for _ in range(rounds):
        for v in variants:
            os.environ["KW_BW_VARIANT"] = v
            go = lambda: L.check(lib.kw_dgemm_bitwise(q.handle(), None, n, n, n, 1.0, A.data(), A.leadingDim(),  # noqa: E731
                                                      B.data(), B.leadingDim(), 0.0, Cb.data(), Cb.leadingDim()))
            go()
            q.wait()
            outs[v] = Cb.download()
            e0, e1 = C.c_void_p(), C.c_void_p()
            lib.kw_event_record(q.handle(), C.byref(e0))
            for _ in range(2):
                go()
            lib.kw_event_record(q.handle(), C.byref(e1))
            q.wait()
            ms = C.c_float()
            L.check(lib.kw_event_elapsed_ms(e0, e1, C.byref(ms)))
            res[v].append(2 * n ** 3 * 2 / (ms.value / 1e3) / 1e12)
    same = all(np.array_equal(outs[v], outs[variants[0]]) for v in variants)
    for v in variants:
        print(json.dumps({"n": n, "variant": v, "median_tflops": round(statistics.median(res[v]), 3),
                          "bitwise_equal_to_first": same}))


if __name__ == "__main__":
    main()
