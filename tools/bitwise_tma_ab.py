"""A/B of the bit-exact DGEMM mode: warp-specialised TMA kernel (KW_BW_TMA=1, default) vs the
cp.async + __syncthreads kernel (KW_BW_TMA=0), interleaved rounds; both must give the same bits.
python tools/bitwise_tma_ab.py [n ...]"""
import os
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402

GPU = kw.BackendKind.GpuCudaRt


def main():
    sizes = [int(v) for v in sys.argv[1:]] or [4096, 8192]
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    for n in sizes:
        rng = np.random.default_rng(n)
        A, B, C0 = (kw.Buffer(dev, kw.IndexVec(n, n), 8) for _ in range(3))
        for b in (A, B, C0):
            b.upload(rng.random((n, n)))
        c_init = C0.download()
        res, outs = {"1": [], "0": []}, {}
        for _ in range(3):
            for v in ("1", "0"):
                os.environ["KW_BW_TMA"] = v
                C0.upload(c_init)
                task = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, n, n, 128), kw.GemmTiledKernel(),
                                     kw.GemmArgs(n, n, n, 1.0, 0.5, A, B, C0, 128, bitwise=True))
                q.enqueue(task)
                q.wait()
                outs[v] = C0.download()
                import time
                reps = max(2, int(2e12 / (2 * n ** 3)))
                t = time.perf_counter()
                for _ in range(reps):
                    q.enqueue(task)
                q.wait()
                res[v].append(2 * n ** 3 * reps / (time.perf_counter() - t) / 1e12)
        same = np.array_equal(outs["1"], outs["0"])
        print({"n": n, "tma_tflops": round(statistics.median(res["1"]), 3),
               "syncthreads_tflops": round(statistics.median(res["0"]), 3), "bitwise_equal": bool(same)}, flush=True)


if __name__ == "__main__":
    main()
