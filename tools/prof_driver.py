"""Small, deterministic launch sequences for ncu (one GPU): `axpy` (fp32 2^28) and
`dgemm <n>` (fp64 n^3), each 3 launches after 1 warm-up, through the C-ABI."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402

GPU = kw.BackendKind.GpuCudaRt


def main():
    what = sys.argv[1]
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    if what == "axpy":
        n = 1 << 28
        x, y = kw.Buffer(dev, kw.IndexVec(n), 4), kw.Buffer(dev, kw.IndexVec(n), 4)
        x.fill_raw(0x3F)
        y.fill_raw(0x3F)
        tpb = int(sys.argv[2]) if len(sys.argv) > 2 else 256
        ept = int(sys.argv[3]) if len(sys.argv) > 3 else 16
        task = kw.createExec(GPU, kw.axpyWorkDiv(GPU, n, tpb, ept), kw.AxpyKernel(), kw.AxpyArgs(n, 1.5, x, y))
    else:
        n = int(sys.argv[2])
        tile = int(sys.argv[3]) if len(sys.argv) > 3 else 128
        rng = np.random.default_rng(0)
        bufs = []
        for _ in range(3):
            b = kw.Buffer(dev, kw.IndexVec(n, n), 8)
            b.upload(rng.random((n, n)))
            bufs.append(b)
        bitwise = len(sys.argv) > 4 and sys.argv[4] == "bitwise"
        task = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, n, n, tile), kw.GemmTiledKernel(),
                             kw.GemmArgs(n, n, n, 1.0, 1.0, *bufs, bitwise=bitwise))
    for _ in range(4):
        q.enqueue(task)
    q.wait()
    print("ok")


if __name__ == "__main__":
    main()
