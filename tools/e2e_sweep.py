"""e2e AXPY (host pinned buffers streamed through the GPU) vs staging chunk size. Run once per
KW_STAGE_CHUNK_MB value (the library reads it at first use)."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    n = 1 << 28
    GPU = kw.BackendKind.GpuCudaRt
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    hx = kw.Buffer(kw.Device.host(), kw.IndexVec(n), 4)
    hy = kw.Buffer(kw.Device.host(), kw.IndexVec(n), 4)
    hx.host_view()[:] = 1.0
    hy.host_view()[:] = 2.0
    task = kw.createExec(GPU, kw.axpyWorkDiv(GPU, n, 512, 4), kw.AxpyKernel(), kw.AxpyArgs(n, 1.0, hx, hy))
    q.enqueue(task)
    q.wait()
    ts = []
    for _ in range(9):
        t = time.perf_counter()
        q.enqueue(task)
        q.wait()
        ts.append(time.perf_counter() - t)
    best, med = min(ts), float(np.median(ts))
    print(f"zerocopy={os.environ.get('KW_AXPY_ZEROCOPY', '0')} chunk_mb={os.environ.get('KW_STAGE_CHUNK_MB', '32')} median {med*1e3:.2f} ms {12*n/med/1e9:.1f} GB/s "
          f"best {12*n/best/1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
