"""e2e DGEMM (host pinned A, B, C through the public API) at n = 4096 and 8192, median of 5
wall-clock steps."""
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def run(n):
    GPU = kw.BackendKind.GpuCudaRt
    q = kw.Queue(kw.Device.gpu(0), kw.QueueFlavor.Async)
    host = kw.Device.host()
    bufs = [kw.Buffer(host, kw.IndexVec(n, n), 8) for _ in range(3)]
    for b in bufs:
        b.host_view()[:, :n] = 1.0
    task = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, n, n, 128), kw.GemmTiledKernel(),
                         kw.GemmArgs(n, n, n, 1.0, 0.5, *bufs))
    q.enqueue(task)
    q.wait()
    ts = []
    for _ in range(8):
        t = time.perf_counter()
        q.enqueue(task)
        q.wait()
        ts.append(time.perf_counter() - t)
    med = statistics.median(ts)
    tag = (f"streamed={os.environ.get('KW_E2E_STREAMED', '1')} panels={os.environ.get('KW_E2E_PANELS', '12')} "
           f"ksplit={os.environ.get('KW_E2E_KSPLIT', 'auto')}")
    print(f"{tag} conn={os.environ.get('CUDA_DEVICE_MAX_CONNECTIONS', '-')} n={n} {med*1e3:.1f} ms {2*n**3/med/1e12:.2f} TFLOP/s steps " + " ".join(f"{t*1e3:.1f}" for t in ts))


if __name__ == "__main__":
    for n in [int(v) for v in os.environ.get("KW_E2E_SIZES", "4096,8192").split(",")]:
        run(n)
