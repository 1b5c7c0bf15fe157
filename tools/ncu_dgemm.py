"""Drives DGEMM launches for an ncu capture: `python tools/ncu_dgemm.py N [cfg] [reps]` runs
kw_dgemm (cfg < 0: the library's own tile choice) `reps` times on N^3 device-resident operands
(pass --launch-skip to ncu to skip the warm-up launches)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    n = int(sys.argv[1])
    cfg = int(sys.argv[2]) if len(sys.argv) > 2 else -1
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    rng = np.random.default_rng(0)
    A, B, Cb = (kw.Buffer(dev, kw.IndexVec(n, n), 8) for _ in range(3))
    for b in (A, B, Cb):
        b.upload(rng.random((n, n)))
    for _ in range(reps):
        if cfg < 0:
            L.check(lib.kw_dgemm(q.handle(), None, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                                 1.0, Cb.data(), Cb.leadingDim()))
        else:
            L.check(lib.kw_dgemm_with_config(q.handle(), cfg, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(),
                                             B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim()))
    q.wait()
    print(f"ok n={n} cfg={cfg} reps={reps}")


if __name__ == "__main__":
    main()
