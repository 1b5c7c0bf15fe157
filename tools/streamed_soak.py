"""Long soak of the streamed e2e DGEMM schedule (ready-flag / done-counter handshake): random
shapes and panel grids, pinned host operands, every result bitwise against the resident launch.
python tools/streamed_soak.py [cases] [seed]"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    os.environ["KW_E2E_MIN_INTENSITY"] = "0"
    lib = L.lib()
    gpu = kw.Device.gpu(0)
    host = kw.Device.host()
    q = kw.Queue(gpu, kw.QueueFlavor.Async)
    t0 = time.time()
    bad = 0
    for case in range(cases):
        m, n, k = (int(v) for v in rng.integers(300, 3000, size=3))
        os.environ["KW_E2E_PANELS"] = str(int(rng.integers(2, 17)))
        os.environ["KW_E2E_KSPLIT"] = str(int(rng.choice([0, 2, 3, 4, 8, 64])))
        os.environ.pop("KW_E2E_KPASSES", None)
        if rng.random() < 0.4:  # several passes: random cumulative percentages
            cuts = sorted(int(v) for v in rng.integers(1, 100, size=int(rng.integers(1, 5))))
            os.environ["KW_E2E_KPASSES"] = ",".join(str(v) for v in cuts)
        a, b, c = rng.standard_normal((m, k)), rng.standard_normal((k, n)), rng.standard_normal((m, n))
        A, B, Cd = (kw.Buffer(gpu, kw.IndexVec(*x.shape), 8) for x in (a, b, c))
        for buf, x in ((A, a), (B, b), (Cd, c)):
            buf.upload(x)
        L.check(lib.kw_dgemm(q.handle(), None, m, n, k, 1.5, A.data(), A.leadingDim(), B.data(), B.leadingDim(),
                             -0.5, Cd.data(), Cd.leadingDim()))
        Ah, Bh, Ch = (kw.Buffer(host, kw.IndexVec(*x.shape), 8) for x in (a, b, c))
        for buf, x in ((Ah, a), (Bh, b), (Ch, c)):
            buf.host_view()[:, : x.shape[1]] = x
        L.check(lib.kw_dgemm(q.handle(), None, m, n, k, 1.5, Ah.data(), Ah.leadingDim(), Bh.data(), Bh.leadingDim(),
                             -0.5, Ch.data(), Ch.leadingDim()))
        q.wait()
        if not np.array_equal(Ch.host_view()[:, :n], Cd.download()):
            bad += 1
            print("MISMATCH", case, m, n, k, os.environ["KW_E2E_PANELS"], os.environ["KW_E2E_KSPLIT"],
                  os.environ.get("KW_E2E_KPASSES"), flush=True)
    print(f"{cases} streamed cases, {bad} mismatches, {time.time() - t0:.1f} s")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
