"""Long soak of the tile configurations the library picks (data-parallel 16/17, SPLIT 18/20/23/24/25,
two-group 26, small tiles 28/29, and kw_dgemm's own choice): random shapes (ragged, small
outputs, small and large k, padded leading dimensions), random
scalars, signed inputs; every configuration must give the bits of config 17, and config 17 must be
within (K+4)u of gemmReference (scaled by |alpha||A||B| + |beta||C| for signed data) on a subset.
python tools/split_soak.py [cases] [seed]"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import oracle as O  # noqa: E402  (test infrastructure: the checker)
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402

CFGS = (16, 18, 20, 23, 24, 25, 26, 28, 29, -1)  # -1: kw_dgemm's own choice (default division)


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 20261019
    rng = np.random.default_rng(seed)
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    t0 = time.time()
    mism = 0
    checked = 0
    for case in range(cases):
        m, n = (int(v) for v in rng.integers(64, 2600, size=2))
        if case % 4 == 3:  # small outputs with long k: the 32 x 32 / 32 x 64 tile picks
            m, n = (int(v) for v in rng.integers(1, 700, size=2))
        k = int(rng.choice([int(rng.integers(1, 64)), int(rng.integers(64, 3000))]))
        align = int(rng.choice([64, 128, 256]))
        alpha = float(rng.choice([1.0, -0.5, 0.75, 2.5]))
        beta = float(rng.choice([0.0, 1.0, -1.25]))
        a, b, c = rng.standard_normal((m, k)), rng.standard_normal((k, n)), rng.standard_normal((m, n))
        outs = {}
        for cfg in (17,) + CFGS:
            A, B, Cd = (kw.Buffer(dev, kw.IndexVec(*x.shape), 8, align) for x in (a, b, c))
            A.upload(a)
            B.upload(b)
            Cd.upload(c)
            if cfg < 0:
                L.check(lib.kw_dgemm(q.handle(), None, m, n, k, alpha, A.data(), A.leadingDim(), B.data(),
                                     B.leadingDim(), beta, Cd.data(), Cd.leadingDim()))
            else:
                L.check(lib.kw_dgemm_with_config(q.handle(), cfg, m, n, k, alpha, A.data(), A.leadingDim(), B.data(),
                                                 B.leadingDim(), beta, Cd.data(), Cd.leadingDim()))
            q.wait()
            outs[cfg] = Cd.download()
        for cfg in CFGS:
            if not np.array_equal(outs[cfg], outs[17]):
                mism += 1
                print(f"MISMATCH case {case} cfg {cfg} m={m} n={n} k={k} align={align}", flush=True)
        if case % 10 == 0:
            ref = O.gemm(alpha, beta, a, b, c, threads=8)
            scale = abs(alpha) * (np.abs(a) @ np.abs(b)) + abs(beta) * np.abs(c)
            assert np.all(np.abs(outs[17] - ref) <= (k + 4) * 2.0 ** -53 * scale), case
            checked += 1
    print(f"{cases} cases x {len(CFGS)} configs vs config 17: {mism} mismatches; oracle checked on {checked}; "
          f"{time.time() - t0:.0f} s")
    return 1 if mism else 0


if __name__ == "__main__":
    sys.exit(main())
