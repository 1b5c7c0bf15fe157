"""SPLIT DGEMM timeline (needs a library built with KW_EXTRA_NVCC_FLAGS=-DKW_SPLIT_TRACE):
`python tools/split_trace.py N cfg` runs 3 launches of kw_dgemm_with_config(cfg) on N^3, traces
the last one (%globaltimer per virtual CTA: start, pieces, end) and prints where the time goes:
kernel span, per-CTA start skew, busy time, time waiting before tail pieces, end skew."""
import ctypes as C
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    n, cfg = int(sys.argv[1]), int(sys.argv[2])
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    A, B, Cb = (kw.Buffer(dev, kw.IndexVec(n, n), 8) for _ in range(3))
    for b in (A, B, Cb):
        b.upload(np.random.default_rng(0).random((n, n)))
    tr = kw.Buffer(dev, kw.IndexVec(4096 * 40), 8)
    tr.fill_raw(0)

    def go():
        L.check(lib.kw_dgemm_with_config(q.handle(), cfg, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(),
                                         B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim()))
    for _ in range(3):
        go()
    q.wait()
    L.check(lib.kw_dgemm_split_trace(tr.data()))
    go()
    q.wait()
    L.check(lib.kw_dgemm_split_trace(None))
    t = tr.download().view(np.uint64).reshape(4096, 40)
    rows = [r for r in t if r[0]]
    t0 = min(int(r[0]) for r in rows)
    starts = [int(r[0]) - t0 for r in rows]
    ends = [int(r[39]) - t0 for r in rows]
    span = max(ends)
    busy, gaps = [], []
    for r in rows:
        b = 0
        prev_end = int(r[0])
        g = 0
        for j in range(18):
            s, e = int(r[2 + 2 * j]), int(r[3 + 2 * j])
            if not s:
                break
            b += e - s
            g += s - prev_end
            prev_end = e
        busy.append(b)
        gaps.append(g)
    flops = 2 * n ** 3
    print(f"n={n} cfg={cfg} virtual CTAs={len(rows)} kernel span {span / 1e3:.1f} us "
          f"({flops / span / 1e3:.2f} TFLOP/s over the span)")
    print(f"  start skew: median {statistics.median(starts) / 1e3:.1f} us, max {max(starts) / 1e3:.1f} us")
    print(f"  end: min {min(ends) / 1e3:.1f} us, median {statistics.median(ends) / 1e3:.1f}, max {max(ends) / 1e3:.1f}")
    print(f"  piece-busy per CTA: median {statistics.median(busy) / 1e3:.1f} us, min {min(busy) / 1e3:.1f}, "
          f"max {max(busy) / 1e3:.1f}")
    print(f"  gaps between pieces (incl. tail waits): median {statistics.median(gaps) / 1e3:.2f} us, "
          f"max {max(gaps) / 1e3:.2f} us")
    # busy time and end per SM (both groups of an SM summed / max), to see whether the spread is
    # per SM (placement) or per CTA
    per_sm = {}
    for r, b, e in zip(rows, busy, ends):
        sm = int(r[1])
        per_sm.setdefault(sm, []).append((b, e))
    line = []
    for sm in sorted(per_sm):
        bs = per_sm[sm]
        line.append(f"{sm}:{max(x[1] for x in bs) / 1e3:.0f}")
    print("  end per SM (sm:us): " + " ".join(line))
    # per-piece durations by kind for the median CTA
    r = rows[len(rows) // 2]
    pieces = []
    for j in range(18):
        s, e = int(r[2 + 2 * j]), int(r[3 + 2 * j])
        if not s:
            break
        pieces.append(f"{(s - t0) / 1e3:.1f}+{(e - s) / 1e3:.1f}")
    print(f"  one CTA (sm {int(r[1])}): start {(int(r[0]) - t0) / 1e3:.1f} us, pieces start+dur: {' '.join(pieces)}, "
          f"end {(int(r[39]) - t0) / 1e3:.1f}")


if __name__ == "__main__":
    main()
