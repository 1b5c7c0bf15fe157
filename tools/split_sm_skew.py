"""Is the SPLIT end-time spread a property of the SMs? (needs a KW_SPLIT_TRACE build, see
split_trace.py): `python tools/split_sm_skew.py N cfg [launches]` traces several launches and
reports, per SM, the busy time (sum of piece durations) of its virtual CTAs; the correlation of
per-SM busy time between launches says whether the same SMs are slow every time."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1602_08477_b200 import _lib as L  # noqa: E402
from paper_1602_08477_b200 import kernelweave as kw  # noqa: E402


def main():
    n, cfg = int(sys.argv[1]), int(sys.argv[2])
    launches = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    lib = L.lib()
    dev = kw.Device.gpu(0)
    q = kw.Queue(dev, kw.QueueFlavor.Async)
    A, B, Cb = (kw.Buffer(dev, kw.IndexVec(n, n), 8) for _ in range(3))
    for b in (A, B, Cb):
        b.upload(np.random.default_rng(0).random((n, n)))
    tr = kw.Buffer(dev, kw.IndexVec(4096 * 40), 8)

    def go():
        L.check(lib.kw_dgemm_with_config(q.handle(), cfg, n, n, n, 1.0, A.data(), A.leadingDim(), B.data(),
                                         B.leadingDim(), 1.0, Cb.data(), Cb.leadingDim()))
    for _ in range(3):
        go()
    q.wait()
    per = []
    for _ in range(launches):
        tr.fill_raw(0)
        L.check(lib.kw_dgemm_split_trace(tr.data()))
        go()
        q.wait()
        L.check(lib.kw_dgemm_split_trace(None))
        t = tr.download().view(np.uint64).reshape(4096, 40)
        rows = [r for r in t if r[0]]
        t0 = min(int(r[0]) for r in rows)
        busy, end = {}, {}
        for r in rows:
            sm = int(r[1])
            b = 0
            for j in range(18):
                s, e = int(r[2 + 2 * j]), int(r[3 + 2 * j])
                if not s:
                    break
                b += e - s
            busy[sm] = busy.get(sm, 0) + b
            end[sm] = max(end.get(sm, 0), int(r[39]) - t0)
        per.append((busy, end))
    sms = sorted(per[0][0])
    bm = np.array([[p[0][s] for s in sms] for p in per], dtype=float) / 1e3
    em = np.array([[p[1][s] for s in sms] for p in per], dtype=float) / 1e3
    print(f"n={n} cfg={cfg} SMs={len(sms)} launches={launches}")
    for i in range(launches):
        print(f"  launch {i}: busy per SM median {np.median(bm[i]):.1f} us, min {bm[i].min():.1f}, max {bm[i].max():.1f}; "
              f"end median {np.median(em[i]):.1f}, min {em[i].min():.1f}, max {em[i].max():.1f}")
    c = np.corrcoef(bm)
    print("  correlation of per-SM busy time between launches:",
          " ".join(f"{c[i, j]:.2f}" for i in range(launches) for j in range(i + 1, launches)))
    mean = bm.mean(axis=0)
    order = np.argsort(mean)
    print("  slowest SMs (mean busy us):", [(sms[i], round(mean[i], 1)) for i in order[-8:]])
    print("  fastest SMs (mean busy us):", [(sms[i], round(mean[i], 1)) for i in order[:8]])
    # by SM-id parity / TPC / rough GPC (smid // 18) buckets
    ids = np.array(sms)
    for name, key in (("smid % 2", ids % 2), ("smid // 16", ids // 16)):
        groups = {int(k): round(float(mean[key == k].mean()), 1) for k in np.unique(key)}
        print(f"  mean busy by {name}: {groups}")


if __name__ == "__main__":
    main()
