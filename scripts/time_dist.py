"""Partitioned path on ONE GPU: build + PCG times of the loopback transport at
P parts (all parts in this process) and of the NCCL transport at world = 1,
for local and global matching. Diagnostic (not the bench): it shows the
algorithmic cost of partitioning, without interconnect time.

usage: python scripts/time_dist.py [spec] [reps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_04221_b200 as pkg  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "randk3d:160,160,160,0"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
A = pkg.from_spec(spec)
dev = pkg.Device(0)


def timed(D):
    out = []
    for r in range(reps + 1):
        dev.synchronize()
        dev.timer_start()
        D.build()
        ts = dev.timer_stop()
        dev.timer_start()
        _, _, rep = D.pcg(want_u=False)
        tv = dev.timer_stop()
        if r:
            out.append((ts, tv, rep["iterations"]))
    a = np.array(out)
    return float(np.median(a[:, 0])), float(np.median(a[:, 1])), int(a[0, 2])


rows = []
uid = pkg.nccl_unique_id()
for matching in ("local", "global"):
    D = pkg.Dist(dev, 1, 0, uid if matching == "local" else pkg.nccl_unique_id(),
                 matching=matching).load(A)
    rows.append(("nccl world=1", matching, *timed(D)))
    del D
    for P in (2, 4, 8):
        D = pkg.Dist(dev, P, matching=matching).load(A)
        rows.append((f"loopback P={P}", matching, *timed(D)))
        del D
print(f"{spec}: n={A.nrows} nnz={A.nnz}")
print(f"{'transport':16s} {'matching':8s} {'setup ms':>9s} {'solve ms':>9s} {'it':>4s} {'ms/it':>7s}")
for t, m, ts, tv, it in rows:
    print(f"{t:16s} {m:8s} {ts:9.2f} {tv:9.2f} {it:4d} {tv / max(it, 1):7.3f}")
