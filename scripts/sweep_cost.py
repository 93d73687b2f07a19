"""Cost of one coarse-level kernel inside the replayed PCG graph: time per PCG
iteration with the coarsest sweep count k (each extra sweep = one more
latency-bound SpMV launch on the 4k-row coarsest level), fixed itmax so the
iteration count is the same. usage: python scripts/sweep_cost.py [spec]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_04221_b200 as pkg

A = pkg.from_spec(sys.argv[1] if len(sys.argv) > 1 else "randk3d:160,160,160,0")
dev = pkg.Device(0)
dA = dev.upload(A)
dh = dev.setup(dA)
db = dev.vec(np.ones(A.nrows))
du = dev.zeros(A.nrows)
res = {}
for rep in range(2):
    for k in (1, 20, 60, 100):
        dev.synchronize()
        dev.timer_start()
        r = dev.pcg_device(dA, dh, db, du, rtol=1e-30, itmax=40, coarsest=k)
        t = dev.timer_stop()
        res[k] = t / r["iterations"]
for k in sorted(res):
    print(f"coarsest sweeps {k:4d}: {res[k]*1e3:8.1f} us / iteration")
print(f"per extra coarsest sweep: {(res[100]-res[20])/80*1e3:.2f} us")
for pre, post in ((0, 1), (1, 1), (2, 2)):
    dev.timer_start()
    r = dev.pcg_device(dA, dh, db, du, rtol=1e-30, itmax=40, pre=pre, post=post)
    print(f"pre/post {pre}/{post}: {dev.timer_stop()/r['iterations']*1e3:8.1f} us / iteration")
