"""Profiling driver (run under ncu via gpurun): one setup + timed kernels or one solve."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_04221_b200 as pkg

mode = sys.argv[1] if len(sys.argv) > 1 else "kernels"
A = pkg.from_spec(os.environ.get("SPEC", "randk3d:160,160,160,0"))
dev = pkg.Device(0)
dA = dev.upload(A)
dh = dev.setup(dA)
if mode == "kernels":
    print("smoother ms", dev.time_smoother(dh, 0, reps=3))
    print("spmv ms", dev.time_spmv(dh, 0, reps=3))
    print("precond ms", dev.time_precond(dh, reps=2))
else:  # one full solve
    db = dev.vec(np.ones(A.nrows)); du = dev.zeros(A.nrows)
    print(dev.pcg_device(dA, dh, db, du))
