"""Device-timed V-cycle (time_precond) and PCG solve repetitions (A/B of solve-path changes)."""
import os, statistics, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_04221_b200 as pkg

spec = os.environ.get("SPEC", "randk3d:160,160,160,0")
A = pkg.from_spec(spec)
dev = pkg.Device(0)
dA = dev.upload(A)
dh = dev.setup(dA)
db = dev.vec(np.ones(A.nrows)); du = dev.zeros(A.nrows)
vc = [dev.time_precond(dh, reps=20) for _ in range(5)]
so = []
for r in range(6):
    dev.timer_start(); rep = dev.pcg_device(dA, dh, db, du); t = dev.timer_stop()
    if r: so.append(t)
print(f"{spec} {os.environ.get('TAG','')} vcycle min {min(vc)*1e3:.1f} med {statistics.median(vc)*1e3:.1f} us | "
      f"solve min {min(so):.2f} med {statistics.median(so):.2f} ms it {rep['iterations']}")
