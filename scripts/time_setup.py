"""Device-timed setup/solve repetitions (min / median) for A/B checks."""
import os, statistics, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_04221_b200 as pkg

spec = os.environ.get("SPEC", "randk3d:160,160,160,0")
reps = int(os.environ.get("REPS", "10"))
A = pkg.from_spec(spec)
dev = pkg.Device(0)
dA = dev.upload(A)
db = dev.vec(np.ones(A.nrows)); du = dev.zeros(A.nrows)
su, so = [], []
for r in range(reps + 2):
    dev.timer_start(); dh = dev.setup(dA); ts = dev.timer_stop()
    dev.timer_start(); rep = dev.pcg_device(dA, dh, db, du, cycle=os.environ.get('CYCLE', 'V')); tv = dev.timer_stop()
    if r >= 2:
        su.append(ts); so.append(tv)
    del dh
if os.environ.get("ALL"): print("setup", [round(x, 1) for x in su], "solve", [round(x, 1) for x in so])
print(f"{spec} {os.environ.get('TAG','')} setup min {min(su):.2f} med {statistics.median(su):.2f} | "
      f"solve min {min(so):.2f} med {statistics.median(so):.2f} it {rep['iterations']}")
