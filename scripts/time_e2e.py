"""End-to-end C-ABI host-buffer solve (mamg_solve_host) repetitions with the
phase split reported by the library (upload / setup / solve / download ms)."""
import os, statistics, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_04221_b200 as pkg

spec = os.environ.get("SPEC", "randk3d:160,160,160,0")
reps = int(os.environ.get("REPS", "5"))
A = pkg.from_spec(spec)
dev = pkg.Device(0)
b = np.ones(A.nrows)
u = np.zeros(A.nrows)
tt, ph = [], []
for r in range(reps + 1):
    t0 = time.perf_counter()
    u, hist, rep = dev.solve_host(A, b=b, out=u)
    dt = (time.perf_counter() - t0) * 1e3
    if r:
        tt.append(dt)
        ph.append((rep["upload_ms"], rep["setup_ms"], rep["solve_ms"], rep["download_ms"]))
m = [statistics.median(x) for x in zip(*ph)]
print(f"{spec} {os.environ.get('TAG','')} e2e min {min(tt):.2f} med {statistics.median(tt):.2f} ms | "
      f"upload {m[0]:.2f} setup {m[1]:.2f} solve {m[2]:.2f} download {m[3]:.2f} it {rep['iterations']}")
