"""Profiling driver: REPS (default 1) device setups (for ncu launch lists of
the setup phase, or MAMG_TRACE=1 phase timings of a warm setup)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_04221_b200 as pkg
A = pkg.from_spec(os.environ.get("SPEC", "randk3d:160,160,160,0"))
dev = pkg.Device(0)
dA = dev.upload(A)
for r in range(int(os.environ.get("REPS", "1"))):
    if r:
        print(f"---- setup {r}", file=sys.stderr, flush=True)
    dh = dev.setup(dA)
    dev.synchronize()
    del dh
print("setup done")
