"""Profiling driver: one device setup (for ncu launch lists of the setup phase)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_04221_b200 as pkg
A = pkg.from_spec(os.environ.get("SPEC", "randk3d:160,160,160,0"))
dev = pkg.Device(0)
dA = dev.upload(A)
dh = dev.setup(dA)
dev.synchronize()
print("setup done, levels", dh.nl)
