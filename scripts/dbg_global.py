"""Debug helper: one global-matching partitioned solve (argv: parts, case)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1810_04221_b200 as pkg

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 8
case = sys.argv[2] if len(sys.argv) > 2 else "aniso"
if case == "aniso":
    A = pkg.gen_anisotropic_3d_q1(16, 16, 16, 1.0, 1.0, 1e-2)
elif case == "elast":
    A = pkg.gen_elasticity_3d(6, 6, 6)
else:
    A = pkg.gen_poisson_2d(96, 96)
dev = pkg.Device(0)
d = pkg.Dist(dev, parts, matching="global").setup(A)
print("info", d.info(), [d.bounds(k) for k in range(d.info()["nl"])])
try:
    u, h, r = d.pcg(itmax=3)
    print("pcg", r["iterations"], h)
except Exception as e:
    print("ERR", e)
