"""Small end-to-end exercise of the device paths for compute-sanitizer:
device generators, setup + PCG (look-back scans), partitioned solves with
peer halos / reductions / overlap (loopback, 3 parts), global matching."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MAMG_DIST_OVERLAP", "1")
import paper_1810_04221_b200 as pkg

dev = pkg.Device(0)
for spec in ["randk3d:10,9,8,1", "aniso27:6,6,6,0.01", "elast3d:3,4,3", "jump3d:9,9,9,4",
             "poisson2d:40,30"]:
    dev.generate(spec)
A = pkg.from_spec("randk3d:24,24,24,1")
u, h, r = dev.solve_host(A)
print("single", r["iterations"])
for matching in ("local", "global"):
    d = pkg.Dist(dev, 3, matching=matching, agglomerate=2000).setup(A)
    ud, hd, rd = d.pcg()
    print(matching, rd["iterations"], bool(np.array_equal(ud.view(np.int64), u.view(np.int64))))
