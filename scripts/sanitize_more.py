"""More compute-sanitizer coverage: W / K cycles, Pairwise mode, the opt-in
one-launch coarsest and tail kernels, NCCL world=1 with the peer paths."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_04221_b200 as pkg

dev = pkg.Device(0)
A = pkg.from_spec("randk3d:20,20,20,1")
for cycle in (0, 1, 2):
    u, h, r = dev.solve_host(A, cycle=cycle)
    print("cycle", cycle, r["iterations"])
u, h, r = dev.solve_host(A, mode=1)
print("pairwise", r["iterations"])
B = pkg.from_spec("elast3d:4,5,4")
u, h, r = dev.solve_host(B)
print("elast", r["iterations"])
d = pkg.Dist(dev, 1, 0, pkg.nccl_unique_id(), matching="global", agglomerate=4000).setup(A)
ud, hd, rd = d.pcg()
print("nccl1", rd["iterations"])
