import sys, time
sys.path.insert(0, '.')
import numpy as np, paper_1810_04221_b200 as pkg
nx = int(sys.argv[1])
dev = pkg.Device(0)
t = time.time(); dA = dev.generate(f"randk3d:{nx},{nx},{nx},0"); dev.synchronize()
print("generated", dA.shape, time.time() - t, flush=True)
t = time.time(); dh = dev.setup(dA); dev.synchronize(); print("setup", time.time() - t, dh.nl, flush=True)
db = dev.vec(np.ones(dA.shape[0])); du = dev.zeros(dA.shape[0])
t = time.time(); rep = dev.pcg_device(dA, dh, db, du); print("solve", time.time() - t, rep["iterations"], rep["final_relres"], flush=True)
