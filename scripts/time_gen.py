"""Generator timing at the BASELINE sizes: host generator (C++, all host
threads; the reference API's CsrMatrix) vs the device generator (matrix
assembled in HBM). usage: python scripts/time_gen.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_04221_b200 as pkg

dev = pkg.Device(0)
for spec in ["poisson2d:512,512", "randk3d:160,160,160,0", "aniso27:128,128,128,0.01",
             "jump3d:200,200,200,8", "elast3d:100,100,100"]:
    t = time.perf_counter()
    A = pkg.from_spec(spec)
    th = time.perf_counter() - t
    del A
    dev.generate(spec)  # warm-up (module load, pool)
    best = 1e9
    for _ in range(3):
        dev.synchronize()
        t = time.perf_counter()
        M = dev.generate(spec)
        dev.synchronize()
        best = min(best, time.perf_counter() - t)
        n, _, nnz = M.shape
        del M
    print(f"{spec:28s} n={n:9d} nnz={nnz:11d}  host {th*1e3:8.1f} ms   device {best*1e3:7.2f} ms")
