import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
r = O.Ref()
A = r.gen_randk3d(160, 160, 160, 0.0, 0)
h = r.build_hierarchy(A)
L = h.levels[-1]
with open('/tmp/coarsest.bin', 'wb') as f:
    np.array([L.A.nrows, L.A.nnz], np.int64).tofile(f)
    np.asarray(L.A.rp, np.int32).tofile(f)
    np.asarray(L.A.ci, np.int32).tofile(f)
    np.asarray(L.A.v, np.float64).tofile(f)
    np.asarray(L.l1, np.float64).tofile(f)
print(L.A.nrows, L.A.nnz)
