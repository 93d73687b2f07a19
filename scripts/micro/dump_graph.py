"""Dump the level-0 weighted graph of a randk3d:nx^3 problem (reference
build_weights) for scripts/micro/suitor_rounds.c: python dump_graph.py nx out.bin"""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from oracle import oracle as O
nx, out = int(sys.argv[1]), sys.argv[2]
r = O.Ref()
A = r.gen_randk3d(nx, nx, nx, 0.0, 0)
xadj, adj, wt, z = r.build_weights(A, np.ones(A.nrows))
with open(out, "wb") as f:
    np.array([A.nrows, len(adj)], np.int64).tofile(f)
    np.asarray(xadj, np.int64).tofile(f)
    np.asarray(adj, np.int32).tofile(f)
    np.asarray(wt, np.float64).tofile(f)
