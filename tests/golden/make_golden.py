"""Generates the committed golden fixtures from the REFERENCE library itself
(oracle/_ref/libmatchamg_ref.so, built from /root/reference/proj/src by
oracle/Makefile). Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Outputs (small, committed):
  tests/golden/kats.json        known-answer vectors of the reference's own
                                tests (proj/tests/*.cpp), evaluated by the
                                reference library
  tests/golden/hierarchies.json per-problem hierarchy + PCG fingerprints:
                                level sizes/nnz, sha256 of every level's
                                A/P/R/l1/w arrays, iterations, residual
                                history and solution hashes — including the
                                BASELINE configs 1 and 2 at full size
The GPU tests and the oracle port are checked against these without needing
/root/reference at run time.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Csr, Ref  # noqa: E402

# generator specs (cli::matrix_from_gen_spec grammar, proj/src/cli.cpp:203-240)
PROBLEMS = {
    "poisson2d:64,64": ("poisson2d", (64, 64)),
    "poisson2d:512,512": ("poisson2d", (512, 512)),          # BASELINE cfg 1
    "randk3d:24,24,24,1": ("randk3d", (24, 24, 24, 1.0, 0)),
    "randk3d:32,32,32,0": ("randk3d", (32, 32, 32, 0.0, 0)),
    "ani:96,96,0.01,0.3": ("ani", (96, 96, 1e-2, 0.3)),
    "ani:128,128,0.001,0.7": ("ani", (128, 128, 1e-3, 0.7)),
    "randk3d:160,160,160,0": ("randk3d", (160, 160, 160, 0.0, 0)),  # BASELINE cfg 2
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_hash(A: Csr) -> str:
    h = hashlib.sha256()
    for a in (np.int64(A.nrows), np.int64(A.ncols), A.rp, A.ci, A.v):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def gen(ref, kind, args):
    return {"poisson2d": ref.gen_poisson2d, "randk3d": ref.gen_randk3d,
            "ani": ref.gen_aniso2d}[kind](*args)


def fingerprint(ref, spec, kind, args):
    A = gen(ref, kind, args)
    h = ref.build_hierarchy(A, keep=True)
    b = np.ones(A.nrows)
    u, hist, rep = ref.pcg(A, h, b)
    st = h.stats()
    return {
        "spec": spec, "n": A.nrows, "nnz": A.nnz, "A_sha": csr_hash(A),
        "nl": h.nl, "sizes": st["sizes"], "level_nnz": st["nnz"], "opcx": st["opcx"],
        "cratio": st["cratio"], "stalled": h.stalled, "zero_edges": h.zero_edges,
        "levels": [{"A": csr_hash(L.A), "P": csr_hash(L.P) if L.P is not None else None,
                    "R": csr_hash(L.R) if L.R is not None else None, "l1": sha(L.l1),
                    "w": sha(L.w)} for L in h.levels],
        "pcg": {"iterations": rep["iterations"], "final_relres": rep["final_relres"],
                "final_relres_hex": float(rep["final_relres"]).hex(),
                "hist_sha": sha(hist), "u_sha": sha(u), "audit_checks": rep["audit_checks"],
                "audit_failures": rep["audit_failures"]},
    }


def kats(ref):
    out = {}
    A = ref.from_triplets(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [2.0, -1.0, -1.0, 2.0])
    g = ref.build_weights(A, np.ones(2))
    out["weights_2x2"] = {"xadj": g[0].tolist(), "adjncy": g[1].tolist(), "weight": g[2].tolist(),
                          "zero": g[3]}
    B = ref.from_triplets(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [2.0, 1.0, 1.0, 2.0])
    out["weights_2x2_sign"] = ref.build_weights(B, np.array([1.0, -1.0]))[2].tolist()
    C3 = ref.from_triplets(3, 3, [0, 0, 1, 1, 1, 2, 2], [0, 1, 0, 1, 2, 1, 2],
                           [2.0, -1.0, -1.0, 2.0, -1.0, -1.0, 2.0])
    g = ref.build_weights(C3, np.array([0.0, 0.0, 1.0]))
    out["weights_zero_den"] = {"weight": g[2].tolist(), "zero": g[3]}
    # suitor KATs (test_matching.cpp:89-101, :150-160)
    out["suitor_path"] = ref.suitor(np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]),
                                    np.array([1.0, 1.0, 2.0, 2.0])).tolist()
    out["suitor_edge"] = ref.suitor(np.array([0, 1, 2]), np.array([1, 0]),
                                    np.array([0.7, 0.7])).tolist()
    out["suitor_zero"] = ref.suitor(np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]),
                                    np.array([0.0, 0.0, 1.0, 1.0])).tolist()
    # aggregation traces (test_coarsening.cpp:40-63)
    for name, mate in [("agg_a", [-1, 2, 1, -1]), ("agg_b", [-1, -1, -1]),
                       ("agg_c", [3, 4, 5, 0, 1, 2])]:
        agg, nc, np_, ns = ref.pairwise_aggregate(np.array(mate))
        out[name] = {"agg_of": agg.tolist(), "n_c": nc, "n_p": np_, "n_s": ns}
    P = ref.build_prolongator(np.array([0, 0]), 1, np.array([1.0, 1.0]))
    out["prolongator_pair"] = P.v.tolist()
    out["prolongator_singleton"] = ref.build_prolongator(np.array([0]), 1, np.array([-3.0])).v.tolist()
    out["restrict_pair"] = ref.restrict_vector(P, np.array([1.0, 1.0])).tolist()
    out["galerkin_2x2"] = ref.galerkin_by_aggregates(A, P).v.tolist()
    # l1 (test_sparse_core.cpp:212-230)
    P5 = ref.from_triplets(5, 5, [0, 0, 1, 1, 1, 2, 2, 2, 3, 3, 3, 4, 4],
                           [0, 1, 0, 1, 2, 1, 2, 3, 2, 3, 4, 3, 4],
                           [2, -1, -1, 2, -1, -1, 2, -1, -1, 2, -1, -1, 2.0])
    out["l1_poisson1d"] = ref.l1_diagonal(P5).tolist()
    # fused triple dot (test_krylov.cpp:21-36)
    out["triple_dot"] = list(ref.triple_dot(np.array([1.0, 2, 3]), np.array([2.0, 3, 1]),
                                            np.array([3.0, 4, 2]), np.array([4.0, 5, 3])))
    # smoother hand iteration (test_multigrid.cpp:40-58)
    out["jacobi_hand"] = ref.l1_jacobi(A, np.array([3.0, 3.0]), np.array([1.0, 1.0]),
                                       np.zeros(2), 1).tolist()
    # blocked reductions across the 2048 boundary, seeded inputs
    rng = np.random.default_rng(2048)
    x = rng.uniform(-1, 1, 5000)
    y = rng.uniform(-1, 1, 5000)
    out["dot_5000_hex"] = float(ref.dot(x, y)).hex()
    out["dot_inputs_seed"] = 2048
    return out


def main():
    ref = Ref()
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats(ref), f, indent=1)
    fps = {}
    for spec, (kind, args) in PROBLEMS.items():
        fps[spec] = fingerprint(ref, spec, kind, args)
        print(spec, fps[spec]["nl"], fps[spec]["pcg"]["iterations"], flush=True)
    with open(os.path.join(HERE, "hierarchies.json"), "w") as f:
        json.dump(fps, f, indent=1)


if __name__ == "__main__":
    main()
