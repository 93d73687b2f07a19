"""ctypes bindings for the two CPU CHECKERS — test infrastructure only.

* ``Ref``  — the unmodified reference library (oracle/_ref/libmatchamg_ref.so,
  built from /root/reference/proj/src by oracle/Makefile, called through
  oracle/ref_shim.cpp).
* ``Port`` — the plain-C restatement (oracle/build/libmamg_oracle.so,
  oracle/matchamg_oracle.c).

Both expose the same Python surface so parity tests can run against either.
Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmatchamg_ref.so")
PORT_SO = os.path.join(HERE, "build", "libmamg_oracle.so")

I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
VP = C.c_void_p


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(I64P)


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(F64P)


@dataclass
class Csr:
    """Host CSR in the reference's API layout (int64 indices, fp64 values)."""

    nrows: int
    ncols: int
    rp: np.ndarray
    ci: np.ndarray
    v: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rp[-1])

    def same(self, other: "Csr") -> bool:
        """Bitwise equality of shape, pattern and values."""
        return (self.nrows == other.nrows and self.ncols == other.ncols
                and np.array_equal(self.rp, other.rp)
                and np.array_equal(self.ci, other.ci)
                and np.array_equal(self.v.view(np.int64), other.v.view(np.int64)))

    def to_dense(self) -> np.ndarray:
        D = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            for k in range(self.rp[i], self.rp[i + 1]):
                D[i, self.ci[k]] += self.v[k]
        return D


class OracleError(Exception):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("final_relres", C.c_double),
                ("converged", C.c_int32), ("pad", C.c_int32),
                ("solve_ms", C.c_double), ("audit_checks", C.c_int64),
                ("audit_failures", C.c_int64), ("audit_max_rel", C.c_double),
                ("breakdown_iteration", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "pad"}


@dataclass
class Level:
    A: Csr
    P: Csr | None
    R: Csr | None
    l1: np.ndarray
    w: np.ndarray


@dataclass
class Hierarchy:
    levels: list
    stalled: bool
    zero_edges: int
    handle: object = None  # keeps the native hierarchy alive (for cycles/pcg)

    @property
    def nl(self):
        return len(self.levels)

    def stats(self):
        nnz = [lv.A.nnz for lv in self.levels]
        opcx = float(np.sum(np.array(nnz, dtype=np.float64))) / float(nnz[0])
        r = 0.0
        for k in range(1, self.nl):
            r += float(self.levels[k - 1].A.nrows) / float(self.levels[k].A.nrows)
        return {"nl": self.nl, "opcx": opcx, "cratio": r / self.nl,
                "sizes": [lv.A.nrows for lv in self.levels], "nnz": nnz}


# ------------------------------------------------------------------------------
class Ref:
    """The reference library itself (oracle/_ref)."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        L = self.L = C.CDLL(path)
        L.mref_last_error.restype = C.c_char_p
        for name in ("mref_csr_from_arrays", "mref_csr_from_triplets", "mref_gen_poisson2d",
                     "mref_gen_aniso2d", "mref_gen_randk3d", "mref_hier_A", "mref_hier_P",
                     "mref_hier_R", "mref_step_P", "mref_step_Ac"):
            getattr(L, name).restype = VP
        L.mref_csr_from_arrays.argtypes = [C.c_int64, C.c_int64, I64P, I64P, F64P]
        L.mref_csr_from_triplets.argtypes = [C.c_int64, C.c_int64, C.c_int64, I64P, I64P, F64P]
        L.mref_gen_poisson2d.argtypes = [C.c_int64, C.c_int64]
        L.mref_gen_aniso2d.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double]
        L.mref_gen_randk3d.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_uint64]
        L.mref_csr_free.argtypes = [VP]
        L.mref_csr_shape.argtypes = [VP, I64P, I64P, I64P]
        L.mref_csr_export.argtypes = [VP, I64P, I64P, F64P]
        L.mref_hier_A.argtypes = L.mref_hier_P.argtypes = L.mref_hier_R.argtypes = [VP, C.c_int]
        L.mref_hier_l1.argtypes = L.mref_hier_w.argtypes = [VP, C.c_int, F64P]
        L.mref_hier_free.argtypes = [VP]
        L.mref_hier_nl.argtypes = [VP]
        L.mref_hier_stats.argtypes = [VP, C.POINTER(C.c_int32), I64P, F64P, F64P]
        L.mref_step_P.argtypes = L.mref_step_Ac.argtypes = [VP]
        L.mref_step_wc.argtypes = [VP, F64P]
        L.mref_step_zero_edges.argtypes = [VP]
        L.mref_step_zero_edges.restype = C.c_int64
        L.mref_step_free.argtypes = [VP]
        L.mref_run_solve.argtypes = [VP, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_int, C.c_double, C.c_int64, F64P, F64P, F64P,
                                     I64P, F64P, C.POINTER(C.c_int), F64P]
        L.mref_dot.restype = L.mref_norm2.restype = C.c_double
        L.mref_matching_weight.restype = C.c_double

    # --- plumbing ---
    def _err(self, st):
        if st:
            raise OracleError(st, self.L.mref_last_error().decode())

    def _wrap(self, A: Csr):
        rp, prp = _i64(A.rp)
        ci, pci = _i64(A.ci)
        v, pv = _f64(A.v)
        h = self.L.mref_csr_from_arrays(A.nrows, A.ncols, prp, pci, pv)
        return h

    def _export(self, h, free=False) -> Csr:
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        self.L.mref_csr_shape(VP(h), C.byref(nr), C.byref(nc), C.byref(nz))
        rp = np.zeros(nr.value + 1, np.int64)
        ci = np.zeros(nz.value, np.int64)
        v = np.zeros(nz.value, np.float64)
        self.L.mref_csr_export(VP(h), rp.ctypes.data_as(I64P), ci.ctypes.data_as(I64P),
                               v.ctypes.data_as(F64P))
        if free:
            self.L.mref_csr_free(VP(h))
        return Csr(nr.value, nc.value, rp, ci, v)

    def set_threads(self, t: int):
        self.L.mref_set_threads(int(t))

    # --- cli::run_solve on a reference-held matrix (bench.py reference arm) ---
    def gen_handle(self, kind, *args):
        """A matrix made by the reference's own generator (src/problems.cpp),
        kept inside the reference (no export): kind = poisson2d | randk3d."""
        if kind == "poisson2d":
            h = self.L.mref_gen_poisson2d(*[int(a) for a in args])
        elif kind == "randk3d":
            nx, ny, nz, sigma, seed = args
            h = self.L.mref_gen_randk3d(int(nx), int(ny), int(nz), float(sigma), int(seed))
        else:
            raise ValueError(kind)
        if not h:
            raise OracleError(1, self.L.mref_last_error().decode())
        return RefMatrix(self, h)

    def wrap(self, A: Csr):
        """Copy a host Csr into the reference (outside any timed region)."""
        return RefMatrix(self, self._wrap(A))

    def run_solve(self, M, threads, max_levels=40, coarse_factor=40.0, mode=2, cycle=0, pre=1,
                  post=1, coarsest=20, rtol=1e-6, itmax=5000, want_u=False):
        """cli::run_solve (proj/src/cli.cpp:242-328): setup_ms = wall time of
        build_hierarchy, solve_ms = SolveReport::solve_ms."""
        sm, vm, wm, rr = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        it, nl = C.c_int64(), C.c_int()
        u = np.zeros(M.nrows) if want_u else None
        self._err(self.L.mref_run_solve(
            VP(M.h), int(threads), int(max_levels), C.c_double(coarse_factor), int(mode),
            int(cycle), int(pre), int(post), int(coarsest), C.c_double(rtol), C.c_int64(itmax),
            C.byref(sm), C.byref(vm), C.byref(wm), C.byref(it), C.byref(rr), C.byref(nl),
            u.ctypes.data_as(F64P) if want_u else None))
        return {"setup_ms": sm.value, "solve_ms": vm.value, "wall_ms": wm.value,
                "iterations": it.value, "final_relres": rr.value, "nl": nl.value, "u": u}

    def max_threads(self) -> int:
        return int(self.L.mref_max_threads())

    # --- generators (src/problems.cpp) ---
    def gen_poisson2d(self, nx, ny) -> Csr:
        h = self.L.mref_gen_poisson2d(nx, ny)
        if not h:
            raise OracleError(1, self.L.mref_last_error().decode())
        return self._export(h, free=True)

    def gen_aniso2d(self, nx, ny, eps, theta) -> Csr:
        h = self.L.mref_gen_aniso2d(nx, ny, eps, theta)
        if not h:
            raise OracleError(1, self.L.mref_last_error().decode())
        return self._export(h, free=True)

    def gen_randk3d(self, nx, ny, nz, sigma, seed=0) -> Csr:
        h = self.L.mref_gen_randk3d(nx, ny, nz, sigma, seed)
        if not h:
            raise OracleError(1, self.L.mref_last_error().decode())
        return self._export(h, free=True)

    def read_mm(self, path) -> Csr:
        self.L.mref_read_mm.restype = VP
        self.L.mref_read_mm.argtypes = [C.c_char_p]
        h = self.L.mref_read_mm(os.fsencode(path))
        if not h:
            raise OracleError(2, self.L.mref_last_error().decode())
        return self._export(h, free=True)

    def write_mm(self, A: Csr, path, symmetric=False):
        self.L.mref_write_mm.argtypes = [VP, C.c_char_p, C.c_int]
        h = self._wrap(A)
        try:
            self._err(self.L.mref_write_mm(VP(h), os.fsencode(path), 1 if symmetric else 0))
        finally:
            self.L.mref_csr_free(VP(h))

    def from_triplets(self, nrows, ncols, rows, cols, vals) -> Csr:
        r, pr = _i64(rows)
        c, pc = _i64(cols)
        v, pv = _f64(vals)
        h = self.L.mref_csr_from_triplets(nrows, ncols, len(r), pr, pc, pv)
        if not h:
            raise OracleError(1, self.L.mref_last_error().decode())
        return self._export(h, free=True)

    # --- kernels ---
    def lane_policy(self, A: Csr) -> int:
        h = self._wrap(A)
        try:
            return int(self.L.mref_lane_policy(VP(h)))
        finally:
            self.L.mref_csr_free(VP(h))

    def spmv(self, A: Csr, x, group=0):
        h = self._wrap(A)
        x, px = _f64(x)
        y = np.zeros(A.nrows)
        try:
            self._err(self.L.mref_spmv(VP(h), int(group), px, y.ctypes.data_as(F64P)))
        finally:
            self.L.mref_csr_free(VP(h))
        return y

    def l1_diagonal(self, A: Csr):
        h = self._wrap(A)
        d = np.zeros(A.nrows)
        try:
            self._err(self.L.mref_l1_diagonal(VP(h), d.ctypes.data_as(F64P)))
        finally:
            self.L.mref_csr_free(VP(h))
        return d

    def has_symmetric_pattern(self, A: Csr) -> bool:
        h = self._wrap(A)
        try:
            return bool(self.L.mref_has_symmetric_pattern(VP(h)))
        finally:
            self.L.mref_csr_free(VP(h))

    def _binop(self, fn, A: Csr, B: Csr | None = None) -> Csr:
        ha = self._wrap(A)
        hb = self._wrap(B) if B is not None else None
        out = VP()
        try:
            st = fn(VP(ha), VP(hb), C.byref(out)) if B is not None else fn(VP(ha), C.byref(out))
            self._err(st)
            return self._export(out.value, free=True)
        finally:
            self.L.mref_csr_free(VP(ha))
            if hb:
                self.L.mref_csr_free(VP(hb))

    def transpose(self, A):
        return self._binop(self.L.mref_transpose, A)

    def spgemm(self, A, B):
        return self._binop(self.L.mref_spgemm, A, B)

    def galerkin_triple(self, A, P):
        return self._binop(self.L.mref_galerkin_triple, A, P)

    def galerkin_by_aggregates(self, A, P):
        return self._binop(self.L.mref_galerkin_by_aggregates, A, P)

    # --- matching ---
    def build_weights(self, A: Csr, w):
        h = self._wrap(A)
        w, pw = _f64(w)
        xadj = np.zeros(A.nrows + 1, np.int64)
        adj = np.zeros(max(A.nnz, 1), np.int64)
        wt = np.zeros(max(A.nnz, 1), np.float64)
        z = C.c_int64()
        try:
            self._err(self.L.mref_build_weights(VP(h), pw, xadj.ctypes.data_as(I64P),
                                                adj.ctypes.data_as(I64P),
                                                wt.ctypes.data_as(F64P), C.byref(z)))
        finally:
            self.L.mref_csr_free(VP(h))
        m = int(xadj[-1])
        return xadj, adj[:m].copy(), wt[:m].copy(), int(z.value)

    def suitor(self, xadj, adjncy, weight):
        n = len(xadj) - 1
        xadj, px = _i64(xadj)
        adjncy, pa = _i64(adjncy if len(adjncy) else np.zeros(1, np.int64))
        weight, pw = _f64(weight if len(weight) else np.zeros(1))
        mate = np.zeros(max(n, 1), np.int64)
        self._err(self.L.mref_suitor(n, px, pa, pw, mate.ctypes.data_as(I64P)))
        return mate[:n]

    def exact_match(self, xadj, adjncy, weight):
        n = len(xadj) - 1
        xadj, px = _i64(xadj)
        adjncy, pa = _i64(adjncy if len(adjncy) else np.zeros(1, np.int64))
        weight, pw = _f64(weight if len(weight) else np.zeros(1))
        mate = np.zeros(max(n, 1), np.int64)
        self._err(self.L.mref_exact_match(n, px, pa, pw, mate.ctypes.data_as(I64P)))
        return mate[:n]

    def matching_weight(self, xadj, adjncy, weight, mate):
        n = len(xadj) - 1
        xadj, px = _i64(xadj)
        adjncy, pa = _i64(adjncy if len(adjncy) else np.zeros(1, np.int64))
        weight, pw = _f64(weight if len(weight) else np.zeros(1))
        mate, pm = _i64(mate)
        return float(self.L.mref_matching_weight(n, px, pa, pw, pm))

    # --- coarsening ---
    def pairwise_aggregate(self, mate):
        n = len(mate)
        mate, pm = _i64(mate)
        agg = np.zeros(max(n, 1), np.int64)
        cnt = np.zeros(3, np.int64)
        self._err(self.L.mref_pairwise_aggregate(n, pm, agg.ctypes.data_as(I64P),
                                                 cnt.ctypes.data_as(I64P)))
        return agg[:n], int(cnt[0]), int(cnt[1]), int(cnt[2])

    def build_prolongator(self, agg, n_c, w) -> Csr:
        n = len(agg)
        agg, pa = _i64(agg)
        w, pw = _f64(w)
        out = VP()
        self._err(self.L.mref_build_prolongator(n, n_c, pa, pw, C.byref(out)))
        return self._export(out.value, free=True)

    def restrict_vector(self, P: Csr, w):
        h = self._wrap(P)
        w, pw = _f64(w)
        wc = np.zeros(P.ncols)
        try:
            self._err(self.L.mref_restrict_vector(VP(h), pw, wc.ctypes.data_as(F64P)))
        finally:
            self.L.mref_csr_free(VP(h))
        return wc

    def coarsen_step(self, A: Csr, w, mode=1):
        h = self._wrap(A)
        w, pw = _f64(w)
        out = VP()
        try:
            self._err(self.L.mref_coarsen_step(VP(h), pw, int(mode), C.byref(out)))
        finally:
            self.L.mref_csr_free(VP(h))
        P = self._export(self.L.mref_step_P(out))
        Ac = self._export(self.L.mref_step_Ac(out))
        wc = np.zeros(Ac.nrows)
        self.L.mref_step_wc(out, wc.ctypes.data_as(F64P))
        z = int(self.L.mref_step_zero_edges(out))
        self.L.mref_step_free(out)
        return P, Ac, wc, z

    def build_hierarchy(self, A: Csr, w=None, max_levels=40, coarse_factor=40.0,
                        mode=2, keep=False, timing=False):
        h = self._wrap(A)
        pw = None
        if w is not None:
            w, pw = _f64(w)
        out = VP()
        ms = C.c_double()
        try:
            self._err(self.L.mref_build_hierarchy(VP(h), pw, int(max_levels),
                                                  C.c_double(coarse_factor), int(mode),
                                                  C.byref(out), C.byref(ms)))
        finally:
            self.L.mref_csr_free(VP(h))
        hier = self._materialize(out) if not timing else None
        if timing:
            return _RefHierHandle(self, out.value), ms.value
        if keep:
            hier.handle = _RefHierHandle(self, out.value)
        else:
            self.L.mref_hier_free(out)
        return hier

    def hier_from_levels(self, levels):
        """Native reference Hierarchy assembled from given levels (for cycles/pcg)."""
        nl = len(levels)
        hs = [self._wrap(L.A) for L in levels]
        ps = [self._wrap(L.P) if L.P is not None else None for L in levels]
        rs = [self._wrap(L.R) if L.R is not None else None for L in levels]
        keep = [(np.ascontiguousarray(L.l1, np.float64), np.ascontiguousarray(L.w, np.float64))
                for L in levels]
        A_arr = (VP * nl)(*hs)
        P_arr = (VP * nl)(*ps)
        R_arr = (VP * nl)(*rs)
        l1_arr = (F64P * nl)(*[k[0].ctypes.data_as(F64P) for k in keep])
        w_arr = (F64P * nl)(*[k[1].ctypes.data_as(F64P) for k in keep])
        out = VP()
        try:
            self._err(self.L.mref_hier_from_levels(nl, A_arr, P_arr, R_arr, l1_arr, w_arr,
                                                   C.byref(out)))
        finally:
            for h in hs + [p for p in ps if p] + [r for r in rs if r]:
                self.L.mref_csr_free(VP(h))
        return _RefHierHandle(self, out.value)

    def _materialize(self, hh):
        nl = self.L.mref_hier_nl(hh)
        levels = []
        for k in range(nl):
            A = self._export(self.L.mref_hier_A(hh, k))
            P = R = None
            if k + 1 < nl:
                P = self._export(self.L.mref_hier_P(hh, k))
                R = self._export(self.L.mref_hier_R(hh, k))
            l1 = np.zeros(A.nrows)
            w = np.zeros(A.nrows)
            self.L.mref_hier_l1(hh, k, l1.ctypes.data_as(F64P))
            self.L.mref_hier_w(hh, k, w.ctypes.data_as(F64P))
            levels.append(Level(A, P, R, l1, w))
        st = C.c_int32()
        z = C.c_int64()
        a, b = C.c_double(), C.c_double()
        self.L.mref_hier_stats(hh, C.byref(st), C.byref(z), C.byref(a), C.byref(b))
        return Hierarchy(levels, bool(st.value), int(z.value))

    # --- multigrid / krylov ---
    def l1_jacobi(self, A: Csr, d, b, x, k):
        h = self._wrap(A)
        d, pd = _f64(d)
        b, pb = _f64(b)
        x = np.array(x, dtype=np.float64)
        try:
            self._err(self.L.mref_l1_jacobi(VP(h), pd, pb, x.ctypes.data_as(F64P), int(k)))
        finally:
            self.L.mref_csr_free(VP(h))
        return x

    def apply_cycle(self, hier: Hierarchy, level, b, x, cycle=0, pre=1, post=1, coarsest=20):
        b, pb = _f64(b)
        x = np.array(x, dtype=np.float64)
        self._err(self.L.mref_apply_cycle(VP(hier.handle.ptr), int(level), pb,
                                          x.ctypes.data_as(F64P), cycle, pre, post, coarsest))
        return x

    def pcg(self, A: Csr, hier: Hierarchy | None, b, u0=None, rtol=1e-6, itmax=5000,
            cycle=0, pre=1, post=1, coarsest=20):
        h = self._wrap(A)
        b, pb = _f64(b)
        pu0 = None
        if u0 is not None:
            u0, pu0 = _f64(u0)
        u = np.zeros(A.nrows)
        hist = np.zeros(itmax + 2)
        rep = _Report()
        hh = VP(hier.handle.ptr) if hier is not None else None
        try:
            st = self.L.mref_pcg(VP(h), hh, cycle, pre, post, coarsest, pb, pu0,
                                 C.c_double(rtol), C.c_int64(itmax), u.ctypes.data_as(F64P),
                                 hist.ctypes.data_as(F64P), C.byref(rep))
        finally:
            self.L.mref_csr_free(VP(h))
        if st:
            raise OracleError(st, self.L.mref_last_error().decode())
        r = rep.as_dict()
        return u, hist[: r["iterations"] + 1].copy(), r

    # --- vector ops ---
    def dot(self, x, y):
        x, px = _f64(x)
        y, py = _f64(y)
        return float(self.L.mref_dot(len(x), px, py))

    def norm2(self, x):
        x, px = _f64(x)
        return float(self.L.mref_norm2(len(x), px))

    def triple_dot(self, w, r, v, q):
        arrs = [_f64(a) for a in (w, r, v, q)]
        out = np.zeros(3)
        self.L.mref_triple_dot(len(w), *[p for _, p in arrs], out.ctypes.data_as(F64P))
        return tuple(out)

    def axpy_pair(self, y1, y2, x, a, b):
        y1 = np.array(y1, dtype=np.float64)
        y2 = np.array(y2, dtype=np.float64)
        x, px = _f64(x)
        self.L.mref_axpy_pair(len(y1), y1.ctypes.data_as(F64P), y2.ctypes.data_as(F64P), px,
                              C.c_double(a), C.c_double(b))
        return y1, y2


class RefMatrix:
    """A CsrMatrix owned by the reference library (freed with it)."""

    def __init__(self, owner, h):
        self.owner, self.h = owner, h
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        owner.L.mref_csr_shape(VP(h), C.byref(nr), C.byref(nc), C.byref(nz))
        self.nrows, self.ncols, self.nnz = nr.value, nc.value, nz.value

    def export(self) -> Csr:
        return self.owner._export(self.h)

    def __del__(self):
        try:
            self.owner.L.mref_csr_free(VP(self.h))
        except Exception:
            pass


class _RefHierHandle:
    def __init__(self, owner, ptr):
        self.owner, self.ptr = owner, ptr

    def __del__(self):
        try:
            self.owner.L.mref_hier_free(self.ptr)
        except Exception:
            pass


# ------------------------------------------------------------------------------
class _OrcCsr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("rp", I64P), ("ci", I64P),
                ("v", F64P)]


class _OrcLevel(C.Structure):
    _fields_ = [("A", C.POINTER(_OrcCsr)), ("P", C.POINTER(_OrcCsr)),
                ("R", C.POINTER(_OrcCsr)), ("l1", F64P), ("w", F64P)]


class _OrcHier(C.Structure):
    _fields_ = [("nl", C.c_int), ("lv", C.POINTER(_OrcLevel)), ("stalled", C.c_int),
                ("zero_edges", C.c_int64)]


ORC_ERR = {1: "non-positive diagonal", 2: "pattern not symmetric", 3: "non-finite weight",
           4: "zero or missing diagonal entry", 5: "smooth vector vanishes on aggregate",
           6: "matrix pattern is not symmetric", 7: "invalid configuration"}


class Port:
    """The C restatement (oracle/matchamg_oracle.c)."""

    kind = "port"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle port`")
        L = self.L = C.CDLL(path)
        CP = C.POINTER(_OrcCsr)
        L.orc_csr_copy_from.restype = CP
        L.orc_csr_copy_from.argtypes = [C.c_int64, C.c_int64, I64P, I64P, F64P]
        L.orc_csr_free.argtypes = [CP]
        for f in ("orc_transpose", "orc_galerkin_by_aggregates"):
            getattr(L, f).restype = CP
        L.orc_transpose.argtypes = [CP]
        L.orc_spgemm.restype = CP
        L.orc_spgemm.argtypes = [CP, CP]
        L.orc_galerkin_by_aggregates.argtypes = [CP, CP]
        L.orc_lane_policy.argtypes = [CP]
        L.orc_spmv.argtypes = [CP, C.c_int, F64P, F64P]
        L.orc_l1_diagonal.argtypes = [CP, F64P]
        L.orc_l1_diagonal.restype = C.c_int64
        L.orc_has_symmetric_pattern.argtypes = [CP]
        L.orc_build_weights.argtypes = [CP, F64P, I64P, I64P, F64P, I64P, I64P]
        L.orc_suitor.argtypes = [C.c_int64, I64P, I64P, F64P, I64P]
        L.orc_pairwise_aggregate.argtypes = [C.c_int64, I64P, I64P, I64P]
        L.orc_build_prolongator.argtypes = [C.c_int64, C.c_int64, I64P, F64P, C.POINTER(CP), I64P]
        L.orc_restrict_vector.argtypes = [CP, F64P, F64P]
        HP = C.POINTER(_OrcHier)
        L.orc_build_hierarchy.argtypes = [CP, F64P, C.c_int, C.c_double, C.c_int,
                                          C.POINTER(HP), I64P]
        L.orc_hier_free.argtypes = [HP]
        L.orc_l1_jacobi.argtypes = [CP, F64P, F64P, F64P, C.c_int]
        L.orc_apply_cycle.argtypes = [HP, C.c_int, F64P, F64P, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_dot.restype = L.orc_norm2.restype = C.c_double
        L.orc_dot.argtypes = [C.c_int64, F64P, F64P]
        L.orc_norm2.argtypes = [C.c_int64, F64P]
        L.orc_triple_dot.argtypes = [C.c_int64, F64P, F64P, F64P, F64P, F64P]
        L.orc_axpy_pair.argtypes = [C.c_int64, F64P, F64P, F64P, C.c_double, C.c_double]
        L.orc_pcg.argtypes = [CP, HP, C.c_int, C.c_int, C.c_int, C.c_int, F64P, F64P,
                              C.c_double, C.c_int64, F64P, F64P, C.POINTER(_Report)]

    def _wrap(self, A: Csr):
        rp, prp = _i64(A.rp)
        ci, pci = _i64(A.ci if len(A.ci) else np.zeros(1, np.int64))
        v, pv = _f64(A.v if len(A.v) else np.zeros(1))
        return self.L.orc_csr_copy_from(A.nrows, A.ncols, prp, pci, pv)

    @staticmethod
    def _read(p) -> Csr:
        s = p.contents
        nr = s.nrows
        rp = np.ctypeslib.as_array(s.rp, shape=(nr + 1,)).copy()
        nz = int(rp[-1])
        ci = np.ctypeslib.as_array(s.ci, shape=(max(nz, 1),))[:nz].copy()
        v = np.ctypeslib.as_array(s.v, shape=(max(nz, 1),))[:nz].copy()
        return Csr(nr, s.ncols, rp, ci, v)

    def _export(self, p) -> Csr:
        A = self._read(p)
        self.L.orc_csr_free(p)
        return A

    def lane_policy(self, A):
        p = self._wrap(A)
        try:
            return int(self.L.orc_lane_policy(p))
        finally:
            self.L.orc_csr_free(p)

    def spmv(self, A, x, group=0):
        p = self._wrap(A)
        g = group if group > 0 else self.L.orc_lane_policy(p)
        x, px = _f64(x)
        y = np.zeros(A.nrows)
        self.L.orc_spmv(p, g, px, y.ctypes.data_as(F64P))
        self.L.orc_csr_free(p)
        return y

    def l1_diagonal(self, A):
        p = self._wrap(A)
        d = np.zeros(A.nrows)
        bad = self.L.orc_l1_diagonal(p, d.ctypes.data_as(F64P))
        self.L.orc_csr_free(p)
        if bad >= 0:
            raise OracleError(1, f"l1_diagonal: zero or missing diagonal entry in row {bad}")
        return d

    def has_symmetric_pattern(self, A):
        p = self._wrap(A)
        try:
            return bool(self.L.orc_has_symmetric_pattern(p))
        finally:
            self.L.orc_csr_free(p)

    def transpose(self, A):
        p = self._wrap(A)
        out = self._export(self.L.orc_transpose(p))
        self.L.orc_csr_free(p)
        return out

    def spgemm(self, A, B):
        pa, pb = self._wrap(A), self._wrap(B)
        r = self.L.orc_spgemm(pa, pb)
        self.L.orc_csr_free(pa)
        self.L.orc_csr_free(pb)
        if not r:
            raise OracleError(1, "spgemm: inner dimensions differ")
        return self._export(r)

    def galerkin_by_aggregates(self, A, P):
        pa, pp = self._wrap(A), self._wrap(P)
        r = self.L.orc_galerkin_by_aggregates(pa, pp)
        self.L.orc_csr_free(pa)
        self.L.orc_csr_free(pp)
        if not r:
            raise OracleError(1, "galerkin_by_aggregates: bad shape")
        return self._export(r)

    def build_weights(self, A, w):
        p = self._wrap(A)
        w, pw = _f64(w)
        xadj = np.zeros(A.nrows + 1, np.int64)
        adj = np.zeros(max(A.nnz, 1), np.int64)
        wt = np.zeros(max(A.nnz, 1))
        z, bad = C.c_int64(), C.c_int64()
        st = self.L.orc_build_weights(p, pw, xadj.ctypes.data_as(I64P), adj.ctypes.data_as(I64P),
                                      wt.ctypes.data_as(F64P), C.byref(z), C.byref(bad))
        self.L.orc_csr_free(p)
        if st:
            raise OracleError(1, f"build_weights: {ORC_ERR[st]} row {bad.value}")
        m = int(xadj[-1])
        return xadj, adj[:m].copy(), wt[:m].copy(), int(z.value)

    def suitor(self, xadj, adjncy, weight):
        n = len(xadj) - 1
        xadj, px = _i64(xadj)
        adjncy, pa = _i64(adjncy if len(adjncy) else np.zeros(1, np.int64))
        weight, pw = _f64(weight if len(weight) else np.zeros(1))
        mate = np.zeros(max(n, 1), np.int64)
        self.L.orc_suitor(n, px, pa, pw, mate.ctypes.data_as(I64P))
        return mate[:n]

    def pairwise_aggregate(self, mate):
        n = len(mate)
        mate, pm = _i64(mate if n else np.zeros(1, np.int64))
        agg = np.zeros(max(n, 1), np.int64)
        cnt = np.zeros(3, np.int64)
        if self.L.orc_pairwise_aggregate(n, pm, agg.ctypes.data_as(I64P), cnt.ctypes.data_as(I64P)):
            raise OracleError(1, "pairwise_aggregate: invalid matching")
        return agg[:n], int(cnt[0]), int(cnt[1]), int(cnt[2])

    def build_prolongator(self, agg, n_c, w):
        n = len(agg)
        agg, pa = _i64(agg)
        w, pw = _f64(w)
        out = C.POINTER(_OrcCsr)()
        bad = C.c_int64()
        st = self.L.orc_build_prolongator(n, n_c, pa, pw, C.byref(out), C.byref(bad))
        if st == 1:
            raise OracleError(1, f"build_prolongator: aggregate id out of range for vertex {bad.value}")
        if st == 2:
            raise OracleError(1, f"build_prolongator: smooth vector vanishes on aggregate {bad.value}")
        return self._export(out)

    def restrict_vector(self, P, w):
        p = self._wrap(P)
        w, pw = _f64(w)
        wc = np.zeros(P.ncols)
        self.L.orc_restrict_vector(p, pw, wc.ctypes.data_as(F64P))
        self.L.orc_csr_free(p)
        return wc

    def build_hierarchy(self, A, w=None, max_levels=40, coarse_factor=40.0, mode=2, keep=False):
        p = self._wrap(A)
        w = np.ones(A.nrows) if w is None else w
        w, pw = _f64(w)
        out = C.POINTER(_OrcHier)()
        bad = C.c_int64()
        st = self.L.orc_build_hierarchy(p, pw, int(max_levels), C.c_double(coarse_factor),
                                        int(mode), C.byref(out), C.byref(bad))
        self.L.orc_csr_free(p)
        if st:
            raise OracleError(1, f"build_hierarchy: {ORC_ERR[st]} ({bad.value})")
        h = out.contents
        levels = []
        for k in range(h.nl):
            lv = h.lv[k]
            A_ = self._read(lv.A)
            P = self._read(lv.P) if lv.P else None
            R = self._read(lv.R) if lv.R else None
            n = A_.nrows
            l1 = np.ctypeslib.as_array(lv.l1, shape=(max(n, 1),))[:n].copy()
            ww = np.ctypeslib.as_array(lv.w, shape=(max(n, 1),))[:n].copy()
            levels.append(Level(A_, P, R, l1, ww))
        hier = Hierarchy(levels, bool(h.stalled), int(h.zero_edges))
        if keep:
            hier.handle = _PortHierHandle(self, out)
        else:
            self.L.orc_hier_free(out)
        return hier

    def l1_jacobi(self, A, d, b, x, k):
        p = self._wrap(A)
        d, pd = _f64(d)
        b, pb = _f64(b)
        x = np.array(x, dtype=np.float64)
        self.L.orc_l1_jacobi(p, pd, pb, x.ctypes.data_as(F64P), int(k))
        self.L.orc_csr_free(p)
        return x

    def apply_cycle(self, hier, level, b, x, cycle=0, pre=1, post=1, coarsest=20):
        b, pb = _f64(b)
        x = np.array(x, dtype=np.float64)
        self.L.orc_apply_cycle(hier.handle.ptr, int(level), pb, x.ctypes.data_as(F64P),
                               cycle, pre, post, coarsest)
        return x

    def pcg(self, A, hier, b, u0=None, rtol=1e-6, itmax=5000, cycle=0, pre=1, post=1,
            coarsest=20):
        p = self._wrap(A)
        b, pb = _f64(b)
        pu0 = None
        if u0 is not None:
            u0, pu0 = _f64(u0)
        u = np.zeros(A.nrows)
        hist = np.zeros(itmax + 2)
        rep = _Report()
        hh = hier.handle.ptr if hier is not None else None
        st = self.L.orc_pcg(p, hh, cycle, pre, post, coarsest, pb, pu0, C.c_double(rtol),
                            C.c_int64(itmax), u.ctypes.data_as(F64P), hist.ctypes.data_as(F64P),
                            C.byref(rep))
        self.L.orc_csr_free(p)
        r = rep.as_dict()
        if st:
            raise OracleError(st, f"pcg breakdown at iteration {r['breakdown_iteration']}")
        return u, hist[: r["iterations"] + 1].copy(), r

    def dot(self, x, y):
        x, px = _f64(x)
        y, py = _f64(y)
        return float(self.L.orc_dot(len(x), px, py))

    def norm2(self, x):
        x, px = _f64(x)
        return float(self.L.orc_norm2(len(x), px))

    def triple_dot(self, w, r, v, q):
        arrs = [_f64(a) for a in (w, r, v, q)]
        out = np.zeros(3)
        self.L.orc_triple_dot(len(w), *[p for _, p in arrs], out.ctypes.data_as(F64P))
        return tuple(out)

    def axpy_pair(self, y1, y2, x, a, b):
        y1 = np.array(y1, dtype=np.float64)
        y2 = np.array(y2, dtype=np.float64)
        x, px = _f64(x)
        self.L.orc_axpy_pair(len(y1), y1.ctypes.data_as(F64P), y2.ctypes.data_as(F64P), px,
                             C.c_double(a), C.c_double(b))
        return y1, y2


class _PortHierHandle:
    def __init__(self, owner, ptr):
        self.owner, self.ptr = owner, ptr

    def __del__(self):
        try:
            self.owner.L.orc_hier_free(self.ptr)
        except Exception:
            pass


def available():
    """(ref_ok, port_ok) — whether each checker library is present."""
    return os.path.exists(REF_SO), os.path.exists(PORT_SO)
