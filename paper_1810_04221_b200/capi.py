"""ctypes binding of the C-ABI (include/mamg_capi.h) exported by
csrc/lib/libmamg_cuda.so — the B200 (sm_100a) implementation of the
reference's AMG-PCG setup/solve path.

This is the Python-side mirror of the reference interface
(/root/reference/proj/include/matchamg/*.hpp): the method names, argument
meaning and exceptions follow the reference's C++ API so that the parity tests
read like the reference's own tests. There is no CPU fallback: importing this
module on a machine without the built library, or calling it without a CUDA
device, raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MAMG_LIB: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("MAMG_LIB") or os.path.join(HERE, "csrc", "lib", "libmamg_cuda.so")

I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
VP = C.c_void_p

MAMG_OK, MAMG_INVALID_ARGUMENT, MAMG_RUNTIME, MAMG_BREAKDOWN, MAMG_CUDA, MAMG_NCCL = range(6)


class MamgError(RuntimeError):
    """Base error carrying the C-ABI status and offending index."""

    def __init__(self, status: int, msg: str, index: int = -1):
        super().__init__(msg)
        self.status = status
        self.index = index


class InvalidArgument(MamgError, ValueError):
    """std::invalid_argument in the reference."""


class BreakdownError(MamgError):
    """matchamg::BreakdownError (proj/include/matchamg/krylov.hpp:52-59)."""

    @property
    def iteration(self) -> int:
        return self.index


class CudaFailure(MamgError):
    pass


_EXC = {MAMG_INVALID_ARGUMENT: InvalidArgument, MAMG_BREAKDOWN: BreakdownError,
        MAMG_CUDA: CudaFailure}


class SetupCfg(C.Structure):
    """SetupConfig (proj/include/matchamg/coarsening.hpp:62-69)."""
    _fields_ = [("max_levels", C.c_int32), ("aggregation", C.c_int32),
                ("coarse_factor", C.c_double)]


class CycleCfg(C.Structure):
    """CycleConfig (proj/include/matchamg/multigrid.hpp:17-24); cycle 0=V, 1=W."""
    _fields_ = [("cycle", C.c_int32), ("pre_sweeps", C.c_int32), ("post_sweeps", C.c_int32),
                ("coarsest_sweeps", C.c_int32)]


class SolveCfg(C.Structure):
    """SolveConfig (proj/include/matchamg/krylov.hpp:29-34)."""
    _fields_ = [("rtol", C.c_double), ("itmax", C.c_int64)]


class Report(C.Structure):
    """SolveReport (proj/include/matchamg/krylov.hpp:36-48) + breakdown info."""
    _fields_ = [("iterations", C.c_int64), ("final_relres", C.c_double),
                ("converged", C.c_int32), ("pad", C.c_int32), ("solve_ms", C.c_double),
                ("audit_checks", C.c_int64), ("audit_failures", C.c_int64),
                ("audit_max_rel", C.c_double), ("breakdown_iteration", C.c_int64),
                ("breakdown_rho", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "pad"}


HOST_PRECOND = C.CFUNCTYPE(None, VP, F64P, F64P, C.c_int64)

# (name, restype, argtypes) for every symbol include/mamg_capi.h declares
SIGNATURES = [
    ("mamg_ctx_create", C.c_int, [C.c_int, C.POINTER(VP)]),
    ("mamg_ctx_destroy", None, [VP]),
    ("mamg_last_error", C.c_char_p, [VP]),
    ("mamg_last_error_index", C.c_int64, [VP]),
    ("mamg_synchronize", C.c_int, [VP]),
    ("mamg_kernel_launches", C.c_int64, [VP]),
    ("mamg_version", C.c_char_p, []),
    ("mamg_dmalloc", C.c_int, [VP, C.c_size_t, C.POINTER(VP)]),
    ("mamg_dfree", C.c_int, [VP, VP]),
    ("mamg_h2d", C.c_int, [VP, VP, VP, C.c_size_t]),
    ("mamg_d2h", C.c_int, [VP, VP, VP, C.c_size_t]),
    ("mamg_csr_upload", C.c_int, [VP, C.c_int64, C.c_int64, I64P, I64P, F64P, C.POINTER(VP)]),
    ("mamg_gen_poisson2d_dev", C.c_int, [VP, C.c_int64, C.c_int64, C.POINTER(VP)]),
    ("mamg_gen_aniso2d_dev", C.c_int, [VP, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                       C.POINTER(VP)]),
    ("mamg_gen_randk3d_dev", C.c_int, [VP, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                       C.c_uint64, C.POINTER(VP)]),
    ("mamg_gen_jump3d_dev", C.c_int, [VP, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                      C.c_double, C.c_double, C.POINTER(VP)]),
    ("mamg_gen_aniso27_dev", C.c_int, [VP, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                       C.c_double, C.c_double, C.POINTER(VP)]),
    ("mamg_gen_elast3d_dev", C.c_int, [VP, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                       C.c_double, C.POINTER(VP)]),
    ("mamg_csr_shape", C.c_int, [VP, I64P, I64P, I64P]),
    ("mamg_csr_download", C.c_int, [VP, VP, I64P, I64P, F64P]),
    ("mamg_mat_destroy", None, [VP]),
    ("mamg_lane_policy", C.c_int, [VP]),
    ("mamg_has_symmetric_pattern", C.c_int, [VP, VP, C.POINTER(C.c_int)]),
    ("mamg_spmv", C.c_int, [VP, VP, C.c_int, VP, VP]),
    ("mamg_l1_diagonal", C.c_int, [VP, VP, VP]),
    ("mamg_transpose", C.c_int, [VP, VP, C.POINTER(VP)]),
    ("mamg_spgemm", C.c_int, [VP, VP, VP, C.POINTER(VP)]),
    ("mamg_galerkin_triple", C.c_int, [VP, VP, VP, C.POINTER(VP)]),
    ("mamg_build_weights", C.c_int, [VP, VP, VP, C.POINTER(VP)]),
    ("mamg_graph_upload", C.c_int, [VP, C.c_int64, I64P, I64P, F64P, C.POINTER(VP)]),
    ("mamg_graph_shape", C.c_int, [VP, I64P, I64P, I64P]),
    ("mamg_graph_download", C.c_int, [VP, VP, I64P, I64P, F64P]),
    ("mamg_graph_destroy", None, [VP]),
    ("mamg_suitor_match", C.c_int, [VP, VP, I64P]),
    ("mamg_pairwise_aggregate", C.c_int, [VP, C.c_int64, I64P, I64P, I64P]),
    ("mamg_build_prolongator", C.c_int, [VP, C.c_int64, C.c_int64, I64P, VP, C.POINTER(VP)]),
    ("mamg_restrict_vector", C.c_int, [VP, VP, VP, VP]),
    ("mamg_galerkin_by_aggregates", C.c_int, [VP, VP, VP, C.POINTER(VP)]),
    ("mamg_coarsen_step", C.c_int, [VP, VP, VP, C.c_int, C.POINTER(VP), C.POINTER(VP),
                                    C.POINTER(VP), I64P]),
    ("mamg_setup", C.c_int, [VP, VP, VP, C.POINTER(SetupCfg), C.POINTER(VP)]),
    ("mamg_hier_from_levels", C.c_int, [VP, C.c_int, C.POINTER(VP), C.POINTER(VP),
                                        C.POINTER(VP), C.POINTER(VP), C.POINTER(VP),
                                        C.POINTER(VP)]),
    ("mamg_hier_destroy", None, [VP]),
    ("mamg_hier_nl", C.c_int, [VP]),
    ("mamg_hier_stats", C.c_int, [VP, C.POINTER(C.c_int), I64P]),
    ("mamg_hier_A", VP, [VP, C.c_int]),
    ("mamg_hier_P", VP, [VP, C.c_int]),
    ("mamg_hier_R", VP, [VP, C.c_int]),
    ("mamg_hier_l1", VP, [VP, C.c_int]),
    ("mamg_hier_w", VP, [VP, C.c_int]),
    ("mamg_l1_jacobi", C.c_int, [VP, VP, VP, VP, VP, C.c_int]),
    ("mamg_apply_cycle", C.c_int, [VP, VP, C.c_int, C.POINTER(CycleCfg), VP, VP]),
    ("mamg_precond_apply", C.c_int, [VP, VP, C.POINTER(CycleCfg), VP, VP]),
    ("mamg_dot", C.c_int, [VP, C.c_int64, VP, VP, F64P]),
    ("mamg_norm2", C.c_int, [VP, C.c_int64, VP, F64P]),
    ("mamg_axpy", C.c_int, [VP, C.c_int64, VP, C.c_double, VP]),
    ("mamg_fused_triple_dot", C.c_int, [VP, C.c_int64, VP, VP, VP, VP, F64P]),
    ("mamg_fused_axpy_pair", C.c_int, [VP, C.c_int64, VP, VP, VP, C.c_double, C.c_double]),
    ("mamg_pcg_solve", C.c_int, [VP, VP, VP, C.POINTER(CycleCfg), HOST_PRECOND, VP, VP, VP,
                                 C.POINTER(SolveCfg), VP, F64P, C.POINTER(Report)]),
    ("mamg_solve_host", C.c_int, [VP, C.c_int64, I64P, I64P, F64P, F64P, F64P,
                                  C.POINTER(SetupCfg), C.POINTER(CycleCfg), C.POINTER(SolveCfg),
                                  F64P, F64P, C.POINTER(Report), C.POINTER(C.c_int), F64P]),
    ("mamg_nccl_unique_id", C.c_int, [VP]),
    ("mamg_dist_create", C.c_int, [VP, C.c_int, C.c_int, VP, C.POINTER(VP)]),
    ("mamg_dist_create_shm", C.c_int, [VP, C.c_int, C.c_int, C.c_char_p, C.POINTER(VP)]),
    ("mamg_group_create", C.c_int, [C.c_int, C.POINTER(VP)]),
    ("mamg_group_destroy", None, [VP]),
    ("mamg_dist_create_group", C.c_int, [VP, VP, C.c_int, C.POINTER(VP)]),
    ("mamg_dist_destroy", None, [VP]),
    ("mamg_dist_last_solve", C.c_int, [VP, C.POINTER(C.c_int)]),
    ("mamg_dist_time", C.c_int, [VP, C.c_int, C.POINTER(CycleCfg), C.c_int, F64P]),
    ("mamg_shm_allgather", C.c_int, [C.c_char_p, C.c_int, C.c_int, I64P, C.c_int64, I64P]),
    ("mamg_dist_set_matching", C.c_int, [VP, C.c_int]),
    ("mamg_dist_set_rebuildable", C.c_int, [VP, C.c_int]),
    ("mamg_dist_set_agglomeration", C.c_int, [VP, C.c_int64]),
    ("mamg_dist_bounds", C.c_int, [C.c_int64, C.c_int, I64P]),
    ("mamg_dist_setup", C.c_int, [VP, C.c_int64, I64P, I64P, F64P, F64P, C.POINTER(SetupCfg)]),
    ("mamg_dist_load", C.c_int, [VP, C.c_int64, I64P, I64P, F64P, F64P]),
    ("mamg_dist_build", C.c_int, [VP, C.POINTER(SetupCfg)]),
    ("mamg_dist_info", C.c_int, [VP, C.POINTER(C.c_int), I64P, I64P, C.POINTER(C.c_int), I64P]),
    ("mamg_dist_level_bounds", C.c_int, [VP, C.c_int, I64P]),
    ("mamg_dist_level_shape", C.c_int, [VP, C.c_int, C.c_int, C.c_int, I64P, I64P]),
    ("mamg_dist_download", C.c_int, [VP, C.c_int, C.c_int, C.c_int, I64P, I64P, F64P]),
    ("mamg_dist_pcg_x0", C.c_int, [VP, F64P, F64P, C.POINTER(CycleCfg), C.POINTER(SolveCfg), F64P,
                                   F64P, C.POINTER(Report)]),
    ("mamg_dist_pcg", C.c_int, [VP, F64P, C.POINTER(CycleCfg), C.POINTER(SolveCfg), F64P, F64P,
                                C.POINTER(Report)]),
    ("mamg_timer_start", C.c_int, [VP]),
    ("mamg_timer_stop", C.c_int, [VP, F64P]),
    ("mamg_time_smoother", C.c_int, [VP, VP, C.c_int, C.c_int, F64P]),
    ("mamg_time_spmv", C.c_int, [VP, VP, C.c_int, C.c_int, F64P]),
    ("mamg_time_precond", C.c_int, [VP, VP, C.POINTER(CycleCfg), C.c_int, F64P]),
]

_LIB = None


def load_library(path: str = LIB_PATH):
    """Load libmamg_cuda.so (raises if it was not built — there is no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with __graft_entry__.build() "
                          "(make -C paper_1810_04221_b200/csrc)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    if a.size == 0:
        a = np.zeros(1, np.int64)
    return a, a.ctypes.data_as(I64P)


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size == 0:
        a = np.zeros(1)
    return a, a.ctypes.data_as(F64P)


@dataclass
class Csr:
    """Host CSR in the reference API layout (proj/include/matchamg/csr.hpp:30-57)."""

    nrows: int
    ncols: int
    rp: np.ndarray
    ci: np.ndarray
    v: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rp[-1])


@dataclass
class Level:
    A: Csr
    P: Csr | None
    R: Csr | None
    l1: np.ndarray
    w: np.ndarray


@dataclass
class Hierarchy:
    """Host materialisation of a device hierarchy (coarsening.hpp:72-94)."""

    levels: list
    stalled: bool
    zero_edges: int
    device: "DeviceHierarchy | None" = field(default=None, repr=False)

    @property
    def nl(self) -> int:
        return len(self.levels)


class DeviceVector:
    """Device fp64 array owned through the C-ABI allocator."""

    def __init__(self, dev: "Device", n: int):
        self.dev, self.n = dev, int(n)
        p = VP()
        dev._check(dev.L.mamg_dmalloc(dev.ctx, max(8 * self.n, 8), C.byref(p)))
        self.ptr = p

    @classmethod
    def from_host(cls, dev, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        v = cls(dev, a.size)
        if a.size:
            dev._check(dev.L.mamg_h2d(dev.ctx, v.ptr, a.ctypes.data_as(VP), 8 * a.size))
        return v

    def to_host(self) -> np.ndarray:
        out = np.zeros(self.n)
        if self.n:
            self.dev._check(self.dev.L.mamg_d2h(self.dev.ctx, out.ctypes.data_as(VP), self.ptr,
                                                8 * self.n))
        return out

    def free(self):
        if self.ptr:
            self.dev.L.mamg_dfree(self.dev.ctx, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class DeviceMatrix:
    """mamg_mat handle (device CSR)."""

    def __init__(self, dev, handle, owned=True):
        self.dev, self.h, self.owned = dev, VP(handle), owned

    @property
    def shape(self):
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        self.dev.L.mamg_csr_shape(self.h, C.byref(nr), C.byref(nc), C.byref(nz))
        return nr.value, nc.value, nz.value

    @property
    def lane_group(self) -> int:
        return int(self.dev.L.mamg_lane_policy(self.h))

    def to_host(self) -> Csr:
        nr, nc, nz = self.shape
        rp = np.zeros(nr + 1, np.int64)
        ci = np.zeros(max(nz, 1), np.int64)
        v = np.zeros(max(nz, 1))
        self.dev._check(self.dev.L.mamg_csr_download(self.dev.ctx, self.h, rp.ctypes.data_as(I64P),
                                                     ci.ctypes.data_as(I64P),
                                                     v.ctypes.data_as(F64P)))
        return Csr(nr, nc, rp, ci[:nz].copy(), v[:nz].copy())

    def __del__(self):
        try:
            if self.owned and self.h:
                self.dev.L.mamg_mat_destroy(self.h)
                self.h = None
        except Exception:
            pass


class DeviceHierarchy:
    """mamg_hier handle: the device-resident multigrid hierarchy."""

    def __init__(self, dev, handle, keep=()):
        self.dev, self.h = dev, VP(handle)
        self._keep = keep

    @property
    def nl(self) -> int:
        return int(self.dev.L.mamg_hier_nl(self.h))

    def stats(self):
        st, z = C.c_int(), C.c_int64()
        self.dev.L.mamg_hier_stats(self.h, C.byref(st), C.byref(z))
        return bool(st.value), int(z.value)

    def level_matrix(self, which: str, k: int) -> DeviceMatrix | None:
        fn = {"A": self.dev.L.mamg_hier_A, "P": self.dev.L.mamg_hier_P,
              "R": self.dev.L.mamg_hier_R}[which]
        p = fn(self.h, k)
        return DeviceMatrix(self.dev, p, owned=False) if p else None

    def level_vector(self, which: str, k: int) -> np.ndarray:
        fn = {"l1": self.dev.L.mamg_hier_l1, "w": self.dev.L.mamg_hier_w}[which]
        p = fn(self.h, k)
        n = self.level_matrix("A", k).shape[0]
        out = np.zeros(n)
        if n:
            self.dev._check(self.dev.L.mamg_d2h(self.dev.ctx, out.ctypes.data_as(VP), VP(p), 8 * n))
        return out

    def materialize(self) -> Hierarchy:
        levels = []
        nl = self.nl
        for k in range(nl):
            A = self.level_matrix("A", k).to_host()
            P = R = None
            if k + 1 < nl:
                P = self.level_matrix("P", k).to_host()
                R = self.level_matrix("R", k).to_host()
            levels.append(Level(A, P, R, self.level_vector("l1", k), self.level_vector("w", k)))
        stalled, z = self.stats()
        return Hierarchy(levels, stalled, z, device=self)

    def __del__(self):
        try:
            if self.h:
                self.dev.L.mamg_hier_destroy(self.h)
                self.h = None
        except Exception:
            pass


def _cycle(cycle="V", pre=1, post=1, coarsest=20) -> CycleCfg:
    c = {"V": 0, "W": 1, "K": 2, 0: 0, 1: 1, 2: 2}[cycle]
    return CycleCfg(c, pre, post, coarsest)


class Device:
    """One mamg_ctx (one CUDA device + stream). Methods mirror the reference API."""

    def __init__(self, device: int = 0):
        self.L = load_library()
        p = VP()
        st = self.L.mamg_ctx_create(int(device), C.byref(p))
        if st != MAMG_OK:
            raise CudaFailure(st, f"mamg_ctx_create({device}) failed: no usable CUDA device")
        self.ctx = p

    def close(self):
        if self.ctx:
            self.L.mamg_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing --
    def _check(self, st):
        if st != MAMG_OK:
            msg = self.L.mamg_last_error(self.ctx).decode()
            idx = int(self.L.mamg_last_error_index(self.ctx))
            raise _EXC.get(st, MamgError)(st, msg, idx)

    @property
    def kernel_launches(self) -> int:
        return int(self.L.mamg_kernel_launches(self.ctx))

    def synchronize(self):
        self._check(self.L.mamg_synchronize(self.ctx))

    def upload(self, A: Csr) -> DeviceMatrix:
        rp, prp = _i64(A.rp)
        ci, pci = _i64(A.ci)
        v, pv = _f64(A.v)
        h = VP()
        self._check(self.L.mamg_csr_upload(self.ctx, A.nrows, A.ncols, prp, pci, pv, C.byref(h)))
        return DeviceMatrix(self, h.value)

    def generate(self, spec: str, seed: int = 0) -> DeviceMatrix:
        """The generator `spec` (problems.from_spec syntax) assembled directly on
        the device: the same matrix bit for bit, no host CSR, no upload."""
        kind, _, rest = spec.partition(":")
        a = [x for x in rest.split(",") if x]
        h = VP()
        L = self.L
        if kind == "poisson2d" and len(a) == 2:
            st = L.mamg_gen_poisson2d_dev(self.ctx, int(a[0]), int(a[1]), C.byref(h))
        elif kind == "ani" and len(a) == 4:
            st = L.mamg_gen_aniso2d_dev(self.ctx, int(a[0]), int(a[1]), float(a[2]), float(a[3]),
                                        C.byref(h))
        elif kind == "randk3d" and len(a) == 4:
            st = L.mamg_gen_randk3d_dev(self.ctx, int(a[0]), int(a[1]), int(a[2]), float(a[3]),
                                        int(seed), C.byref(h))
        elif kind == "aniso27" and len(a) == 4:
            st = L.mamg_gen_aniso27_dev(self.ctx, int(a[0]), int(a[1]), int(a[2]), 1.0, 1.0,
                                        float(a[3]), C.byref(h))
        elif kind == "jump3d" and len(a) == 4:
            st = L.mamg_gen_jump3d_dev(self.ctx, int(a[0]), int(a[1]), int(a[2]), int(a[3]),
                                       int(seed), 1e-3, 1e3, C.byref(h))
        elif kind == "elast3d" and len(a) == 3:
            st = L.mamg_gen_elast3d_dev(self.ctx, int(a[0]), int(a[1]), int(a[2]), 0.42, 1.7,
                                        C.byref(h))
        else:
            raise ValueError(f"bad generator spec `{spec}`")
        self._check(st)
        return DeviceMatrix(self, h.value)

    def vec(self, a) -> DeviceVector:
        return DeviceVector.from_host(self, a)

    def zeros(self, n) -> DeviceVector:
        return DeviceVector.from_host(self, np.zeros(n))

    def _mat(self, A):
        return A if isinstance(A, DeviceMatrix) else self.upload(A)

    # -- device-event timing --
    def timer_start(self):
        self._check(self.L.mamg_timer_start(self.ctx))

    def timer_stop(self) -> float:
        ms = C.c_double()
        self._check(self.L.mamg_timer_stop(self.ctx, C.byref(ms)))
        return ms.value

    def time_smoother(self, hier: "DeviceHierarchy", level=0, reps=20) -> float:
        ms = C.c_double()
        self._check(self.L.mamg_time_smoother(self.ctx, hier.h, level, reps, C.byref(ms)))
        return ms.value

    def time_spmv(self, hier: "DeviceHierarchy", level=0, reps=20) -> float:
        ms = C.c_double()
        self._check(self.L.mamg_time_spmv(self.ctx, hier.h, level, reps, C.byref(ms)))
        return ms.value

    def time_precond(self, hier: "DeviceHierarchy", reps=10, cycle=0, pre=1, post=1,
                     coarsest=20) -> float:
        ms = C.c_double()
        cfg = _cycle(cycle, pre, post, coarsest)
        self._check(self.L.mamg_time_precond(self.ctx, hier.h, C.byref(cfg), reps, C.byref(ms)))
        return ms.value

    def pcg_device(self, dA: DeviceMatrix, dh: "DeviceHierarchy", db: DeviceVector,
                   du: DeviceVector, rtol=1e-6, itmax=5000, cycle=0, pre=1, post=1, coarsest=20):
        """pcg_solve on device-resident data (no host copies of vectors)."""
        cfg = SolveCfg(float(rtol), int(itmax))
        cyc = _cycle(cycle, pre, post, coarsest)
        rep = Report()
        self._check(self.L.mamg_pcg_solve(self.ctx, dA.h, dh.h, C.byref(cyc), HOST_PRECOND(), None,
                                          db.ptr, None, C.byref(cfg), du.ptr, None, C.byref(rep)))
        return rep.as_dict()

    # -- kernels (kernels.hpp) --
    def spmv(self, A, x, group=0) -> np.ndarray:
        dA = self._mat(A)
        dx = self.vec(x)
        dy = self.zeros(dA.shape[0])
        self._check(self.L.mamg_spmv(self.ctx, dA.h, int(group), dx.ptr, dy.ptr))
        return dy.to_host()

    def lane_policy(self, A) -> int:
        return self._mat(A).lane_group

    def l1_diagonal(self, A) -> np.ndarray:
        dA = self._mat(A)
        d = self.zeros(dA.shape[0])
        self._check(self.L.mamg_l1_diagonal(self.ctx, dA.h, d.ptr))
        return d.to_host()

    def has_symmetric_pattern(self, A) -> bool:
        out = C.c_int()
        dA = self._mat(A)
        self._check(self.L.mamg_has_symmetric_pattern(self.ctx, dA.h, C.byref(out)))
        return bool(out.value)

    def _unary(self, fn, *mats) -> Csr:
        out = VP()
        dms = [self._mat(m) for m in mats]  # keep the handles alive across the call
        self._check(fn(self.ctx, *[d.h for d in dms], C.byref(out)))
        return DeviceMatrix(self, out.value).to_host()

    def transpose(self, A) -> Csr:
        return self._unary(self.L.mamg_transpose, A)

    def spgemm(self, A, B) -> Csr:
        return self._unary(self.L.mamg_spgemm, A, B)

    def galerkin_triple(self, A, P) -> Csr:
        return self._unary(self.L.mamg_galerkin_triple, A, P)

    def galerkin_by_aggregates(self, A, P) -> Csr:
        return self._unary(self.L.mamg_galerkin_by_aggregates, A, P)

    # -- matching (matching.hpp) --
    def build_weights(self, A, w):
        dA = self._mat(A)
        dw = self.vec(w)
        g = VP()
        self._check(self.L.mamg_build_weights(self.ctx, dA.h, dw.ptr, C.byref(g)))
        try:
            return self._graph_to_host(g)
        finally:
            self.L.mamg_graph_destroy(g)

    def _graph_to_host(self, g):
        n, m, z = C.c_int64(), C.c_int64(), C.c_int64()
        self.L.mamg_graph_shape(g, C.byref(n), C.byref(m), C.byref(z))
        xadj = np.zeros(n.value + 1, np.int64)
        adj = np.zeros(max(m.value, 1), np.int64)
        wt = np.zeros(max(m.value, 1))
        self._check(self.L.mamg_graph_download(self.ctx, g, xadj.ctypes.data_as(I64P),
                                               adj.ctypes.data_as(I64P), wt.ctypes.data_as(F64P)))
        return xadj, adj[: m.value].copy(), wt[: m.value].copy(), int(z.value)

    def suitor(self, xadj, adjncy, weight) -> np.ndarray:
        n = len(xadj) - 1
        xa, px = _i64(xadj)
        ad, pa = _i64(adjncy)
        wt, pw = _f64(weight)
        g = VP()
        self._check(self.L.mamg_graph_upload(self.ctx, n, px, pa, pw, C.byref(g)))
        try:
            mate = np.zeros(max(n, 1), np.int64)
            self._check(self.L.mamg_suitor_match(self.ctx, g, mate.ctypes.data_as(I64P)))
            return mate[:n]
        finally:
            self.L.mamg_graph_destroy(g)

    # -- coarsening (coarsening.hpp) --
    def pairwise_aggregate(self, mate):
        n = len(mate)
        m, pm = _i64(mate)
        agg = np.zeros(max(n, 1), np.int64)
        cnt = np.zeros(3, np.int64)
        self._check(self.L.mamg_pairwise_aggregate(self.ctx, n, pm, agg.ctypes.data_as(I64P),
                                                   cnt.ctypes.data_as(I64P)))
        return agg[:n], int(cnt[0]), int(cnt[1]), int(cnt[2])

    def build_prolongator(self, agg, n_c, w) -> Csr:
        n = len(agg)
        a, pa = _i64(agg)
        dw = self.vec(w)
        out = VP()
        self._check(self.L.mamg_build_prolongator(self.ctx, n, int(n_c), pa, dw.ptr, C.byref(out)))
        return DeviceMatrix(self, out.value).to_host()

    def restrict_vector(self, P, w) -> np.ndarray:
        dP = self._mat(P)
        dw = self.vec(w)
        wc = self.zeros(dP.shape[1])
        self._check(self.L.mamg_restrict_vector(self.ctx, dP.h, dw.ptr, wc.ptr))
        return wc.to_host()

    def coarsen_step(self, A, w, mode=1):
        dA = self._mat(A)
        dw = self.vec(w)
        P, Ac, wc = VP(), VP(), VP()
        z = C.c_int64()
        self._check(self.L.mamg_coarsen_step(self.ctx, dA.h, dw.ptr, int(mode), C.byref(P),
                                             C.byref(Ac), C.byref(wc), C.byref(z)))
        Ph = DeviceMatrix(self, P.value).to_host()
        Ach = DeviceMatrix(self, Ac.value).to_host()
        out = np.zeros(Ach.nrows)
        if Ach.nrows:
            self._check(self.L.mamg_d2h(self.ctx, out.ctypes.data_as(VP), wc, 8 * Ach.nrows))
        self.L.mamg_dfree(self.ctx, wc)
        return Ph, Ach, out, int(z.value)

    def setup(self, A, w=None, max_levels=40, coarse_factor=40.0, mode=2) -> DeviceHierarchy:
        """build_hierarchy (coarsening.cpp:194-238) -> device-resident hierarchy."""
        dA = self._mat(A)
        dw = self.vec(w) if w is not None else None
        cfg = SetupCfg(int(max_levels), int(mode), float(coarse_factor))
        h = VP()
        self._check(self.L.mamg_setup(self.ctx, dA.h, dw.ptr if dw else None, C.byref(cfg),
                                      C.byref(h)))
        return DeviceHierarchy(self, h.value)

    def build_hierarchy(self, A, w=None, max_levels=40, coarse_factor=40.0, mode=2,
                        keep=True) -> Hierarchy:
        return self.setup(A, w, max_levels, coarse_factor, mode).materialize()

    # -- multigrid (multigrid.hpp) --
    def l1_jacobi(self, A, d, b, x, k):
        dA = self._mat(A)
        dd, db, dx = self.vec(d), self.vec(b), self.vec(x)
        self._check(self.L.mamg_l1_jacobi(self.ctx, dA.h, dd.ptr, db.ptr, dx.ptr, int(k)))
        return dx.to_host()

    def apply_cycle(self, hier, level, b, x, cycle=0, pre=1, post=1, coarsest=20):
        dh = hier.device if isinstance(hier, Hierarchy) else hier
        cfg = _cycle(cycle, pre, post, coarsest)
        db, dx = self.vec(b), self.vec(x)
        self._check(self.L.mamg_apply_cycle(self.ctx, dh.h, int(level), C.byref(cfg), db.ptr,
                                            dx.ptr))
        return dx.to_host()

    def precond_apply(self, hier, r, cycle=0, pre=1, post=1, coarsest=20):
        dh = hier.device if isinstance(hier, Hierarchy) else hier
        cfg = _cycle(cycle, pre, post, coarsest)
        dr = self.vec(r)
        dz = self.zeros(len(r))
        self._check(self.L.mamg_precond_apply(self.ctx, dh.h, C.byref(cfg), dr.ptr, dz.ptr))
        return dz.to_host()

    # -- vector ops (vector_ops.hpp) --
    def dot(self, x, y) -> float:
        dx, dy = self.vec(x), self.vec(y)
        out = C.c_double()
        self._check(self.L.mamg_dot(self.ctx, len(x), dx.ptr, dy.ptr, C.byref(out)))
        return out.value

    def norm2(self, x) -> float:
        dx = self.vec(x)
        out = C.c_double()
        self._check(self.L.mamg_norm2(self.ctx, len(x), dx.ptr, C.byref(out)))
        return out.value

    def triple_dot(self, w, r, v, q):
        dv = [self.vec(a) for a in (w, r, v, q)]
        out = np.zeros(3)
        self._check(self.L.mamg_fused_triple_dot(self.ctx, len(w), *[d.ptr for d in dv],
                                                 out.ctypes.data_as(F64P)))
        return tuple(out)

    def axpy_pair(self, y1, y2, x, a, b):
        d1, d2, dx = self.vec(y1), self.vec(y2), self.vec(x)
        self._check(self.L.mamg_fused_axpy_pair(self.ctx, len(y1), d1.ptr, d2.ptr, dx.ptr,
                                                C.c_double(a), C.c_double(b)))
        return d1.to_host(), d2.to_host()

    # -- Krylov (krylov.hpp) --
    def pcg(self, A, hier, b, u0=None, rtol=1e-6, itmax=5000, cycle=0, pre=1, post=1,
            coarsest=20, host_precond=None):
        """pcg_solve (krylov.cpp:43-141). hier: Hierarchy/DeviceHierarchy or None;
        host_precond: optional python callable z = f(r) (a host PrecondFn)."""
        dA = self._mat(A)
        dh = None
        if hier is not None:
            dh = hier.device if isinstance(hier, Hierarchy) else hier
        n = dA.shape[0]
        db = self.vec(b)
        du0 = self.vec(u0) if u0 is not None else None
        du = self.zeros(n)
        cfg = SolveCfg(float(rtol), int(itmax))
        cyc = _cycle(cycle, pre, post, coarsest)
        hist = np.zeros(int(itmax) + 2)
        rep = Report()
        cb = HOST_PRECOND()
        if host_precond is not None:
            def _tramp(user, r, z, nn):
                rr = np.ctypeslib.as_array(r, shape=(nn,))
                zz = np.ctypeslib.as_array(z, shape=(nn,))
                zz[:] = host_precond(rr.copy())
            cb = HOST_PRECOND(_tramp)
        st = self.L.mamg_pcg_solve(self.ctx, dA.h, dh.h if dh else None, C.byref(cyc), cb, None,
                                   db.ptr, du0.ptr if du0 else None, C.byref(cfg), du.ptr,
                                   hist.ctypes.data_as(F64P), C.byref(rep))
        self._check(st)
        r = rep.as_dict()
        return du.to_host(), hist[: r["iterations"] + 1].copy(), r

    def solve_host(self, A: Csr, w=None, b=None, rtol=1e-6, itmax=5000, max_levels=40,
                   coarse_factor=40.0, mode=2, cycle=0, pre=1, post=1, coarsest=20, out=None):
        """The end-to-end cli::run_solve path on host buffers (one C-ABI call).
        `out`: optional caller-owned float64 array of n receiving u."""
        rp, prp = _i64(A.rp)
        ci, pci = _i64(A.ci)
        v, pv = _f64(A.v)
        pw = pb = None
        if w is not None:
            w, pw = _f64(w)
        if b is not None:
            b, pb = _f64(b)
        if out is not None:
            if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != A.nrows:
                raise ValueError("solve_host: out must be a contiguous float64 array of n")
            u = out
        else:
            u = np.zeros(A.nrows)
        hist = np.zeros(int(itmax) + 2)
        rep = Report()
        nl = C.c_int()
        times = np.zeros(4)
        scfg = SetupCfg(int(max_levels), int(mode), float(coarse_factor))
        ccfg = _cycle(cycle, pre, post, coarsest)
        cfg = SolveCfg(float(rtol), int(itmax))
        self._check(self.L.mamg_solve_host(self.ctx, A.nrows, prp, pci, pv, pw, pb, C.byref(scfg),
                                           C.byref(ccfg), C.byref(cfg),
                                           u.ctypes.data_as(F64P), hist.ctypes.data_as(F64P),
                                           C.byref(rep), C.byref(nl),
                                           times.ctypes.data_as(F64P)))
        r = rep.as_dict()
        r.update({"nl": nl.value, "setup_ms": times[0], "upload_ms": times[2],
                  "download_ms": times[3]})
        return u, hist[: r["iterations"] + 1].copy(), r


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it)."""
    L = load_library()
    buf = (C.c_char * 128)()
    if L.mamg_nccl_unique_id(C.cast(buf, VP)) != MAMG_OK:
        raise MamgError(MAMG_NCCL, "ncclGetUniqueId failed")
    return bytes(buf)


def shm_allgather(name: str, world: int, rank: int, values) -> np.ndarray:
    """The shm transport's host collective alone (mamg_shm_allgather; no GPU):
    every rank passes the same fresh `name` and len(values) int64 -> a
    (world, len) array in rank order."""
    L = load_library()
    v = np.ascontiguousarray(values, np.int64)
    out = np.zeros(world * len(v), np.int64)
    rc = L.mamg_shm_allgather(name.encode(), int(world), int(rank), v.ctypes.data_as(I64P),
                              len(v), out.ctypes.data_as(I64P))
    if rc != MAMG_OK:
        raise MamgError(rc, L.mamg_last_error(None).decode())
    return out.reshape(world, len(v))


def partition_bounds(n: int, world: int) -> list:
    """Level-0 row-block boundaries of the partitioned path (2048-aligned)."""
    L = load_library()
    out = np.zeros(world + 1, np.int64)
    if L.mamg_dist_bounds(int(n), int(world), out.ctypes.data_as(I64P)) != MAMG_OK:
        raise InvalidArgument(MAMG_INVALID_ARGUMENT, "bad partition request")
    return out.tolist()


class ThreadGroup:
    """An in-process rank group (mamg_group_create): ranks as threads of this
    process, one Device (context) each, passed to Dist(..., group=g)."""

    def __init__(self, world: int):
        L = load_library()
        self.L, self.world = L, int(world)
        h = VP()
        if L.mamg_group_create(self.world, C.byref(h)) != MAMG_OK:
            raise MamgError(MAMG_RUNTIME, "mamg_group_create failed")
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.L.mamg_group_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Dist:
    """Row-block partitioned hierarchy + PCG (include/mamg_capi.h, mamg_dist_*).

    rank = -1: all `world` parts in this context (loopback transport, one GPU);
    rank >= 0: this process owns part `rank` (NCCL transport; `uid` from
    nccl_unique_id() on rank 0), or — with shm="<name>" — the NCCL-free
    multi-process transport (host collectives in a POSIX shared-memory
    segment, device data through CUDA IPC; ranks may share one GPU).
    matching = "local": Suitor on each part's own graph block (aggregates never
    straddle parts); "global": one Suitor over the whole graph across parts
    (cross-part aggregates, hierarchy bit-identical to the unpartitioned one)."""

    AGGLOMERATE = 262144  # device default (mamg_dist_set_agglomeration)

    def __init__(self, dev: Device, world: int, rank: int = -1, uid: bytes | None = None,
                 matching: str = "local", agglomerate: int | None = None,
                 shm: str | None = None, group: "ThreadGroup | None" = None):
        self.dev, self.world, self.rank = dev, int(world), int(rank)
        if matching not in ("local", "global"):
            raise ValueError("matching must be 'local' or 'global'")
        h = VP()
        if group is not None:
            dev._check(dev.L.mamg_dist_create_group(dev.ctx, group.h, self.rank, C.byref(h)))
        elif shm is not None:
            dev._check(dev.L.mamg_dist_create_shm(dev.ctx, self.world, self.rank,
                                                  shm.encode(), C.byref(h)))
        else:
            ub = C.create_string_buffer(uid, 128) if uid is not None else None
            dev._check(dev.L.mamg_dist_create(dev.ctx, self.world, self.rank,
                                              C.cast(ub, VP) if ub is not None else None,
                                              C.byref(h)))
        self.h = h
        self.matching = matching
        dev._check(dev.L.mamg_dist_set_matching(h, 1 if matching == "global" else 0))
        self.agglomerate = self.AGGLOMERATE if agglomerate is None else int(agglomerate)
        dev._check(dev.L.mamg_dist_set_agglomeration(h, self.agglomerate))

    def __del__(self):
        try:
            if self.h:
                self.dev.L.mamg_dist_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def local_ranks(self):
        return list(range(self.world)) if self.rank < 0 else [self.rank]

    def setup(self, A: Csr, w=None, max_levels=40, coarse_factor=40.0, mode=2):
        rp, prp = _i64(A.rp)
        ci, pci = _i64(A.ci)
        v, pv = _f64(A.v)
        pw = None
        if w is not None:
            w, pw = _f64(w)
        cfg = SetupCfg(int(max_levels), int(mode), float(coarse_factor))
        self.dev._check(self.dev.L.mamg_dist_setup(self.h, A.nrows, prp, pci, pv, pw, C.byref(cfg)))
        self.n = A.nrows
        return self

    def load(self, A: Csr, w=None):
        """H2D of this process's row blocks (kept device-resident)."""
        rp, prp = _i64(A.rp)
        ci, pci = _i64(A.ci)
        v, pv = _f64(A.v)
        pw = None
        if w is not None:
            w, pw = _f64(w)
        self.dev._check(self.dev.L.mamg_dist_load(self.h, A.nrows, prp, pci, pv, pw))
        self.n = A.nrows
        return self

    def build(self, max_levels=40, coarse_factor=40.0, mode=2):
        """Partition-aware build_hierarchy on the loaded blocks (device only)."""
        cfg = SetupCfg(int(max_levels), int(mode), float(coarse_factor))
        self.dev._check(self.dev.L.mamg_dist_build(self.h, C.byref(cfg)))
        return self

    def info(self):
        nl, st = C.c_int(), C.c_int()
        ln = np.zeros(64, np.int64)
        lz = np.zeros(64, np.int64)
        z = C.c_int64()
        self.dev.L.mamg_dist_info(self.h, C.byref(nl), ln.ctypes.data_as(I64P),
                                  lz.ctypes.data_as(I64P), C.byref(st), C.byref(z))
        k = nl.value
        return {"nl": k, "sizes": ln[:k].tolist(), "nnz": lz[:k].tolist(), "stalled": bool(st.value),
                "zero_edges": int(z.value)}

    def time(self, what: str = "precond", reps: int = 20, cycle=0, pre=1, post=1,
             coarsest=20) -> float:
        """Device ms per launch (collective): 'sweep' = the level-0 l1-Jacobi
        sweep of the local rows, 'precond' = one cycle from zero with halos."""
        ms = C.c_double()
        cyc = _cycle(cycle, pre, post, coarsest)
        self.dev._check(self.dev.L.mamg_dist_time(self.h, {"sweep": 0, "precond": 1}[what],
                                                  C.byref(cyc), int(reps), C.byref(ms)))
        return ms.value

    def local_shape(self, level: int = 0, rank: int | None = None):
        """(rows, nnz) of a local part's level matrix."""
        nr, nz = C.c_int64(), C.c_int64()
        r = self.local_ranks[0] if rank is None else rank
        self.dev._check(self.dev.L.mamg_dist_level_shape(self.h, r, level, 0, C.byref(nr),
                                                         C.byref(nz)))
        return nr.value, nz.value

    def last_solve(self) -> dict:
        """How the last pcg() ran (mamg_dist_last_solve)."""
        f = (C.c_int * 4)()
        self.dev._check(self.dev.L.mamg_dist_last_solve(self.h, f))
        return {"peer_reduce": bool(f[0]), "peer_halo": bool(f[1]), "overlap": bool(f[2]),
                "graphs": bool(f[3])}

    def bounds(self, level: int):
        out = np.zeros(self.world + 1, np.int64)
        self.dev._check(self.dev.L.mamg_dist_level_bounds(self.h, level, out.ctypes.data_as(I64P)))
        return out.tolist()

    def download(self, rank: int, level: int, which: int):
        nr, nz = C.c_int64(), C.c_int64()
        self.dev._check(self.dev.L.mamg_dist_level_shape(self.h, rank, level, which, C.byref(nr),
                                                         C.byref(nz)))
        rp = np.zeros(nr.value + 1, np.int64)
        ci = np.zeros(max(nz.value, 1), np.int64)
        v = np.zeros(max(nz.value, 1))
        self.dev._check(self.dev.L.mamg_dist_download(self.h, rank, level, which,
                                                      rp.ctypes.data_as(I64P),
                                                      ci.ctypes.data_as(I64P),
                                                      v.ctypes.data_as(F64P)))
        if which >= 3:
            return v[: nr.value].copy()
        return rp, ci[: nz.value].copy(), v[: nz.value].copy()

    def gather_level(self, level: int) -> Level:
        """Full level (all parts must be local: loopback) with global indices."""
        info = self.info()
        nl = info["nl"]

        def cat(which, ncols):
            rps, cis, vs = [0], [], []
            for r in self.local_ranks:
                rp, ci, v = self.download(r, level, which)
                base = rps[-1]
                rps.extend((rp[1:] + base).tolist())
                cis.append(ci)
                vs.append(v)
            return Csr(len(rps) - 1, ncols, np.array(rps, np.int64), np.concatenate(cis),
                       np.concatenate(vs))
        n = info["sizes"][level]
        A = cat(0, n)
        P = R = None
        if level + 1 < nl:
            nc = info["sizes"][level + 1]
            P = cat(1, nc)
            R = cat(2, n)
        l1 = np.concatenate([self.download(r, level, 3) for r in self.local_ranks])
        w = np.concatenate([self.download(r, level, 4) for r in self.local_ranks])
        return Level(A, P, R, l1, w)

    def pcg(self, b=None, rtol=1e-6, itmax=5000, cycle=0, pre=1, post=1, coarsest=20,
            want_u=True, u0=None):
        pb = pu0 = None
        if b is not None:
            b, pb = _f64(b)
        if u0 is not None:
            u0, pu0 = _f64(u0)
        u = np.zeros(self.n if want_u else 1)
        hist = np.zeros(int(itmax) + 2)
        rep = Report()
        cyc = _cycle(cycle, pre, post, coarsest)
        cfg = SolveCfg(float(rtol), int(itmax))
        self.dev._check(self.dev.L.mamg_dist_pcg_x0(self.h, pb, pu0, C.byref(cyc), C.byref(cfg),
                                                    u.ctypes.data_as(F64P) if want_u else None,
                                                    hist.ctypes.data_as(F64P), C.byref(rep)))
        r = rep.as_dict()
        return u, hist[: r["iterations"] + 1].copy(), r

