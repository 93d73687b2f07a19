"""Model-problem generators (proj/include/matchamg/problems.hpp) through the
host library's C entry points (include/mamg_host.h). Bit-identical to the
reference's generators; these are the inputs of every bench and parity run."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .capi import Csr, HERE

HOST_LIB = os.path.join(HERE, "csrc", "lib", "libmatchamg.so")


class _HostCsr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("rp", C.POINTER(C.c_int64)), ("ci", C.POINTER(C.c_int64)),
                ("v", C.POINTER(C.c_double))]


_L = None


def _lib():
    global _L
    if _L is None:
        if not os.path.exists(HOST_LIB):
            raise ImportError(f"{HOST_LIB} missing: run __graft_entry__.build()")
        L = C.CDLL(HOST_LIB)
        L.mamg_gen_poisson2d.argtypes = [C.c_int64, C.c_int64, C.POINTER(_HostCsr)]
        L.mamg_gen_aniso2d.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double,
                                       C.POINTER(_HostCsr)]
        L.mamg_gen_randk3d.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                                       C.POINTER(_HostCsr)]
        L.mamg_gen_aniso27.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                       C.c_double, C.POINTER(_HostCsr)]
        L.mamg_gen_jump3d.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                      C.c_double, C.c_double, C.POINTER(_HostCsr)]
        L.mamg_gen_elast3d.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                       C.POINTER(_HostCsr)]
        L.mamg_read_mm.argtypes = [C.c_char_p, C.POINTER(_HostCsr)]
        L.mamg_write_mm.argtypes = [C.c_int64, C.c_int64, C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_char_p,
                                    C.c_int]
        L.mamg_host_csr_free.argtypes = [C.POINTER(_HostCsr)]
        L.mamg_host_last_error.restype = C.c_char_p
        _L = L
    return _L


def _take(st, h: _HostCsr) -> Csr:
    L = _lib()
    if st != 0:
        raise ValueError(L.mamg_host_last_error().decode())
    n, nz = h.nrows, h.nnz
    rp = np.ctypeslib.as_array(h.rp, shape=(n + 1,)).copy()
    ci = np.ctypeslib.as_array(h.ci, shape=(max(nz, 1),))[:nz].copy()
    v = np.ctypeslib.as_array(h.v, shape=(max(nz, 1),))[:nz].copy()
    L.mamg_host_csr_free(C.byref(h))
    return Csr(n, h.ncols, rp, ci, v)


def gen_poisson_2d(nx: int, ny: int) -> Csr:
    """proj/src/problems.cpp:67-69 (5-point Laplacian)."""
    h = _HostCsr()
    return _take(_lib().mamg_gen_poisson2d(nx, ny, C.byref(h)), h)


def gen_anisotropic_2d(nx: int, ny: int, epsilon: float, theta: float) -> Csr:
    """proj/src/problems.cpp:58-65 (9-point anisotropic stencil)."""
    h = _HostCsr()
    return _take(_lib().mamg_gen_aniso2d(nx, ny, epsilon, theta, C.byref(h)), h)


def gen_poisson_3d_randk(nx: int, ny: int, nz: int, sigma: float = 1.0, seed: int = 0) -> Csr:
    """proj/src/problems.cpp:115-193 (FV, lognormal permeability; sigma=0 -> 7-point)."""
    h = _HostCsr()
    return _take(_lib().mamg_gen_randk3d(nx, ny, nz, sigma, seed, C.byref(h)), h)


def gen_anisotropic_3d_q1(nx: int, ny: int, nz: int, kx: float = 1.0, ky: float = 1.0,
                          kz: float = 1.0) -> Csr:
    """BASELINE cfg 3: Q1 27-point -div(K grad u), K = diag(kx, ky, kz), Dirichlet (new)."""
    h = _HostCsr()
    return _take(_lib().mamg_gen_aniso27(nx, ny, nz, kx, ky, kz, C.byref(h)), h)


def gen_jump_3d(nx: int, ny: int, nz: int, block: int = 8, seed: int = 0, lo: float = 1e-3,
                hi: float = 1e3) -> Csr:
    """BASELINE cfg 4: 7-point FV with K in {lo, 1, hi} on seeded block^3 sub-cubes (new)."""
    h = _HostCsr()
    return _take(_lib().mamg_gen_jump3d(nx, ny, nz, block, seed, lo, hi, C.byref(h)), h)


def gen_elasticity_3d(nx: int, ny: int, nz: int, mu: float = 0.42, lam: float = 1.7) -> Csr:
    """BASELINE cfg 5: Q1 Lame elasticity, 3 interleaved dofs per node, clamped x=0 (new)."""
    h = _HostCsr()
    return _take(_lib().mamg_gen_elast3d(nx, ny, nz, mu, lam, C.byref(h)), h)


class MatrixMarketError(RuntimeError):
    """read/write_matrix_market failures (std::runtime_error in the C++ API)."""


def read_matrix_market(path: str) -> Csr:
    """matchamg::read_matrix_market (proj/include/matchamg/matrix_market.hpp)."""
    L = _lib()
    h = _HostCsr()
    st = L.mamg_read_mm(os.fsencode(path), C.byref(h))
    if st == 2:
        raise MatrixMarketError(L.mamg_host_last_error().decode())
    return _take(st, h)


def write_matrix_market(A: Csr, path: str, symmetric: bool = False) -> None:
    """matchamg::write_matrix_market (%.16e values, exact round trip)."""
    L = _lib()
    rp = np.ascontiguousarray(A.rp, dtype=np.int64)
    ci = np.ascontiguousarray(A.ci, dtype=np.int64)
    v = np.ascontiguousarray(A.v, dtype=np.float64)
    st = L.mamg_write_mm(A.nrows, A.ncols, rp.ctypes.data_as(C.POINTER(C.c_int64)),
                         ci.ctypes.data_as(C.POINTER(C.c_int64)),
                         v.ctypes.data_as(C.POINTER(C.c_double)), os.fsencode(path),
                         1 if symmetric else 0)
    if st == 1:
        raise ValueError(L.mamg_host_last_error().decode())
    if st == 2:
        raise MatrixMarketError(L.mamg_host_last_error().decode())


def from_spec(spec: str, seed: int = 0) -> Csr:
    """cli::matrix_from_gen_spec grammar (proj/src/cli.cpp:203-240):
    "poisson2d:NX,NY", "ani:NX,NY,EPS,THETA", "randk3d:NX,NY,NZ,SIGMA"; extended with
    the BASELINE cfg 3-5 generators "aniso27:NX,NY,NZ,EPS" (K = diag(1,1,EPS)),
    "jump3d:NX,NY,NZ,BLOCK" and "elast3d:NX,NY,NZ"."""
    kind, _, args = spec.partition(":")
    a = args.split(",") if args else []
    if kind == "poisson2d" and len(a) == 2:
        return gen_poisson_2d(int(a[0]), int(a[1]))
    if kind == "ani" and len(a) == 4:
        return gen_anisotropic_2d(int(a[0]), int(a[1]), float(a[2]), float(a[3]))
    if kind == "randk3d" and len(a) == 4:
        return gen_poisson_3d_randk(int(a[0]), int(a[1]), int(a[2]), float(a[3]), seed)
    if kind == "aniso27" and len(a) == 4:
        return gen_anisotropic_3d_q1(int(a[0]), int(a[1]), int(a[2]), 1.0, 1.0, float(a[3]))
    if kind == "jump3d" and len(a) == 4:
        return gen_jump_3d(int(a[0]), int(a[1]), int(a[2]), int(a[3]), seed)
    if kind == "elast3d" and len(a) == 3:
        return gen_elasticity_3d(int(a[0]), int(a[1]), int(a[2]))
    raise ValueError(f"bad generator spec `{spec}`")
