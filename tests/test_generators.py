"""BASELINE cfg 3-5 generators (new; matchamg/problems.hpp) and the oracle
port on their matrices. CPU-only: the reference library (oracle/_ref) is the
checker for the port; the GPU parity of the same matrices is in
tests/test_gpu_configs.py."""
import numpy as np
import pytest

import paper_1810_04221_b200 as pkg
from conftest import bits, same_csr


def to_oracle(O, A):
    return O.Csr(A.nrows, A.ncols, A.rp, A.ci, A.v)


SPECS = ["aniso27:7,6,5,0.01", "jump3d:12,11,10,4", "elast3d:5,6,4"]


@pytest.mark.parametrize("spec", SPECS)
def test_generator_symmetric_spd_sorted(O, spec):
    A = to_oracle(O, pkg.from_spec(spec, seed=3))
    D = A.to_dense()
    assert np.array_equal(bits(D), bits(D.T))          # exactly symmetric values
    assert np.linalg.eigvalsh(D).min() > 0.0          # SPD
    for i in range(A.nrows):                          # sorted unique columns, diagonal present
        cols = A.ci[A.rp[i]:A.rp[i + 1]]
        assert np.all(np.diff(cols) > 0) and i in cols
    off = D - np.diag(np.diag(D))
    assert np.count_nonzero(off) == A.nnz - A.nrows   # exact zeros dropped off the diagonal


def test_generator_shapes_and_stencils(O):
    A = pkg.gen_anisotropic_3d_q1(9, 9, 9, 1.0, 1.0, 1e-2)
    assert A.nrows == 729 and np.diff(A.rp).max() == 27
    # constant coefficients: an interior row sums to zero (Q1 stiffness kills constants)
    mid = (4 * 9 + 4) * 9 + 4
    assert abs(A.v[A.rp[mid]:A.rp[mid + 1]].sum()) < 1e-12 * A.v[A.rp[mid]:A.rp[mid + 1]].max()
    J = pkg.gen_jump_3d(16, 16, 16, 4, seed=1)
    assert J.nrows == 4096 and np.diff(J.rp).max() == 7
    # the off-diagonal couplings take the harmonic means of {1e-3, 1, 1e3} pairs only
    assert np.unique(np.round(J.v[J.v < 0] / J.v[J.v < 0].min(), 9)).size <= 6
    E = pkg.gen_elasticity_3d(6, 6, 6)
    assert E.nrows == 648 and np.diff(E.rp).max() == 51
    # translations in y are rigid motions: rows of nodes away from the clamp
    # (i >= 1) annihilate u = (0, 1, 0) everywhere
    u = np.zeros(E.nrows)
    u[1::3] = 1.0
    Eo = to_oracle(O, E)
    y = Eo.to_dense() @ u
    nodes = np.arange(E.nrows) // 3
    far = (nodes % 6) >= 1
    assert np.abs(y[far]).max() < 1e-10 * np.abs(E.v).max()


def test_generator_spec_and_errors():
    assert pkg.from_spec("jump3d:8,8,8,2", seed=5).nrows == 512
    a = pkg.from_spec("jump3d:8,8,8,2", seed=5)
    b = pkg.from_spec("jump3d:8,8,8,2", seed=6)
    assert not np.array_equal(a.v, b.v)
    for bad in ("aniso27:1,4,4,0.1", "aniso27:4,4,4,0", "jump3d:4,4,4,0", "elast3d:4,1,4"):
        with pytest.raises(ValueError):
            pkg.from_spec(bad)


@pytest.mark.parametrize("spec", ["aniso27:14,13,12,0.01", "jump3d:20,20,20,4", "elast3d:8,8,8"])
def test_port_matches_reference_on_new_configs(O, ref, port, spec):
    A = to_oracle(O, pkg.from_spec(spec))
    hr = ref.build_hierarchy(A)
    hp = port.build_hierarchy(A)
    assert hr.nl == hp.nl and hr.nl >= 2
    for a, b in zip(hr.levels, hp.levels):
        assert same_csr(a.A, b.A)
        assert np.array_equal(bits(a.w), bits(b.w))
    b = np.ones(A.nrows)
    hr = ref.build_hierarchy(A, keep=True)
    hp = port.build_hierarchy(A, keep=True)
    ur, histr, rr = ref.pcg(A, hr, b)
    up, histp, rp = port.pcg(A, hp, b)
    assert rr["iterations"] == rp["iterations"] and rr["converged"] == 1
    assert np.array_equal(bits(ur), bits(up))
