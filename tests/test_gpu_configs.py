"""GPU parity on BASELINE cfg 3-5 matrix families (27-point anisotropic Q1,
jump-coefficient FV, 3-dof Q1 elasticity) at reduced sizes: hierarchy, cycle
and PCG bit-identical to the reference library on the same matrix. These
stress the long-row paths (G = 32 lane-strided sums, rows > 32 entries,
coarse Galerkin rows of 60-90 entries)."""
import numpy as np
import pytest

import paper_1810_04221_b200 as pkg
from conftest import bits, same_csr

pytestmark = pytest.mark.gpu

SPECS = ["aniso27:32,32,32,0.01", "jump3d:40,40,40,8", "elast3d:16,16,16", "elast3d:24,24,24",
         "aniso27:64,64,64,0.01"]


def load(O, spec):
    A = pkg.from_spec(spec)
    return O.Csr(A.nrows, A.ncols, A.rp, A.ci, A.v)


@pytest.mark.parametrize("spec", SPECS)
def test_hierarchy_and_pcg_bitwise(dev, ref, O, spec):
    A = load(O, spec)
    hd = dev.build_hierarchy(A)
    hr = ref.build_hierarchy(A)
    assert hd.nl == hr.nl and hd.stalled == hr.stalled and hd.zero_edges == hr.zero_edges
    for k, (a, b) in enumerate(zip(hd.levels, hr.levels)):
        assert same_csr(a.A, b.A), (spec, k)
        assert np.array_equal(bits(a.l1), bits(b.l1)), (spec, k)
        assert np.array_equal(bits(a.w), bits(b.w)), (spec, k)
        if b.P is not None:
            assert same_csr(a.P, b.P) and same_csr(a.R, b.R), (spec, k)
    b = np.ones(A.nrows)
    hs = dev.setup(A)
    hk = ref.build_hierarchy(A, keep=True)
    ud, hsd, rd = dev.pcg(A, hs, b)
    ur, hsr, rr = ref.pcg(A, hk, b)
    assert rd["iterations"] == rr["iterations"] and rr["converged"] == 1, spec
    assert np.array_equal(bits(hsd), bits(hsr)), spec
    assert np.array_equal(bits(ud), bits(ur)), spec


def test_spmv_long_rows_every_group(dev, ref, O):
    A = load(O, "elast3d:10,10,10")
    x = np.random.default_rng(3).uniform(-1, 1, A.ncols)
    for g in (0, 1, 2, 4, 8, 16, 32):
        assert np.array_equal(bits(dev.spmv(A, x, g)), bits(ref.spmv(A, x, g))), g


@pytest.mark.parametrize("spec", ["elast3d:12,12,12", "aniso27:20,20,20,0.01"])
def test_wcycle_and_pairwise_mode(dev, ref, O, spec):
    A = load(O, spec)
    hd = dev.build_hierarchy(A, mode=1)
    hr = ref.build_hierarchy(A, mode=1)
    assert hd.nl == hr.nl
    for a, b in zip(hd.levels, hr.levels):
        assert same_csr(a.A, b.A)
    hs = dev.setup(A)
    hk = ref.build_hierarchy(A, keep=True)
    rng = np.random.default_rng(5)
    r = rng.uniform(-1, 1, A.nrows)
    for cyc in (0, 1):
        zd = dev.precond_apply(hs, r, cyc, 1, 1, 20)
        zr = ref.apply_cycle(hk, 0, r, np.zeros(A.nrows), cyc, 1, 1, 20)
        assert np.array_equal(bits(zd), bits(zr)), cyc


def irregular_spd(n, rng, hubs=6, hub_deg=700):
    """SPD with heavy-tailed degrees: a banded core plus random long-range
    couplings and a few hub rows of ~hub_deg entries — exercises the tile
    overflow (global-read) SpMV path, long coarse Galerkin rows (mid and
    CTA-per-row paths) and irregular Suitor candidate lists."""
    import scipy.sparse as sp
    rows, cols, vals = [], [], []
    for off in (1, 2, 17):
        i = np.arange(n - off)
        rows.append(i); cols.append(i + off); vals.append(-rng.uniform(0.2, 1.0, n - off))
    m = 4 * n
    i = rng.integers(0, n, m); j = rng.integers(0, n, m)
    keep = i != j
    rows.append(i[keep]); cols.append(j[keep]); vals.append(-rng.uniform(0.01, 0.3, keep.sum()))
    for h in rng.choice(n, hubs, replace=False):
        j = rng.choice(n, hub_deg, replace=False)
        j = j[j != h]
        rows.append(np.full(j.size, h)); cols.append(j); vals.append(-rng.uniform(0.01, 0.1, j.size))
    r = np.concatenate(rows); c = np.concatenate(cols); v = np.concatenate(vals)
    U = sp.coo_matrix((v, (r, c)), shape=(n, n)).tocsr()
    U.sum_duplicates()
    S = (U + U.T).tocsr()
    S.sort_indices()
    d = np.asarray(abs(S).sum(axis=1)).ravel() + rng.uniform(0.1, 1.0, n)
    A = (S + sp.diags(d)).tocsr()
    A.sort_indices()
    from oracle.oracle import Csr
    return Csr(n, n, A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data.astype(np.float64))


@pytest.mark.parametrize("seed", [1, 2])
def test_irregular_spd_bitwise(dev, ref, seed):
    rng = np.random.default_rng(seed)
    A = irregular_spd(60000, rng)
    hd = dev.build_hierarchy(A)
    hr = ref.build_hierarchy(A)
    assert hd.nl == hr.nl
    for k, (a, b) in enumerate(zip(hd.levels, hr.levels)):
        assert same_csr(a.A, b.A), k
        if b.P is not None:
            assert same_csr(a.P, b.P), k
    x = rng.uniform(-1, 1, A.nrows)
    for g in (0, 8, 32):
        assert np.array_equal(bits(dev.spmv(A, x, g)), bits(ref.spmv(A, x, g))), g
    b = np.ones(A.nrows)
    hs = dev.setup(A)
    hk = ref.build_hierarchy(A, keep=True)
    ud, hsd, rd = dev.pcg(A, hs, b)
    ur, hsr, rr = ref.pcg(A, hk, b)
    assert rd["iterations"] == rr["iterations"] and rr["converged"] == 1
    assert np.array_equal(bits(ud), bits(ur))
