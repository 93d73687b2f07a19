"""BASELINE-size parity (north star: bit-exact aggregates and coarse-matrix
patterns at 160^3). Builds the cfg-2 hierarchy (3D 7-point Poisson 160^3,
4,096,000 rows, the reference's own generator) on the device and compares
EVERY level with the reference library's (proj/src/coarsening.cpp:194-242):
A (pattern and value bits), P (the aggregates and the prolongator values),
R, l1 and w — then the full PCG solve (iterations, history, solution bits).
The cfg-1 2D case runs the same check (latency-bound size)."""
import numpy as np
import pytest

from conftest import bits, same_csr

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("spec", [("randk3d", (160, 160, 160, 0.0, 0)), ("poisson2d", (512, 512))])
def test_baseline_hierarchy_every_level_bitwise(dev, ref, spec):
    kind, args = spec
    A = ref.gen_randk3d(*args) if kind == "randk3d" else ref.gen_poisson2d(*args)
    hr = ref.build_hierarchy(A)
    hd = dev.build_hierarchy(A)
    assert hd.nl == hr.nl and hd.stalled == hr.stalled and hd.zero_edges == hr.zero_edges
    for k, (a, b) in enumerate(zip(hd.levels, hr.levels)):
        assert a.A.nrows == b.A.nrows and a.A.nnz == b.A.nnz, k
        assert same_csr(a.A, b.A), k
        assert np.array_equal(bits(a.l1), bits(b.l1)), k
        assert np.array_equal(bits(a.w), bits(b.w)), k
        if b.P is not None:
            assert same_csr(a.P, b.P) and same_csr(a.R, b.R), k
    del hr, hd
    b = np.ones(A.nrows)
    hs = dev.setup(A)
    hk = ref.build_hierarchy(A, keep=True)
    ud, hsd, rd = dev.pcg(A, hs, b)
    ur, hsr, rr = ref.pcg(A, hk, b)
    assert rd["iterations"] == rr["iterations"] and rr["converged"] == 1
    assert np.array_equal(bits(hsd), bits(hsr))
    assert np.array_equal(bits(ud), bits(ur))


def test_large_block_recycling_across_contexts(ref):
    """Large device blocks (>= 32 MB) are recycled per context stream
    (bigblock.cu). Two contexts build hierarchies of a 6.9M-entry matrix
    alternately (its values alone are 55 MB), one context is destroyed in
    between (its cached blocks are freed), and every hierarchy stays
    bit-identical to the reference's."""
    import paper_1810_04221_b200 as pkg
    A = ref.gen_randk3d(100, 100, 100, 0.0, 0)
    hr = ref.build_hierarchy(A)

    def check(d):
        hd = d.build_hierarchy(A)
        assert hd.nl == hr.nl
        for a, b in zip(hd.levels, hr.levels):
            assert same_csr(a.A, b.A)
            if b.P is not None:
                assert same_csr(a.P, b.P)

    d1, d2 = pkg.Device(0), pkg.Device(0)
    check(d1)
    check(d2)
    check(d1)
    d1.close()
    check(d2)
    d3 = pkg.Device(0)
    check(d3)
    check(d2)
    d2.close()
    d3.close()


def test_more_than_2pow30_entries(dev):
    """1.1e9 entries (3D 7-point 540^3, assembled on the device): the row
    bisections' midpoints stay in int32 past 2^30 entry offsets (a setup of
    >= 1.07e9 entries used to hang). Pinned against the row-block partitioned
    build of the same matrix (two parts of 5.5e8 entries, global matching —
    bit-identical by construction): level sizes, iterations, final residual."""
    import numpy as np
    dA = dev.generate("randk3d:540,540,540,0")
    assert dA.shape[2] == 1100498400
    dh = dev.setup(dA)
    sizes = [dh.level_matrix("A", k).shape[0] for k in range(dh.nl)]
    assert sizes == [157464000, 39366005, 9841802, 2460637, 616259, 154521, 38903, 9799]
    n = dA.shape[0]
    rep = dev.pcg_device(dA, dh, dev.vec(np.ones(n)), dev.zeros(n))
    assert rep["iterations"] == 89 and rep["converged"]
    assert abs(rep["final_relres"] - 8.464e-07) < 1e-10
    del dh, dA
