"""Device-side generators: every BASELINE generator
assembled directly on the GPU must equal the host generator's matrix bit for
bit (row pointers, columns, value bits) — the host generators are themselves
pinned to the reference's (tests/test_generators.py)."""
import numpy as np
import pytest

import paper_1810_04221_b200 as pkg
from conftest import bits

pytestmark = pytest.mark.gpu

SPECS = [("poisson2d:37,29", 0), ("poisson2d:512,512", 0), ("ani:33,41,0.01,0.7", 0),
         ("randk3d:12,10,9,0", 0), ("randk3d:12,10,9,1.5", 3), ("randk3d:20,20,20,1", 7),
         ("aniso27:9,8,7,0.01", 0), ("aniso27:16,16,16,1", 0),
         ("jump3d:17,15,13,4", 2), ("jump3d:24,24,24,8", 0),
         ("elast3d:5,6,4", 0), ("elast3d:1,3,3", 0), ("randk3d:160,160,160,0", 0)]


@pytest.mark.parametrize("spec,seed", SPECS)
def test_device_generator_bitwise(dev, spec, seed):
    H = pkg.from_spec(spec, seed)
    D = dev.generate(spec, seed).to_host()
    assert (D.nrows, D.ncols) == (H.nrows, H.ncols), spec
    assert np.array_equal(np.asarray(D.rp, np.int64), np.asarray(H.rp, np.int64)), spec
    assert np.array_equal(np.asarray(D.ci, np.int64), np.asarray(H.ci, np.int64)), spec
    assert np.array_equal(bits(D.v), bits(H.v)), spec


def test_device_generated_matrix_solves_like_uploaded(dev):
    """setup + PCG on a device-generated matrix = on the uploaded host one."""
    spec = "aniso27:24,24,24,0.01"
    dA = dev.generate(spec)
    dB = dev.upload(pkg.from_spec(spec))
    n = dA.shape[0]
    out = []
    for M in (dA, dB):
        h = dev.setup(M)
        b = dev.vec(np.ones(n))
        u = dev.zeros(n)
        rep = dev.pcg_device(M, h, b, u)
        out.append((rep["iterations"], u.to_host()))
    assert out[0][0] == out[1][0] and np.array_equal(bits(out[0][1]), bits(out[1][1]))


def test_device_generator_errors(dev):
    with pytest.raises(pkg.InvalidArgument, match="grid must be"):
        dev.generate("randk3d:1,4,4,0")
    with pytest.raises(ValueError):
        dev.generate("nosuch:3,3")
