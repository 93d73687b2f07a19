"""MatrixMarket I/O (matchamg/matrix_market.hpp, the input side of the path):
the parallel reader/writer of the host library against the reference
library's own read_matrix_market / write_matrix_market (oracle/_ref), and the
reference tests' cases (proj/tests/test_problems_io.cpp:133-238). CPU only."""
import os

import numpy as np
import pytest

import paper_1810_04221_b200 as pkg
from conftest import bits, random_sparse, random_spd, same_csr


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_reference_cases(tmp_path):
    p = write(tmp_path, "one.mtx", "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 2.0\n")
    A = pkg.read_matrix_market(p)
    assert A.nrows == 1 and len(A.v) == 1 and A.v[0] == 2.0
    p = write(tmp_path, "sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n"
              "% lower triangle only\n3 3 4\n1 1 2.0\n2 1 -1.0\n2 2 2.0\n3 3 2.0\n")
    A = pkg.read_matrix_market(p)
    assert A.rp.tolist() == [0, 2, 4, 5] and A.ci.tolist() == [0, 1, 0, 1, 2]
    assert A.v.tolist() == [2.0, -1.0, -1.0, 2.0, 2.0]
    p = write(tmp_path, "dup.mtx", "%%MatrixMarket matrix coordinate real general\n"
              "2 2 3\n1 2 1.5\n1 2 0.25\n2 2 1.0\n")
    A = pkg.read_matrix_market(p)
    assert len(A.v) == 2 and A.v[0] == 1.75
    p = write(tmp_path, "bad.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(pkg.MatrixMarketError, match=":3:"):
        pkg.read_matrix_market(p)
    p = write(tmp_path, "badh.mtx", "%%MatrixMarket matrix array real general\n2 2\n")
    with pytest.raises(pkg.MatrixMarketError):
        pkg.read_matrix_market(p)
    with pytest.raises(pkg.MatrixMarketError, match="cannot open"):
        pkg.read_matrix_market("/nonexistent/missing.mtx")


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 2.0\n",
    "%%MatrixMarket matrix coordinate real general\n% c\n\n2 2 1\n\n1 1 +1.5e3\n",
    "%%MatrixMarket matrix coordinate real general\r\n2 2 2\r\n1 1 1.0\r\n2 2 -0.5\r\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n",
])
def test_messages_and_values_match_reference(tmp_path, ref, O, text):
    p = write(tmp_path, "case.mtx", text)
    try:
        r = ref.read_mm(p)
        rerr = None
    except O.OracleError as e:
        r, rerr = None, str(e)
    try:
        d = pkg.read_matrix_market(p)
        derr = None
    except pkg.MatrixMarketError as e:
        d, derr = None, str(e)
    assert (rerr is None) == (derr is None), (rerr, derr)
    if rerr is None:
        assert same_csr(O.Csr(d.nrows, d.ncols, d.rp, d.ci, d.v), r)
    else:
        assert derr in rerr or rerr.endswith(derr), (rerr, derr)


def test_round_trip_and_reference_bitwise(tmp_path, ref, O):
    rng = np.random.default_rng(4)
    for A, sym in [(random_sparse(300, 300, 6, rng), False), (random_spd(200, 4, rng), True),
                   (ref.gen_randk3d(20, 20, 20, 1.0, 3), True)]:
        p = str(tmp_path / "a.mtx")
        q = str(tmp_path / "b.mtx")
        pkg.write_matrix_market(A, p, symmetric=sym)
        ref.write_mm(A, q, symmetric=sym)
        assert open(p, "rb").read() == open(q, "rb").read()   # identical text
        d = pkg.read_matrix_market(p)
        r = ref.read_mm(p)
        assert same_csr(O.Csr(d.nrows, d.ncols, d.rp, d.ci, d.v), r)
        assert same_csr(r, A)


def test_large_parallel_read_with_duplicates(tmp_path, ref, O):
    # many body chunks (> 1 MiB) plus duplicate entries: the duplicate sums
    # follow the reference's from_triplets order
    rng = np.random.default_rng(7)
    n, m = 4000, 60000
    i = rng.integers(1, n + 1, m)
    j = rng.integers(1, n + 1, m)
    v = rng.uniform(-1, 1, m)
    lines = [f"{a} {b} {c:.17g}" for a, b, c in zip(i, j, v)]
    p = write(tmp_path, "big.mtx", "%%MatrixMarket matrix coordinate real general\n"
              f"{n} {n} {m}\n" + "\n".join(lines) + "\n")
    d = pkg.read_matrix_market(p)
    r = ref.read_mm(p)
    assert same_csr(O.Csr(d.nrows, d.ncols, d.rp, d.ci, d.v), r)
