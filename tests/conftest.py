"""Shared fixtures. `-m gpu` tests need a B200 and call the product through
its C-ABI (paper_1810_04221_b200.capi); the checkers (oracle/) are test
infrastructure only."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: full-size (BASELINE) configurations")


def _ensure_oracle():
    from oracle import oracle as O
    ref_ok, port_ok = O.available()
    if not port_ok:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)
    if not ref_ok and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    return O


@pytest.fixture(scope="session")
def O():
    return _ensure_oracle()


@pytest.fixture(scope="session")
def ref(O):
    return O.Ref()


@pytest.fixture(scope="session")
def port(O):
    return O.Port()


@pytest.fixture(scope="session")
def dev():
    from paper_1810_04221_b200 import Device
    return Device(0)


# ------------------------------------------------------------ generators --
def csr_from_dense(D):
    from oracle.oracle import Csr
    n, m = D.shape
    rp = [0]
    ci, v = [], []
    for i in range(n):
        for j in range(m):
            if D[i, j] != 0.0:
                ci.append(j)
                v.append(D[i, j])
        rp.append(len(ci))
    return Csr(n, m, np.array(rp, np.int64), np.array(ci, np.int64), np.array(v))


def csr_from_rows(n, m, rows):
    """rows: list of dict col->val; columns sorted."""
    from oracle.oracle import Csr
    rp = [0]
    ci, v = [], []
    for r in rows:
        for j in sorted(r):
            ci.append(j)
            v.append(r[j])
        rp.append(len(ci))
    return Csr(n, m, np.array(rp, np.int64), np.array(ci, np.int64), np.array(v, np.float64))


def random_sparse(n, m, per_row, rng):
    rows = []
    for _ in range(n):
        cols = rng.choice(m, size=min(per_row, m), replace=False)
        rows.append({int(j): float(rng.uniform(-1, 1)) for j in cols})
    return csr_from_rows(n, m, rows)


def random_spd(n, off_per_row, rng):
    """Symmetric pattern, mirrored values, diagonal above the row |sums|
    (the reference tests' random_spd, proj/tests/support/generators.hpp:64-85)."""
    rows = [dict() for _ in range(n)]
    rowsum = np.zeros(n)
    for i in range(n):
        want = min(off_per_row, n - 1 - i)
        cols = set()
        while len(cols) < want:
            j = int(rng.integers(0, n))
            if j > i:
                cols.add(j)
        for j in sorted(cols):
            val = float(rng.uniform(-1, 1))
            rows[i][j] = val
            rows[j][i] = val
            rowsum[i] += abs(val)
            rowsum[j] += abs(val)
    for i in range(n):
        rows[i][i] = rowsum[i] + float(rng.uniform(0.5, 2.0))
    return csr_from_rows(n, n, rows)


def random_graph(n, p, rng, wlo=0.05, whi=2.0, discrete=False):
    """Symmetric weighted graph with mirrored weights (generators.hpp:87-114)."""
    adj = [dict() for _ in range(n)]
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < p:
                c = float(rng.uniform(wlo, whi))
                if discrete:
                    c = 1.0 if c < 1.0 else 2.0
                adj[i][j] = c
                adj[j][i] = c
    xadj = [0]
    a, w = [], []
    for v in range(n):
        for u in sorted(adj[v]):
            a.append(u)
            w.append(adj[v][u])
        xadj.append(len(a))
    return np.array(xadj, np.int64), np.array(a, np.int64), np.array(w)


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.int64)


def same_csr(a, b):
    return (a.nrows == b.nrows and a.ncols == b.ncols and np.array_equal(a.rp, b.rp)
            and np.array_equal(a.ci, b.ci) and np.array_equal(bits(a.v), bits(b.v)))
