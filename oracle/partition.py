"""Partition-aware oracle — TEST INFRASTRUCTURE ONLY.

The reference has no partitioned path. The B200 build's row-block
partitioned setup matches on local graph blocks only, so its parity target is
the reference's own public functions composed as follows (no reference code
is modified): in every pairwise step, build_weights runs on A with the
inter-block entries masked out (diagonal kept), then suitor_match and
pairwise_aggregate; build_prolongator, galerkin_by_aggregates and
restrict_vector use the FULL A (proj/src/coarsening.cpp:163-185). Aggregates
never straddle blocks, so coarse levels stay contiguous row blocks: block r of
the coarse level holds the aggregates led by block r's rows. The level loop
mirrors build_hierarchy (proj/src/coarsening.cpp:194-238).

Agglomeration (the device default): the first level below the finest with at
most `agglom` rows is replicated on every rank, so it and all coarser steps
are unpartitioned (one block [0, n) reported as rank 0's).
"""
from __future__ import annotations

import numpy as np

from .oracle import Csr, Hierarchy, Level, Ref

ALIGN = 2048  # level-0 block boundaries on 2048-row multiples (bit-exact dots)
AGGLOM = 262144  # device default of mamg_dist_set_agglomeration


def partition_bounds(n: int, parts: int, align: int = ALIGN) -> list[int]:
    """Level-0 row-block boundaries: multiples of `align` (the last is n)."""
    b = [0]
    for r in range(1, parts):
        cut = int(np.floor(r * n / parts / align + 0.5)) * align  # llround
        b.append(min(max(cut, b[-1]), n))
    b.append(n)
    return b


def block_of(bounds, n):
    owner = np.zeros(n, np.int64)
    for r in range(len(bounds) - 1):
        owner[bounds[r]:bounds[r + 1]] = r
    return owner


def mask_cross(A: Csr, bounds) -> Csr:
    """A with every entry (i, j) whose row and column lie in different blocks removed."""
    owner = block_of(bounds, A.nrows)
    rows = np.repeat(np.arange(A.nrows), np.diff(A.rp))
    keep = owner[rows] == owner[A.ci]
    rp = np.zeros(A.nrows + 1, np.int64)
    np.add.at(rp, rows[keep] + 1, 1)
    rp = np.cumsum(rp)
    return Csr(A.nrows, A.ncols, rp, A.ci[keep].copy(), A.v[keep].copy())


def pairwise_step(ref: Ref, A: Csr, w, bounds):
    Am = mask_cross(A, bounds)
    xadj, adj, wt, zero = ref.build_weights(Am, w)
    mate = ref.suitor(xadj, adj, wt)
    agg, nc, _, _ = ref.pairwise_aggregate(mate)
    P = ref.build_prolongator(agg, nc, w)
    Ac = ref.galerkin_by_aggregates(A, P)
    wc = ref.restrict_vector(P, w)
    cb = [int(agg[b]) if b < A.nrows else nc for b in bounds[:-1]] + [nc]
    return P, Ac, wc, zero, cb


def double_pairwise(ref: Ref, A: Csr, w, bounds):
    P1, A1, w1, z1, b1 = pairwise_step(ref, A, w, bounds)
    P2, A2, w2, z2, b2 = pairwise_step(ref, A1, w1, b1)
    return ref.spgemm(P1, P2), A2, w2, z1 + z2, b2


def build_hierarchy(ref: Ref, A: Csr, parts: int, w=None, max_levels=40, coarse_factor=40.0,
                    mode=2, keep=True, agglom=AGGLOM):
    """Partition-aware build_hierarchy; returns (Hierarchy, per-level block bounds)."""
    n = A.nrows
    w = np.ones(n) if w is None else np.asarray(w, np.float64)
    bounds = partition_bounds(n, parts)
    bound = coarse_factor * np.cbrt(float(n))
    levels = [Level(A, None, None, ref.l1_diagonal(A), w)]
    all_bounds = [bounds]
    stalled, zero = False, 0
    while float(levels[-1].A.nrows) > bound and len(levels) < max_levels:
        fine = levels[-1]
        if agglom and len(levels) > 1 and fine.A.nrows <= agglom:
            all_bounds[-1] = [0] + [fine.A.nrows] * parts   # replicated from here on
        step = double_pairwise if mode == 2 else pairwise_step
        P, Ac, wc, z, cb = step(ref, fine.A, fine.w, all_bounds[-1])
        zero += z
        if Ac.nrows == fine.A.nrows:
            stalled = True
            break
        fine.P = P
        fine.R = ref.transpose(P)
        levels.append(Level(Ac, None, None, ref.l1_diagonal(Ac), wc))
        all_bounds.append(cb)
    h = Hierarchy(levels, stalled, zero)
    if keep:
        h.handle = ref.hier_from_levels(levels)
    return h, all_bounds
