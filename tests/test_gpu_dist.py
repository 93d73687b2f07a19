"""GPU parity of the row-block partitioned path run with the
in-process loopback transport (all parts on the one available B200): every
level's A, P, R, l1 and w and the whole PCG trajectory must be bit-identical
to the partition-aware oracle — the reference's own functions composed with
masked matching (oracle/partition.py)."""
import numpy as np
import pytest

from conftest import bits, same_csr

pytestmark = pytest.mark.gpu

CASES = [("poisson2d:96x96", lambda r: r.gen_poisson2d(96, 96)),
         ("poisson2d:512x512", lambda r: r.gen_poisson2d(512, 512)),
         ("randk3d:24^3 s=1", lambda r: r.gen_randk3d(24, 24, 24, 1.0, 0)),
         ("randk3d:48^3 s=1", lambda r: r.gen_randk3d(48, 48, 48, 1.0, 0)),
         ("ani:128x128", lambda r: r.gen_aniso2d(128, 128, 1e-2, 0.4))]


@pytest.mark.parametrize("agglom", [0, 4096, None])
@pytest.mark.parametrize("parts", [2, 4])
@pytest.mark.parametrize("name,gen", CASES)
def test_partitioned_hierarchy_and_pcg_bitwise(dev, ref, name, gen, parts, agglom):
    """agglom: 0 = every level partitioned; 4096 / None (default 262144) = the
    coarse levels from the first one at or below that size replicated."""
    from oracle import partition as PA
    import paper_1810_04221_b200 as pkg
    A = gen(ref)
    ag = PA.AGGLOM if agglom is None else agglom
    ho, obounds = PA.build_hierarchy(ref, A, parts, agglom=ag)
    d = pkg.Dist(dev, parts, agglomerate=agglom).setup(A)
    info = d.info()
    assert info["nl"] == ho.nl, (name, parts)
    assert info["sizes"] == [L.A.nrows for L in ho.levels]
    assert info["zero_edges"] == ho.zero_edges and info["stalled"] == ho.stalled
    for k in range(ho.nl):
        assert d.bounds(k) == obounds[k], (name, parts, k)
        g = d.gather_level(k)
        o = ho.levels[k]
        assert same_csr(g.A, o.A), (name, parts, k)
        assert np.array_equal(bits(g.l1), bits(o.l1)) and np.array_equal(bits(g.w), bits(o.w))
        if o.P is not None:
            assert same_csr(g.P, o.P) and same_csr(g.R, o.R), (name, parts, k)
    b = np.ones(A.nrows)
    ud, hd, rd = d.pcg()
    uo, hsto, ro = ref.pcg(A, ho, b)
    assert rd["iterations"] == ro["iterations"], (name, parts)
    assert np.array_equal(bits(hd), bits(hsto)) and np.array_equal(bits(ud), bits(uo))


def test_partitioned_one_part_equals_unpartitioned(dev, ref):
    import paper_1810_04221_b200 as pkg
    A = ref.gen_randk3d(20, 20, 20, 1.0, 3)
    d = pkg.Dist(dev, 1).setup(A)
    ud, hd, rd = d.pcg()
    ur, hr, rr = ref.pcg(A, ref.build_hierarchy(A, keep=True), np.ones(A.nrows))
    assert rd["iterations"] == rr["iterations"] and np.array_equal(bits(ud), bits(ur))


@pytest.mark.parametrize("parts", [4, 8])
def test_partitioned_wcycle_and_empty_parts(dev, ref, parts):
    """1600 rows < 2048: at 4 parts parts 1..3 are empty, at 8 parts all but
    part 6 (part 0 empty: the sweeps' halo decision must not hinge on it)."""
    from oracle import partition as PA
    import paper_1810_04221_b200 as pkg
    A = ref.gen_poisson2d(40, 40)
    ho, _ = PA.build_hierarchy(ref, A, parts, agglom=0)
    d = pkg.Dist(dev, parts, agglomerate=0).setup(A)
    for cycle in (1, 0):
        ud, hd, rd = d.pcg(cycle=cycle)
        uo, ho_hist, ro = ref.pcg(A, ho, np.ones(A.nrows), cycle=cycle)
        assert rd["iterations"] == ro["iterations"] and np.array_equal(bits(ud), bits(uo))


def test_partitioned_rejects_asymmetric_pattern(dev):
    import paper_1810_04221_b200 as pkg
    from conftest import csr_from_rows
    n = 5000
    rows = [{i: 4.0} for i in range(n)]
    rows[10][4500] = -1.0   # cross-part entry without its mirror
    A = csr_from_rows(n, n, rows)
    with pytest.raises(pkg.InvalidArgument, match="not symmetric"):
        pkg.Dist(dev, 2).setup(A)


def test_nccl_transport_single_rank(dev, ref):
    """The NCCL transport (rank >= 0) with world = 1 on the one GPU: exercises
    ncclCommInitRank / allgather / broadcast paths end to end."""
    import paper_1810_04221_b200 as pkg
    A = ref.gen_randk3d(16, 16, 16, 1.0, 2)
    d = pkg.Dist(dev, 1, 0, pkg.nccl_unique_id()).setup(A)
    ud, hd, rd = d.pcg()
    ur, hr, rr = ref.pcg(A, ref.build_hierarchy(A, keep=True), np.ones(A.nrows))
    assert rd["iterations"] == rr["iterations"] and np.array_equal(bits(ud), bits(ur))


def test_partitioned_load_then_rebuild(dev, ref):
    """load once, build twice (bench protocol): identical hierarchies and solves."""
    import paper_1810_04221_b200 as pkg
    A = ref.gen_poisson2d(128, 128)
    d = pkg.Dist(dev, 2).load(A)
    d.build()
    u1, h1, r1 = d.pcg()
    d.build()
    u2, h2, r2 = d.pcg(want_u=True)
    assert r1["iterations"] == r2["iterations"] and np.array_equal(bits(u1), bits(u2))


# ---- global (cross-part) matching, SURVEY.md §8f rank 1 -------------------
# One Suitor over the whole graph (suitor words addressed across parts), so
# the mate array is the unpartitioned one and aggregates straddle parts: the
# hierarchy and the PCG must equal the UNPARTITIONED reference bit for bit
# at every part count.
GCASES = CASES + [("aniso27:16^3", lambda r: _pk().gen_anisotropic_3d_q1(16, 16, 16, 1.0, 1.0, 1e-2)),
                  ("elast3d:6^3", lambda r: _pk().gen_elasticity_3d(6, 6, 6))]


def _pk():
    import paper_1810_04221_b200 as pkg
    return pkg


def _check_global(dev, ref, A, parts, cycle=0, agglom=None):
    import paper_1810_04221_b200 as pkg
    ho = ref.build_hierarchy(A, keep=True)
    d = pkg.Dist(dev, parts, matching="global", agglomerate=agglom).setup(A)
    info = d.info()
    assert info["nl"] == ho.nl
    assert info["sizes"] == [L.A.nrows for L in ho.levels]
    assert info["zero_edges"] == ho.zero_edges and info["stalled"] == ho.stalled
    for k in range(ho.nl):
        g = d.gather_level(k)
        o = ho.levels[k]
        assert same_csr(g.A, o.A), k
        assert np.array_equal(bits(g.l1), bits(o.l1)) and np.array_equal(bits(g.w), bits(o.w)), k
        if o.P is not None:
            assert same_csr(g.P, o.P), k
            assert same_csr(g.R, o.R), k
    b = np.ones(A.nrows)
    ud, hd, rd = d.pcg(cycle=cycle)
    uo, hsto, ro = ref.pcg(A, ho, b, cycle=cycle)
    assert rd["iterations"] == ro["iterations"]
    assert np.array_equal(bits(hd), bits(hsto)) and np.array_equal(bits(ud), bits(uo))


@pytest.mark.parametrize("agglom", [0, None])
@pytest.mark.parametrize("parts", [2, 3, 4, 8])
@pytest.mark.parametrize("name,gen", GCASES)
def test_global_matching_equals_unpartitioned(dev, ref, name, gen, parts, agglom):
    _check_global(dev, ref, gen(ref), parts, agglom=agglom)


def test_global_matching_wcycle_pairwise_and_empty_parts(dev, ref):
    import paper_1810_04221_b200 as pkg
    _check_global(dev, ref, ref.gen_poisson2d(40, 40), 4, cycle=1)   # parts 1..3 empty
    _check_global(dev, ref, ref.gen_poisson2d(40, 40), 8, cycle=1, agglom=0)  # part 0 empty
    _check_global(dev, ref, ref.gen_randk3d(24, 24, 24, 1.0, 1), 4, cycle=1, agglom=2000)
    A = ref.gen_randk3d(20, 20, 20, 1.0, 5)
    ho = ref.build_hierarchy(A, mode=1, keep=True)
    d = pkg.Dist(dev, 3, matching="global").setup(A, mode=1)
    assert d.info()["sizes"] == [L.A.nrows for L in ho.levels]
    ud, hd, rd = d.pcg()
    uo, _, ro = ref.pcg(A, ho, np.ones(A.nrows))
    assert rd["iterations"] == ro["iterations"] and np.array_equal(bits(ud), bits(uo))


def test_global_matching_differs_from_local_on_cfg2_family(dev, ref):
    """Local-block matching changes the hierarchy (iteration delta); global
    matching restores the unpartitioned one."""
    import paper_1810_04221_b200 as pkg
    A = ref.gen_randk3d(32, 32, 32, 0.0, 0)
    loc = pkg.Dist(dev, 4).setup(A).info()
    glo = pkg.Dist(dev, 4, matching="global").setup(A).info()
    ho = ref.build_hierarchy(A)
    assert glo["sizes"] == [L.A.nrows for L in ho.levels]
    assert loc["sizes"] != glo["sizes"]


@pytest.mark.parametrize("peer", [False, True])
def test_global_matching_nccl_single_rank(dev, ref, peer, monkeypatch):
    """NCCL transport with world = 1: the IPC shared-block and barrier paths
    (global Suitor; with MAMG_DIST_PEER=1 also the peer reductions, halo
    mailboxes and agglomeration gather, which world = 1 skips by default)."""
    import paper_1810_04221_b200 as pkg
    if peer:
        monkeypatch.setenv("MAMG_DIST_PEER", "1")
    A = ref.gen_randk3d(40, 40, 40, 1.0, 2)
    d = pkg.Dist(dev, 1, 0, pkg.nccl_unique_id(), matching="global", agglomerate=8000).setup(A)
    ud, hd, rd = d.pcg()
    ur, hr, rr = ref.pcg(A, ref.build_hierarchy(A, keep=True), np.ones(A.nrows))
    assert rd["iterations"] == rr["iterations"] and np.array_equal(bits(ud), bits(ur))


@pytest.mark.parametrize("agglom", [0, None])
@pytest.mark.parametrize("parts", [3, 8])
def test_irregular_spd_partitioned_both_matchings(dev, ref, parts, agglom):
    """Random long-range couplings and hub rows: every part exchanges with
    every other (halo plans, tplan, straddling aggregates between far parts,
    hub rows in the shipped Galerkin rows)."""
    from oracle import partition as PA
    import paper_1810_04221_b200 as pkg
    from test_gpu_configs import irregular_spd
    A = irregular_spd(30000, np.random.default_rng(parts), hubs=4, hub_deg=400)
    _check_global(dev, ref, A, parts, agglom=agglom)
    ag = PA.AGGLOM if agglom is None else agglom
    ho, obounds = PA.build_hierarchy(ref, A, parts, agglom=ag)
    d = pkg.Dist(dev, parts, agglomerate=agglom).setup(A)
    assert d.info()["sizes"] == [L.A.nrows for L in ho.levels]
    for k in range(ho.nl):
        assert d.bounds(k) == obounds[k]
        g = d.gather_level(k)
        assert same_csr(g.A, ho.levels[k].A), k
    ud, hd, rd = d.pcg()
    uo, _, ro = ref.pcg(A, ho, np.ones(A.nrows))
    assert rd["iterations"] == ro["iterations"] and np.array_equal(bits(ud), bits(uo))


@pytest.mark.parametrize("matching", ["local", "global"])
def test_bench_partitioned_branch_runs(matching):
    """bench.py's N > 1 branch (run_partitioned) at one GPU (--partitioned:
    NCCL transport, world = 1): the contract keys of its JSON line are there
    and the solve converges as on the single-device path."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--partitioned",
                        "--matching", matching, "--config", "cfg1", "--steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["iterations"] == 59 and d["gpu_launches"] > 0
    assert d["matching"] == matching
    for k in ("roofline", "vcycle", "setup_cold_s", "strong_scaling_same_run", "parity"):
        assert k in d, k
    assert d["parity"]["iterations"] == d["parity"]["iterations_ref"]
    assert d["parity"]["history_bitwise"] and d["parity"]["solution_bitwise_equal"]


@pytest.mark.parametrize("matching", ["local", "global"])
def test_partitioned_check_failures_name_global_rows(dev, ref, matching):
    """A check failure inside one part (non-positive diagonal in part 1's
    rows) is raised with the reference's message and the GLOBAL row."""
    import paper_1810_04221_b200 as pkg
    A = ref.gen_poisson2d(64, 64)          # 4096 rows: parts [0, 2048), [2048, 4096)
    v = A.v.copy()
    row = 3000
    for k in range(A.rp[row], A.rp[row + 1]):
        if A.ci[k] == row:
            v[k] = -1.0
    from oracle.oracle import Csr
    B = Csr(A.nrows, A.ncols, A.rp, A.ci, v)
    with pytest.raises(pkg.InvalidArgument, match=f"row {row}"):
        pkg.Dist(dev, 2, matching=matching, agglomerate=0).setup(B)


@pytest.mark.parametrize("spec", ["aniso27:48,48,48,0.01", "elast3d:16,16,16", "jump3d:48,48,48,8"])
@pytest.mark.parametrize("parts,agglom", [(3, 0), (4, None), (8, 0)])
def test_global_matching_medium_cfg_families(dev, spec, parts, agglom):
    """BASELINE cfg 3-5 families at medium size: global matching on the
    partitioned path reproduces the single-device hierarchy sizes, iteration
    count and solution bits (the single-device path is bitwise to the
    reference; tests/test_gpu_configs.py)."""
    import paper_1810_04221_b200 as pkg
    A = pkg.from_spec(spec)
    u1, h1, r1 = dev.solve_host(A)
    d = pkg.Dist(dev, parts, matching="global", agglomerate=agglom).setup(A)
    ud, hd, rd = d.pcg()
    assert rd["iterations"] == r1["iterations"], spec
    assert np.array_equal(bits(hd), bits(h1)) and np.array_equal(bits(ud), bits(u1)), spec


@pytest.mark.parametrize("name,gen", CASES[1:4])
@pytest.mark.parametrize("matching", ["local", "global"])
def test_halo_interior_overlap_bitwise(dev, ref, name, gen, matching, monkeypatch):
    """Halos on a second stream overlapped with every part's interior rows
    (forced on the loopback; default where halos cross GPUs): solution and
    history bits unchanged."""
    import paper_1810_04221_b200 as pkg
    A = gen(ref)
    base = pkg.Dist(dev, 4, matching=matching, agglomerate=0).setup(A).pcg()
    monkeypatch.setenv("MAMG_DIST_OVERLAP", "1")
    d = pkg.Dist(dev, 4, matching=matching, agglomerate=0).setup(A)
    for cycle in (0, 1):
        ub, hb, rb = base if cycle == 0 else pkg.Dist(dev, 4, matching=matching,
                                                     agglomerate=0).setup(A).pcg(cycle=1)
        uo, ho, ro = d.pcg(cycle=cycle)
        assert ro["iterations"] == rb["iterations"], (name, cycle)
        assert np.array_equal(bits(uo), bits(ub)) and np.array_equal(bits(ho), bits(hb)), (name, cycle)


@pytest.mark.parametrize("parts", [3, 8])
@pytest.mark.parametrize("name,gen", [CASES[1], CASES[3], CASES[4]])
def test_local_matching_oracle_more_parts(dev, ref, name, gen, parts):
    """Local matching vs the partition-aware oracle at 3 and 8 parts
    (hierarchy, history and solution bits)."""
    from oracle import partition as PA
    import paper_1810_04221_b200 as pkg
    A = gen(ref)
    ho, obounds = PA.build_hierarchy(ref, A, parts, agglom=PA.AGGLOM)
    d = pkg.Dist(dev, parts).setup(A)
    assert d.info()["sizes"] == [L.A.nrows for L in ho.levels]
    for k in range(ho.nl):
        assert d.bounds(k) == obounds[k], (name, parts, k)
        assert same_csr(d.gather_level(k).A, ho.levels[k].A), (name, parts, k)
    ud, hd, rd = d.pcg()
    uo, hsto, ro = ref.pcg(A, ho, np.ones(A.nrows))
    assert rd["iterations"] == ro["iterations"]
    assert np.array_equal(bits(hd), bits(hsto)) and np.array_equal(bits(ud), bits(uo))


@pytest.mark.parametrize("parts", [5, 7, 16])
def test_global_matching_odd_and_max_part_counts(dev, ref, parts):
    _check_global(dev, ref, ref.gen_randk3d(40, 40, 40, 1.0, 4), parts, agglom=0)


@pytest.mark.parametrize("matching", ["local", "global"])
def test_partitioned_pairwise_mode_and_custom_w(dev, ref, matching):
    """Pairwise (single-step) aggregation and a non-constant smooth vector w
    through the partitioned build: local matching vs the partition oracle,
    global matching vs the unpartitioned reference."""
    from oracle import partition as PA
    import paper_1810_04221_b200 as pkg
    A = ref.gen_randk3d(24, 24, 24, 1.0, 9)
    w = 1.0 + 0.5 * np.sin(np.arange(A.nrows) * 0.37)
    for mode in (1, 2):
        if matching == "local":
            ho, _ = PA.build_hierarchy(ref, A, 3, w=w, mode=mode, agglom=0)
        else:
            ho = ref.build_hierarchy(A, w=w, mode=mode, keep=True)
        d = pkg.Dist(dev, 3, matching=matching, agglomerate=0).setup(A, w=w, mode=mode)
        assert d.info()["sizes"] == [L.A.nrows for L in ho.levels], mode
        for k in range(ho.nl):
            g = d.gather_level(k)
            assert same_csr(g.A, ho.levels[k].A), (mode, k)
            assert np.array_equal(bits(g.w), bits(ho.levels[k].w)), (mode, k)
        ud, hd, rd = d.pcg()
        uo, _, ro = ref.pcg(A, ho, np.ones(A.nrows))
        assert rd["iterations"] == ro["iterations"] and np.array_equal(bits(ud), bits(uo)), mode
