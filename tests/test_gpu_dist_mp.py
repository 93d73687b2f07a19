"""The partitioned path across PROCESSES: one rank per
process, `pkg.Dist(..., rank, shm=name)` — the NCCL-free multi-process
transport (host collectives in a POSIX shared-memory segment, device data
through CUDA IPC). All ranks share the one B200, so every cross-process
protocol of the solve runs for real: the CUDA-IPC halo mailboxes with their
two-parity epochs and system-scope arrival counters (peer_halo.cu), the peer
reductions storing dot partials into every rank's buffer + k_fold_peer
(solve.cu), the agglomeration gather, and — with matching="global" — the
128-bit system-scope Suitor CAS on peer suitor words (matching.cu
k_suitor_glob). Checked bit for bit against

  * local matching: the partition-aware oracle (oracle/partition.py: the
    reference's own functions composed with block-masked matching);
  * global matching: the UNPARTITIONED reference (proj/src/coarsening.cpp:
    194-242 + proj/src/krylov.cpp), since one Suitor over the whole graph has
    the unique greedy fixed point (proj/include/matchamg/matching.hpp:51-57).

Dot products keep the reference's 2048-block order across ranks
(proj/src/vector_ops.cpp:16-25), so the residual history must match too."""
import multiprocessing as mp
import os
import uuid

import numpy as np
import pytest

from conftest import bits, same_csr

pytestmark = pytest.mark.gpu

TIMEOUT = 240


def _worker(rank, world, name, A, kw, env, q):
    try:
        os.environ.update(env)
        import paper_1810_04221_b200 as pkg
        dev = pkg.Device(0)
        Ap = pkg.Csr(A[0], A[1], A[2], A[3], A[4])
        d = pkg.Dist(dev, world, rank, shm=name, matching=kw.get("matching", "local"),
                     agglomerate=kw.get("agglom"))
        d.setup(Ap, mode=kw.get("mode", 2))
        info = d.info()
        levels = []
        for k in range(info["nl"]):
            lv = {"bounds": d.bounds(k), "A": d.download(rank, k, 0),
                  "l1": d.download(rank, k, 3), "w": d.download(rank, k, 4)}
            if k + 1 < info["nl"]:
                lv["P"] = d.download(rank, k, 1)
                lv["R"] = d.download(rank, k, 2)
            levels.append(lv)
        runs = []
        for cyc in kw.get("cycles", [0]):
            u, h, r = d.pcg(cycle=cyc)
            runs.append((u, h, r, d.last_solve()))
        # a second build + solve on the same Dist (IPC blocks / mailboxes reused)
        if kw.get("rebuild"):
            d.build(mode=kw.get("mode", 2))
            runs.append(d.pcg(cycle=kw.get("cycles", [0])[0]) + (d.last_solve(),))
        q.put((rank, "ok", {"info": info, "levels": levels, "runs": runs}))
    except BaseException as e:  # report, never hang the parent
        import traceback
        q.put((rank, "err", traceback.format_exc()))


def run_ranks(A, world, env=None, **kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = "mamg_test_" + uuid.uuid4().hex[:12]
    At = (A.nrows, A.ncols, np.asarray(A.rp, np.int64), np.asarray(A.ci, np.int64),
          np.asarray(A.v, np.float64))
    e = {"MAMG_SHM_TIMEOUT": "120"}
    e.update(env or {})
    procs = [ctx.Process(target=_worker, args=(r, world, name, At, kw, e, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            rank, status, payload = q.get(timeout=TIMEOUT)
            out[rank] = (status, payload)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    errs = [f"rank {r}: {p}" for r, (s, p) in out.items() if s != "ok"]
    assert not errs, "\n".join(errs)
    return [out[r][1] for r in range(world)]


def _cat(parts, which, ncols):
    from oracle.oracle import Csr
    rps, cis, vs = [0], [], []
    for rp, ci, v in parts:
        rps.extend((np.asarray(rp[1:]) + rps[-1]).tolist())
        cis.append(ci)
        vs.append(v)
    return Csr(len(rps) - 1, ncols, np.array(rps, np.int64), np.concatenate(cis), np.concatenate(vs))


def check(res, ho, ref, A, cycles=(0,), bounds=None, peer_reduce=True, peer_halo=True):
    info = res[0]["info"]
    for r in res:
        assert r["info"] == info  # every rank agrees on the global level sizes
    assert info["nl"] == ho.nl
    assert info["sizes"] == [L.A.nrows for L in ho.levels]
    assert info["zero_edges"] == ho.zero_edges and info["stalled"] == ho.stalled
    for k in range(ho.nl):
        o = ho.levels[k]
        if bounds is not None:
            assert res[0]["levels"][k]["bounds"] == bounds[k], k
        n = info["sizes"][k]
        gA = _cat([r["levels"][k]["A"] for r in res], 0, n)
        assert same_csr(gA, o.A), k
        l1 = np.concatenate([r["levels"][k]["l1"] for r in res])
        w = np.concatenate([r["levels"][k]["w"] for r in res])
        assert np.array_equal(bits(l1), bits(o.l1)) and np.array_equal(bits(w), bits(o.w)), k
        if o.P is not None:
            nc = info["sizes"][k + 1]
            assert same_csr(_cat([r["levels"][k]["P"] for r in res], 1, nc), o.P), k
            assert same_csr(_cat([r["levels"][k]["R"] for r in res], 2, n), o.R), k
    b = np.ones(A.nrows)
    nruns = len(res[0]["runs"])
    for j in range(nruns):
        cyc = cycles[j] if j < len(cycles) else cycles[0]
        uo, ho_hist, ro = ref.pcg(A, ho, b, cycle=cyc)
        bnd = res[0]["levels"][0]["bounds"]
        u = np.zeros(A.nrows)
        for rk, r in enumerate(res):
            ur, hr, rr, how = r["runs"][j]
            # the cross-process peer paths really ran (eager: host-waiting transport)
            assert how["peer_reduce"] == peer_reduce and how["graphs"] is False, how
            if ho.nl > 1 and res[0]["info"]["sizes"][0] > 0:
                assert how["peer_halo"] == peer_halo, how
            assert rr["iterations"] == ro["iterations"], (j, rk)
            assert np.array_equal(bits(hr), bits(ho_hist)), (j, rk)
            u[bnd[rk]:bnd[rk + 1]] = ur[bnd[rk]:bnd[rk + 1]]
        assert np.array_equal(bits(u), bits(uo)), j


LCASES = [("poisson2d:96x96", lambda r: r.gen_poisson2d(96, 96)),
          ("randk3d:24^3 s=1", lambda r: r.gen_randk3d(24, 24, 24, 1.0, 0)),
          ("ani:128x128", lambda r: r.gen_aniso2d(128, 128, 1e-2, 0.4))]


@pytest.mark.parametrize("agglom", [0, 4096])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,gen", LCASES)
def test_mp_local_matching_bitwise_vs_partition_oracle(ref, name, gen, world, agglom):
    from oracle import partition as PA
    A = gen(ref)
    ho, obounds = PA.build_hierarchy(ref, A, world, agglom=agglom)
    res = run_ranks(A, world, agglom=agglom)
    check(res, ho, ref, A, bounds=obounds)


@pytest.mark.parametrize("agglom", [0, 4096])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,gen", LCASES[:2])
def test_mp_global_matching_bitwise_vs_unpartitioned(ref, name, gen, world, agglom):
    A = gen(ref)
    ho = ref.build_hierarchy(A, keep=True)
    res = run_ranks(A, world, matching="global", agglom=agglom)
    check(res, ho, ref, A)


@pytest.mark.parametrize("env", [{"MAMG_DIST_NCCL_HALO": "1"}, {"MAMG_DIST_NCCL_REDUCE": "1"},
                                 {"MAMG_DIST_NO_OVERLAP": "1"}])
def test_mp_transport_variants(ref, env):
    """The Comm's own halo / allgathered partials instead of the peer paths,
    and the peer halos without the interior overlap."""
    from oracle import partition as PA
    A = ref.gen_randk3d(24, 24, 24, 1.0, 2)
    ho, _ = PA.build_hierarchy(ref, A, 2, agglom=0)
    check(run_ranks(A, 2, env=env, agglom=0), ho, ref, A,
          peer_reduce="MAMG_DIST_NCCL_REDUCE" not in env, peer_halo="MAMG_DIST_NCCL_HALO" not in env)


def test_mp_wcycle_rebuild_and_empty_rank(ref):
    """W and V cycles on one build, a rebuild on the same Dist (IPC mailboxes
    and shared blocks reused), and 1600 rows < 2048: ranks 1, 2 own nothing."""
    from oracle import partition as PA
    A = ref.gen_poisson2d(40, 40)
    ho, _ = PA.build_hierarchy(ref, A, 3, agglom=0)
    res = run_ranks(A, 3, agglom=0, cycles=[1, 0], rebuild=True)
    check(res, ho, ref, A, cycles=(1, 0))


def test_mp_global_pairwise_mode(ref):
    A = ref.gen_randk3d(20, 20, 20, 1.0, 5)
    ho = ref.build_hierarchy(A, mode=1, keep=True)
    res = run_ranks(A, 2, matching="global", mode=1)
    check(res, ho, ref, A)


# ---- ranks as THREADS of this process (mamg_dist_create_group) ---------------
def run_threads(A, world, matching="local", agglom=None, u0=None):
    """Every rank: its own Device (context) on GPU 0, one thread, one group;
    ctypes releases the GIL, so the ranks really run concurrently."""
    import threading
    import paper_1810_04221_b200 as pkg
    g = pkg.ThreadGroup(world)
    devs = [pkg.Device(0) for _ in range(world)]
    Ap = pkg.Csr(A.nrows, A.ncols, np.asarray(A.rp, np.int64), np.asarray(A.ci, np.int64),
                 np.asarray(A.v, np.float64))
    out, errs = [None] * world, []

    def body(r):
        try:
            d = pkg.Dist(devs[r], world, r, matching=matching, agglomerate=agglom, group=g)
            d.setup(Ap)
            u, h, rep = d.pcg(u0=u0)
            out[r] = (d.info(), d.bounds(0), u, h, rep, d.last_solve())
        except BaseException as e:  # surfaced below
            errs.append((r, repr(e)))
    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=TIMEOUT)
    assert not errs, errs
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,gen", LCASES[:2])
def test_threads_global_matching_bitwise_vs_unpartitioned(ref, name, gen, world):
    A = gen(ref)
    ho = ref.build_hierarchy(A, keep=True)
    out = run_threads(A, world, matching="global")
    uo, hsto, ro = ref.pcg(A, ho, np.ones(A.nrows))
    u = np.zeros(A.nrows)
    for r, (info, bnd, ur, hr, rep, how) in enumerate(out):
        assert info["sizes"] == [L.A.nrows for L in ho.levels]
        assert rep["iterations"] == ro["iterations"] and np.array_equal(bits(hr), bits(hsto))
        # ranks of one process sharing a device keep the Comm's halos / allgathers
        assert how["peer_reduce"] is False and how["peer_halo"] is False
        u[bnd[r]:bnd[r + 1]] = ur[bnd[r]:bnd[r + 1]]
    assert np.array_equal(bits(u), bits(uo))


def test_threads_local_matching_and_initial_guess(ref):
    """local matching vs the partition-aware oracle, from a nonzero u0
    (pcg_solve's u0, proj/src/krylov.cpp:73-84)"""
    from oracle import partition as PA
    A = ref.gen_randk3d(24, 24, 24, 1.0, 3)
    ho, _ = PA.build_hierarchy(ref, A, 2, agglom=0)
    u0 = np.sin(np.arange(A.nrows) * 0.01)
    out = run_threads(A, 2, agglom=0, u0=u0)
    uo, hsto, ro = ref.pcg(A, ho, np.ones(A.nrows), u0=u0)
    u = np.zeros(A.nrows)
    for r, (info, bnd, ur, hr, rep, how) in enumerate(out):
        assert rep["iterations"] == ro["iterations"] and np.array_equal(bits(hr), bits(hsto))
        u[bnd[r]:bnd[r + 1]] = ur[bnd[r]:bnd[r + 1]]
    assert np.array_equal(bits(u), bits(uo))
