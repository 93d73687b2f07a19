#!/usr/bin/env python
"""AMG-PCG setup+solve benchmark (BASELINE.json metric) on B200.

A "step" is one pass of the hot path over the synthetic workload: the
device-resident setup (build_hierarchy, proj/src/coarsening.cpp:194-238) plus
the AMG-preconditioned CG solve to rtol 1e-6 (pcg_solve, proj/src/krylov.cpp),
b = w = ones, V(1,1) cycle, 20 coarsest sweeps — the reference defaults.
N=1 workload: BASELINE configs[1], 3D 7-point Poisson 160^3 (4,096,000 rows).

  value   : setup+solve seconds with the matrix resident in HBM (CUDA events)
  e2e     : the same through the C-ABI host-buffer call mamg_solve_host
            (H2D of A and b, setup, solve, D2H of u inside the timed region)
  roofline: the level-0 fused l1-Jacobi sweep kernel (SpMV + update), the
            dominant solve kernel, against the measured HBM copy bandwidth
  cpu_baseline: the reference library (oracle/_ref, built from
            /root/reference) timed on this host's cores on the same matrix

`--impl reference` times the reference CPU implementation instead (rank 0).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# rank 0 prints exactly one JSON line on stdout: keep NCCL's banner off it
os.environ.setdefault("NCCL_DEBUG", "WARN")

METRIC = "AMG-PCG setup+solve time (s) and V-cycle GB/s vs HBM peak, 1/2/4/8 B200"
CONFIGS = {
    "cfg1": ("poisson2d:512,512", "BASELINE cfg1: 2D Poisson 5-point 512x512 (262,144 rows)"),
    "cfg2": ("randk3d:160,160,160,0", "BASELINE cfg2: 3D Poisson 7-point 160^3 (4,096,000 rows)"),
    # BASELINE cfg 3-5: measured with --config, parity-tested at reduced sizes
    "cfg3": ("aniso27:128,128,128,0.01",
             "BASELINE cfg3: 3D anisotropic Q1 27-point 128^3, K = diag(1,1,1e-2) (2,097,152 rows)"),
    "cfg4": ("jump3d:200,200,200,8",
             "BASELINE cfg4: 3D jump-coefficient FV 7-point 200^3, K in {1e-3,1,1e3} on 8^3 "
             "sub-cubes (8,000,000 rows)"),
    "cfg5": ("elast3d:100,100,100",
             "BASELINE cfg5: 3D Q1 linear elasticity, 3 dof/node, 100^3 nodes (3,000,000 rows)"),
}
DATA = {"cfg1": "2D 5-point Laplacian", "cfg2": "sigma=0 -> constant 7-point",
        "cfg3": "Q1 trilinear FEM, Dirichlet", "cfg4": "seeded (0) piecewise-constant K",
        "cfg5": "Q1 Lame mu=0.42 lambda=1.7, clamped x=0"}
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.lines = device, None, []

    def __enter__(self):
        if os.environ.get("MAMG_BENCH_NO_CLOCKS"):
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def mark(self):
        return len(self.lines)

    def summary(self, lo=0, hi=None):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines[lo:hi] if hi is not None and hi > lo else self.lines[lo:]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def vcycle_bytes(levels):
    """Algorithmic bytes of one V(1,1) cycle from zero:
    sum_{k<L} [24n (pre from 0) + (12nnz + 28n) (residual) + (20n + 12n') (R)
    + (32n + 8n') (prolong+correct) + (12nnz + 36n) (post)]
    + 24n_L + 19 (12nnz_L + 36n_L) (coarsest)."""
    tot = 0
    L = len(levels) - 1
    for k in range(L):
        n, nnz = levels[k]
        nc = levels[k + 1][0]
        tot += 24 * n + (12 * nnz + 28 * n) + (20 * n + 12 * nc) + (32 * n + 8 * nc) + (12 * nnz + 36 * n)
    n, nnz = levels[L]
    tot += 24 * n + 19 * (12 * nnz + 36 * n)
    return tot


def load_profile_traffic():
    p = os.path.join(ROOT, "profiles", "smoother_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


def cpu_model():
    """CPU model name and logical CPU count of this host (lscpu's 'Model name')."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    if model is None:
        try:
            with open("/proc/cpuinfo") as f:
                for ln in f:
                    if ln.startswith("model name"):
                        model = ln.split(":", 1)[1].strip()
                        break
        except Exception:
            pass
    return {"model": model, "logical_cpus": os.cpu_count()}


def config_for(args, n, nnz, world):
    """The `config` dict — identical in the B200 arm and the reference arm."""
    spec, label = CONFIGS[args.config]
    return {"workload": label, "spec": spec, "n": n, "nnz": nnz,
            "cycle": "V(1,1), 20 coarsest sweeps", "rtol": 1e-6, "rhs": "b = w = ones",
            "parallelism": "1 GPU" if world == 1 else f"row-block partition over {world} GPUs",
            "l2": (("inputs larger than L2 (A = %.0f MB > 126 MB), no flush"
                    if 12 * nnz + 4 * n > 126e6 else
                    "A = %.0f MB fits in the 126 MB L2 (no flush; a latency-bound size)")
                   % ((12 * nnz + 4 * n) / 1e6))}


def ref_matrix(ref, args):
    """BASELINE matrix made by the REFERENCE's own generator (src/problems.cpp)
    and kept inside it; cfg 3-5 have no reference generator: the repo's host
    generator builds them (the only product code the reference arm touches)."""
    spec, _ = CONFIGS[args.config]
    kind, rest = spec.split(":")
    vals = [float(x) for x in rest.split(",")]
    if kind == "poisson2d":
        return ref.gen_handle("poisson2d", int(vals[0]), int(vals[1])), "reference generator"
    if kind == "randk3d":
        return (ref.gen_handle("randk3d", int(vals[0]), int(vals[1]), int(vals[2]), vals[3], 0),
                "reference generator")
    import paper_1810_04221_b200 as pkg
    return ref.wrap(pkg.from_spec(spec)), "repo host generator (no reference generator)"


def reference_checker():
    from oracle import oracle as O
    ref_ok, _ = O.available()
    if not ref_ok:
        raise RuntimeError("oracle/_ref missing: build it with `make -C oracle ref`")
    return O.Ref()


def run_reference(args):
    """The reference's own CPU implementation of the path (oracle/_ref = the
    unmodified proj/src compiled here), timed like cli::run_solve
    (proj/src/cli.cpp:273-275 + SolveReport::solve_ms, krylov.cpp:54-64) on the
    reference's own matrix: no marshalling inside the timers, nothing from
    paper_1810_04221_b200 loaded (cfg 1-2)."""
    rank, _, world = env_rank()
    if rank != 0:
        return
    ref = reference_checker()
    M, source = ref_matrix(ref, args)
    threads = os.cpu_count() or 1
    steps = []
    for s in range(args.warmup + args.steps):
        r = ref.run_solve(M, threads)
        if s >= args.warmup:
            steps.append(r)
    setup = statistics.mean(r["setup_ms"] for r in steps)
    solve = statistics.mean(r["solve_ms"] for r in steps)
    wall = statistics.mean(r["wall_ms"] for r in steps)
    v = (setup + solve) / 1e3
    one = None
    if not args.no_single_thread:
        one = ref.run_solve(M, 1)
        ref.set_threads(threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: {CONFIGS[args.config][0]} ({DATA[args.config]}), b = w = ones; "
                f"matrix from the {source}",
        "config": config_for(args, M.nrows, M.nnz, world),
        "setup_s": setup / 1e3, "solve_s": solve / 1e3, "wall_s": wall / 1e3,
        "iterations": steps[-1]["iterations"], "final_relres": steps[-1]["final_relres"],
        "levels": steps[-1]["nl"],
        "step_ms": [round(r["setup_ms"] + r["solve_ms"], 3) for r in steps],
        "cpu_baseline": {"value": v, "unit": "s", "cores": threads, "kind": "reference",
                         "sample": "one full cli::run_solve setup+solve per step (setup_ms around "
                                   "build_hierarchy + SolveReport::solve_ms)",
                         "cpu": cpu_model()},
        "cpu_1thread": (None if one is None else
                        {"value": (one["setup_ms"] + one["solve_ms"]) / 1e3, "unit": "s",
                         "cores": 1, "setup_s": one["setup_ms"] / 1e3,
                         "solve_s": one["solve_ms"] / 1e3, "iterations": one["iterations"]}),
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def _digest(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def hierarchy_digests(levels):
    """Per level: sizes and SHA-256 prefixes of A, P (= the aggregates and
    prolongator values), R, l1 and w — bits, not approximate values."""
    out = []
    for L in levels:
        csr = lambda M: None if M is None else _digest(np.asarray(M.rp, np.int64),
                                                        np.asarray(M.ci, np.int64),
                                                        np.asarray(M.v, np.float64))
        out.append({"n": int(L.A.nrows), "nnz": int(L.A.nnz), "A": csr(L.A), "P": csr(L.P),
                    "R": csr(L.R), "l1": _digest(np.asarray(L.l1, np.float64)),
                    "w": _digest(np.asarray(L.w, np.float64))})
    return out


def run_b200(args):
    rank, local, world = env_rank()
    dist = None
    if world > 1 or args.partitioned:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if world == 1:  # --partitioned on one GPU: a one-rank group
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("gloo", rank=0, world_size=1)
        else:
            dist.init_process_group("nccl")

    def barrier():
        if dist:
            dist.barrier()

    def allmax(x):
        if not dist or world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    import paper_1810_04221_b200 as pkg
    if world > 1 or args.partitioned:
        return run_partitioned(args, rank, local, world, dist, barrier, allmax)
    spec, label = CONFIGS[args.config]
    t_gen = time.perf_counter()
    A = pkg.from_spec(spec)
    host_gen_ms = (time.perf_counter() - t_gen) * 1e3
    n, nnz = A.nrows, A.nnz
    dev = pkg.Device(local)
    # the same matrix assembled on the device (informational: the input side)
    dev.generate(spec)
    dev.synchronize()
    t_gen = time.perf_counter()
    dG = dev.generate(spec)
    dev.synchronize()
    dev_gen_ms = (time.perf_counter() - t_gen) * 1e3
    del dG
    dA = dev.upload(A)
    db = dev.vec(np.ones(n))
    du = dev.zeros(n)

    def step():
        dev.timer_start()
        dh = dev.setup(dA)
        t_setup = dev.timer_stop()
        dev.timer_start()
        rep = dev.pcg_device(dA, dh, db, du)
        t_solve = dev.timer_stop()
        return dh, rep, t_setup, t_solve

    # the clock sampler starts before the warm-up so its NVML start-up cost is
    # outside the timed region; only samples taken during the timed steps count
    clk = Clocks(local).__enter__()
    for _ in range(args.warmup):
        dh, rep, _, _ = step()
        del dh
    barrier()
    dev.synchronize()
    l0 = dev.kernel_launches
    setups, solves = [], []
    c0 = clk.mark()
    for _ in range(args.steps):
        dh, rep, ts, tv = step()
        setups.append(ts)
        solves.append(tv)
        if _ + 1 < args.steps:
            del dh
    dev.synchronize()
    c1 = clk.mark()
    time.sleep(0.25)
    clk.__exit__(None, None, None)
    barrier()
    launches = dev.kernel_launches - l0
    step_ms = [a + b for a, b in zip(setups, solves)]
    ms_step = allmax(statistics.mean(step_ms))
    setup_ms = allmax(statistics.mean(setups))
    solve_ms = allmax(statistics.mean(solves))
    value = ms_step / 1e3

    # kernel roofline: level-0 fused l1-Jacobi sweep (SpMV + update)
    hbm, hbm_src = measured_hbm()
    lv = []
    for k in range(dh.nl):
        nr, nc, nz = dh.level_matrix("A", k).shape
        lv.append((nr, nz))
    sm_ms = dev.time_smoother(dh, 0, reps=50)
    sm_bytes = 12 * nnz + 36 * n
    sm_gbs = sm_bytes / (sm_ms * 1e-3) / 1e9
    spmv_ms = dev.time_spmv(dh, 0, reps=50)
    spmv_bytes = 12 * nnz + 4 * (n + 1) + 16 * n
    vc_ms = dev.time_precond(dh, reps=20)
    vc_bytes = vcycle_bytes(lv)
    traffic = load_profile_traffic()

    # end-to-end through the C-ABI host-buffer call (host timer); release the
    # device-resident objects first so the e2e path starts from the same pool
    # the last timed step's hierarchy, downloaded for the level-by-level parity check
    dig_dev = (hierarchy_digests(dh.materialize().levels)
               if rank == 0 and world == 1 and not args.no_cpu_baseline else None)
    del dh, dA, db
    dev.synchronize()
    e2e = []
    u_e2e = None
    b_host = np.ones(n)  # the caller's right-hand side (pageable host memory, like A)
    u_host = np.zeros(n)  # the caller's solution buffer, reused across calls
    for r in range(1 + min(args.steps, 3)):
        t0 = time.perf_counter()
        u_e2e, hist, rep_e2e = dev.solve_host(A, b=b_host, out=u_host)
        dt = time.perf_counter() - t0
        if r > 0:
            e2e.append(dt)
    e2e_v = allmax(statistics.mean(e2e))
    h2d = 8 * (n + 1) + 8 * nnz + 8 * nnz + 8 * n  # rp, ci, v (int64/fp64 API layout), b
    d2h = 8 * n

    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
        "scaling": "weak" if world > 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: {spec} ({DATA[args.config]}), b = w = ones",
        "config": config_for(args, n, nnz, world), "levels": len(lv),
        "setup_s": setup_ms / 1e3, "solve_s": solve_ms / 1e3,
        "iterations": rep["iterations"], "final_relres": rep["final_relres"],
        "e2e": {"value": e2e_v, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "upload_ms": rep_e2e["upload_ms"], "setup_ms": rep_e2e["setup_ms"],
                "solve_ms": rep_e2e["solve_ms"], "download_ms": rep_e2e["download_ms"]},
        "roofline": {"kernel": "l1-Jacobi sweep (fused SpMV+update), level 0", "bound": "hbm",
                     "achieved": sm_gbs, "peak": hbm, "unit": "GB/s", "frac": sm_gbs / hbm,
                     "peak_source": hbm_src, "bytes_per_launch": sm_bytes, "ms_per_launch": sm_ms,
                     "frac_of_8TBs": sm_gbs / 8000.0,
                     "traffic": (traffic or {}).get("bytes_per_launch")},
        "spmv": {"ms": spmv_ms, "bytes": spmv_bytes, "gbs": spmv_bytes / (spmv_ms * 1e-3) / 1e9},
        "vcycle": {"ms": vc_ms, "bytes": vc_bytes, "gbs": vc_bytes / (vc_ms * 1e-3) / 1e9,
                   "frac": vc_bytes / (vc_ms * 1e-3) / 1e9 / hbm},
        "gpu_launches": launches,
        "clocks": clk.summary(c0, c1 + 2),
        "generate": {"host_ms": round(host_gen_ms, 2), "device_ms": round(dev_gen_ms, 3),
                     "note": "matrix generation before the timed step (host C++ generator vs "
                             "the bit-identical device generator); not part of value or e2e"},
        "step_ms": [round(a + b, 3) for a, b in zip(setups, solves)],
        "setup_ms_steps": [round(a, 3) for a in setups],
        "solve_ms_steps": [round(b, 3) for b in solves],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference (oracle/_ref) on this host's cores, timed like
        # cli::run_solve on the same matrix (copied in outside the timers)
        ref = reference_checker()
        threads = os.cpu_count() or 1
        ref.run_solve(ref.gen_handle("randk3d", 12, 12, 12, 0.0, 0), threads)  # OpenMP warm-up
        M = ref.wrap(A)
        rr = ref.run_solve(M, threads, want_u=True)
        u_ref = rr["u"]
        line["cpu_baseline"] = {"value": (rr["setup_ms"] + rr["solve_ms"]) / 1e3, "unit": "s",
                                "cores": threads, "kind": "reference",
                                "setup_s": rr["setup_ms"] / 1e3, "solve_s": rr["solve_ms"] / 1e3,
                                "sample": f"one full cli::run_solve setup+solve of {label}",
                                "cpu": cpu_model()}
        u_dev = du.to_host()
        # full-size hierarchy parity, level by level (bits of A, P, R, l1, w)
        dig_ref = hierarchy_digests(ref.build_hierarchy(A).levels)
        per_level = [a == b for a, b in zip(dig_dev, dig_ref)]
        line["parity"] = {"iterations_ref": rr["iterations"], "iterations": rep["iterations"],
                          "levels_ref": len(dig_ref), "levels": len(dig_dev),
                          "hierarchy_bitwise": bool(len(dig_dev) == len(dig_ref) and all(per_level)),
                          "hierarchy_levels_bitwise": per_level,
                          "hierarchy_digests": dig_dev,
                          "solution_bitwise_equal": bool(np.array_equal(u_dev.view(np.int64),
                                                                        u_ref.view(np.int64))),
                          "e2e_solution_bitwise_equal": bool(np.array_equal(
                              u_e2e.view(np.int64), u_ref.view(np.int64))),
                          "max_rel_diff": float(np.max(np.abs(u_dev - u_ref)) /
                                                max(np.max(np.abs(u_ref)), 1e-300))}
    if rank == 0:
        emit(line)
    if dist:
        dist.destroy_process_group()


def run_partitioned(args, rank, local, world, dist, barrier, allmax):
    """N > 1: the row-block partitioned path (one rank per GPU, NCCL transport).
    Strong scaling: the whole problem is split into `world` row blocks;
    matching runs on local blocks (partition-aware hierarchy) or,
    with --matching global, as one Suitor across the parts (hierarchy identical
    to the single-GPU one).

    Also reported: the cold setup (first build of the Dist: IPC mappings,
    scratch growth) beside the warm one; the level-0 sweep roofline of the
    slowest rank; the partitioned V-cycle GB/s; parity of the iterations and
    the residual history against the partition-aware oracle (local) or the
    unpartitioned reference (global); and T1 / (p Tp) with T1 = the
    single-GPU path timed on rank 0 in the same run."""
    import paper_1810_04221_b200 as pkg
    spec, label = CONFIGS[args.config]
    A = pkg.from_spec(spec)
    n, nnz = A.nrows, A.nnz
    dev = pkg.Device(local)
    obj = [pkg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    D = pkg.Dist(dev, world, rank, obj[0], matching=args.matching).load(A)

    def step():
        dev.timer_start()
        D.build()
        ts = dev.timer_stop()
        dev.timer_start()
        _, hist, rep = D.pcg(want_u=False)
        tv = dev.timer_stop()
        return rep, hist, ts, tv

    def allmin(x):
        return -allmax(-x)

    clk = Clocks(local).__enter__()
    barrier()
    dev.timer_start()
    D.build()  # cold: the first build of this Dist
    cold_setup_ms = allmax(dev.timer_stop())
    D.pcg(want_u=False)
    for _ in range(args.warmup - 1):
        step()
    barrier()
    dev.synchronize()
    l0 = dev.kernel_launches
    c0 = clk.mark()
    setups, solves = [], []
    for _ in range(args.steps):
        rep, hist, ts, tv = step()
        setups.append(ts)
        solves.append(tv)
    dev.synchronize()
    c1 = clk.mark()
    clk.__exit__(None, None, None)
    barrier()
    launches = dev.kernel_launches - l0
    ms_step = allmax(statistics.mean([a + b for a, b in zip(setups, solves)]))
    setup_ms = allmax(statistics.mean(setups))
    solve_ms = allmax(statistics.mean(solves))
    how = D.last_solve()
    info = D.info()
    # kernel roofline (level-0 sweep of this rank's rows; the slowest rank)
    hbm, hbm_src = measured_hbm()
    ln, lz = D.local_shape(0)
    sw_ms = D.time("sweep", reps=50)
    sw_bytes = 12 * lz + 36 * ln
    sw_gbs = allmin(sw_bytes / (sw_ms * 1e-3) / 1e9 if sw_ms > 0 else 0.0)
    sw_ms = allmax(sw_ms)
    vc_ms = allmax(D.time("precond", reps=20))
    vc_bytes = vcycle_bytes(list(zip(info["sizes"], info["nnz"])))
    vc_gbs = vc_bytes / (vc_ms * 1e-3) / 1e9
    # end to end: H2D of this rank's blocks + build + solve + D2H of its rows
    e2e = []
    for r in range(1 + min(args.steps, 3)):
        barrier()
        t0 = time.perf_counter()
        D.load(A)
        D.build()
        u, hist_e, rep_e = D.pcg()
        dt = allmax(time.perf_counter() - t0)
        if r > 0:
            e2e.append(dt)
    line = {
        "metric": METRIC, "value": ms_step / 1e3, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: {spec} ({DATA[args.config]}), b = w = ones",
        "config": config_for(args, n, nnz, world), "levels": info["nl"],
        "matching": args.matching,
        "transport": "NCCL setup collectives; solve halos / dot partials / agglomeration "
                     "gather over CUDA-IPC peer memory" if how["peer_reduce"] else "NCCL",
        "solve_paths": how,
        "setup_s": setup_ms / 1e3, "solve_s": solve_ms / 1e3, "setup_cold_s": cold_setup_ms / 1e3,
        "iterations": rep["iterations"], "final_relres": rep["final_relres"],
        "e2e": {"value": statistics.mean(e2e), "unit": "s",
                "h2d_bytes_per_step": 8 * (n + 1) + 16 * nnz,
                "d2h_bytes_per_step": 8 * n},
        "roofline": {"kernel": "l1-Jacobi sweep (fused SpMV+update), level 0, local rows; "
                               "slowest rank", "bound": "hbm", "achieved": sw_gbs, "peak": hbm,
                     "unit": "GB/s", "frac": sw_gbs / hbm, "peak_source": hbm_src,
                     "ms_per_launch": sw_ms, "bytes_per_launch_rank0": sw_bytes,
                     "traffic": None},
        "vcycle": {"ms": vc_ms, "bytes": vc_bytes, "gbs": vc_gbs, "gbs_per_gpu": vc_gbs / world,
                   "frac_per_gpu": vc_gbs / world / hbm},
        "gpu_launches": launches,
        "clocks": clk.summary(c0, c1 + 2),
        "step_ms": [round(a + b, 3) for a, b in zip(setups, solves)],
    }
    # T1: the single-GPU path on rank 0, same matrix, same run (others wait)
    if rank == 0:
        dA = dev.upload(A)
        db = dev.vec(np.ones(n))
        du = dev.zeros(n)
        t1 = []
        for r in range(4):
            dev.timer_start()
            dh = dev.setup(dA)
            dev.pcg_device(dA, dh, db, du)
            t = dev.timer_stop()
            del dh
            if r > 0:
                t1.append(t)
        t1_ms = statistics.mean(t1)
        line["strong_scaling_same_run"] = {"t1_s": t1_ms / 1e3, "tp_s": ms_step / 1e3,
                                           "efficiency": t1_ms / (world * ms_step),
                                           "note": "T1 / (p Tp), T1 = single-GPU path on rank 0"}
        del dA, db, du
    if rank == 0 and not args.no_cpu_baseline:
        ref = reference_checker()
        from oracle import oracle as O
        Ao = O.Csr(A.nrows, A.ncols, A.rp, A.ci, A.v)
        if args.matching == "local":
            from oracle import partition as PA
            ho, _ = PA.build_hierarchy(ref, Ao, world, agglom=D.agglomerate)
            target = "partition-aware oracle (oracle/partition.py)"
        else:
            ho = ref.build_hierarchy(Ao, keep=True)
            target = "unpartitioned reference"
        uo, ho_hist, ro = ref.pcg(Ao, ho, np.ones(n))
        b0, b1 = D.bounds(0)[0], D.bounds(0)[1]
        line["parity"] = {"target": target, "iterations_ref": ro["iterations"],
                          "iterations": rep["iterations"],
                          "levels_ref": ho.nl, "levels": info["nl"],
                          "sizes_equal": info["sizes"] == [L.A.nrows for L in ho.levels],
                          "history_bitwise": bool(np.array_equal(
                              np.asarray(hist).view(np.int64), ho_hist.view(np.int64))),
                          # rank 0's rows (each rank holds its own block)
                          "solution_bitwise_equal": bool(np.array_equal(
                              u[b0:b1].view(np.int64), uo[b0:b1].view(np.int64)))}
    barrier()
    if rank == 0:
        emit(line)
    dist.destroy_process_group()


# the one JSON line goes to the process's real stdout; everything else that
# reaches file descriptor 1 while the bench runs (NCCL's version banner when
# NCCL_DEBUG is preset in the environment, library prints) goes to stderr
_JSON_FD = None


def emit(line):
    sys.stdout.flush()
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    # (not restored: NCCL may still log while communicators are torn down at exit)
    _main()
    sys.stdout.flush()


def _main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-single-thread", action="store_true",
                    help="reference arm: skip the extra 1-thread reference run")
    ap.add_argument("--matching", choices=["local", "global"], default="local",
                    help="partitioned path (--gpus > 1): Suitor per part or across parts")
    ap.add_argument("--partitioned", action="store_true",
                    help="run the partitioned (NCCL) path even at one GPU (checks that path)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
