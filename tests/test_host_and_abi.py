"""CPU tests of the product's host side: the C-ABI library loads and exports
every symbol include/mamg_capi.h declares (no compute without a GPU), the host
facade exports the matchamg C++ API, and the host generators reproduce the
reference's matrices bit for bit."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, bits


def header_functions(path):
    txt = open(path).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(mamg_\w+)\s*\(", txt, flags=re.M)
    return sorted(set(n for n in names if not n.endswith("_t")))


def test_capi_exports_every_declared_symbol():
    import paper_1810_04221_b200 as pkg
    lib = pkg.load_library()
    names = header_functions(os.path.join(ROOT, "include", "mamg_capi.h"))
    assert len(names) > 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    bound = {n for n, _, _ in pkg.capi.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound
    assert lib.mamg_version().decode().startswith("matchamg-b200")


def test_capi_reports_no_device_cleanly():
    import paper_1810_04221_b200 as pkg
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(pkg.MamgError):
        pkg.Device(0)


def test_cuda_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1810_04221_b200", "csrc", "lib", "libmamg_cuda.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # TMA bulk copies in the SpMV/smoother kernels


def test_host_facade_exports_matchamg_api():
    so = os.path.join(ROOT, "paper_1810_04221_b200", "csrc", "lib", "libmatchamg.so")
    out = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True, text=True).stdout
    for sym in ["matchamg::build_hierarchy(", "matchamg::pcg_solve(", "matchamg::spmv(",
                "matchamg::suitor_match(", "matchamg::galerkin_by_aggregates(",
                "matchamg::MultigridPreconditioner::apply(", "matchamg::apply_cycle(",
                "matchamg::fused_triple_dot(", "matchamg::build_weights(",
                "matchamg::gen_poisson_3d_randk(", "matchamg::l1_jacobi_sweeps(",
                "matchamg::hierarchy_stats(", "matchamg::double_pairwise(",
                "matchamg::spgemm(", "matchamg::transpose(", "mamg_gen_randk3d"]:
        assert sym in out, sym


@pytest.mark.parametrize("spec", ["poisson2d:512,512", "ani:33,17,0.01,0.7", "randk3d:20,17,9,1.3",
                                  "randk3d:12,12,12,0"])
def test_generators_bitwise_vs_reference(ref, spec):
    import paper_1810_04221_b200 as pkg
    A = pkg.from_spec(spec, seed=7)
    kind, args = spec.split(":")
    a = args.split(",")
    if kind == "poisson2d":
        B = ref.gen_poisson2d(int(a[0]), int(a[1]))
    elif kind == "ani":
        B = ref.gen_aniso2d(int(a[0]), int(a[1]), float(a[2]), float(a[3]))
    else:
        B = ref.gen_randk3d(int(a[0]), int(a[1]), int(a[2]), float(a[3]), 7)
    assert np.array_equal(A.rp, B.rp) and np.array_equal(A.ci, B.ci)
    assert np.array_equal(bits(A.v), bits(B.v))


def test_generator_spec_errors():
    import paper_1810_04221_b200 as pkg
    with pytest.raises(ValueError):
        pkg.from_spec("poisson2d:4")
    with pytest.raises(ValueError):
        pkg.from_spec("randk3d:1,4,4,0")
    with pytest.raises(ValueError):
        pkg.from_spec("ani:8,8,0,0")


def test_vcycle_byte_model():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    # cfg 2 V-cycle = 1,715.2 MB (level sizes from the golden)
    import json
    fp = json.load(open(os.path.join(ROOT, "tests", "golden", "hierarchies.json")))
    c2 = fp["randk3d:160,160,160,0"]
    b = bench.vcycle_bytes(list(zip(c2["sizes"], c2["level_nnz"])))
    assert abs(b / 1e6 - 1715.2) < 0.5
