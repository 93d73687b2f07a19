"""matchamg-b200: B200-native (sm_100a) AMG-PCG based on compatible weighted
matching (arXiv 1810.04221), a drop-in for the reference's setup/solve path.

The product is the CUDA library csrc/lib/libmamg_cuda.so (C-ABI in
include/mamg_capi.h) and the host C++ facade csrc/lib/libmatchamg.so (the
reference's matchamg API, include/matchamg/*.hpp). This package exposes both
to Python via ctypes; there is no CPU fallback.
"""
from .capi import (BreakdownError, Csr, Device, DeviceHierarchy, Dist, Hierarchy, InvalidArgument,
                   Level, LIB_PATH, MamgError, load_library, nccl_unique_id, partition_bounds,
                   shm_allgather, ThreadGroup)
from .problems import (HOST_LIB, from_spec, gen_anisotropic_2d, gen_anisotropic_3d_q1,
                       gen_elasticity_3d, gen_jump_3d, gen_poisson_2d, gen_poisson_3d_randk,
                       MatrixMarketError, read_matrix_market, write_matrix_market)

__all__ = ["BreakdownError", "Csr", "Device", "DeviceHierarchy", "Dist", "Hierarchy", "InvalidArgument",
           "nccl_unique_id", "partition_bounds", "shm_allgather", "ThreadGroup",
           "Level", "LIB_PATH", "MamgError", "load_library", "HOST_LIB", "from_spec",
           "gen_anisotropic_2d", "gen_poisson_2d", "gen_poisson_3d_randk",
           "gen_anisotropic_3d_q1", "gen_jump_3d", "gen_elasticity_3d",
           "read_matrix_market", "write_matrix_market", "MatrixMarketError"]
