"""B200-native selected inversion of block-banded Dyson matrices (RGF / nRGF / DDRGF).

The compute path is libbbsi_cuda.so (sm_100a DMMA kernels) behind the C ABI in
include/bbsi_cuda.h; this package is the host-side mirror of the reference
``bbsi`` interface plus the BASELINE Dyson workloads. No CPU fallback.
"""
from .bbsi import (BlockBandedMatrix, BlockLayout, CudaError, DomainPlan, ExtendedInverse,  # noqa: F401
                   InvalidArgumentError, KernelCounters, SingularMatrixError, ddrgf, make_layout, random_spd_like,
                   read_bbm, rgf_extended, rgf_fused, rgf_many, rgf_ndiag, rgf_tridiag, write_bbm)

__all__ = ["BlockBandedMatrix", "BlockLayout", "CudaError", "DomainPlan", "ExtendedInverse", "InvalidArgumentError",
           "KernelCounters", "SingularMatrixError", "ddrgf", "make_layout", "random_spd_like", "read_bbm",
           "rgf_extended", "rgf_fused", "rgf_many", "rgf_ndiag", "rgf_tridiag", "write_bbm"]
