"""B200-native (sm_100a) CT normal operator R*M*MR = F_NU F_NU^* and the CG / split-Bregman
solves around it (arXiv 1705.07497's hot path), behind the C ABI in include/tomo_b200.h.

The compute lives in libtomo_b200.so (hand-written CUDA for sm_100a + a C++ host runtime);
this package is the Python mirror of the reference's operator/solver API.
"""
from .tomo import (  # noqa: F401
    CgStats, ConfigError, CudaError, Error, Geometry, IoError, NormalBackend, NumericalError, SolveTrace,
    SolverConfig, apply_normal, apply_normal_real, generate_shepp_logan, grad, grad_adjoint, kernel_launches,
    make_direct_backend, make_fused_backend, make_surrogate_backend, nccl_unique_id, load_sparse_info, radial_density_weights, random_ellipses, shrink,
    split_bregman_tv, tikhonov_solve,
)

__all__ = [
    "Geometry", "NormalBackend", "SolverConfig", "SolveTrace", "CgStats", "make_direct_backend", "make_fused_backend", "load_sparse_info",
    "make_surrogate_backend", "apply_normal", "apply_normal_real", "split_bregman_tv", "tikhonov_solve",
    "grad", "grad_adjoint", "shrink", "generate_shepp_logan", "random_ellipses", "radial_density_weights",
    "nccl_unique_id", "kernel_launches", "Error", "ConfigError", "NumericalError", "IoError", "CudaError",
]
