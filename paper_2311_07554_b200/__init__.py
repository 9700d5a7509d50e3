"""B200-native PaC-IM hot path (arXiv 2311.07554): Python binding of libpacim.so.

The binding only marshals arguments into the C ABI declared in
include/pacim.h; every step of the path runs in the library's sm_100a
kernels.  Importing succeeds without a GPU, but any call that reaches the
library fails loudly if libpacim.so is missing or no CUDA device exists —
there is no CPU fallback.
"""
from .binding import (  # noqa: F401
    PACIM_GEN_ER,
    PACIM_GEN_GRID,
    PACIM_GEN_RMAT,
    PACIM_P_CONST,
    PACIM_P_WIC,
    PACIM_P_UNIFORM,
    Context,
    PacimError,
    lib,
    lib_path,
    pacim_nccl_unique_id,
    pacim_threshold_from_p,
    pacim_threshold_uniform,
    pacim_version,
)
