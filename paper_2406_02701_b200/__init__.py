"""B200-native MPCR engine: multi-precision dense linear algebra on sm_100a.

The compute path is ``libmpcr_b200.so`` (hand-written CUDA for sm_100a behind
the C ABI ``include/mpcr_b200.h``); this package is its host-side mirror of
the reference API (``mpnum`` / MPCRTile).  Importing does not touch the GPU;
the first call loads the library and fails loudly if it is missing.
"""
from ._lib import LIB_PATH, MPError, lib  # noqa: F401
from .mpcr import (  # noqa: F401
    BinaryOp,
    Context,
    KernelKey,
    MPArray,
    MPCRTile,
    Precision,
    ProcessGrid,
    ReduceOp,
    Side,
    UnaryOp,
    default_context,
    diag,
    dispatch,
    dist_owner,
    dist_schedule,
    ew_binary,
    ew_scalar,
    ew_unary,
    gaussian_nll,
    linalg,
    matern_mle,
    nccl_unique_id,
    parse_precision,
    promote,
    random_uniform_matrix,
    reduce,
    rng_normal,
    rng_uniform,
    tile_chol,
    tile_gemm,
    tile_trsm,
    transpose,
)

__all__ = [
    "BinaryOp", "Context", "KernelKey", "dispatch", "MPArray", "MPCRTile", "MPError", "Precision", "ProcessGrid", "ReduceOp", "Side",
    "UnaryOp", "default_context", "diag", "dist_owner", "dist_schedule", "nccl_unique_id", "ew_binary", "ew_scalar", "ew_unary", "gaussian_nll", "linalg", "matern_mle",
    "parse_precision", "promote", "random_uniform_matrix", "reduce", "rng_normal", "rng_uniform", "tile_chol", "tile_gemm", "tile_trsm", "transpose",
    "lib", "LIB_PATH",
]
