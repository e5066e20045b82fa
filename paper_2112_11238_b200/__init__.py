"""B200-native mu-mode product / Tucker engine (arXiv 2112.11238 hot path).

Public API mirrors the reference's ``mumode::core`` / ``mumode::ops`` hot-path
operators; see ``api.py``. Compute lives in ``libmumode_b200.so`` (sm_100a).
"""
from .api import (  # noqa: F401
    ArgumentError,
    ContractError,
    CudaError,
    FactorizedStack,
    Handle,
    KronSumSolver,
    MumodeError,
    NumericalError,
    Rng,
    SizeError,
    colmajor_empty,
    cttucker,
    dematricize,
    expint,
    expm,
    extract_tridiag,
    get_handle,
    is_colmajor,
    itucker,
    kronsumv,
    launch_count,
    matricize,
    mode_action,
    mode_product,
    to_colmajor,
    tucker,
    symtridiag_eig,
    tucker_sequential,
    tuckerfun,
)

__version__ = "0.1.0"
