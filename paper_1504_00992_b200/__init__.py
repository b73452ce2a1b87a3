"""paper_1504_00992_b200 — B200-native (sm_100a) TEBD two-site decimation with randomized SVD.

The compute path is librrsvd_b200.so (hand-written CUDA for sm_100a behind the C ABI in
include/rrsvd_b200.h).  This package is the host-side mirror of the reference C++ API
(rrsvd:: / rrsvd::tebd::) for tests, benchmarks and Python users.  There is no CPU fallback.
"""
from ._lib import (CONTRACT_VIOLATION, CUDA_ERROR, NUMERIC_FAILURE, OMEGA_PHILOX,  # noqa: F401
                   OMEGA_REFERENCE, Context, ContractViolation, CudaError, NumericFailure, lib)
from .api import *  # noqa: F401,F403

__all__ = [n for n in dir() if not n.startswith("_")]
