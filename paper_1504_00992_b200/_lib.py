"""ctypes binding of ``lib/librrsvd_b200.so`` (the C ABI declared in include/rrsvd_b200.h).

There is no fallback: importing this module on a machine without the built library raises, and
``Context()`` raises when no sm_100 device is present.  Arrays may be numpy (host memory → the
library stages them, the reference-facing end-to-end path) or torch CUDA tensors (device
pointers, no copies).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# (RRSVD_B200_LIB: an alternative in-tree build, for A/B timing of kernel variants)
LIB_PATH = os.environ.get("RRSVD_B200_LIB") or os.path.join(_HERE, "lib", "librrsvd_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "rrsvd_b200.h")

OK, CONTRACT_VIOLATION, NUMERIC_FAILURE, CUDA_ERROR = 0, 1, 2, 3
OP_N, OP_C = 0, 1
OMEGA_REFERENCE, OMEGA_PHILOX = 0, 1

_lib = None


class RrsvdError(RuntimeError):
    code = CUDA_ERROR


class ContractViolation(RrsvdError, ValueError):
    """rrsvd::contract_violation (errors.hpp:11-14)."""
    code = CONTRACT_VIOLATION


class NumericFailure(RrsvdError):
    """rrsvd::numeric_failure (errors.hpp:17-25)."""
    code = NUMERIC_FAILURE


class CudaError(RrsvdError):
    code = CUDA_ERROR


class Backend(C.Structure):
    _fields_ = [("kind", C.c_int), ("target_rank", C.c_uint64), ("oversampling", C.c_uint64),
                ("power_iterations", C.c_uint64), ("accuracy_check", C.c_int),
                ("epsilon", C.c_double), ("probe_count", C.c_uint64),
                ("det_crossover", C.c_uint64), ("seed", C.c_uint64)]


class DecimInfo(C.Structure):
    _fields_ = [("discarded", C.c_double), ("chi", C.c_uint64), ("randomized_path", C.c_int),
                ("tolerance_certified", C.c_int), ("pseudo_inverse_applied", C.c_int)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built — run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (no CPU fallback exists)")
        _lib = C.CDLL(LIB_PATH)
        _lib.rrsvd_b200_version.restype = C.c_char_p
        _lib.rrsvd_b200_last_error.restype = C.c_char_p
        _lib.rrsvd_b200_last_error.argtypes = [C.c_void_p]
        _lib.rrsvd_b200_launch_count.restype = C.c_uint64
        _lib.rrsvd_b200_launch_count.argtypes = [C.c_void_p]
        _lib.rrsvd_b200_ctx_destroy.argtypes = [C.c_void_p]
    return _lib


def header_symbols() -> list[str]:
    """Every function the public header declares (used by the ABI-surface test)."""
    import re
    txt = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(rrsvd_b200_[a-z0-9_]+)\s*\(", txt)))


class Context:
    """An rrsvd_b200_ctx bound to a device and a CUDA stream."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = C.c_void_p()
        rc = lib().rrsvd_b200_ctx_create(C.c_int(device), C.c_void_p(stream), C.byref(h))
        if rc != OK:
            raise CudaError(f"rrsvd_b200_ctx_create failed (code {rc}): no usable sm_100 device")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().rrsvd_b200_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc == OK:
            return
        msg = lib().rrsvd_b200_last_error(self.h).decode()
        raise {CONTRACT_VIOLATION: ContractViolation, NUMERIC_FAILURE: NumericFailure}.get(
            rc, CudaError)(msg)

    @property
    def launches(self) -> int:
        return int(lib().rrsvd_b200_launch_count(self.h))

    def synchronize(self):
        self.check(lib().rrsvd_b200_synchronize(self.h))

    def set_stream(self, stream: int):
        self.check(lib().rrsvd_b200_set_stream(self.h, C.c_void_p(stream)))


# ------------------------------------------------------------------------------- pointers

def ptr(x):
    """Raw pointer of a numpy array (host) or torch tensor (device or host); None → NULL."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous, "arrays must be C-contiguous"
        return C.c_void_p(x.ctypes.data)
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous(), "tensors must be contiguous"
        return C.c_void_p(x.data_ptr())
    raise TypeError(type(x))


def sz(v) -> C.c_size_t:
    return C.c_size_t(int(v))
