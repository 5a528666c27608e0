"""Batched tridiagonal solves on the GPU (BASELINE configs[1]).

thomas_solve_inplace (tridiagonal.hpp:25-42) over many independent systems,
in the line-contiguous or the strided (interleaved) layout. Arguments are
torch CUDA float64 tensors.
"""
from __future__ import annotations

import ctypes as C

from . import _native as N
from .errors import DeviceError, LineError

CONTIGUOUS, STRIDED = N.LAYOUT_CONTIGUOUS, N.LAYOUT_STRIDED


def thomas_solve_batch(lower, diag, upper, rhs, x, n: int, batch: int, layout: int = CONTIGUOUS,
                       exact: bool = True, stream: int = 0) -> None:
    lib = N.load()
    for t in (lower, diag, upper, rhs, x):
        if not t.is_cuda or t.numel() != n * batch:
            raise ValueError("bands must be CUDA tensors with n*batch elements")
    failed = C.c_int64(-1)
    rc = lib.pcgpu_tridiag_batch(*(C.c_void_p(t.data_ptr()) for t in (lower, diag, upper, rhs, x)),
                                 n, batch, layout, 1 if exact else 0, C.c_void_p(stream),
                                 C.byref(failed))
    if rc == N.ERR_ZERO_PIVOT:
        raise LineError(failed.value, "thomas_solve: zero pivot")
    if rc != N.OK:
        raise DeviceError(f"pcgpu_tridiag_batch failed ({rc})")
