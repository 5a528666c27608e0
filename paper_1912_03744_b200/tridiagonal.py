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
                       exact: bool = True, stream=None) -> None:
    """Solves `batch` systems of length `n`; the five arguments are contiguous
    float64 CUDA tensors of n*batch elements on one device. `stream`: a CUDA
    stream handle (default: torch's current stream on that device, so the
    solve is ordered with the caller's torch work). x may alias rhs."""
    import torch
    lib = N.load()
    if n < 1 or batch < 1:
        raise ValueError("n and batch must be >= 1")
    if layout not in (CONTIGUOUS, STRIDED):
        raise ValueError("layout must be CONTIGUOUS or STRIDED")
    ts = (lower, diag, upper, rhs, x)
    dev = diag.device if isinstance(diag, torch.Tensor) else None
    for t in ts:
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError("bands must be CUDA tensors")
        if t.dtype != torch.float64:
            raise ValueError("bands must be float64")
        if not t.is_contiguous() or t.numel() != n * batch:
            raise ValueError("bands must be contiguous with n*batch elements")
        if t.device != dev:
            raise ValueError("bands must be on one device")
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    failed = C.c_int64(-1)
    with torch.cuda.device(dev):
        rc = lib.pcgpu_tridiag_batch(*(C.c_void_p(t.data_ptr()) for t in ts), n, batch, layout,
                                     1 if exact else 0, C.c_void_p(stream), C.byref(failed))
    if rc == N.ERR_ZERO_PIVOT:
        raise LineError(failed.value, "thomas_solve: zero pivot")
    if rc != N.OK:
        raise DeviceError(f"pcgpu_tridiag_batch failed ({rc})")
