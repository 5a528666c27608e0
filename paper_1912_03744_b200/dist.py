"""Partitioned ADI stepper across the B200s of one node.

One process per GPU (torchrun), torch.distributed for the plumbing: rank 0
creates the NCCL unique id through the library, the process group broadcasts
it, and every rank builds a `pcgpu_dist` (include/pcgpu.h). The library then
runs the z-slab radial sweep, the all-to-all transposes and the per-iteration
allreduce(max) of the Picard norm itself (NCCL on the library's stream).
With ``emulate=P`` the library runs P virtual ranks in this process on one
GPU -- the same code path minus NCCL -- which is how the partitioned path is
validated on a single GPU (bit-identical to the single-GPU stepper).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from .desc import build_desc
from .errors import ConfigError, DeviceError, TauFloorError
from .solver import DevicePlan, _step_result


def slab_plan(grid, mats, source, timing, cfg, nranks: int) -> Tuple[List[int], List[int]]:
    """Slab boundaries (host only, no GPU): rank p owns radial lines
    [zb[p], zb[p+1]) and axial lines [rb[p], rb[p+1])."""
    lib = N.load()
    desc, keep = build_desc(grid, mats, source, timing, cfg, N.MODE_EXACT, 0)
    zb = (C.c_int32 * (nranks + 1))()
    rb = (C.c_int32 * (nranks + 1))()
    rc = lib.pcgpu_dist_plan(C.byref(desc), nranks, zb, rb)
    if rc != N.OK:
        raise ConfigError("pcgpu_dist_plan failed")
    return list(zb), list(rb)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    if N.load().pcgpu_nccl_unique_id(buf) != N.OK:
        raise DeviceError("ncclGetUniqueId failed")
    return bytes(buf)


def share_unique_id(rank: int, device=None) -> bytes:
    """Rank 0 creates the id, torch.distributed broadcasts it."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend()
    dev = device if (device is not None and backend == "nccl") else "cpu"
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, src=0)
    return bytes(t.cpu().numpy().tobytes())


def allgather_bytes(mine: bytes) -> bytes:
    """Every rank's equal-length byte block, concatenated in rank order
    (torch.distributed all_gather; CUDA tensors under NCCL, CPU under gloo)."""
    import torch
    import torch.distributed as dist
    t = torch.frombuffer(bytearray(mine), dtype=torch.uint8)
    dev = f"cuda:{torch.cuda.current_device()}" if dist.get_backend() == "nccl" else "cpu"
    parts = [torch.zeros(len(mine), dtype=torch.uint8, device=dev)
             for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t.to(dev))
    return b"".join(bytes(p.cpu().numpy().tobytes()) for p in parts)


class PartitionedAdi:
    """z-slab / r-slab partitioned AdiStepper.

    The exact kernels on dense slabs -- bit-identical to the single-GPU
    stepper (and so to the reference)."""

    def __init__(self, grid, mats, source, timing, cfg, device: int = 0,
                 rank: int = 0, world: int = 1, emulate: Optional[int] = None,
                 unique_id: Optional[bytes] = None, mode: str = "exact"):
        self._lib = N.load()
        cfg.validate()
        timing.validate()
        self._grid = grid
        self._nr, self._nz = grid.nr(), grid.nz()
        if mode != "exact":
            raise ConfigError(f"exec.mode: unknown mode {mode!r} (only 'exact' exists)")
        self.mode = mode
        self._desc, self._keep = build_desc(grid, mats, source, timing, cfg, N.MODE_EXACT,
                                            device)
        h = C.c_void_p()
        if emulate is not None:
            rc = self._lib.pcgpu_dist_create(C.byref(self._desc), 0, int(emulate), None,
                                              C.byref(h))
        else:
            if unique_id is None:
                raise ValueError("unique_id required for a multi-process partitioned run")
            idbuf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
            rc = self._lib.pcgpu_dist_create(C.byref(self._desc), rank, world, idbuf, C.byref(h))
        if rc != N.OK:
            msg = self._lib.pcgpu_dist_last_error(None).decode()
            raise (ConfigError if rc == N.ERR_CONFIG else DeviceError)(msg)
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.pcgpu_dist_destroy(self._h)
            self._h = None

    def _check(self, rc):
        if rc == N.OK:
            return
        msg = self._lib.pcgpu_dist_last_error(self._h).decode()
        if rc == N.ERR_TAU_FLOOR:
            raise TauFloorError(msg)
        raise DeviceError(f"pcgpu_dist error {rc}: {msg}")

    def slabs(self):
        v = [C.c_int32() for _ in range(4)]
        self._lib.pcgpu_dist_slabs(self._h, *(C.byref(x) for x in v))
        return tuple(x.value for x in v)

    def set_field(self, field_dev) -> None:
        self._check(self._lib.pcgpu_dist_set_field(self._h, C.c_void_p(field_dev.data_ptr())))

    def get_field(self, field_dev) -> None:
        self._check(self._lib.pcgpu_dist_get_field(self._h, C.c_void_p(field_dev.data_ptr())))

    @staticmethod
    def _host_ptr(field, nr: int, nz: int, writable: bool):
        a = field
        if getattr(a, "shape", None) != (nr, nz) or a.dtype != "float64" or \
                not a.flags["F_CONTIGUOUS"] or (writable and not a.flags["WRITEABLE"]):
            raise ValueError("host field: a writable (nr, nz) float64 Fortran-ordered array")
        return C.c_void_p(a.ctypes.data)

    def set_field_host(self, field) -> None:
        """Exact mode: this rank's state lines (r-slab columns) from a host
        field ((nr, nz) float64, Fortran order; pinned for full PCIe speed)."""
        nr, nz = self._nr, self._nz
        self._check(self._lib.pcgpu_dist_set_field_host(self._h, self._host_ptr(field, nr, nz, False)))

    def get_field_host(self, field) -> None:
        """Exact mode: this rank's state lines into the host field."""
        nr, nz = self._nr, self._nz
        self._check(self._lib.pcgpu_dist_get_field_host(self._h, self._host_ptr(field, nr, nz, True)))

    def run(self, t0: float, nsteps: int, keep_results: bool = False):
        res = (N.StepResultC * nsteps)() if keep_results and nsteps > 0 else None
        st = N.RunStats()
        rc = self._lib.pcgpu_dist_run(self._h, t0, int(nsteps), res, C.byref(st))
        stats = {k: getattr(st, k) for k, _ in N.RunStats._fields_}
        self._check(rc)
        return float(st.t_end), stats, ([_step_result(r) for r in res] if res is not None else [])

    def transport(self) -> str:
        """'peer' (fused slab passes store into the owners' slabs) or 'nccl'
        (all-to-all transposes)."""
        return "peer" if self._lib.pcgpu_dist_transport(self._h) == 1 else "nccl"

    def enable_peer_transport(self) -> None:
        """Exact mode, one process per GPU: map every rank's slabs into this
        process (CUDA IPC handles all-gathered over torch.distributed), so the
        fused K3/K4 passes store straight into the peers over NVLink."""
        mine = (C.c_uint8 * N.DIST_IPC_BYTES)()
        self._check(self._lib.pcgpu_dist_ipc_export(self._h, mine))
        blob = allgather_bytes(bytes(mine))
        allh = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        rc = self._lib.pcgpu_dist_ipc_import(self._h, allh)
        # every rank must use the same transport: agree on the outcome
        ok = allgather_bytes(bytes([1 if rc == N.OK else 0]))
        if all(ok):
            return True
        self._check(self._lib.pcgpu_dist_peer_off(self._h))
        import warnings
        warnings.warn("pcgpu: CUDA IPC peer mapping failed on rank(s) "
                      f"{[r for r, v in enumerate(ok) if not v]}; using the NCCL transport")
        return False

    def stream(self) -> int:
        return int(self._lib.pcgpu_dist_stream(self._h) or 0)

    def launch_count(self) -> int:
        return int(self._lib.pcgpu_dist_launch_count(self._h))

    def enable_timing(self, on: bool = True) -> None:
        self._lib.pcgpu_dist_enable_timing(self._h, 1 if on else 0)

    def timing(self) -> dict:
        tm, rm, am = C.c_double(), C.c_double(), C.c_double()
        tn, an = C.c_int64(), C.c_int64()
        self._lib.pcgpu_dist_timing(self._h, C.byref(tm), C.byref(tn), C.byref(an), C.byref(rm),
                                    C.byref(am))
        return {"transpose_ms": tm.value, "transposes": tn.value, "allreduces": an.value,
                "radial_ms": rm.value, "axial_ms": am.value}
