"""Snapshot and trace writers (pulsecell snapshot_io.hpp / snapshot_io.cpp),
SURVEY 8(f)-2.

* SnapshotWriter: device fields written off the critical path -- a
  device-to-device copy into a slot on the stepping stream, a pinned-memory
  copy on the writer's copy stream and the formatting on a writer thread in
  libpcgpu.so (pcgpu_writer_*). Byte-identical to the reference's
  write_snapshot (CSV and VTK legacy structured grid).
* write_snapshot / write_trace / write_phase_trace / read_snapshot_csv: the
  reference's formats for host data ("%.17g"), restated here.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import _native as N
from .desc import build_desc
from .errors import DeviceError


class SnapshotFormat(enum.IntEnum):  # snapshot_io.hpp:12
    Csv = 0
    VtkStructured = 1


@dataclass
class SnapshotRow:  # snapshot_io.hpp:14-18
    r: float
    z: float
    layer: int
    T: float


def _g(v: float) -> str:
    """printf("%.17g") (snapshot_io.cpp:12-16)."""
    return "%.17g" % v


def write_snapshot(grid, field: np.ndarray, path: str, fmt: SnapshotFormat, header: str) -> None:
    """snapshot_io.cpp:26-60 for a host field (column-major (nr, nz))."""
    nr, nz = grid.nr(), grid.nz()
    out: List[str] = []
    if fmt == SnapshotFormat.Csv:
        out.append(f"# {header}\n")
        out.append("r,z,layer,T\n")
        for j in range(nz):
            zc = _g(grid.z_center(j))
            for i in range(grid.row_extent(j)):
                out.append(f"{_g(grid.r_center(i))},{zc},{grid.layer(i)},{_g(field[i, j])}\n")
    else:
        out.append("# vtk DataFile Version 3.0\n")
        out.append(f"{header}\n")
        out.append("ASCII\nDATASET STRUCTURED_GRID\n")
        out.append(f"DIMENSIONS {nr} {nz} 1\n")
        out.append(f"POINTS {nr * nz} double\n")
        for j in range(nz):
            zc = _g(grid.z_center(j))
            for i in range(nr):
                out.append(f"{_g(grid.r_center(i))} {zc} 0\n")
        out.append(f"POINT_DATA {nr * nz}\n")
        out.append("SCALARS temperature double 1\nLOOKUP_TABLE default\n")
        for j in range(nz):
            for i in range(nr):
                out.append(_g(field[i, j] if grid.in_mask(i, j) else math.nan) + "\n")
        out.append("SCALARS layer int 1\nLOOKUP_TABLE default\n")
        for j in range(nz):
            for i in range(nr):
                out.append(f"{grid.layer(i)}\n")
        out.append("SCALARS mask int 1\nLOOKUP_TABLE default\n")
        for j in range(nz):
            for i in range(nr):
                out.append("1\n" if grid.in_mask(i, j) else "0\n")
    with open(path, "w", newline="") as f:
        f.write("".join(out))


def read_snapshot_csv(path: str) -> List[SnapshotRow]:  # snapshot_io.cpp:62-86
    rows: List[SnapshotRow] = []
    saw = False
    with open(path) as f:
        for line in f:
            line = line.rstrip("\n")
            if not line or line[0] == "#":
                continue
            if not saw:
                if line != "r,z,layer,T":
                    raise ValueError(f"{path}: unexpected column header")
                saw = True
                continue
            p = line.split(",")
            if len(p) != 4:
                raise ValueError(f"{path}: malformed row: {line}")
            rows.append(SnapshotRow(float(p[0]), float(p[1]), int(p[2]), float(p[3])))
    return rows


def write_trace(trace, probe_count: int, path: str, header: str) -> None:
    """snapshot_io.cpp:88-101: columns t, probe_1..probe_k."""
    out = [f"# {header}\n", "t" + "".join(f",probe_{k}" for k in range(1, probe_count + 1)) + "\n"]
    for e in trace:
        out.append(_g(e.t) + "".join("," + _g(v) for v in e.values) + "\n")
    with open(path, "w", newline="") as f:
        f.write("".join(out))


def write_phase_trace(periods: Sequence[np.ndarray], t_per: float, path: str,
                      header: str) -> None:
    """snapshot_io.cpp:103-117: columns period, phase_index, phase_t, value."""
    out = [f"# {header}\n", "period,phase_index,phase_t,value\n"]
    for p, row in enumerate(periods):
        s = len(row)
        for q in range(s):
            phase_t = (float(p) + float(q) / s) * t_per
            out.append(f"{p},{q},{_g(phase_t)},{_g(row[q])}\n")
    with open(path, "w", newline="") as f:
        f.write("".join(out))


class SnapshotWriter:
    """Asynchronous writer of device snapshots (pcgpu_writer_*)."""

    def __init__(self, stepper, slots: int = 2):
        self._lib = N.load()
        g = stepper.grid()
        self._grid = g
        self._stepper = stepper
        desc, self._keep = build_desc(g, stepper._mats, stepper._source, stepper._timing,
                                      stepper._cfg, stepper._plan.mode_id(),
                                      stepper._plan.device)
        self._zc = np.array([g.z_center(j) for j in range(g.nz())], dtype=np.float64)
        h = C.c_void_p()
        rc = self._lib.pcgpu_writer_create(C.byref(desc), self._zc.ctypes.data, int(slots),
                                           C.byref(h))
        if rc != N.OK:
            raise DeviceError(f"pcgpu_writer_create failed ({rc})")
        self._h = h

    def submit(self, field_dev_ptr: int, path: str, fmt: SnapshotFormat, header: str,
               stream: int = 0) -> None:
        """Queue a device field (raw pointer, column-major nr x nz) for writing;
        `stream`: the stream that produced it (default: the stepper's)."""
        st = stream or self._stepper.stream()
        rc = self._lib.pcgpu_writer_submit(self._h, C.c_void_p(field_dev_ptr), C.c_void_p(st),
                                           path.encode(), int(fmt), header.encode())
        if rc != N.OK:
            raise DeviceError(f"pcgpu_writer_submit failed ({rc})")

    def flush(self) -> int:
        n = C.c_int64()
        rc = self._lib.pcgpu_writer_flush(self._h, C.byref(n))
        if rc != N.OK:
            raise DeviceError(self._lib.pcgpu_writer_last_error(self._h).decode())
        return int(n.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self.flush()
            self._lib.pcgpu_writer_destroy(self._h)
            self._h = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.pcgpu_writer_destroy(h)
            self._h = None
