"""Marshal the host objects into the C-ABI descriptor (include/pcgpu.h).

The reference's C++ wrapper does the same from pulsecell::Grid et al.
(include/pulsecell_gpu/adi_stepper.hpp); this is the Python-side equivalent.
"""
from __future__ import annotations

import ctypes as C
from typing import Any, List, Tuple

import numpy as np

from . import _native as N
from .geometry import Grid
from .materials import LayerMaterials, PropertyTable
from .source import FieldSource, JouleSource, NullSource, SourceModel, SourceSpec


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _table(t: PropertyTable, keep: List[Any]) -> N.Table:
    tt = np.ascontiguousarray(t.t, dtype=np.float64)
    vv = np.ascontiguousarray(t.v, dtype=np.float64)
    keep += [tt, vv]
    return N.Table(int(tt.size), _dptr(tt), _dptr(vv))


def source_kind(source: SourceModel) -> int:
    if isinstance(source, JouleSource):
        return N.SOURCE_JOULE
    if isinstance(source, FieldSource):
        return N.SOURCE_FIELD
    if isinstance(source, NullSource):
        return N.SOURCE_NULL
    raise TypeError(f"unsupported SourceModel {type(source).__name__}: the device supports "
                    "NullSource, JouleSource and FieldSource (T-independent per-cell power)")


def build_desc(grid: Grid, mats: LayerMaterials, source: SourceModel, timing: SourceSpec,
               cfg, mode: int = N.MODE_EXACT, device: int = 0,
               explicit_extents: bool = False) -> Tuple[N.Desc, List[Any]]:
    """pcgpu_desc of a problem. The masked extents are passed as arrays for a
    generalised stepped domain (or when explicit_extents is set); otherwise
    the library derives them from nr_core / nz_shared like the reference."""
    keep: List[Any] = []
    layer = np.ascontiguousarray(grid.layer_arr, dtype=np.int32)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
            (grid.r_centers, grid.gap_r_arr, grid.width_z_arr, grid.gap_z_arr)]
    keep += [layer] + arrs
    m_arr = (N.Material * max(1, len(mats)))()
    for k, m in enumerate(mats):
        if m is None:
            m_arr[k] = N.Material(0.0, N.Table(), N.Table(), N.Table())
            continue
        m_arr[k] = N.Material(m.rho(), _table(m.cv, keep), _table(m.lam, keep),
                              _table(m.chi, keep))
    keep.append(m_arr)
    d = N.Desc()
    d.abi_version = N.PCGPU_ABI_VERSION
    d.nr, d.nz = grid.nr(), grid.nz()
    d.nr_core, d.nz_shared = grid.nr_core(), grid.nz_shared()
    d.layer = layer.ctypes.data_as(C.POINTER(C.c_int32))
    d.r_center, d.gap_r, d.width_z, d.gap_z = (_dptr(a) for a in arrs)
    # one material per layer is validated by the library (solver.cpp:135-136)
    d.n_layers = len(mats) if len(mats) == grid.domain().layer_count() else -1
    d.materials = C.cast(m_arr, C.POINTER(N.Material))
    d.source_kind = source_kind(source)
    d.source_layer = getattr(source, "source_layer", grid.domain().source_layer)
    d.amplitude = getattr(source, "amplitude", 0.0)
    d.t_per, d.t_src, d.t_trs = timing.t_per, timing.t_src, timing.t_trs
    d.xi, d.zeta, d.waveform = timing.xi, timing.zeta, int(timing.waveform)
    d.epsilon, d.max_iter, d.tau_min = cfg.epsilon, cfg.max_iter, cfg.tau_min
    d.tau_transient_divisor = cfg.tau_transient_divisor
    d.tau_source_divisor = cfg.tau_source_divisor
    d.halfpoint_rule, d.range_policy = int(cfg.halfpoint_rule), int(cfg.range_policy)
    d.all_neumann = 1 if cfg.all_neumann else 0
    d.T0, d.t_ceiling = cfg.T0, cfg.t_ceiling
    d.mode, d.device = int(mode), int(device)
    if explicit_extents or not grid.domain().is_two_level():  # explicit extents
        re = np.ascontiguousarray(grid.row_extents(), dtype=np.int32)
        ce = np.ascontiguousarray(grid.col_extents(), dtype=np.int32)
        keep += [re, ce]
        d.row_extent = re.ctypes.data_as(C.POINTER(C.c_int32))
        d.col_extent = ce.ctypes.data_as(C.POINTER(C.c_int32))
    return d, keep
