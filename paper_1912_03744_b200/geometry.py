"""Stepped multilayer cylinder grid -- host mirror of pulsecell::Grid.

Restates proj/include/pulsecell/geometry.hpp:14-125 and proj/src/geometry.cpp:
every metric is computed with the same IEEE double operations in the same
order, so the arrays are bit-identical to the reference Grid's (checked
against the reference build in tests/test_host_mirror.py). The grid is host
data; the kernels receive its metric arrays through the C-ABI.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .errors import ConfigError


def _llround(x: float) -> int:
    """std::llround (round half away from zero)."""
    r = math.floor(abs(x))
    if abs(x) - r >= 0.5:
        r += 1
    return int(r if x >= 0 else -r)


@dataclass
class DomainSpec:
    """geometry.hpp:14-27."""
    layer_radii: List[float] = field(default_factory=list)
    core_length: float = 0.0
    outer_length: float = 0.0
    layer_materials: List[str] = field(default_factory=list)
    source_layer: int = 0
    # Generalised stepped domain (beyond the reference): the
    # axial length of every layer, non-increasing outward, the core's being
    # core_length and the shortest outer_length. None: the reference's two
    # levels (core_length for layer 0, outer_length for the others).
    layer_lengths: Optional[List[float]] = None

    def validate(self) -> None:  # geometry.cpp:7-22
        if not self.layer_radii:
            raise ConfigError("domain.layer_radii: empty")
        prev = 0.0
        for r in self.layer_radii:
            if not r > prev:
                raise ConfigError("domain.layer_radii: must be strictly increasing and positive")
            prev = r
        if not self.core_length > 0:
            raise ConfigError("domain.core_length: must be > 0")
        if not self.outer_length > 0:
            raise ConfigError("domain.outer_length: must be > 0")
        if self.outer_length > self.core_length:
            raise ConfigError("domain.outer_length: exceeds core_length")
        if len(self.layer_materials) != len(self.layer_radii):
            raise ConfigError("domain.layer_materials: needs one entry per layer")
        if self.source_layer < 0 or self.source_layer >= self.layer_count():
            raise ConfigError("domain.source_layer: out of range")
        if self.layer_lengths is not None:
            L = list(self.layer_lengths)
            if len(L) != self.layer_count():
                raise ConfigError("domain.layer_lengths: needs one entry per layer")
            if any(not (b <= a) for a, b in zip(L, L[1:])):
                raise ConfigError("domain.layer_lengths: must be non-increasing outward")
            if L[0] != self.core_length or min(L) != self.outer_length:
                raise ConfigError("domain.layer_lengths: must span outer_length .. core_length")

    def lengths(self) -> List[float]:
        """Axial length of every layer."""
        if self.layer_lengths is not None:
            return list(self.layer_lengths)
        return [self.core_length] + [self.outer_length] * (self.layer_count() - 1)

    def is_two_level(self) -> bool:
        """True when the layer lengths are the reference's own rule."""
        return self.layer_lengths is None or list(self.layer_lengths) == (
            [self.core_length] + [self.outer_length] * (self.layer_count() - 1))

    def layer_count(self) -> int:
        return len(self.layer_radii)

    def r_max(self) -> float:
        return self.layer_radii[-1]

    def layer_inner_radius(self, m: int) -> float:
        return 0.0 if m == 0 else self.layer_radii[m - 1]

    def source_cross_section(self) -> float:  # geometry.cpp:24-29
        ro = self.layer_radii[self.source_layer]
        ri = self.layer_inner_radius(self.source_layer)
        return math.pi * (ro * ro - ri * ri)


@dataclass
class GridSpec:
    """geometry.hpp:29-35."""
    radial_divisions: List[int] = field(default_factory=list)
    axial_divisions_core: int = 1
    axial_divisions_outer: int = 1

    def validate(self, domain: DomainSpec) -> None:  # geometry.cpp:31-40
        if len(self.radial_divisions) != len(domain.layer_radii):
            raise ConfigError("grid.radial_divisions: needs one entry per layer")
        if any(n < 1 for n in self.radial_divisions):
            raise ConfigError("grid.radial_divisions: all counts must be >= 1")
        if self.axial_divisions_core < 1:
            raise ConfigError("grid.axial_divisions_core: must be >= 1")
        if self.axial_divisions_outer < 1:
            raise ConfigError("grid.axial_divisions_outer: must be >= 1")


@dataclass
class CellMetrics:
    r: float
    hbar: float
    etabar: float
    r_lo: float
    r_hi: float


class Grid:
    """Cell-centred shifted grid over the stepped domain (geometry.hpp:45-115)."""

    def __init__(self, domain: DomainSpec, spec: GridSpec):
        domain.validate()
        spec.validate(domain)
        self._domain, self._spec = domain, spec
        r_center, width_r, layer = [], [], []
        for m in range(domain.layer_count()):  # geometry.cpp:47-58
            lo = domain.layer_inner_radius(m)
            hi = domain.layer_radii[m]
            n = spec.radial_divisions[m]
            w = (hi - lo) / n
            for q in range(n):
                r_center.append(lo + (q + 0.5) * w)
                width_r.append(w)
                layer.append(m)
        self._nr_core = spec.radial_divisions[0]
        z0, zmax = domain.outer_length, domain.core_length  # geometry.cpp:60-82
        self._nz_shared = spec.axial_divisions_outer
        z_center, width_z = [], []
        w = z0 / spec.axial_divisions_outer
        for q in range(spec.axial_divisions_outer):
            z_center.append((q + 0.5) * w)
            width_z.append(w)
        # Segments above the shared region: the reference's single extension
        # [outer_length, core_length], or one per distinct layer length of a
        # generalised domain, each sized with the core's axial step.
        levels = sorted(set(domain.lengths()))
        seg_end = [spec.axial_divisions_outer]  # z cells up to each level
        core_step = zmax / spec.axial_divisions_core
        for lo, hi in zip(levels, levels[1:]):
            n_ext = max(1, _llround((hi - lo) / core_step))
            w = (hi - lo) / n_ext
            for q in range(n_ext):
                z_center.append(lo + (q + 0.5) * w)
                width_z.append(w)
            seg_end.append(len(z_center))
        # masked extents: layer m spans the z cells below its length
        lens = domain.lengths()
        col_of_layer = [seg_end[levels.index(L)] for L in lens]
        self._col_ext = np.array([col_of_layer[m] for m in layer], dtype=np.int32)
        self._row_ext = np.array([int(np.sum(self._col_ext > j)) for j in range(len(z_center))],
                                 dtype=np.int32)
        gap_r = [0.0] * (len(r_center) + 1)  # geometry.cpp:84-94
        gap_r[0], gap_r[-1] = width_r[0], width_r[-1]
        for i in range(1, len(r_center)):
            gap_r[i] = r_center[i] - r_center[i - 1]
        gap_z = [0.0] * (len(z_center) + 1)
        gap_z[0], gap_z[-1] = width_z[0], width_z[-1]
        for j in range(1, len(z_center)):
            gap_z[j] = z_center[j] - z_center[j - 1]
        f8 = np.float64
        self.r_centers = np.array(r_center, dtype=f8)
        self.z_centers = np.array(z_center, dtype=f8)
        self.width_r_arr = np.array(width_r, dtype=f8)
        self.width_z_arr = np.array(width_z, dtype=f8)
        self.gap_r_arr = np.array(gap_r, dtype=f8)
        self.gap_z_arr = np.array(gap_z, dtype=f8)
        self.layer_arr = np.array(layer, dtype=np.int32)
        self._active = sum(self.col_extent(i) for i in range(self.nr()))

    def domain(self) -> DomainSpec:
        return self._domain

    def spec(self) -> GridSpec:
        return self._spec

    def nr(self) -> int:
        return len(self.r_centers)

    def nz(self) -> int:
        return len(self.z_centers)

    def nr_core(self) -> int:
        return self._nr_core

    def nz_shared(self) -> int:
        return self._nz_shared

    def r_center(self, i: int) -> float:
        return float(self.r_centers[i])

    def z_center(self, j: int) -> float:
        return float(self.z_centers[j])

    def width_r(self, i: int) -> float:
        return float(self.width_r_arr[i])

    def width_z(self, j: int) -> float:
        return float(self.width_z_arr[j])

    def gap_r(self, i: int) -> float:
        return float(self.gap_r_arr[i])

    def gap_z(self, j: int) -> float:
        return float(self.gap_z_arr[j])

    def row_extent(self, j: int) -> int:
        return int(self._row_ext[j])

    def col_extent(self, i: int) -> int:
        return int(self._col_ext[i])

    def row_extents(self) -> np.ndarray:
        return self._row_ext

    def col_extents(self) -> np.ndarray:
        return self._col_ext

    def in_mask(self, i: int, j: int) -> bool:
        return 0 <= i < self.nr() and 0 <= j < self.col_extent(i)

    def active_cells(self) -> int:
        return self._active

    def layer(self, i: int) -> int:
        return int(self.layer_arr[i])

    def control_r(self, i: int) -> float:
        return 0.5 * (self.gap_r(i) + self.gap_r(i + 1))

    def control_z(self, j: int) -> float:
        return 0.5 * (self.gap_z(j) + self.gap_z(j + 1))

    def face_r_lo(self, i: int) -> float:
        return 0.0 if i == 0 else 0.5 * (self.r_center(i - 1) + self.r_center(i))

    def face_r_hi(self, i: int, n: int) -> float:
        if i == n - 1:
            return self.r_center(i) + 0.5 * self.width_r(i)
        return 0.5 * (self.r_center(i) + self.r_center(i + 1))

    def mask(self) -> np.ndarray:
        """Boolean (nr, nz) array of in-mask cells."""
        m = np.zeros((self.nr(), self.nz()), dtype=bool)
        for i in range(self.nr()):
            m[i, : self._col_ext[i]] = True
        return m


def build_grid(domain: DomainSpec, spec: GridSpec) -> Grid:
    return Grid(domain, spec)


def cell_metrics(grid: Grid, i: int, j: int) -> CellMetrics:  # geometry.cpp:103-110
    if not grid.in_mask(i, j):
        raise ConfigError(f"cell_metrics: index ({i},{j}) outside the domain mask")
    n = grid.row_extent(j)
    return CellMetrics(grid.r_center(i), grid.control_r(i), grid.control_z(j),
                       grid.face_r_lo(i), grid.face_r_hi(i, n))


def layer_index(grid: Grid, i: int, j: int) -> int:
    if not grid.in_mask(i, j):
        raise ConfigError(f"layer_index: index ({i},{j}) outside the domain mask")
    return grid.layer(i)
