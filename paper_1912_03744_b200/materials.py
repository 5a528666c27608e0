"""Material property tables -- host mirror of proj/include/pulsecell/materials.hpp.

Tables are host data marshalled to the device (where the hot path evaluates
them, adi_device.cuh). The host-side ``eval`` below exists for configuration
checks and diagnostics only; it restates materials.hpp:39-46 exactly.
"""
from __future__ import annotations

import enum
from typing import Dict, List, Optional, Sequence

import numpy as np

from .errors import ConfigError, TableRangeError


class Property(enum.IntEnum):  # materials.hpp:12
    HeatCapacity = 0
    Conductivity = 1
    Resistivity = 2


class RangePolicy(enum.IntEnum):  # materials.hpp:13
    Clamp = 0
    Strict = 1


class HalfPointRule(enum.IntEnum):  # materials.hpp:16-20
    MeanTemperature = 0
    MeanLambda = 1
    TwoSidedHarmonic = 2


class PropertyTable:
    """Piecewise-linear curve over strictly increasing knots (materials.hpp:24-53)."""

    def __init__(self, knots_T: Optional[Sequence[float]] = None,
                 values: Optional[Sequence[float]] = None):
        t = np.asarray([] if knots_T is None else knots_T, dtype=np.float64)
        v = np.asarray([] if values is None else values, dtype=np.float64)
        if t.shape != v.shape:
            raise ConfigError("property table: knot/value size mismatch")
        if t.size > 1 and not np.all(t[1:] > t[:-1]):
            raise ConfigError("property table: temperature knots must be strictly increasing")
        self.t = np.ascontiguousarray(t)
        self.v = np.ascontiguousarray(v)

    def empty(self) -> bool:
        return self.t.size == 0

    def size(self) -> int:
        return int(self.t.size)

    def t_min(self) -> float:
        return float(self.t[0])

    def t_max(self) -> float:
        return float(self.t[-1])

    def covers(self, lo: float, hi: float) -> bool:
        return (not self.empty()) and self.t_min() <= lo and hi <= self.t_max()

    def in_range(self, T: float) -> bool:
        return (not self.empty()) and T >= self.t[0] and T <= self.t[-1]

    def __call__(self, T: float) -> float:  # materials.hpp:39-46
        t, v = self.t, self.v
        if T <= t[0]:
            return float(v[0])
        if T >= t[-1]:
            return float(v[-1])
        k = 1
        while t[k] < T:
            k += 1
        w = (T - float(t[k - 1])) / (float(t[k]) - float(t[k - 1]))
        return float(v[k - 1]) + w * (float(v[k]) - float(v[k - 1]))

    def knots(self) -> np.ndarray:
        return self.t

    def values(self) -> np.ndarray:
        return self.v


class MaterialTable:
    """One layer's material (materials.hpp:57-95, materials.cpp:19-58)."""

    def __init__(self, name: str, rho: float, cv: PropertyTable, lam: PropertyTable,
                 chi: Optional[PropertyTable] = None):
        self._name, self._rho = name, float(rho)
        self.cv, self.lam, self.chi = cv, lam, chi if chi is not None else PropertyTable()
        if not self._rho > 0:
            raise ConfigError(f"material {name}: rho must be > 0")
        if cv.empty():
            raise ConfigError(f"material {name}: missing heat capacity table")
        if lam.empty():
            raise ConfigError(f"material {name}: missing conductivity table")
        if not np.all(cv.v > 0):
            raise ConfigError(f"material {name}: heat capacity values must be > 0")
        if not np.all(lam.v > 0):
            raise ConfigError(f"material {name}: conductivity values must be > 0")
        if not np.all(self.chi.v >= 0):
            raise ConfigError(f"material {name}: resistivity values must be >= 0")

    def name(self) -> str:
        return self._name

    def rho(self) -> float:
        return self._rho

    def table(self, which: Property) -> PropertyTable:
        return {Property.HeatCapacity: self.cv, Property.Conductivity: self.lam,
                Property.Resistivity: self.chi}[Property(which)]

    def has_resistivity(self) -> bool:
        return not self.chi.empty()

    def eval(self, which: Property, T: float, policy: RangePolicy = RangePolicy.Clamp) -> float:
        t = self.table(which)
        if t.empty():
            raise TableRangeError(f"material {self._name}: property table missing")
        if not t.in_range(T) and policy == RangePolicy.Strict:
            raise TableRangeError(f"material {self._name}: T={T} outside table range "
                                  f"[{t.t_min()}, {t.t_max()}]")
        return t(T)


class MaterialSet:
    """Named material collection (materials.hpp:127-139)."""

    def __init__(self) -> None:
        self._tables: List[MaterialTable] = []

    def add(self, table: MaterialTable) -> None:
        if self.contains(table.name()):
            raise ConfigError(f"duplicate material name: {table.name()}")
        self._tables.append(table)

    def by_name(self, name: str) -> MaterialTable:
        for t in self._tables:
            if t.name() == name:
                return t
        raise ConfigError(f"unknown material: {name}")

    def contains(self, name: str) -> bool:
        return any(t.name() == name for t in self._tables)

    def size(self) -> int:
        return len(self._tables)

    def tables(self) -> List[MaterialTable]:
        return list(self._tables)


LayerMaterials = List[MaterialTable]


def resolve_layers(mset: MaterialSet, layer_names: Sequence[str]) -> LayerMaterials:
    return [mset.by_name(n) for n in layer_names]
