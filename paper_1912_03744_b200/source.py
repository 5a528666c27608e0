"""Pulsed Joule source -- host mirror of proj/include/pulsecell/source.hpp.

pulse_value is a host scalar per half-step (bind_time); the per-cell power
chi(T) * amplitude * pulse is evaluated on the device inside the line kernels.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import ConfigError
from .geometry import _llround
from .materials import MaterialTable, Property, RangePolicy


class Waveform(enum.IntEnum):  # source.hpp:9
    Rectangular = 0
    Transient = 1


@dataclass
class SourceSpec:
    """source.hpp:14-29."""
    t_per: float = 0.0
    t_src: float = 0.0
    t_trs: float = 0.0
    xi: float = 4.0
    zeta: float = 2.0
    I0: float = 0.0
    S_C: float = 0.0
    waveform: Waveform = Waveform.Transient
    joule_dimensional: bool = False

    def validate(self) -> None:  # source.cpp:9-17
        if not self.t_per > 0:
            raise ConfigError("source.t_per: must be > 0")
        if not (self.t_src > 0 and self.t_src <= self.t_per):
            raise ConfigError("source.t_src: must satisfy 0 < t_src <= t_per")
        if not (self.t_trs > 0 and self.t_trs < self.t_src):
            raise ConfigError("source.t_trs: must satisfy 0 < t_trs < t_src")
        if not self.xi > 0:
            raise ConfigError("source.xi: must be > 0")
        if not self.zeta > 0:
            raise ConfigError("source.zeta: must be > 0")
        if self.I0 < 0:
            raise ConfigError("source.I0: must be >= 0")

    def current_factor(self) -> float:  # source.hpp:26-28
        if self.joule_dimensional:
            return self.I0 * self.I0 / (self.S_C * self.S_C)
        return self.I0 * self.I0 / self.S_C


def pulse_rect(t: float, spec: SourceSpec) -> float:  # source.cpp:18-21
    phase = math.fmod(t, spec.t_per)
    return 1.0 if phase < spec.t_src else 0.0


def pulse_transient(t: float, spec: SourceSpec) -> float:  # source.cpp:23-40
    phase = math.fmod(t, spec.t_per)
    margin = spec.t_trs / spec.zeta * (1.0 + 6.5 / spec.xi)
    elapsed = _llround((t - phase) / spec.t_per)
    back_hi = min(elapsed, 1 + int(math.ceil((spec.t_src + margin) / spec.t_per)))
    scale = spec.xi * spec.zeta / spec.t_trs
    s = 0.0
    for m in range(-1, back_hi + 1):
        u = phase + float(m) * spec.t_per
        s += math.erf(scale * u - spec.xi) - math.erf(scale * (u - spec.t_src) - spec.xi)
    return 0.5 * s


def pulse_value(t: float, spec: SourceSpec) -> float:  # source.cpp:42-45
    return pulse_rect(t, spec) if spec.waveform == Waveform.Rectangular else pulse_transient(t, spec)


class SourceModel:
    """Per-cell power hook (source.hpp:48-55). Device-native kinds are
    NullSource / JouleSource; T-independent models subclass FieldSource."""

    kind = -1

    def bind_time(self, t: float) -> None:
        raise NotImplementedError


class NullSource(SourceModel):  # source.hpp:57-61
    kind = 0

    def bind_time(self, t: float) -> None:
        pass


class JouleSource(SourceModel):  # source.hpp:63-83, source.cpp:47-58
    kind = 1

    def __init__(self, spec: SourceSpec, source_layer: int, source_material: MaterialTable,
                 policy: RangePolicy = RangePolicy.Clamp):
        self.spec = spec
        self.source_layer = source_layer
        self.material = source_material
        self.policy = policy
        self.amplitude = spec.current_factor() if spec.S_C > 0 else float("nan")
        spec.validate()
        if not spec.S_C > 0:
            raise ConfigError("source.S_C: must be > 0")
        if spec.I0 > 0 and not source_material.has_resistivity():
            raise ConfigError(f"material {source_material.name()}: source layer needs a "
                              "resistivity table")
        self.pulse = 0.0

    def bind_time(self, t: float) -> None:
        self.pulse = pulse_value(t, self.spec)


class FieldSource(SourceModel):
    """T-independent per-cell power (e.g. the acceptance suite's manufactured
    source, acceptance_main.cpp:262-274). Subclasses implement
    ``power_field(grid, t) -> (nr, nz) array``; the stepper binds it to the
    device once per half-step at t + tau/2."""

    kind = 2

    def __init__(self, grid):
        self.grid = grid

    def bind_time(self, t: float) -> None:
        pass

    def power_field(self, grid, t: float) -> np.ndarray:
        raise NotImplementedError
