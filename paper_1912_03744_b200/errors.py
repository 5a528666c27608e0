"""Exception hierarchy of the reference (proj/include/pulsecell/errors.hpp:10-54)."""
from __future__ import annotations


class Error(RuntimeError):
    """pulsecell::Error."""


class ConfigError(Error):
    """Invalid run configuration or violated spec invariant (errors.hpp:16-20)."""


class TableRangeError(Error):
    """Temperature outside a property table's knot range in strict mode (errors.hpp:22-26)."""


class TauFloorError(Error):
    """Adaptive halving drove the time step below the floor (errors.hpp:28-42)."""

    def __init__(self, message: str, tau: float = float("nan"), floor: float = float("nan"),
                 time: float = float("nan")):
        super().__init__(message)
        self.tau, self.floor, self.time = tau, floor, time


class LineError(Error):
    """A line body failed; carries the lowest failing line index (errors.hpp:45-54)."""

    def __init__(self, line: int, what: str, cause: type | None = None):
        super().__init__(f"line {line} failed: {what}")
        self.line = line
        self.cause = cause


class DeviceError(Error):
    """CUDA runtime failure inside libpcgpu (no reference equivalent)."""
