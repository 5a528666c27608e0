"""pulsecell-b200: B200-native (sm_100a, FP64) ADI hot path of arXiv 1912.03744.

Drop-in for pulsecell::AdiStepper; see DESIGN.md and include/pcgpu.h.
"""
from .errors import (ConfigError, DeviceError, Error, LineError, TableRangeError,  # noqa: F401
                     TauFloorError)
from .geometry import CellMetrics, DomainSpec, Grid, GridSpec, build_grid, cell_metrics  # noqa: F401
from .materials import (HalfPointRule, MaterialSet, MaterialTable, Property,  # noqa: F401
                        PropertyTable, RangePolicy, resolve_layers)
from .source import (FieldSource, JouleSource, NullSource, SourceModel, SourceSpec,  # noqa: F401
                     Waveform, pulse_rect, pulse_transient, pulse_value)
from .solver import (AdiStepper, DevicePlan, HalfStepOutcome, SolverConfig,  # noqa: F401
                     StepResult, initial_tau, make_field)

__version__ = "0.1.0"
