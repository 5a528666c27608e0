"""Shared helpers for the parity tests."""
from __future__ import annotations

import numpy as np

from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan, make_field
from paper_1912_03744_b200.source import FieldSource, JouleSource, NullSource


make_source = configs.make_source


def gpu_stepper(case, mode="exact", source=None):
    g = case.grid()
    src = source if source is not None else make_source(case, g)
    return AdiStepper(g, case.materials, src, case.timing, case.solver,
                      DevicePlan(device=0, mode=mode))


def to_dev(f: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(f.T)).cuda().t()


def to_host(t) -> np.ndarray:
    return np.asfortranarray(t.t().contiguous().cpu().numpy().T)


def rel_linf(a: np.ndarray, b: np.ndarray, mask: np.ndarray) -> float:
    return float(np.max(np.abs(a[mask] - b[mask])) / np.max(np.abs(b[mask])))
