"""Snapshot / trace writers against the reference's own
writers (snapshot_io.cpp, compiled into oracle/_ref/libpcref.so), byte for
byte: the host restatements here (CPU), the asynchronous device writer on the
GPU, and evolve() sending its snapshots through that writer."""
import os

import numpy as np
import pytest

from oracle.oracle import RefStepper, ref_evolve
from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.runner import ProbeSpec, RunnerConfig, TraceEntry
from paper_1912_03744_b200.snapshot_io import (SnapshotFormat, SnapshotWriter, read_snapshot_csv,
                                               write_phase_trace, write_snapshot, write_trace)
from paper_1912_03744_b200.solver import make_field


def _case():
    return configs.scaled(configs.cfg4(), [44, 5, 13, 3], 128, 87)


def _ref_snapshot(ref, f, path, fmt, header):
    ref._check(ref.lib.pcref_write_snapshot(ref.h, f.ctypes.data, path.encode(), int(fmt),
                                            header.encode()))


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("fmt", list(SnapshotFormat))
def test_host_write_snapshot_matches_reference(tmp_path, fmt):
    case = _case()
    g = case.grid()
    f = configs.smooth_field(g, 7.0)
    f[3, 4] = np.pi * 1e-7
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    write_snapshot(g, f, a, fmt, "t=0.5 snapshot")
    _ref_snapshot(RefStepper(case), f, b, fmt, "t=0.5 snapshot")
    assert _bytes(a) == _bytes(b)
    if fmt == SnapshotFormat.Csv:
        rows = read_snapshot_csv(a)
        assert len(rows) == g.active_cells() and rows[0].T == f[0, 0]


def test_host_trace_writers_match_reference(tmp_path):
    case = _case()
    ref = RefStepper(case)
    rng = np.random.default_rng(3)
    tr = [TraceEntry(float(t), 1e-3, list(rng.uniform(4, 9, 3))) for t in np.cumsum(rng.uniform(0, 1e-3, 40))]
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    write_trace(tr, 3, a, "trace")
    ts = np.array([e.t for e in tr])
    vs = np.array([v for e in tr for v in e.values])
    ref._check(ref.lib.pcref_write_trace(ref.h, ts.ctypes.data, vs.ctypes.data, len(tr), 3,
                                         b.encode(), b"trace"))
    assert _bytes(a) == _bytes(b)
    rows = [rng.uniform(4, 9, 16) for _ in range(3)]
    write_phase_trace(rows, 0.3, a, "phase")
    flat = np.concatenate(rows)
    ref._check(ref.lib.pcref_write_phase_trace(ref.h, flat.ctypes.data, 3, 16, 0.3, b.encode(),
                                               b"phase"))
    assert _bytes(a) == _bytes(b)


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", list(SnapshotFormat))
def test_device_writer_matches_reference(cuda, tmp_path, fmt):
    from helpers import gpu_stepper, to_dev
    case = _case()
    g = case.grid()
    f = configs.smooth_field(g, 7.0)
    gpu = gpu_stepper(case, "exact")
    w = SnapshotWriter(gpu, slots=2)
    fd = to_dev(f)
    paths = [str(tmp_path / f"s{k}") for k in range(5)]
    for p in paths:  # more submissions than slots: submit waits for a free slot
        w.submit(fd.data_ptr(), p, fmt, "device snapshot")
    assert w.flush() == 5
    w.close()
    ref = str(tmp_path / "ref")
    _ref_snapshot(RefStepper(case), f, ref, fmt, "device snapshot")
    for p in paths:
        assert _bytes(p) == _bytes(ref)


@pytest.mark.gpu
def test_evolve_snapshots_through_writer(cuda, tmp_path):
    """evolve's at-time / post-off snapshots go to the async writer; the files
    equal the reference writer's output for the reference evolve's snapshots."""
    from helpers import gpu_stepper, to_dev
    case = configs.step_cell(True, tau_transient_divisor=10.0, tau_source_divisor=20.0)
    g = case.grid()
    cfg = RunnerConfig(t_end=0.25, probes=[ProbeSpec(0.2, 0.3)], snapshot_times=[0.05, 0.15],
                       snapshot_pre_on=True, snapshot_post_off=True)
    gpu = gpu_stepper(case, "exact")
    w = SnapshotWriter(gpu, slots=2)
    names = {0: "pre_on", 1: "post_off", 2: "at"}

    def target(kind, t, k):
        return (str(tmp_path / f"{names[kind]}_{k}.csv"), SnapshotFormat.Csv, f"t={float(t)!r}")

    res = gpu.evolve(case.timing, to_dev(make_field(g, case.solver.T0)), cfg.t_end, cfg, w,
                     target)
    w.close()
    ref = RefStepper(case)
    want = ref_evolve(ref, make_field(g, case.solver.T0), cfg.t_end, cfg, case.timing.I0)
    assert len(res.at_times) == len(want["at_times"]) == 2
    for k, (snap, (t, fr)) in enumerate(zip(res.at_times, want["at_times"])):
        assert snap.t == t and snap.path and os.path.exists(snap.path)
        rp = str(tmp_path / f"ref_at_{k}.csv")
        _ref_snapshot(ref, fr, rp, SnapshotFormat.Csv, f"t={float(t)!r}")
        assert _bytes(snap.path) == _bytes(rp)
