"""The C restatement against the committed golden fixtures (generated from
the reference itself by tests/golden/make_golden.py). Runs everywhere,
including where /root/reference is absent."""
import glob
import os

import numpy as np
import pytest

from oracle.oracle import PortStepper, port_available, port_thomas_batch

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
pytestmark = pytest.mark.skipif(not port_available(), reason="oracle/_build not built")


def golden_cases():
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(GOLD, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    return mg.CASES


@pytest.mark.parametrize("case_def", golden_cases(), ids=lambda c: c[0])
def test_port_reproduces_golden(case_def):
    name, build, init, steps, t0 = case_def
    z = np.load(os.path.join(GOLD, f"{name}.npz"))
    case = build()
    port = PortStepper(case)
    f = np.asfortranarray(z["initial"])
    t_end, stats, res = port.run(f, float(z["t0"]), int(z["steps"]))
    seq = np.array([[r.tau_used, r.halvings, r.radial.iterations, r.axial.iterations,
                     r.radial.last_delta, r.axial.last_delta] for r in res])
    assert np.array_equal(seq, z["seq"])
    assert t_end == float(z["t_end"])
    m = case.grid().mask()
    assert np.array_equal(f[m], z["final"][m])
    assert port.clamp_events() == [int(v) for v in z["clamp"]]


def test_port_thomas_golden():
    z = np.load(os.path.join(GOLD, "thomas_batch.npz"))
    batch, n = z["x"].shape
    flat = [np.ascontiguousarray(z[k].reshape(-1)) for k in ("lower", "diag", "upper", "rhs")]
    rc, x, _ = port_thomas_batch(*flat, n, batch, 0)
    assert rc == 0 and np.array_equal(x.reshape(batch, n), z["x"])
    # strided layout of the same systems
    tr = [np.ascontiguousarray(z[k].T.reshape(-1)) for k in ("lower", "diag", "upper", "rhs")]
    rc, xs, _ = port_thomas_batch(*tr, n, batch, 1)
    assert rc == 0 and np.array_equal(xs.reshape(n, batch).T, z["x"])
