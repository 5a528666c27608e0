"""The C++ drop-in (include/pulsecell_gpu/adi_stepper.hpp) against the
reference's own AdiStepper, side by side in one native process on the
reference's own objects (tests/native/dropin_test.cpp): bit-identical steps
in exact mode, the reference exception types, and the device path of the
reference's simulate / bench commands (include/pulsecell_gpu/cli_device.hpp,
SURVEY 8(f)-4): simulate's output files byte-identical to the CPU run's."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "native", "_build", "dropin_test")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/native not built (needs the reference headers)")
def test_cpp_dropin_bitwise_vs_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "masked cells differing 0" in r.stdout
    assert "evolve" in r.stdout and "identical" in r.stdout
    assert "differing 0, bench --device ok" in r.stdout
