"""div_rn (the exact kernels' division by a per-row constant with a
precomputed reciprocal) is bit-identical to the IEEE division on 2^32 random
pairs across wide exponent ranges and on the special values
(tests/native/divcheck.cu); rcp_rn_nb (the line solvers' branch-free
reciprocal) is bit-identical to __drcp_rn wherever it does not flag its input,
and flags every special value (tests/native/rcp_check.cu)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "native", "_build", "divcheck")
RCP_BIN = os.path.join(HERE, "native", "_build", "rcp_check")


@pytest.mark.gpu
def test_div_rn_matches_ieee_division():
    if not os.path.exists(BIN):
        pytest.fail("tests/native/_build/divcheck not built (run __graft_entry__.build())")
    out = subprocess.run([BIN, str(1 << 32)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    n, bad = (int(v) for v in out.stdout.split()[:2])
    assert n == 1 << 32 and bad == 0


@pytest.mark.gpu
def test_rcp_rn_nb_matches_drcp_rn():
    if not os.path.exists(RCP_BIN):
        pytest.fail("tests/native/_build/rcp_check not built (run __graft_entry__.build())")
    out = subprocess.run([RCP_BIN, str(1 << 34)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    words = out.stdout.split()
    assert int(words[1]) == 1 << 34 and int(words[3]) == 0 and int(words[7]) == 0
