"""configs[1]'s data generator (tools/cfg1_gen.c) draws exactly the stream
SURVEY 8(d) specifies: std::mt19937_64(2024) with
std::uniform_real_distribution<double> (checked against <random> itself)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_cfg1_generator_matches_std_random(tmp_path):
    obj = tmp_path / "gen.o"
    exe = tmp_path / "check"
    subprocess.run(["gcc", "-O2", "-c", os.path.join(ROOT, "tools", "cfg1_gen.c"), "-o", str(obj)],
                   check=True)
    subprocess.run(["g++", "-O2", os.path.join(ROOT, "tools", "test_cfg1_gen.cpp"), str(obj), "-o",
                    str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr
