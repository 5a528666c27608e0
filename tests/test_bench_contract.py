"""bench.py's reference arm on the CPU: one JSON line with the driver's keys
(the reference's own AdiStepper from oracle/_ref on the host cores, or the C
restatement when the reference library is absent)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--cpu-nz", "64"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "FP64 ADI cell-updates/s (incl. Picard iters)"
    assert d["unit"] == "cell-updates/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["dtype"] == "f64"
    assert d["config"]["workload"].startswith("cfg3")
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("reference", "port") and cb["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_stdout_is_only_the_json_line():
    """Whatever this process or its libraries write to fd 1 (NCCL prints its
    version banner there) goes to stderr; stdout holds the one JSON line."""
    code = (
        "import os, sys, json\n"
        "sys.path.insert(0, %r)\n"
        "import bench\n"
        "bench.claim_stdout()\n"
        "os.write(1, b'NCCL version 2.28.9+cuda12.9\\n')\n"   # a C library writing to fd 1
        "print('a python print')\n"
        "bench.emit({'metric': 'm', 'value': 1.0})\n"
    ) % ROOT
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.splitlines() == [json.dumps({"metric": "m", "value": 1.0})]
    assert "NCCL version" in r.stderr and "a python print" in r.stderr
