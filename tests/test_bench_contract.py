"""The driver's bench contract on CPU: the reference arm (the oracle on the host cores) prints
one JSON line with the keys the driver reads, for a small workload."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--workload", "cfg1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the unmodified reference package when baseline/_ref is installed, else the oracle port
    kind = "reference" if (ROOT / "baseline" / "_ref" / "fastcdf").is_dir() else "port"
    assert d["cpu_baseline"]["kind"] == kind and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"] == "cfg1"
    # a measurement of the stated sample, not a projection: ms_per_step x steps is wall time
    assert d["ms_per_step"] > 0 and "sample" in d["cpu_baseline"]


def test_reference_arm_nonzero_rank_is_silent():
    env = {"RANK": "1", "WORLD_SIZE": "2", "PATH": "/usr/bin:/bin"}
    import os

    env = {**os.environ, **env}
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--workload", "cfg1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0
    assert not [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
