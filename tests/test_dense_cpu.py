"""The optional dense fp32 all-cores CPU context figure (BASELINE.md §3.2,
oracle/dense_cpu.cpp): it builds, runs a 1-layer step and reports JSON."""
import json
import subprocess
from pathlib import Path

import pytest

EXE = Path(__file__).resolve().parents[1] / "oracle/_ref/dense_cpu"


@pytest.mark.skipif(not EXE.exists(), reason="oracle/_ref/dense_cpu not built")
def test_dense_cpu_runs():
    r = subprocess.run([str(EXE), "1", "64", "1", "2"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    assert out["layers"] == 1 and out["ctx"] == 64 and out["threads"] == 2
    assert out["tokens_per_s"] > 0 and 0 <= out["token"] < 128256
