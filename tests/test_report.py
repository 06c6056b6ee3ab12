"""ExecutionReport serialisation (drop-in C++ API, reference
proj/include/uopsim/machine.hpp:84-87): compiled against the in-tree
libvdc.so and run on the CPU (no GPU calls)."""
import os
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
NJ = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


def test_report_json_kv_chrome_roundtrip(tmp_path):
    lib = ROOT / "paper_2605_03190_b200" / "lib"
    exe = tmp_path / "report_roundtrip"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include", f"-I{NJ}",
                    str(ROOT / "tests" / "cpp" / "report_roundtrip.cpp"), "-o", str(exe), f"-L{lib}", "-lvdc",
                    f"-Wl,-rpath,{lib}", "-L/usr/local/cuda/lib64", "-lcudart"], check=True, capture_output=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60, env=dict(os.environ))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "report round trip ok" in r.stdout
