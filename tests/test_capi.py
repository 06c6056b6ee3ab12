"""The C-ABI library (include/vdc.h) loads on a CPU-only host and exports
every entry point the header declares; no compute calls are made here."""
import ctypes
import re
from pathlib import Path

from paper_2605_03190_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared(header):
    text = (ROOT / "include" / header).read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(vdc_[a-z0-9_]+)\s*\(", text, re.M)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    names = declared("vdc.h")
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_native.EXPORTS) <= set(names)


def test_errors_cross_the_boundary_as_status_codes():
    import json
    h = ctypes.c_void_p()
    rc = _native.lib().vdc_program_build(json.dumps({"workload": {"tensors": [], "operators": []}, "profile": {"builtin": "nope"}}).encode(), ctypes.byref(h))
    assert rc == _native.VDC_ERR_INPUT
    assert _native.lib().vdc_last_error()


def test_cpp_dropin_header_compiles(tmp_path):
    """include/uopsim/machine.hpp (the reference executor API over the
    C-ABI) builds against libvdc.so from a C++ caller (examples/)."""
    import subprocess
    r = subprocess.run(["make", "-B", "-C", str(ROOT / "examples"), "machine_demo"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
