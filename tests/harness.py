"""Shared test helpers: run a program through the CPU oracle (oracle/_ref,
TEST INFRASTRUCTURE) and through the device engine, and compare."""
from __future__ import annotations

import json
import os
import subprocess
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_INTERP = ROOT / "oracle/_ref/oracle_interp"
REF_CLI = ROOT / "oracle/_ref/ref_cli"


def oracle_available() -> bool:
    return ORACLE_INTERP.exists()


def run_oracle(program_json: dict, seed: int = 0, step=None, inputs: bytes | None = None):
    """Returns (index, inputs{name: f32}, outputs{name: f32}, meta)."""
    with tempfile.TemporaryDirectory() as d:
        pj = os.path.join(d, "prog.json")
        with open(pj, "w") as f:
            json.dump(program_json, f)
        args = [str(ORACLE_INTERP), pj, d, str(seed), ",".join(str(int(s)) for s in (step or [0]))]
        if inputs is not None:
            ip = os.path.join(d, "given.bin")
            with open(ip, "wb") as f:
                f.write(inputs)
            args.append(ip)
        r = subprocess.run(args, capture_output=True, text=True)
        with open(os.path.join(d, "index.json")) as f:
            idx = json.load(f)
        inp = np.fromfile(os.path.join(d, "inputs.bin"), dtype=np.float32)
        out = np.fromfile(os.path.join(d, "outputs.bin"), dtype=np.float32)
    ins = {e["name"]: inp[e["offset"]: e["offset"] + e["count"]] for e in idx["tensors"]}
    outs = {e["name"]: out[e["offset"]: e["offset"] + e["count"]] for e in idx["tensors"]}
    idx["returncode"] = r.returncode
    idx["stdout"] = r.stdout
    return idx, ins, outs


def compare(dev: dict, ref: dict, rel: float, names=None):
    """max|dev-ref| <= rel * max(|ref|) per tensor; returns list of failures."""
    bad = []
    for name in names or ref.keys():
        a, b = np.asarray(dev[name], np.float64), np.asarray(ref[name], np.float64)
        scale = max(np.abs(b).max(), 1e-30) if b.size else 1.0
        err = np.abs(a - b).max() if b.size else 0.0
        if not np.isfinite(err) or err > rel * scale:
            bad.append((name, float(err), float(scale)))
    return bad
