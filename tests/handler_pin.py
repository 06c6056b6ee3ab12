"""Driver of oracle/_ref/handler_pin (TEST INFRASTRUCTURE): recomposes each
decode operator from the reference's own HandlerState arithmetic
(reference src/handlers.cpp, compiled unmodified). `pin(tensors, cfg,
token, pos)` returns the reference-handler value of every operator output,
evaluated on the given inputs of that operator; chain=True runs a whole
decode step on the handlers' own intermediates."""
from __future__ import annotations

import json
import struct
import subprocess
import tempfile
from pathlib import Path

import numpy as np

EXE = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "handler_pin"
NAMES = ("attn_norm", "wqkv", "q", "kc", "vc", "wo", "attn", "x1", "mlp_norm", "wgu", "a", "wd", "x2")


def _write(path, arrays: dict):
    with open(path, "wb") as f:
        for k, v in arrays.items():
            v = np.ascontiguousarray(v, dtype=np.float32).reshape(-1)
            b = k.encode()
            f.write(struct.pack("<I", len(b)) + b + struct.pack("<Q", v.size) + v.tobytes())


def _read(path) -> dict:
    out = {}
    data = Path(path).read_bytes()
    i = 0
    while i < len(data):
        (nl,) = struct.unpack_from("<I", data, i)
        name = data[i + 4: i + 4 + nl].decode()
        (n,) = struct.unpack_from("<Q", data, i + 4 + nl)
        i += 12 + nl
        out[name] = np.frombuffer(data, dtype=np.float32, count=n, offset=i).copy()
        i += 4 * n
    return out


def pin(T: dict, cfg: dict, token: int, pos: int, chain: bool = False) -> dict:
    d = cfg["hidden"]
    arrays = {"x.in": T["embed.table"].reshape(-1, d)[token], "final_norm": T["final_norm"], "lm_head": T["lm_head"]}
    for l in range(cfg["layers"]):
        for n in NAMES:
            if f"L{l}.{n}" in T:
                arrays[f"L{l}.{n}"] = T[f"L{l}.{n}"]
    conf = {k: cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn", "vocab", "theta", "gu_block")}
    conf.update(pos=int(pos), chain=chain)
    with tempfile.TemporaryDirectory() as td:
        fi, fo = Path(td, "in.bin"), Path(td, "out.bin")
        _write(fi, arrays)
        r = subprocess.run([str(EXE), str(fi), str(fo), json.dumps(conf)], capture_output=True, text=True, timeout=300)
        if r.returncode != 0:
            raise RuntimeError(r.stderr)
        return _read(fo)
