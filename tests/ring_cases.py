"""Ring-engine test cases shared by the GPU tests and the smoke entry point:
model requests, deterministic synthetic inputs and the dense-reference check
(decode_ref.py — test infrastructure)."""
from __future__ import annotations

import numpy as np

import decode_ref

TINY = {"model": {"preset": "tiny"}, "layout": {"ctx_pages": 1, "max_ctx": 64, "gu_block": 16, "pages_per_job": 1}}
MID = {"model": {"preset": "llama3-8b", "layers": 2, "hidden": 1024, "heads": 8, "kv_heads": 2, "ffn": 2816,
                 "vocab": 4096},
       "layout": {"ctx_pages": 8, "max_ctx": 512, "pages_per_job": 2, "gu_block": 4}}


def request(base: dict, sm_count: int | None = None, ring_slots: int = 12) -> dict:
    r = {"engine": "ring", "model": dict(base["model"]), "layout": dict(base["layout"]), "ring_slots": ring_slots,
         "profile": {"builtin": "b200"}}
    if sm_count:
        r["profile"]["sm_count"] = sm_count
    return r


def model_cfg(info: dict, req: dict) -> dict:
    """decode_ref config from the program's graph (shapes) and the request."""
    g = {t["name"]: t for t in info["graph"]["tensors"]}
    kc = g["L0.kc"]["shape"]
    d = g["embed.table"]["shape"][1]
    hd = kc[2]
    q = g["L0.q"]["shape"][0]
    nodes = {n["id"]: n for n in info["graph"]["operators"]}
    eps = float(nodes["L0.qkv"]["attrs"]["eps"])
    theta = float(nodes["L0.qkv"]["attrs"]["theta"])
    layers = sum(1 for n in info["graph"]["operators"] if n["id"].endswith(".qkv"))
    dtype = [x["dtype"] for x in info["descriptors"] if x["name"] == "L0.wqkv"][0]
    return {"hidden": d, "heads": q // hd, "kv_heads": kc[0], "head_dim": hd, "ffn": g["L0.a"]["shape"][0],
            "eps": eps, "theta": theta, "layers": layers, "gu_block": req["layout"]["gu_block"], "dtype": dtype,
            "qk_norm": "L0.q_norm" in g,
            # ring programs stage bf16(x * w) and apply 1/rms to the GEMV output
            # (reference-form programs normalise before the MATVEC)
            "norm_scale_after": req.get("engine") == "ring"}


def synth_inputs(info: dict, seed: int = 0) -> dict:
    """Weights uniform in [-1,1)/sqrt(fan_in) (bf16-rounded for bf16 tensors),
    norms ones, KV caches uniform, activations zero."""
    rng = np.random.default_rng(seed)
    out = {}
    for d in info["descriptors"]:
        if d["view_of"] >= 0:
            continue
        n = int(np.prod(d["shape"]))
        if d["init"] == 2:
            a = np.ones(n, np.float32)
        elif d["external"] or d["state"]:
            fan = d["shape"][-1]
            a = (rng.random(n, np.float32) * 2 - 1) / np.float32(np.sqrt(fan))
        else:
            a = np.zeros(n, np.float32)
        if d["name"].endswith("q_norm") or d["name"].endswith("k_norm"):  # non-trivial QK-norm weights
            a = (1.0 + 0.25 * (rng.random(n, np.float32) * 2 - 1)).astype(np.float32)
        if d["dtype"] == "bf16":
            a = decode_ref.bf16(a)
        out[d["name"]] = a
    return out


def check_against_dense(info: dict, req: dict, ins: dict, host: dict, token: int, pos: int, cfg: dict | None = None) -> dict:
    """Errors of the device results vs the dense numpy reference."""
    cfg = cfg or model_cfg(info, req)
    ref = decode_ref.decode_step(ins, cfg, token, pos)
    lg, rl = host["logits"].astype(np.float64), ref["logits"].astype(np.float64)
    res = {"logits_max_abs": float(np.abs(lg - rl).max()), "logits_rms": float(np.sqrt(np.mean(rl ** 2))),
           "logits_max": float(np.abs(rl).max()), "argmax_equal": int(np.argmax(lg)) == int(np.argmax(rl))}
    hkv, hd = cfg["kv_heads"], cfg["head_dim"]
    kv = 0.0
    for l in range(cfg["layers"]):
        for name, r in (("kc", ref["k"][l]), ("vc", ref["v"][l])):
            c = host[f"L{l}.{name}"].reshape(hkv, -1, hd)[:, pos].reshape(-1)
            kv = max(kv, float(np.abs(c - r).max() / max(np.abs(r).max(), 1e-30)))
    res["kv_rel"] = kv
    return res
