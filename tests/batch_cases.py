"""Batched-decode test cases (SURVEY §8 C3 shape: B requests with their own
contexts over a paged KV pool): requests, step blocks and the per-request
check against the dense numpy reference (decode_ref.py, test
infrastructure). Each request of a batched step is an independent decode
step of the same model, so request b is checked against
decode_ref.decode_step on its own gathered cache pages."""
from __future__ import annotations

import numpy as np

import decode_ref
import ring_cases as rc

MID_MODEL = {"preset": "llama3-8b", "layers": 2, "hidden": 1024, "heads": 8, "kv_heads": 2, "ffn": 2816, "vocab": 4096}


def request(model: dict, req_pages: list, pages_per_job: int = 4, sm_count: int | None = None) -> dict:
    r = {"engine": "ring", "model": dict(model),
         "layout": {"batch": len(req_pages), "req_pages": list(req_pages), "pages_per_job": pages_per_job,
                    "gu_block": 128, "page_rows": 64},
         "profile": {"builtin": "b200"}}
    if sm_count:
        r["profile"]["sm_count"] = sm_count
    return r


def model_cfg(info: dict) -> dict:
    g = {t["name"]: t for t in info["graph"]["tensors"]}
    kc = g["L0.kc"]["shape"]
    hd, hkv = kc[2], kc[1] // 64
    nodes = {n["id"]: n for n in info["graph"]["operators"]}
    layers = sum(1 for n in info["graph"]["operators"] if n["id"].endswith(".qkv"))
    return {"hidden": g["embed.table"]["shape"][1], "heads": g["L0.q"]["shape"][1] // hd, "kv_heads": hkv, "head_dim": hd,
            "ffn": g["L0.a"]["shape"][1], "eps": float(nodes["L0.qkv"]["attrs"]["eps"]),
            "theta": float(nodes["L0.qkv"]["attrs"]["theta"]), "layers": layers, "gu_block": 128, "dtype": "bf16",
            # batched programs store the RMSNorm operand as bf16(x * w) and scale
            # the GEMM output by 1/rms (decode_ref documents both conventions)
            "norm_scale_after": True, "qk_norm": "L0.q_norm" in g}


def step_block(info: dict, tokens, pos) -> np.ndarray:
    """[token, pos, ctx] per request, then the page table (request-major)."""
    b = info["batch"]
    st = np.zeros(int(info["step_scalars"]), np.int64)
    for i in range(b["nb"]):
        st[3 * i: 3 * i + 3] = (tokens[i], pos[i], pos[i] + 1)
    pt = np.asarray(b["page_table"], np.int64)
    st[b["page_table_off"]: b["page_table_off"] + pt.size] = pt
    return st


def request_view(info: dict, T: dict, b: int, cfg: dict) -> dict:
    """Single-request tensors of request b: shared weights + its cache pages
    gathered into the (hkv, pages*64, hd) layout decode_ref expects."""
    nbi = info["batch"]
    maxp = nbi["maxp"]
    pt = np.asarray(nbi["page_table"], np.int64).reshape(nbi["nb"], maxp)
    g = {t["name"]: t for t in info["graph"]["tensors"]}
    npages = sum(1 for p in range(maxp) if p == 0 or pt[b, p] != 0)
    hkv, hd = cfg["kv_heads"], cfg["head_dim"]
    out = dict(T)
    for l in range(cfg["layers"]):
        for c in ("kc", "vc"):
            pool = T[f"L{l}.{c}"].reshape(g[f"L{l}.{c}"]["shape"][0], hkv, 64, hd)
            pages = pool[pt[b, :npages]]                      # (np, hkv, 64, hd)
            out[f"L{l}.{c}"] = np.ascontiguousarray(pages.transpose(1, 0, 2, 3)).reshape(-1)
    return out


def appended_rows(info: dict, host: dict, b: int, pos: int, cfg: dict, l: int):
    nbi = info["batch"]
    pt = np.asarray(nbi["page_table"], np.int64).reshape(nbi["nb"], nbi["maxp"])
    g = {t["name"]: t for t in info["graph"]["tensors"]}
    hkv, hd = cfg["kv_heads"], cfg["head_dim"]
    rows = []
    for c in ("kc", "vc"):
        pool = host[f"L{l}.{c}"].reshape(g[f"L{l}.{c}"]["shape"][0], hkv, 64, hd)
        rows.append(pool[pt[b, pos // 64], :, pos % 64, :].reshape(-1))
    return rows


def check_batch(info: dict, state: dict, host: dict, tokens, pos, cfg: dict | None = None) -> list:
    """Per-request errors of the device step vs the dense reference."""
    cfg = cfg or model_cfg(info)
    nb = info["batch"]["nb"]
    V = host["logits"].size // nb
    out = []
    for b in range(nb):
        ref = decode_ref.decode_step(request_view(info, state, b, cfg), cfg, int(tokens[b]), int(pos[b]))
        lg = host["logits"].reshape(nb, V)[b].astype(np.float64)
        rl = ref["logits"].astype(np.float64)
        res = {"logits_max_abs": float(np.abs(lg - rl).max()), "logits_rms": float(np.sqrt(np.mean(rl ** 2))),
               "argmax_equal": int(np.argmax(lg)) == int(np.argmax(rl)),
               # how far the device's greedy choice is from the reference's best logit
               "argmax_gap": float(rl.max() - rl[int(np.argmax(lg))])}
        # appended K/V rows, max |d| / max |ref|: layer 0 (fed by the embedding
        # row only) and the deeper layers, which inherit upstream bf16 rounding
        # flips of the attention / hidden activations (see test_gpu_batch)
        kv = [0.0, 0.0]
        for l in range(cfg["layers"]):
            k, v = appended_rows(info, host, b, int(pos[b]), cfg, l)
            for got, r in ((k, ref["k"][l]), (v, ref["v"][l])):
                kv[min(l, 1)] = max(kv[min(l, 1)], float(np.abs(got - r).max() / max(np.abs(r).max(), 1e-30)))
        res["kv_rel"], res["kv_rel_deep"] = kv
        # the same step under the single-request rounding convention
        # (bf16(x * inv * w) operand): a looser cross-check of the model math
        alt = decode_ref.decode_step(request_view(info, state, b, cfg), dict(cfg, norm_scale_after=False), int(tokens[b]),
                                     int(pos[b]))["logits"].astype(np.float64)
        res["logits_max_abs_alt"] = float(np.abs(lg - alt).max())
        out.append(res)
    return out


synth_inputs = rc.synth_inputs


def readback(info: dict, tens: dict) -> dict:
    """Device tensors -> host float32 arrays in logical (row-major) order
    (packed weight tiles are unpacked)."""
    from paper_2605_03190_b200.engine import to_logical

    shapes = {d["name"]: d for d in info["descriptors"]}
    return {k: to_logical(shapes[k], v.float().cpu().numpy()) for k, v in tens.items()}
