"""Dense numpy reference of one decode step (TEST INFRASTRUCTURE).

Independent of the µop machinery: evaluates the model definition of
include/uopsim/decode.hpp directly from the tensors (fused wqkv / wgu
layouts, interleaved-pair RoPE with double-precision angles, fused RMSNorm
with bf16 rounding of the normalised vector when the model is bf16, GQA
attention over the cache + the appended row, SwiGLU, residual adds,
fp32 logits). Used to pin the oracle interpreter and the decode lowering.
"""
from __future__ import annotations

import numpy as np


def bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 -> bf16 (RNE) -> float32, like the engine's stores."""
    x = np.asarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def decode_step(T: dict, cfg: dict, token: int, pos: int) -> dict:
    """T: name -> float32 array (row-major, shapes per the graph). Returns
    logits and the appended k/v rows per layer."""
    d, hq, hkv, hd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"]
    ffn, eps, theta, layers = cfg["ffn"], cfg["eps"], cfg["theta"], cfg["layers"]
    gu_block = cfg["gu_block"]
    is_bf16 = cfg["dtype"] == "bf16"
    rnd = bf16 if is_bf16 else (lambda a: np.asarray(a, np.float32))
    f32 = np.float32
    ctx = pos + 1
    grp = hq // hkv

    # batched programs store the normalised operand as bf16(x * w) and apply
    # the per-request 1/rms to the GEMM output (cfg["norm_scale_after"])
    scale_after = cfg.get("norm_scale_after", False)

    def rmsnorm(x, w):
        ss = np.float32(np.sum(x.astype(np.float64) ** 2))
        inv = f32(1.0) / np.sqrt(ss / f32(x.size) + f32(eps))
        if scale_after:
            return rnd(x * w), inv
        return rnd(x * inv * w), f32(1.0)

    def mv(W, h):
        hv, s = h
        return (W.astype(np.float64) @ hv.astype(np.float64)).astype(np.float32) * s

    def rope(v, row0):
        out = v.copy()
        for i in range(0, v.size, 2):
            dd = (row0 + i) % hd
            ang = pos * theta ** (-dd / hd)
            c, s = np.float32(np.cos(ang)), np.float32(np.sin(ang))
            a, b = v[i], v[i + 1]
            out[i], out[i + 1] = a * c - b * s, a * s + b * c
        return out

    x = rnd(T["embed.table"].reshape(-1, d)[token])
    res = {"k": [], "v": []}
    for l in range(layers):
        L = f"L{l}."
        h = rmsnorm(x, T[L + "attn_norm"].reshape(-1))
        qkv = mv(T[L + "wqkv"].reshape(-1, d), h)
        if cfg.get("qk_norm"):
            # Qwen3: q / k stored as bf16, per-head RMSNorm (bf16) then the rotary
            def headnorm(v, w):
                v = rnd(v).reshape(-1, hd)
                ss = np.sum(v.astype(np.float32) * v.astype(np.float32), axis=1, dtype=np.float32)
                inv = (f32(1.0) / np.sqrt(ss / f32(hd) + f32(eps))).astype(np.float32)
                return rnd(v * inv[:, None] * w.reshape(1, hd)).reshape(-1)
            q = rnd(rope(headnorm(qkv[: hq * hd], T[L + "q_norm"]), 0))
            k = rnd(rope(headnorm(qkv[hq * hd: (hq + hkv) * hd], T[L + "k_norm"]), hq * hd))
        else:
            q = rnd(rope(qkv[: hq * hd], 0))
            k = rnd(rope(qkv[hq * hd: (hq + hkv) * hd], hq * hd))
        v = rnd(qkv[(hq + hkv) * hd:])
        Kc = T[L + "kc"].reshape(hkv, -1, hd).copy()
        Vc = T[L + "vc"].reshape(hkv, -1, hd).copy()
        Kc[:, pos, :] = k.reshape(hkv, hd)
        Vc[:, pos, :] = v.reshape(hkv, hd)
        res["k"].append(k.copy())
        res["v"].append(v.copy())
        att = np.zeros(hq * hd, np.float32)
        for hh in range(hq):
            g = hh // grp
            s = (Kc[g, :ctx].astype(np.float64) @ q[hh * hd:(hh + 1) * hd].astype(np.float64)) / np.sqrt(hd)
            p = np.exp(s - s.max())
            att[hh * hd:(hh + 1) * hd] = (p @ Vc[g, :ctx].astype(np.float64)) / p.sum()
        att = rnd(att)
        x1 = rnd(x + (T[L + "wo"].reshape(d, -1).astype(np.float64) @ att.astype(np.float64)).astype(np.float32))
        h2 = rmsnorm(x1, T[L + "mlp_norm"].reshape(-1))
        gu = mv(T[L + "wgu"].reshape(-1, d), h2)
        gu = gu.reshape(-1, gu_block)
        gate, up = gu[:, : gu_block // 2].reshape(-1), gu[:, gu_block // 2:].reshape(-1)
        a = rnd(gate / (1.0 + np.exp(-gate)) * up)
        x = rnd(x1 + (T[L + "wd"].reshape(d, -1).astype(np.float64) @ a.astype(np.float64)).astype(np.float32))
    hf = rmsnorm(x, T["final_norm"].reshape(-1))
    res["logits"] = mv(T["lm_head"].reshape(-1, d), hf)
    return res
