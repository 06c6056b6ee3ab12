"""fp32 dense decode reference on the GPU (TEST INFRASTRUCTURE, the checker).

An independent evaluation of the model a decode program describes, written
from the model definition (include/uopsim/decode.hpp; Llama-3 / Qwen3
decoder layers) in plain PyTorch fp32 — no µop machinery, no engine code.
Used for parity at the benchmarked configurations (full 32-layer C2 at ctx
4096, 32-layer C3 batch 32, 36-layer Qwen3-8B, Llama-3-70B shapes under TP),
where the numpy reference (decode_ref.py) would take hours.

Arithmetic: bf16 weights converted to fp32, every matmul / softmax / norm in
fp32 (TF32 off), RoPE angles in double precision (the reference handler's
interleaved pairs, handlers.cpp:88-100), attention by the exact softmax
(the limit of the online softmax of handlers.cpp:54-87). The engine's
*stored* activations are bf16 (the program's descriptors say so), so the
reference rounds to bf16 exactly where a tensor is stored (SURVEY §8(d):
"the oracle runs fp32 on the same bf16-rounded weights and bf16-rounded
stored activations"): the residual stream, the RMSNorm operand (bf16(x·inv·w),
or bf16(x·w) with 1/rms applied to the GEMM output when the program stores
that operand — batched programs), q/k/v, the attention output and the
SwiGLU product. The reference carries its OWN KV cache across steps (a copy
of the synthetic history plus the rows it appends itself): multi-step runs
measure the drift of the engine against an independent decode, teacher-forced
with the engine's tokens.
"""
from __future__ import annotations

import math

import numpy as np


def _torch():
    import torch

    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    return torch


def bf16r(x):
    """round an fp32 tensor to bf16 values (RNE), kept in fp32"""
    return x.to(_torch().bfloat16).float()


def unpack_sw128(t, rows: int, cols: int):
    """packed pre-swizzled 128 x 64 tiles (ring_abi.h VDC_DESC_PACKED_SW128) -> (rows, cols)"""
    torch = _torch()
    x = t.view(rows // 128, cols // 64, 128, 8, 8)  # rb, kt, r, physical chunk, e
    r = torch.arange(128, device=t.device)[:, None]
    c = torch.arange(8, device=t.device)[None, :]
    x = x[:, :, r, c ^ (r & 7), :]                  # logical chunk c of row r lives at c ^ (r % 8)
    return x.permute(0, 2, 1, 3, 4).reshape(rows, cols)


KPAGE_SWZ = 0x40000000  # ring_abi.h VDC_DESC_KPAGE_SWZ


def unswizzle_k(t, hd: int):
    """swizzled K/V page rows (VDC_DESC_KPAGE_SWZ) -> logical (..., 64, hd)"""
    torch = _torch()
    x = t.view(-1, 64, hd // 8, 8)
    r = torch.arange(64, device=t.device)[:, None]
    c = torch.arange(hd // 8, device=t.device)[None, :]
    pc = (c & 8) | ((c & 7) ^ (r & 7))
    return x[:, r, pc, :].reshape(t.shape)


class DenseDecoder:
    """W: name -> 2-D (or 1-D norm) torch tensor in logical row-major order
    (bf16 or fp32 values); caches: per request, per layer (K, V) bf16 tensors
    of shape (hkv, >= ctx + steps, hd) in logical order."""

    def __init__(self, W: dict, cfg: dict, caches: list, compute=None):
        self.W, self.cfg, self.caches = W, cfg, caches
        self.torch = _torch()
        self.ct = compute or self.torch.float32  # float64: the precision-floor probe (same rounding points)

    def _f(self, t):
        return t.to(self.ct)

    def _norm(self, x, w):
        """stored RMSNorm operand + the scale applied to the GEMM output"""
        inv = 1.0 / self.torch.sqrt((x * x).mean(dim=1, keepdim=True) + self.cfg["eps"])
        if self.cfg.get("norm_scale_after"):
            return self._r(x * self._f(w)[None, :]), inv
        return self._r(x * inv * self._f(w)[None, :]), None

    def _mm(self, h, name):
        hv, s = h
        y = hv @ self._f(self.W[name]).t()
        return y * s if s is not None else y

    def _rope(self, v, pos, hd):
        """interleaved pairs (2i, 2i+1) of each head; angles in double precision"""
        torch = self.torch
        B = v.shape[0]
        x = v.view(B, -1, hd // 2, 2)
        i = torch.arange(hd // 2, device=v.device, dtype=torch.float64)
        p = torch.tensor(pos, device=v.device, dtype=torch.float64)[:, None]
        ang = p * torch.pow(torch.tensor(self.cfg["theta"], dtype=torch.float64, device=v.device), -(2 * i) / hd)[None, :]
        c, s = torch.cos(ang).float().to(self.ct)[:, None, :], torch.sin(ang).float().to(self.ct)[:, None, :]
        a, b = x[..., 0], x[..., 1]
        return torch.stack((a * c - b * s, a * s + b * c), dim=-1).reshape(v.shape)

    def _headnorm(self, v, w, hd):
        x = self._r(v).view(v.shape[0], -1, hd)
        inv = 1.0 / self.torch.sqrt((x * x).mean(dim=2, keepdim=True) + self.cfg["eps"])
        return self._r(x * inv * self._f(w).view(1, 1, hd)).reshape(v.shape)

    def _r(self, x):
        """a stored bf16 activation"""
        return x.to(self.torch.bfloat16).to(self.ct)

    def step(self, tokens, pos) -> dict:
        torch = self.torch
        c = self.cfg
        d, hq, hkv, hd, L = c["hidden"], c["heads"], c["kv_heads"], c["head_dim"], c["layers"]
        gub = c["gu_block"]
        B = len(tokens)
        grp = hq // hkv
        tok = torch.tensor([int(t) for t in tokens], device=self.W["embed.table"].device)
        x = self._f(self.W["embed.table"][tok])  # (B, d), bf16 values
        out = {"k": [], "v": []}
        for l in range(L):
            P = f"L{l}."
            qkv = self._mm(self._norm(x, self.W[P + "attn_norm"]), P + "wqkv")
            q, k, v = qkv[:, : hq * hd], qkv[:, hq * hd: (hq + hkv) * hd], qkv[:, (hq + hkv) * hd:]
            if c.get("qk_norm"):
                q, k = self._headnorm(q, self.W[P + "q_norm"], hd), self._headnorm(k, self.W[P + "k_norm"], hd)
            q, k, v = self._r(self._rope(q, pos, hd)), self._r(self._rope(k, pos, hd)), self._r(v)
            out["k"].append(k)
            out["v"].append(v)
            att = torch.empty(B, hq * hd, device=x.device, dtype=self.ct)
            for b in range(B):
                Kc, Vc = self.caches[b][l]
                p0 = int(pos[b])
                Kc[:, p0, :] = k[b].view(hkv, hd).to(Kc.dtype)
                Vc[:, p0, :] = v[b].view(hkv, hd).to(Vc.dtype)
                Kf, Vf = self._f(Kc[:, : p0 + 1, :]), self._f(Vc[:, : p0 + 1, :])   # (hkv, ctx, hd)
                qh = q[b].view(hkv, grp, hd)
                s = torch.einsum("kgd,ktd->kgt", qh, Kf) / math.sqrt(hd)
                pr = torch.softmax(s, dim=-1)
                att[b] = torch.einsum("kgt,ktd->kgd", pr, Vf).reshape(-1)
            att = self._r(att)
            x1 = self._r(x + att @ self._f(self.W[P + "wo"]).t())
            gu = self._mm(self._norm(x1, self.W[P + "mlp_norm"]), P + "wgu").view(B, -1, gub)
            g, u = gu[:, :, : gub // 2].reshape(B, -1), gu[:, :, gub // 2:].reshape(B, -1)
            a = self._r(g / (1.0 + torch.exp(-g)) * u)
            x = self._r(x1 + a @ self._f(self.W[P + "wd"]).t())
        out["logits"] = self._mm(self._norm(x, self.W["final_norm"]), "lm_head")[:, : c["vocab"]]
        return out


# ----------------------------------------------------------------------------
# building the reference from engine tensors


def _shape(d):
    return [int(s) for s in d["shape"]]


def weights_single(info: dict, tens: dict, cfg: dict) -> dict:
    """single-request program: row-major device tensors, viewed (no copies)"""
    descs = {d["name"]: d for d in info["descriptors"]}
    d = cfg["hidden"]
    W = {}
    for name, t in tens.items():
        if name.endswith((".kc", ".vc")) or descs[name]["dtype"] == "i64":
            continue
        if name.endswith("norm"):
            W[name] = t.view(-1)
        else:
            W[name] = t.view(-1, _shape(descs[name])[-1] if name != "lm_head" else d)
    return W


def caches_single(info: dict, tens: dict, cfg: dict, extra: int = 0) -> list:
    """request 0's cache copies (hkv, T, hd) per layer"""
    descs = {d["name"]: d for d in info["descriptors"]}
    hkv, hd = cfg["kv_heads"], cfg["head_dim"]
    out = []
    for l in range(cfg["layers"]):
        T = _shape(descs[f"L{l}.kc"])[1]
        pair = []
        for c in ("kc", "vc"):
            t = tens[f"L{l}.{c}"].view(hkv, T, hd)
            if descs[f"L{l}.{c}"].get("tma") == KPAGE_SWZ:  # swizzled page rows -> logical
                t = unswizzle_k(t.contiguous(), hd)
            pair.append(t.clone())
        out.append(tuple(pair))
    return [out]


def weights_batched(info: dict, tens: dict, cfg: dict) -> dict:
    """batched program: packed weights unpacked into new bf16 tensors"""
    descs = {d["name"]: d for d in info["descriptors"]}
    W = {}
    for name, t in tens.items():
        dd = descs[name]
        if name.endswith((".kc", ".vc")) or dd["dtype"] != "bf16" or dd.get("symmetric"):
            continue
        if dd["tma"] == 0x80000000:
            W[name] = unpack_sw128(t, *_shape(dd))
        elif name.endswith("norm"):
            W[name] = t.view(-1)
        elif name == "embed.table":
            W[name] = t.view(_shape(dd))
    return W


def caches_batched(info: dict, tens: dict, cfg: dict, page_table: np.ndarray, req_pages: list, extra_pages: int = 1,
                   cap_pages: int = 0) -> list:
    """per request: its pages gathered into logical (hkv, pages * 64, hd)
    copies, padded by extra_pages (or up to cap_pages) empty pages"""
    torch = _torch()
    descs = {d["name"]: d for d in info["descriptors"]}
    hkv, hd = cfg["kv_heads"], cfg["head_dim"]
    out = []
    for b, npg in enumerate(req_pages):
        pages = torch.as_tensor(page_table[b, :npg].astype(np.int64), device=next(iter(tens.values())).device)
        per = []
        for l in range(cfg["layers"]):
            pair = []
            for c in ("kc", "vc"):
                pool = tens[f"L{l}.{c}"].view(_shape(descs[f"L{l}.{c}"])[0], hkv, 64, hd)
                if descs[f"L{l}.{c}"].get("tma") == KPAGE_SWZ:  # swizzled page rows (K and V)
                    pool = unswizzle_k(pool, hd)
                g = pool[pages].permute(1, 0, 2, 3).reshape(hkv, npg * 64, hd)
                npad = max(cap_pages - npg, 0) if cap_pages else extra_pages
                pad = torch.zeros(hkv, npad * 64, hd, dtype=g.dtype, device=g.device)
                pair.append(torch.cat([g, pad], dim=1).contiguous())
            per.append(tuple(pair))
        out.append(per)
    return out


def errors(dev_logits, ref: dict) -> dict:
    """per request: max|d| / rms(ref), rms(d) / rms(ref), argmax agreement"""
    rl = ref["logits"].double()
    lg = dev_logits.double()[:, : rl.shape[1]]
    rms = (rl * rl).mean(dim=1).sqrt()
    d = lg - rl
    return {"max": (d.abs().max(dim=1).values / rms).cpu().numpy(), "rms": ((d * d).mean(dim=1).sqrt() / rms).cpu().numpy(),
            "argmax_equal": (lg.argmax(dim=1) == rl.argmax(dim=1)).cpu().numpy()}


def assemble_tp(Wr: list, cfg_rank: dict, world: int) -> dict:
    """the single-device model equivalent to `world` Megatron shards
    (csrc/host/decode_graph.cpp tp split): q|k|v rows and gate/up blocks
    column-parallel, o / down row-parallel, vocab-parallel lm_head (rows past
    the vocabulary are zero padding at the end), replicated embedding/norms"""
    torch = _torch()
    hd = cfg_rank["head_dim"]
    qr, kvr = cfg_rank["heads"] * hd, cfg_rank["kv_heads"] * hd
    full = {k: v for k, v in Wr[0].items() if k == "embed.table" or k.endswith("norm")}
    for l in range(cfg_rank["layers"]):
        P = f"L{l}."
        wq = [w[P + "wqkv"] for w in Wr]
        full[P + "wqkv"] = torch.cat([w[:qr] for w in wq] + [w[qr:qr + kvr] for w in wq] + [w[qr + kvr:] for w in wq])
        full[P + "wo"] = torch.cat([w[P + "wo"] for w in Wr], dim=1)
        full[P + "wgu"] = torch.cat([w[P + "wgu"] for w in Wr])
        full[P + "wd"] = torch.cat([w[P + "wd"] for w in Wr], dim=1)
    full["lm_head"] = torch.cat([w["lm_head"] for w in Wr])
    return full


def vocab_of(info: dict) -> int:
    return int([t for t in info["graph"]["tensors"] if t["name"] == "embed.table"][0]["shape"][0])
