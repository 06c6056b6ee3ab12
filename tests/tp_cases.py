"""Tensor-parallel test harness (ring engine). Builds the W rank programs of a
model (Megatron split), synthesizes per-rank weight shards plus replicated
tensors, assembles the equivalent single-device model for the dense
reference (decode_ref), and runs the W ranks on ONE GPU: each rank is its own
engine context on 148 // W SMs, launched concurrently on its own stream, with
the symmetric exchange buffers as plain device allocations (the same peer
protocol that runs over NVLink across GPUs)."""
from __future__ import annotations

import numpy as np

import decode_ref
import ring_cases as rc

REPLICATED = ("embed.table",)  # everything else is either sharded or norm-ones / zero-initialised


def rank_request(base: dict, world: int, rank: int, sms: int | None = None) -> dict:
    req = rc.request(base, sms if sms is not None else 148 // world)
    req["layout"]["tp_world"] = world
    req["layout"]["tp_rank"] = rank
    req["layout"]["argmax"] = True  # fused sampling with the cross-rank (max, index) exchange
    return req


def synth_rank_inputs(infos: list, seed: int = 0) -> list:
    """per-rank arrays; replicated tensors identical on every rank"""
    outs = [rc.synth_inputs(info, seed + 1000 * r) for r, info in enumerate(infos)]
    for name in REPLICATED:
        for o in outs[1:]:
            o[name] = outs[0][name].copy()
    return outs


def assemble_full(infos: list, ins: list, cfg_full: dict) -> dict:
    """the single-device model equivalent to the W shards"""
    W = len(infos)
    d, hd = cfg_full["hidden"], cfg_full["head_dim"]
    hq, hkv = cfg_full["heads"] // W, cfg_full["kv_heads"] // W
    qr, kvr = hq * hd, hkv * hd
    full = {"embed.table": ins[0]["embed.table"], "final_norm": ins[0]["final_norm"]}
    shapes = {dd["name"]: dd["shape"] for dd in infos[0]["descriptors"]}
    for l in range(cfg_full["layers"]):
        L = f"L{l}."
        full[L + "attn_norm"] = ins[0][L + "attn_norm"]
        full[L + "mlp_norm"] = ins[0][L + "mlp_norm"]
        wq = [x[L + "wqkv"].reshape(-1, d) for x in ins]
        full[L + "wqkv"] = np.concatenate([w[:qr] for w in wq] + [w[qr:qr + kvr] for w in wq] + [w[qr + kvr:] for w in wq]).reshape(-1)
        T = shapes[L + "kc"][1]
        for c in ("kc", "vc"):
            full[L + c] = np.concatenate([x[L + c].reshape(hkv, T, hd) for x in ins]).reshape(-1)
        full[L + "wo"] = np.concatenate([x[L + "wo"].reshape(d, qr) for x in ins], axis=1).reshape(-1)
        full[L + "wgu"] = np.concatenate([x[L + "wgu"].reshape(-1, d) for x in ins]).reshape(-1)
        ffn_r = shapes[L + "a"][0]
        full[L + "wd"] = np.concatenate([x[L + "wd"].reshape(d, ffn_r) for x in ins], axis=1).reshape(-1)
    full["lm_head"] = np.concatenate([x["lm_head"].reshape(-1, d) for x in ins]).reshape(-1)
    return full


def run_emulated(base: dict, world: int, steps=((17, 40),), seed: int = 0, capi_tp: bool = False):
    """returns (per-step dense-reference errors, full cfg)"""
    import torch
    from paper_2605_03190_b200 import Program
    from paper_2605_03190_b200.engine import Engine

    reqs = [rank_request(base, world, r) for r in range(world)]
    progs = [Program.build(q) for q in reqs]
    infos = [p.info() for p in progs]
    ins = synth_rank_inputs(infos, seed)
    engines, tens = [], []
    for p, x in zip(progs, ins):
        e = Engine(p, watchdog_ms=5000)
        tens.append(e.bind_inputs_nonsym(x))
        engines.append(e)
    keep = []
    if capi_tp:  # the library allocates, exports and binds (vdc_tp_alloc / vdc_tp_bind), no torch buffers
        blobs = [e.tp_alloc() for e in engines]
        for r, e in enumerate(engines):
            e.tp_bind(blobs, r)
    else:  # symmetric buffers: one per rank per symmetric tensor, shared by pointer
        for d in [d for d in infos[0]["descriptors"] if d.get("symmetric")]:
            nbytes = 128 + int(np.prod(d["shape"])) * 4
            bufs = [torch.zeros(nbytes // 4, dtype=torch.float32, device="cuda") for _ in range(world)]
            keep.append(bufs)
            for r, e in enumerate(engines):
                e.bind_symmetric(d["name"], [b.data_ptr() for b in bufs], world, r)
    step_t = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(world)]
    for e, st in zip(engines, step_t):
        e.bind_step(st)
    streams = [torch.cuda.Stream() for _ in range(world)]
    cfg_full = rc.model_cfg(infos[0], reqs[0])
    cfg_full.update({"heads": cfg_full["heads"] * world, "kv_heads": cfg_full["kv_heads"] * world,
                     "ffn": cfg_full["ffn"] * world})
    state = [{k: v.copy() for k, v in x.items()} for x in ins]
    results = []
    for token, pos in steps:
        for st in step_t:
            st[0], st[1], st[2] = token, pos, pos + 1
        torch.cuda.synchronize()
        for e, s in zip(engines, streams):
            e.launch(s)
        reps = [e.wait() for e in engines]
        for rep in reps:
            assert rep.status == 0, rep.message
        host = [e.host_arrays(t) for e, t in zip(engines, tens)]
        full_in = assemble_full(infos, state, cfg_full)
        full_dev = {"logits": np.concatenate([h["logits"] for h in host])}
        want = int(np.argmax(full_dev["logits"]))  # every rank sampled the argmax of the whole vocabulary
        assert all(int(h["next_token"].reshape(-1)[0]) == want for h in host), [h["next_token"] for h in host]
        hd = cfg_full["head_dim"]
        T = {dd["name"]: dd["shape"] for dd in infos[0]["descriptors"]}["L0.kc"][1]
        for l in range(cfg_full["layers"]):
            for c in ("kc", "vc"):
                full_dev[f"L{l}.{c}"] = np.concatenate([h[f"L{l}.{c}"].reshape(-1, T, hd) for h in host]).reshape(-1)
        results.append(rc.check_against_dense(infos[0], reqs[0], full_in, full_dev, token, pos, cfg=cfg_full))
        state = [{k: v.copy() for k, v in h.items()} for h in host]
    return results, cfg_full
