"""Batched decode with tensor parallelism (SURVEY §8 e, C4/C5 shape): the W
rank programs of a batched model (column-parallel qkv / gate-up, row-parallel
o / down into symmetric fp32 exchange buffers, in-kernel batched
ALLREDUCE_ADD, vocab-parallel lm_head) run as W concurrent engine contexts
on one B200 (148 // W SMs each, own streams; the exchange buffers are plain
device allocations, the protocol is the cross-GPU one). The concatenated
logits and the appended K/V rows are checked per request against the dense
reference of the assembled single-device model (batch_cases tolerances)."""
import numpy as np
import pytest

import batch_cases as bc
import test_gpu_batch as tb
from paper_2605_03190_b200 import Program

pytestmark = pytest.mark.gpu


def assemble(infos, ins, cfg):
    W = len(infos)
    d, hd = cfg["hidden"], cfg["head_dim"]
    qr, kvr = cfg["heads"] // W * hd, cfg["kv_heads"] // W * hd
    shapes = {x["name"]: x["shape"] for x in infos[0]["descriptors"]}
    full = {k: v for k, v in ins[0].items() if not k.startswith("L") or k.endswith("norm")}
    # vocab shards are padded to whole 128-row blocks: the first `vocab` rows of
    # the concatenation are the vocabulary (in rank order)
    vocab = ins[0]["embed.table"].size // d
    full["lm_head"] = np.concatenate([x["lm_head"].reshape(-1, d) for x in ins])[:vocab].reshape(-1)
    for l in range(cfg["layers"]):
        L = f"L{l}."
        wq = [x[L + "wqkv"].reshape(-1, d) for x in ins]
        full[L + "wqkv"] = np.concatenate([w[:qr] for w in wq] + [w[qr:qr + kvr] for w in wq] +
                                          [w[qr + kvr:] for w in wq]).reshape(-1)
        P = shapes[L + "kc"][0]
        for c in ("kc", "vc"):
            full[L + c] = np.concatenate([x[L + c].reshape(P, -1, hd) for x in ins], axis=1).reshape(-1)
        full[L + "wo"] = np.concatenate([x[L + "wo"].reshape(d, qr) for x in ins], axis=1).reshape(-1)
        full[L + "wgu"] = np.concatenate([x[L + "wgu"].reshape(-1, d) for x in ins]).reshape(-1)
        ffn_r = shapes[L + "a"][1]
        full[L + "wd"] = np.concatenate([x[L + "wd"].reshape(d, ffn_r) for x in ins], axis=1).reshape(-1)
        for n in ("attn_norm", "mlp_norm"):
            if L + n in ins[0]:
                full[L + n] = ins[0][L + n]
    return full


def run_tp(model, req_pages, steps, world):
    import torch
    from paper_2605_03190_b200.engine import Engine

    reqs = []
    for r in range(world):
        q = bc.request(model, req_pages, 4, 148 // world)
        q["layout"]["tp_world"], q["layout"]["tp_rank"] = world, r
        q["layout"]["argmax"] = True  # fused sampling with the cross-rank (max, index) exchange
        reqs.append(q)
    progs = [Program.build(q) for q in reqs]
    infos = [p.info() for p in progs]
    ins = [bc.synth_inputs(info, 1000 * r) for r, info in enumerate(infos)]
    for x in ins[1:]:  # replicated tensors: embedding and every norm weight (incl. QK-norm)
        for k in ins[0]:
            if k == "embed.table" or k.endswith("norm"):
                x[k] = ins[0][k].copy()
    engines, tens = [], []
    for p, x in zip(progs, ins):
        e = Engine(p, watchdog_ms=5000)
        tens.append(e.bind_inputs_nonsym(x))
        engines.append(e)
    keep = []
    for dsc in [x for x in infos[0]["descriptors"] if x.get("symmetric")]:
        nbytes = 128 + int(np.prod(dsc["shape"])) * 4
        bufs = [torch.zeros(nbytes // 4, dtype=torch.float32, device="cuda") for _ in range(world)]
        keep.append(bufs)
        for r, e in enumerate(engines):
            e.bind_symmetric(dsc["name"], [b.data_ptr() for b in bufs], world, r)
    sts = [torch.zeros(int(infos[0]["step_scalars"]), dtype=torch.int64, device="cuda") for _ in range(world)]
    for e, st in zip(engines, sts):
        e.bind_step(st)
    streams = [torch.cuda.Stream() for _ in range(world)]
    cfg = bc.model_cfg(infos[0])
    cfg.update({"heads": cfg["heads"] * world, "kv_heads": cfg["kv_heads"] * world, "ffn": cfg["ffn"] * world})
    state = [dict(x) for x in ins]
    out = []
    for tokens, pos in steps:
        blk = torch.from_numpy(bc.step_block(infos[0], tokens, pos))
        for st in sts:
            st.copy_(blk)
        torch.cuda.synchronize()
        for e, s in zip(engines, streams):
            e.launch(s)
        for e in engines:
            rep = e.wait()
            assert rep.status == 0, rep.message
        host = [bc.readback(info, t) for info, t in zip(infos, tens)]
        full_state = assemble(infos, state, cfg)
        full_host = assemble(infos, host, cfg)
        nb = len(req_pages)
        vocab = ins[0]["embed.table"].size // cfg["hidden"]
        full_host["logits"] = np.concatenate([h["logits"].reshape(nb, -1) for h in host], axis=1)[:, :vocab].reshape(-1)
        # every rank sampled the argmax of the whole (unpadded) vocabulary
        want = [int(i) for i in np.argmax(full_host["logits"].reshape(nb, vocab), axis=1)]
        for h in host:
            assert [int(t) for t in h["next_token"].reshape(-1)[:nb]] == want
        out.append(bc.check_batch(infos[0], full_state, full_host, tokens, pos, cfg=cfg))
        state = host
    return out


@pytest.mark.parametrize("world", [1, 2])
def test_mid_batch6_tp(cuda, world):
    rng = np.random.default_rng(7)
    pages = [int(p) for p in rng.integers(1, 6, 6)]
    pos0 = [int(rng.integers(0, 64 * p - 2)) for p in pages]
    steps = [([int(t) for t in rng.integers(0, 4096, 6)], [p + s for p in pos0]) for s in range(2)]
    for rs in run_tp(bc.MID_MODEL, pages, steps, world):
        tb.assert_close(rs)


def test_qwen3_layer_batch8_tp4(cuda):
    """C4 shape: Qwen3-8B layer (QK-norm, 32/8 heads, ffn 12288), batch 8,
    tensor parallel over 4 ranks (8 q heads / 2 kv heads / 3072 ffn rows
    and 8192 vocab columns per rank)"""
    model = {"preset": "qwen3-8b", "layers": 1, "vocab": 32768}
    rng = np.random.default_rng(8)
    pages = [int(p) for p in rng.integers(1, 9, 8)]
    pos = [int(rng.integers(0, 64 * p)) for p in pages]
    tokens = [int(t) for t in rng.integers(0, 32768, 8)]
    for rs in run_tp(model, pages, [(tokens, pos)], 4):
        tb.assert_close(rs)


def test_mid_batch4_tp2_padded_vocab(cuda):
    """a vocabulary that does not split into whole 128-row blocks per rank
    (4000 / 2 = 2000 -> 2048-row shards, zero-padded): logits past the
    vocabulary are dropped (Llama-3 128256 / 8 and Qwen3 151936 / 4 shards)"""
    model = dict(bc.MID_MODEL, vocab=4000)
    rng = np.random.default_rng(9)
    pages = [2, 3, 1, 2]
    pos = [int(rng.integers(0, 64 * p)) for p in pages]
    tokens = [int(t) for t in rng.integers(0, 4000, 4)]
    for rs in run_tp(model, pages, [(tokens, pos)], 2):
        tb.assert_close(rs)
