"""Prefill chunk on the batched path: the rows of one
launch are consecutive positions of ONE sequence sharing its KV pages
(layout.prefill); the qkv BGEMM appends all their K/V rows and every row
attends causally to its own prefix, including the rows appended in the same
launch. Checked against the dense reference run token by token (decode_ref,
the cache updated with the reference's own rows): every row's logits, and
every appended K/V row (each row checked as one step on the device's
history, as the multi-step decode tests do)."""
import numpy as np
import pytest

import batch_cases as bc
import decode_ref
from paper_2605_03190_b200 import Program

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p0,S", [(0, 20), (70, 32), (100, 64)])
def test_prefill_chunk_matches_sequential(cuda, p0, S):
    import torch
    from paper_2605_03190_b200.engine import Engine

    pages = (p0 + S + 63) // 64 + 1
    req = bc.request(bc.MID_MODEL, [pages] * S, 4, None)
    req["layout"]["prefill"] = True
    prog = Program.build(req)
    info = prog.info()
    ins = bc.synth_inputs(info, 3)
    eng = Engine(prog, watchdog_ms=5000)
    tens = eng.bind_inputs(ins)
    rng = np.random.default_rng(p0 + S)
    toks = [int(t) for t in rng.integers(0, 4096, S)]
    pos = [p0 + b for b in range(S)]
    st = torch.from_numpy(bc.step_block(info, toks, pos)).cuda()
    eng.bind_step(st)
    rep = eng.run()
    assert rep.status == 0, rep.message
    host = bc.readback(info, tens)
    cfg = bc.model_cfg(info)
    # sequential reference over the shared pages (request 0's view = the sequence)
    T = bc.request_view(info, ins, 0, cfg)
    hkv, hd = cfg["kv_heads"], cfg["head_dim"]
    V = host["logits"].size // S
    for b in range(S):
        ref = decode_ref.decode_step(T, cfg, toks[b], pos[b])
        lg = host["logits"].reshape(S, V)[b].astype(np.float64)
        rl = ref["logits"].astype(np.float64)
        rms = float(np.sqrt(np.mean(rl ** 2)))
        assert np.abs(lg - rl).max() <= 2e-2 * rms, (b, np.abs(lg - rl).max(), rms)
        # greedy choice agrees up to near-ties (both conventions round differently)
        assert rl[int(np.argmax(lg))] >= rl.max() - 2e-2 * rms, b
        for l in range(cfg["layers"]):
            k, v = bc.appended_rows(info, host, 0, pos[b], cfg, l)
            for got, r in ((k, ref["k"][l]), (v, ref["v"][l])):
                assert np.abs(got - r).max() <= 1e-2 * max(np.abs(r).max(), 1e-30), (b, l)
            # the next row's reference sees the device's appended rows (as the
            # multi-step decode tests carry the device state): each row is
            # checked as one step on the same history
            for c, r in (("kc", k), ("vc", v)):
                a = T[f"L{l}.{c}"].reshape(hkv, -1, hd)
                a[:, pos[b], :] = r.reshape(hkv, hd)
