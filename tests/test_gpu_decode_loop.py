"""Multi-step decode on the device: greedy sampling fused
into the lm_head epilogue writes the token back into the step block and
advances the position, so consecutive launches decode consecutive tokens
with no host round trip. Checked against the host-driven loop (host reads
next_token, writes the step block): identical token sequences and identical
KV caches, single-request and batched."""
import numpy as np
import pytest

import batch_cases as bc
import ring_cases as rc
from paper_2605_03190_b200 import Program

pytestmark = pytest.mark.gpu

STEPS = 5


def engine(req, seed=0):
    from paper_2605_03190_b200.engine import Engine

    prog = Program.build(req)
    info = prog.info()
    eng = Engine(prog, watchdog_ms=5000)
    tens = eng.bind_inputs(rc.synth_inputs(info, seed))
    return eng, tens, info


def test_single_request_device_loop(cuda):
    import torch

    tokens = {}
    caches = {}
    for mode in ("host", "device"):
        base = {"model": dict(rc.MID["model"]), "layout": dict(rc.MID["layout"], argmax=True, feedback=mode == "device")}
        eng, tens, info = engine(rc.request(base))
        st = torch.tensor([17, 100, 101, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
        eng.bind_step(st)
        seq = []
        for k in range(STEPS):
            rep = eng.run()
            assert rep.status == 0, rep.message
            tok = int(tens["next_token"].item())
            seq.append(tok)
            if mode == "host":
                st[0], st[1], st[2] = tok, 101 + k, 102 + k
            else:
                assert [int(x) for x in st[:3].tolist()] == [tok, 101 + k, 102 + k]
        tokens[mode] = seq
        caches[mode] = {k: v.float().cpu().numpy() for k, v in tens.items() if k.endswith(("kc", "vc"))}
    assert tokens["host"] == tokens["device"]
    for k in caches["host"]:
        assert np.array_equal(caches["host"][k], caches["device"][k]), k


def test_batched_device_loop(cuda):
    import torch

    pages = [2, 3, 1, 4, 2, 2]
    pos0 = [60, 120, 10, 180, 70, 64]
    tok0 = [5, 77, 901, 3, 1234, 42]
    tokens = {}
    for mode in ("host", "device"):
        req = bc.request(bc.MID_MODEL, pages, 4, None)
        req["layout"].update(argmax=True, feedback=mode == "device")
        eng, tens, info = engine(req)
        st = torch.from_numpy(bc.step_block(info, tok0, pos0)).cuda()
        eng.bind_step(st)
        seq = []
        for k in range(STEPS):
            rep = eng.run()
            assert rep.status == 0, rep.message
            tk = [int(x) for x in tens["next_token"].view(-1).tolist()]
            seq.append(tk)
            if mode == "host":
                st.copy_(torch.from_numpy(bc.step_block(info, tk, [p + k + 1 for p in pos0])))
        tokens[mode] = seq
    assert tokens["host"] == tokens["device"]
