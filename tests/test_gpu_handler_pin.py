"""Per-µop pin of the device's decode arithmetic to the reference's own
HandlerState (reference src/handlers.cpp:17-168, oracle/handler_pin.cpp):
one decode step of the C1 tiny fp32 model on the ring engine, then every
operator output recomputed from the reference handlers on the DEVICE's own
inputs to that operator:

  qkv (RMS_GEMV + rotary + KV append)  RMSNORM, MATVEC, ROPE
  ATTN_DECODE (split-KV + fused combine)  ATTN over the whole context
  o (GEMV_ADD)                          MATVEC + ELEMWISE add
  gate/up (RMS_GEMV + SwiGLU)           RMSNORM, MATVEC, ELEMWISE silu, ELEMWISE mul
  down (GEMV_ADD)                       MATVEC + ELEMWISE add
  head (RMS_GEMV)                       RMSNORM, MATVEC

fp32 throughout; tolerance 1e-5 of the output's max magnitude (the device
sums in a different association)."""
import numpy as np
import pytest

import handler_pin
import ring_cases as rc
from paper_2605_03190_b200 import Program

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not handler_pin.EXE.exists(), reason="oracle/_ref not built")
@pytest.mark.parametrize("token,pos", [(17, 40), (250, 63)])
def test_every_decode_uop_matches_reference_handlers(cuda, token, pos):
    import torch
    from paper_2605_03190_b200.engine import Engine

    req = rc.request(rc.TINY)
    prog = Program.build(req)
    info = prog.info()
    cfg = rc.model_cfg(info, req)
    cfg["vocab"] = info["descriptors"][0]["shape"][0]
    ins = rc.synth_inputs(info, seed=0)
    eng = Engine(prog, device=0, watchdog_ms=5000)
    tens = eng.bind_inputs(ins)
    eng.bind_step(torch.tensor([token, pos, pos + 1, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda:0"))
    rep = eng.run()
    assert rep.status == 0, rep.message
    dev = eng.host_arrays(tens)
    hp = handler_pin.pin(dev, cfg, token, pos)
    hkv, hd = cfg["kv_heads"], cfg["head_dim"]

    def close(name, got, want):
        err = float(np.abs(got - want).max())
        assert err <= 1e-5 * max(1.0, float(np.abs(want).max())), (name, err, float(np.abs(want).max()))

    for l in range(cfg["layers"]):
        L = f"L{l}."
        close(L + "q", dev[L + "q"], hp[L + "q"])
        close(L + "k_row", dev[L + "kc"].reshape(hkv, -1, hd)[:, pos].reshape(-1), hp[L + "k_row"])
        close(L + "v_row", dev[L + "vc"].reshape(hkv, -1, hd)[:, pos].reshape(-1), hp[L + "v_row"])
        for n in ("attn", "x1", "a", "x2"):
            close(L + n, dev[L + n], hp[L + n])
    close("logits", dev["logits"], hp["logits"])
