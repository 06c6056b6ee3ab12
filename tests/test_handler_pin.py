"""The dense decode reference (tests/decode_ref.py) that every GPU parity test
compares against, pinned to the reference's own handler arithmetic: one full
decode step of the C1 tiny fp32 model recomposed from HandlerState
(RMSNORM / MATVEC / ROPE / ATTN / ELEMWISE, reference src/handlers.cpp:17-168,
oracle/handler_pin.cpp) must give the same logits and appended K/V rows.
CPU only (oracle/_ref is built from /root/reference by __graft_entry__.build)."""
import numpy as np
import pytest

import decode_ref
import handler_pin
import ring_cases as rc
from paper_2605_03190_b200 import Program


@pytest.mark.skipif(not handler_pin.EXE.exists(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("token,pos", [(17, 40), (3, 0), (500, 63)])
def test_dense_reference_matches_reference_handlers(token, pos):
    req = rc.request(rc.TINY)
    info = Program.build(req).info()
    cfg = rc.model_cfg(info, req)
    cfg["vocab"] = info["descriptors"][0]["shape"][0]
    ins = rc.synth_inputs(info, seed=0)
    ref = decode_ref.decode_step(ins, cfg, token, pos)
    hp = handler_pin.pin(ins, cfg, token, pos, chain=True)
    scale = np.abs(ref["logits"]).max()
    assert np.abs(hp["logits"] - ref["logits"]).max() <= 1e-5 * scale
    for l in range(cfg["layers"]):
        for key, name in (("k", "k_row"), ("v", "v_row")):
            r = ref[key][l]
            assert np.abs(hp[f"L{l}.{name}"] - r).max() <= 1e-5 * max(1.0, np.abs(r).max()), (l, key)
