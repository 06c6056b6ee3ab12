"""The CPU oracle (TEST INFRASTRUCTURE) pinned against an independent dense
numpy evaluation of the decode model (tests/decode_ref.py): the oracle
interpreter executes the lowered µop program of the tiny C1 decoder with the
reference's own HandlerState arithmetic (oracle/interp.cpp), decode_ref
evaluates the model equations directly. Tolerance: C1 fp32, max|d| <=
1e-5 * max|ref| on logits — relaxed to 1e-4 here because the
dense reference accumulates in fp64."""
import numpy as np
import pytest

import decode_ref
import harness
from paper_2605_03190_b200 import Program

TINY = {"hidden": 256, "heads": 4, "kv_heads": 4, "head_dim": 64, "ffn": 512, "eps": 1e-5, "theta": 10000.0,
        "layers": 2, "gu_block": 16, "dtype": "f32"}


def tiny_request(sm_count=4, ctx_pages=1, max_ctx=64):
    return {"model": {"preset": "tiny"},
            "layout": {"ctx_pages": ctx_pages, "max_ctx": max_ctx, "job_rows": 16, "gu_block": 16},
            "profile": {"builtin": "b200", "sm_count": sm_count}}


def shaped(info, arrays):
    return {d["name"]: arrays[d["name"]] for d in info["descriptors"] if d["view_of"] < 0}


@pytest.mark.skipif(not harness.oracle_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("token,pos", [(17, 16), (3, 40), (0, 0), (511, 63)])
def test_oracle_matches_dense_reference(token, pos):
    prog = Program.build(tiny_request())
    idx, ins, outs = harness.run_oracle(prog.text(True), seed=5, step=[token, pos, pos + 1])
    assert idx["returncode"] == 0 and idx["completed"]
    ref = decode_ref.decode_step(shaped(prog.info(), ins), TINY, token, pos)
    lg = outs["logits"]
    assert np.abs(lg - ref["logits"]).max() <= 1e-4 * np.abs(ref["logits"]).max()
    for l in range(TINY["layers"]):
        kc = outs[f"L{l}.kc"].reshape(4, 64, 64)[:, pos].reshape(-1)
        vc = outs[f"L{l}.vc"].reshape(4, 64, 64)[:, pos].reshape(-1)
        assert np.abs(kc - ref["k"][l]).max() <= 1e-4 * max(1.0, np.abs(ref["k"][l]).max())
        assert np.abs(vc - ref["v"][l]).max() <= 1e-4 * max(1.0, np.abs(ref["v"][l]).max())
