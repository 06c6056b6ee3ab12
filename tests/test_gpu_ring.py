"""Device parity of the ring engine (the decode hot path: one persistent
sm_100a kernel, include/uopsim/ring_abi.h) through the C-ABI.

Checks, on identical synthetic inputs:
  * against the dense numpy decode (tests/decode_ref.py; itself pinned to
    the CPU oracle by test_decode_oracle.py): logits and the appended K/V
    rows. Tolerances: fp32 model (C1 tiny) max|d| <= 1e-5 *
    max|ref|; bf16 models max|d logits| <= 2e-2 * rms(ref logits), KV rows
    rel <= 1e-2 (one bf16 ulp is 7.8e-3), argmax equal.
  * against the CPU oracle interpreter running the reference-form µop
    program of the same graph (oracle/_ref/oracle_interp): same bound.
  * a multi-step decode (device KV cache carried across launches, positions
    advancing) against the dense reference step by step.
"""
import numpy as np
import pytest

import decode_ref
import harness
import ring_cases as rc
from paper_2605_03190_b200 import Program

pytestmark = pytest.mark.gpu

LLAMA_1L = {"model": {"preset": "llama3-8b", "layers": 1, "vocab": 32000},
            "layout": {"ctx_pages": 16, "max_ctx": 1024, "pages_per_job": 4, "gu_block": 4}}


def run(base, sms=None, steps=((17, 40),), seed=0, ring_slots=12):
    from paper_2605_03190_b200.engine import Engine
    import torch

    req = rc.request(base, sms, ring_slots)
    prog = Program.build(req)
    info = prog.info()
    ins = rc.synth_inputs(info, seed)
    eng = Engine(prog, watchdog_ms=5000)
    tens = eng.bind_inputs(ins)
    st = torch.zeros(8, dtype=torch.int64, device="cuda")
    eng.bind_step(st)
    outs = []
    state = {k: v.copy() for k, v in ins.items()}
    for token, pos in steps:
        st[0], st[1], st[2] = token, pos, pos + 1
        rep = eng.run()
        assert rep.status == 0, rep.message
        host = eng.host_arrays(tens)
        res = rc.check_against_dense(info, req, state, host, token, pos)
        outs.append((res, host))
        state = {k: v.copy() for k, v in host.items()}  # the device caches feed the next step
    return info, req, ins, outs


def assert_close(res, fp32):
    if fp32:
        assert res["logits_max_abs"] <= 1e-5 * res["logits_max"], res
        assert res["kv_rel"] <= 1e-5, res
    else:
        assert res["logits_max_abs"] <= 2e-2 * res["logits_rms"], res
        assert res["kv_rel"] <= 1e-2, res
    assert res["argmax_equal"], res


@pytest.mark.parametrize("sms", [4, 148])
@pytest.mark.parametrize("token,pos", [(17, 40), (3, 0), (500, 63)])
def test_tiny_fp32_matches_dense(cuda, sms, token, pos):
    _, _, _, outs = run(rc.TINY, sms, ((token, pos),))
    assert_close(outs[0][0], fp32=True)


@pytest.mark.parametrize("token,pos", [(17, 300), (3, 0), (4095, 511)])
def test_mid_bf16_matches_dense(cuda, token, pos):
    _, _, _, outs = run(rc.MID, None, ((token, pos),))
    assert_close(outs[0][0], fp32=False)


@pytest.mark.parametrize("slots", [8, 10, 11])
def test_mid_bf16_other_ring_depths(cuda, slots):
    """rings of 8, 10 and 11 slots: the memory core's lanes walk the folded
    stream (ring_abi.h vdc_run) with stride R, so every run entry is entered
    at other offsets than with 12 slots; two steps carry the caches"""
    _, _, _, outs = run(rc.MID, None, ((17, 300), (18, 301)), ring_slots=slots)
    for res, _ in outs:
        assert_close(res, fp32=False)


def test_fused_argmax_matches_logits(cuda):
    """greedy sampling fused into the lm_head epilogue: next_token equals the
    argmax of the device logits (first index on ties) and of the reference"""
    base = {"model": dict(rc.MID["model"]), "layout": dict(rc.MID["layout"], argmax=True)}
    for token, pos in ((17, 300), (4095, 511)):
        info, req, ins, outs = run(base, None, ((token, pos),))
        res, host = outs[0]
        assert_close(res, fp32=False)
        assert int(host["next_token"][0]) == int(np.argmax(host["logits"])), (host["next_token"], np.argmax(host["logits"]))


@pytest.mark.parametrize("token,pos", [(17, 300), (3, 0), (4095, 511)])
def test_mid_qwen3_qk_norm_matches_dense(cuda, token, pos):
    """Qwen3 QK-norm (per-head RMSNorm of q and k before the rotary, applied
    by the attention µop; the appended k row is written back normalised)"""
    base = {"model": dict(rc.MID["model"], qk_norm=True, eps=1e-6, theta=1e6), "layout": dict(rc.MID["layout"])}
    _, _, _, outs = run(base, None, ((token, pos), (token + 1, pos + 1)) if pos < 511 else ((token, pos),))
    for res, _ in outs:
        assert_close(res, fp32=False)


def test_llama3_8b_layer_matches_dense(cuda):
    _, _, _, outs = run(LLAMA_1L, None, ((1234, 777),))
    assert_close(outs[0][0], fp32=False)


def test_multi_step_decode_carries_the_kv_cache(cuda):
    steps = [(17, 100), (5, 101), (99, 102), (7, 103)]
    _, _, _, outs = run(rc.MID, None, steps)
    for res, _ in outs:
        assert_close(res, fp32=False)


@pytest.mark.skipif(not harness.oracle_available(), reason="oracle/_ref not built")
def test_tiny_matches_oracle_interpreter(cuda):
    """ring device result vs the CPU oracle executing the reference-form
    program (LOAD_WAIT/ALLOC/FREE/STORE streams + reference handlers)"""
    token, pos = 21, 33
    info, req, ins, outs = run(rc.TINY, None, ((token, pos),))
    ref_req = {"model": req["model"], "layout": {k: v for k, v in req["layout"].items()},
               "profile": {"builtin": "b200", "sm_count": 4}}
    ref_req["layout"]["job_rows"] = 16
    ref_prog = Program.build(ref_req)
    rinfo = ref_prog.info()
    names = [d["name"] for d in rinfo["descriptors"] if d["view_of"] < 0]
    blob = b"".join(np.ascontiguousarray(ins[n], np.float32).tobytes() for n in names)
    idx, _, ref_out = harness.run_oracle(ref_prog.text(True), step=[token, pos, pos + 1], inputs=blob)
    assert idx["returncode"] == 0 and idx["completed"]
    host = outs[0][1]
    scale = np.abs(ref_out["logits"]).max()
    assert np.abs(host["logits"] - ref_out["logits"]).max() <= 1e-5 * scale
    for l in range(2):
        for c in ("kc", "vc"):
            a = host[f"L{l}.{c}"].reshape(4, 64, 64)[:, pos]
            b = ref_out[f"L{l}.{c}"].reshape(4, 64, 64)[:, pos]
            assert np.abs(a - b).max() <= 1e-5 * max(1.0, np.abs(b).max())


def test_cpp_machine_dropin_runs(cuda):
    """the reference's simulate()/Machine call sites, unchanged, on the device"""
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    subprocess.run(["make", "-C", str(root / "examples"), "all"], check=True, capture_output=True)
    r = subprocess.run([str(root / "examples" / "machine_demo")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fig4: status=completed" in r.stdout and "tiny decode (ring): status=completed" in r.stdout
    # ExecutionReport serialisations + device conservation counts, and the
    # wait-for edge of a program stuck on a dep queue nobody produces
    assert "json_roundtrip=exact" in r.stdout and "queues_drained=1 slots_all_free=1" in r.stdout, r.stdout
    assert "stuck program: status=deadlock" in r.stdout and "named=yes" in r.stdout, r.stdout
    # a batched program driven from C++: step block sized by the program,
    # page table from the vdc_kv_* block allocator, fused sampling
    b = subprocess.run([str(root / "examples" / "batched_demo")], capture_output=True, text=True, timeout=120)
    assert b.returncode == 0, b.stdout + b.stderr
    assert b.stdout.count("status=completed") == 4, b.stdout
