"""Input synthesis parity: the reference synthesize_inputs
stream (workload.cpp:411-435, util.hpp:15-33, incl. the [-1, 3) unit_float
quirk, finding 8).

CPU: the numpy restatement (synth_ref.py) reproduces the reference's own
outputs bit for bit (golden vectors from oracle/_ref/ref_cli).
GPU: the device synthesizer (vdc_program_synthesize) produces exactly the
restatement's values for every storage tensor of single-request and batched
decode programs, in their device layouts (packed / swizzled tensors are
compared after to_logical)."""
import json
from pathlib import Path

import numpy as np
import pytest

import synth_ref as sr

GOLD = json.loads((Path(__file__).parent / "golden" / "synth_golden.json").read_text())


@pytest.mark.parametrize("case", range(len(GOLD["cases"])))
def test_restatement_matches_reference_synthesize_inputs(case):
    c = GOLD["cases"][case]
    outputs = {o for op in GOLD["workload"]["operators"] for o in op["outputs"]}
    specs = {t["name"]: t for t in GOLD["workload"]["tensors"]}
    assert len(c["tensors"]) == len(specs)
    for t in c["tensors"]:
        s = specs[t["name"]]
        n = int(np.prod(s["shape"]))
        assert t["n"] == n
        init = "zeros" if t["name"] in outputs else s["init"]
        v = sr.synthesize(t["name"], n, init, seed=c["seed"])
        assert [int(x) for x in v[: len(t["head_bits"])].view(np.uint32)] == t["head_bits"], t["name"]
        assert sr.bits_fnv1a(v) == int(t["fnv1a_bits"]), t["name"]


def test_unit_float_range_quirk():
    u = sr.unit_float(sr.draws(12345, 1 << 16))
    assert u.min() >= -1.0 and u.max() < 3.0 and u.max() > 2.9  # [-1, 3), not the commented [-1, 1)


def test_offset_draws_continue_the_stream():
    a = sr.synthesize("w", 100, seed=3)
    b = sr.synthesize("w", 60, seed=3, start=40)
    assert np.array_equal(a[40:], b)


@pytest.mark.gpu
@pytest.mark.parametrize("batched", [False, True])
def test_device_synthesis_matches_restatement(cuda, batched):
    import ring_cases as rc
    import batch_cases as bc
    from paper_2605_03190_b200 import Program
    from paper_2605_03190_b200.engine import Engine, to_logical

    req = bc.request(bc.MID_MODEL, [3, 1, 5, 2], 4) if batched else rc.request(rc.MID)
    req["model"]["scaled_init"] = True
    prog = Program.build(req)
    eng = Engine(prog)
    tens = eng.synthesize(seed=11)
    descs = {d["name"]: d for d in prog.info()["descriptors"]}
    seen_layouts = set()
    for name, t in tens.items():
        d = descs[name]
        got = to_logical(d, t.float().cpu().numpy())
        init = d["init"] if (d["external"] or d["state"]) and not d["symmetric"] else 1
        want = sr.synthesize(name, got.size, init, seed=11, scale=d["init_scale"], dtype=d["dtype"])
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), name
        seen_layouts.add(d["tma"] if d["tma"] in (0x80000000, 0x40000000) else 0)
    if batched:
        assert seen_layouts == {0, 0x80000000, 0x40000000}
