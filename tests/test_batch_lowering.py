"""Batched ring lowering (decode.hpp LayoutConfig::batch),
checked on the CPU: the structural contract of batched programs the sm_100a
kernel relies on.

* every (row block, k tile) of every BGEMM operator is streamed exactly once,
  and each SM streams an equal share (+-1 tile: stream-K);
* stream-K pieces of a row block have consecutive partial slots, piece
  indices 0..n-1 and one arrival counter; complete blocks have none;
* every (request, kv head, logical page) is read exactly once, through the
  program's page table; attention jobs start their K tiles on even ring
  indices (a 16-byte pad tile realigns them);
* the page table is contiguous per request and the step block has room for
  it; readiness targets: one publish per row block per operator;
* tensor-parallel rank programs agree on the exchange buffers and split
  the vocabulary."""
import collections

import numpy as np
import pytest

import batch_cases as bc
from paper_2605_03190_b200 import Program

BGEMM, ATTN, ALLRED = 0x2D, 0x2A, 0x2C


def build(model, pages, sms=16, ppj=4, **layout):
    req = bc.request(model, pages, ppj, sms)
    req["layout"].update(layout)
    p = Program.build(req)
    return p.info(), p.text(False)


def stream_tiles(text, sm):
    out = []
    for l in text["streams"][f"sm{sm}.vmc"].splitlines():
        if l.startswith("LOAD"):
            out.append(l.split("addr=")[1].split()[0])
    return out


@pytest.mark.parametrize("pages,sms", [([3, 1, 5, 2], 16), ([1] * 17, 8), ([7, 2], 148)])
def test_batched_program_invariants(pages, sms):
    info, text = build(bc.MID_MODEL, pages, sms)
    assert text["certificate_ok"]
    jobs = info["jobs"]
    b = info["batch"]
    assert b["nb"] == len(pages) and b["npad"] == (16 if len(pages) <= 16 else 32) and b["maxp"] == max(pages)
    pt = np.asarray(b["page_table"]).reshape(len(pages), b["maxp"])
    nxt = 0
    for r, n in enumerate(pages):  # contiguous allocation, request-major
        assert list(pt[r, :n]) == list(range(nxt, nxt + n))
        nxt += n
    assert info["step_scalars"] >= b["page_table_off"] + pt.size

    # BGEMM: every (row block, k tile) exactly once per weight; balanced shares
    seen = collections.Counter()
    blocks = collections.defaultdict(list)
    for j in jobs:
        if j["op"] != BGEMM:
            continue
        kt0, kt1 = j["kt"]
        for kt in range(kt0, kt1):
            seen[(j["r0"] // 128, kt, j["k"], j["o"][0])] += 1
        blocks[(j["o"][0], j["r0"])].append(j)
    assert seen and max(seen.values()) == 1
    for (out, r0), ps in blocks.items():
        ps.sort(key=lambda j: j["split"])
        need = len(ps)
        assert [j["split"] for j in ps] == list(range(need))
        assert all(j["arrive"][1] == need for j in ps)
        if need > 1:
            assert len({j["arrive"][0] for j in ps}) == 1
            slots = [j["part"][1] for j in ps]
            assert slots == list(range(slots[0], slots[0] + need))
        kts = sorted((j["kt"][0], j["kt"][1]) for j in ps)
        assert kts[0][0] == 0 and all(a[1] == b2[0] for a, b2 in zip(kts, kts[1:]))
        assert kts[-1][1] == ps[0]["k"] // 64

    # attention: every (request, kv head, page) exactly once, K on even ring index
    att = collections.Counter()
    for j in jobs:
        if j["op"] == ATTN:
            h = j["a"][1] // (64 * 128)
            for p in range(j["r0"], j["r1"]):
                att[(j["req"], h, p)] += 1
    hkv = bc.MID_MODEL["kv_heads"]
    assert set(att) == {(r, h, p) for r, n in enumerate(pages) for h in range(hkv) for p in range(n)}
    assert set(att.values()) == {bc.MID_MODEL["layers"]}  # once per layer
    for sm in range(sms):
        g = 0
        for l in text["streams"][f"sm{sm}.vcc0"].splitlines():
            if l.startswith(("#", "HALT")):
                continue
            size = int(l.split("size=")[1].split()[0])
            j = jobs[int(l.split("imm=")[1].split()[0]) if "imm=" in l else 0]
            if j["op"] == ATTN:
                assert (g + j["lead_pad"]) % 2 == 0, "K tiles must start on an even ring index"
            g += size


def test_stream_k_balance_llama_shapes():
    """the Llama-3-8B gate/up operator over 148 SMs: every SM streams the same
    number of weight tiles (+-1)"""
    info, text = build({"preset": "llama3-8b", "layers": 1, "vocab": 32000}, [4] * 32, 148, 16)
    gu = [j for j in info["jobs"] if j["op"] == BGEMM and (j["flags"] & 0x04)]
    per_sm = collections.Counter()
    sm_of = {}
    for sm in range(148):
        for l in text["streams"][f"sm{sm}.vcc0"].splitlines():
            if not l.startswith(("#", "HALT")):
                sm_of[int(l.split("imm=")[1].split()[0]) if "imm=" in l else 0] = sm
    for i, j in enumerate(info["jobs"]):
        if j["op"] == BGEMM and (j["flags"] & 0x04):
            per_sm[sm_of[i]] += j["kt"][1] - j["kt"][0]
    assert gu and max(per_sm.values()) - min(per_sm.values()) <= 1
    assert sum(per_sm.values()) == (2 * 14336 // 128) * (4096 // 64)


def test_tp_rank_programs_agree():
    infos = []
    for r in range(2):
        info, text = build(bc.MID_MODEL, [3, 2], 16, tp_world=2, tp_rank=r)
        assert text["certificate_ok"]
        infos.append(info)
    sym = [[d["name"] for d in i["descriptors"] if d.get("symmetric")] for i in infos]
    assert sym[0] == sym[1] and len(sym[0]) == 2 * bc.MID_MODEL["layers"]
    shapes = [{d["name"]: d["shape"] for d in i["descriptors"]} for i in infos]
    assert shapes[0]["logits"][1] * 2 == bc.MID_MODEL["vocab"]
    ar = [[j for j in i["jobs"] if j["op"] == ALLRED] for i in infos]
    assert [j["x"][2] for j in ar[0]] == [j["x"][2] for j in ar[1]]  # identical readiness targets on both ranks


def test_qk_norm_jobs():
    info, _ = build(dict(bc.MID_MODEL, qk_norm=True), [2, 3], 16)
    att = [j for j in info["jobs"] if j["op"] == ATTN]
    assert att and all(j["flags"] & 0x1000 for j in att)
    qkv = [j for j in info["jobs"] if j["op"] == BGEMM and (j["flags"] & 0x80)]
    assert qkv and all(j["flags"] & 0x1000 for j in qkv)


def test_prefill_chunk_shares_pages():
    info, text = build(bc.MID_MODEL, [3] * 10, 16, prefill=True)
    assert text["certificate_ok"]
    b = info["batch"]
    pt = np.asarray(b["page_table"]).reshape(10, b["maxp"])
    assert (pt == pt[0]).all() and list(pt[0]) == [0, 1, 2]
    shapes = {d["name"]: d["shape"] for d in info["descriptors"]}
    assert shapes["L0.kc"][0] == 3  # one sequence's pages
    att = [j for j in info["jobs"] if j["op"] == ATTN]
    assert att and all(j["flags"] & 0x4000 for j in att)
    with pytest.raises(Exception):
        build(bc.MID_MODEL, [3, 2], 16, prefill=True)  # rows of a chunk share one allocation
