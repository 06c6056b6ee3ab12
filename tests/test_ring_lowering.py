"""Ring-mode lowering (host/ring_lower.cpp) invariants, checked on the CPU.

The ring program is the decode path's µop program: per SM a memory stream of
LOAD [send] tile words and a compute stream of operand-block µops
(include/uopsim/ring_abi.h). These tests pin the structural contract the
device engine relies on: every compute µop's tiles are exactly the LOADs of
its SM's memory stream in order; each GEMV operator's output rows are
covered exactly once; every KV page of every kv head is read exactly once;
readiness targets equal the number of producing µops; per-SM work is
balanced; and operators appear in topological order on every SM
(deadlock freedom of the counter waits)."""
import collections

import pytest

import bench
import ring_cases as rc
from paper_2605_03190_b200 import Program, VdcError

OP = {"GEMV": 0x27, "RMS_GEMV": 0x28, "GEMV_ADD": 0x29, "ATTN_DECODE": 0x2A}


def build(req):
    p = Program.build(req)
    return p, p.info(), p.text(False)


def parse_stream(text):
    out = []
    for line in text.splitlines():
        if line.startswith("#"):
            continue
        name = line.split()[0]
        f = dict(kv.split("=", 1) for kv in line.split()[2:] if "=" in kv) if "[" in line else {}
        out.append((name, line, f))
    return out


CASES = {"tiny": rc.request(rc.TINY), "tiny4": rc.request(rc.TINY, 4), "mid": rc.request(rc.MID),
         "llama3-8b-2l": bench.model_request(2)}


@pytest.mark.parametrize("name", sorted(CASES))
def test_ring_program_invariants(name):
    prog, info, text = build(CASES[name])
    assert text["certificate_ok"], "validate_ring_program reported a violation"
    jobs = info["jobs"]
    descs = info["descriptors"]
    sms = info["sm_count"]
    # per SM: compute µops consume exactly the memory stream's LOADs
    for sm in range(sms):
        mem = [l for l in text["streams"][f"sm{sm}.vmc"].splitlines() if l.startswith("LOAD")]
        comp = [l for l in text["streams"][f"sm{sm}.vcc0"].splitlines() if not l.startswith(("#", "HALT"))]
        used = 0
        for l in comp:
            size = int(l.split("size=")[1].split()[0])
            imm = int(l.split("imm=")[1].split()[0]) if "imm=" in l else 0
            j = jobs[imm]
            used += size
            if j["op"] in (OP["GEMV"], OP["RMS_GEMV"], OP["GEMV_ADD"]):
                tr, tc = j["tile"]
                assert size == (j["r1"] - j["r0"]) // tr * (j["k"] // tc)
            elif j["op"] == OP["ATTN_DECODE"]:
                assert size == 2 * (j["r1"] - j["r0"]) + j["lead_pad"] if "lead_pad" in j else True
        assert used == len(mem), f"sm{sm}: {used} tiles consumed, {len(mem)} loaded"
    # GEMV rows covered exactly once per (weight tensor)
    cover = collections.defaultdict(list)
    for j in jobs:
        if j["op"] in (OP["GEMV"], OP["RMS_GEMV"], OP["GEMV_ADD"]):
            key = (j["o"][0], j["k"], j["flags"] & 0x1, j["x"][0])
            cover[key].append((j["r0"], j["r1"]))
    for key, rs in cover.items():
        rs.sort()
        for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
            assert a1 <= b0, f"overlapping GEMV rows {rs}"
    # readiness targets: number of µops producing the storage tensor
    writers = collections.Counter()
    for j in jobs:
        if j["flags"] & 0x80:  # fused q|k|v rows: publishes every region it touches
            qrows, kvr = j["block"], j["split"]
            if j["r0"] < qrows:
                writers[j["o"][0]] += 1
            if j["r0"] < qrows + kvr and j["r1"] > qrows:
                writers[j["b"][0]] += 1
            if j["r1"] > qrows + kvr:
                writers[j["o2"][0]] += 1
        else:
            writers[j["o"][0]] += 1
    for j in jobs:
        for key in ("x", "a", "b"):
            t, _, need = j[key]
            if t >= 0 and need:
                assert need == writers[t] or descs[t]["name"].endswith((".attn",)), (key, j)


@pytest.mark.parametrize("name", ["tiny", "llama3-8b-2l"])
def test_ring_balance(name):
    prog, info, text = build(CASES[name])
    loads = [sum(1 for l in text["streams"][f"sm{s}.vmc"].splitlines() if l.startswith("LOAD"))
             for s in range(info["sm_count"])]
    if name.startswith("llama"):
        # equal bytes per SM within 5% (weights split to +-1 tile per operator;
        # the attention pages sit on 128 of the 148 SMs)
        mean = sum(loads) / len(loads)
        assert (max(loads) - min(loads)) / mean < 0.05, (min(loads), max(loads), mean)


@pytest.mark.parametrize("slots", [6, 9, 13])
def test_ring_slots_give_every_slot_one_consumer_warp(slots):
    req = dict(CASES["tiny"], ring_slots=slots)
    with pytest.raises(VdcError):
        Program.build(req)


def test_attention_pages_read_once():
    prog, info, text = build(CASES["llama3-8b-2l"])
    kv = {f"t{d['index']}@" for d in info["descriptors"] if d["name"] in ("L0.kc", "L0.vc")}
    pages = collections.Counter()
    for sm in range(info["sm_count"]):
        for l in text["streams"][f"sm{sm}.vmc"].splitlines():
            addr = l.split("addr=")[1].split()[0] if l.startswith("LOAD") else ""
            if any(addr.startswith(t) for t in kv):
                pages[addr] += 1
    # every (kv head, page) of L0.kc / L0.vc loaded once (a lead pad may repeat one)
    assert len(pages) == 2 * 8 * 64
    assert sum(pages.values()) - len(pages) <= info["sm_count"]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_tp_rank_programs_shard_the_model(world):
    """Megatron split of Llama-3-8B: every rank holds 1/world of the
    projection rows/columns and of the vocabulary, the o and down GEMVs write
    this rank's slot of a symmetric (W*D) partial buffer, and one
    ALLREDUCE_ADD per block sums the slots in rank order."""
    totals = collections.Counter()
    for rank in range(world):
        req = bench.model_request(2)
        req["layout"]["tp_world"], req["layout"]["tp_rank"] = world, rank
        req["profile"]["sm_count"] = 148
        prog = Program.build(req)
        info = prog.info()
        assert prog.text(False)["certificate_ok"]
        ds = {d["name"]: d for d in info["descriptors"]}
        assert ds["L0.wqkv"]["shape"][0] == (4096 + 2 * 1024) // world
        assert ds["L0.wo"]["shape"] == [4096, 4096 // world]
        assert ds["L0.wd"]["shape"] == [4096, 14336 // world]
        assert ds["L0.o.part"]["symmetric"] and ds["L0.o.part"]["shape"] == [world * 4096, 1]
        ar = [j for j in info["jobs"] if j["op"] == 0x2C]
        assert sum(j["r1"] - j["r0"] for j in ar) == 2 * 2 * 4096  # 2 allreduces x 2 layers x D rows
        sym_out = [j for j in info["jobs"] if j["flags"] & 0x100]
        assert all(j["o"][1] == rank * 4096 for j in sym_out)
        totals["lm_head"] += ds["lm_head"]["shape"][0] * ds["lm_head"]["shape"][1] if len(ds["lm_head"]["shape"]) == 2 else \
            ds["lm_head"]["shape"][0] * ds["lm_head"]["shape"][1] * ds["lm_head"]["shape"][2]
    assert totals["lm_head"] == 128256 * 4096
