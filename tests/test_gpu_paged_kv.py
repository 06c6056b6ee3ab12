"""Paged KV with a host block allocator: a shared page
pool smaller than the requests' total capacity, pages reserved on demand
between launches (vdc_kv_reserve -> the step block's page table), 100
device-fed decode steps (fused argmax + feedback) that cross page
boundaries, and a request that finishes, releases its pages and restarts
at position 0 on recycled pages (stale contents must not leak: pages past
the context are never loaded, rows past it are masked). Every step is
checked against the fp64 / fp32 torch checkers (torch_ref.py) that keep
their own per-request caches. Plus: appending at a position without a page
fails loudly (fault 7) instead of writing another request's page."""
import numpy as np
import pytest

import batch_cases as bc
import torch_ref as tr
from paper_2605_03190_b200 import KvPages, Program

pytestmark = pytest.mark.gpu


def _setup(ctxs, cap_pages, pool_pages, seed=5):
    import torch
    from paper_2605_03190_b200.engine import Engine

    req = bc.request(dict(bc.MID_MODEL, scaled_init=True), [cap_pages] * len(ctxs), 4)
    req["layout"].update(argmax=True, feedback=True, pool_pages=pool_pages)
    prog = Program.build(req)
    info = prog.info()
    eng = Engine(prog, watchdog_ms=5000)
    tens = eng.synthesize(seed=seed)
    bi = info["batch"]
    kv = KvPages(pool_pages, bi["nb"], bi["maxp"])
    return torch, eng, tens, info, kv


def _write_table(st, info, kv):
    import torch
    bi = info["batch"]
    off = bi["page_table_off"]
    st[off: off + bi["nb"] * bi["maxp"]].copy_(torch.tensor(kv.table(), dtype=torch.int64))


def test_shared_pool_growth_release_restart(cuda):
    ctxs = [60, 120, 10, 180, 70, 64]
    cap, steps = 6, 100
    torch, eng, tens, info, kv = _setup(ctxs, cap, pool_pages=24)
    B = len(ctxs)
    for b, c in enumerate(ctxs):
        kv.reserve(b, c)
    cfg = dict(bc.model_cfg(info), vocab=tr.vocab_of(info))
    W = tr.weights_batched(info, tens, cfg)
    pt0 = np.asarray(kv.table(), np.int64).reshape(B, -1)
    held0 = kv.stats()[1]
    refs = [tr.DenseDecoder(W, cfg, tr.caches_batched(info, tens, cfg, pt0, held0, cap_pages=cap), ct)
            for ct in (torch.float64, torch.float32)]
    toks = [int(5 + 101 * b) for b in range(B)]
    pos = [c - 1 for c in ctxs]
    st = torch.from_numpy(bc.step_block(info, toks, pos)).cuda()
    agree = total = 0
    crossed = 0
    for k in range(steps):
        if k == 50:  # request 2 finishes; its row restarts a new sequence at position 0 on recycled pages
            kv.release(2)
            toks[2], pos[2] = 7, 0
            st[6], st[7], st[8] = 7, 0, 1
            for r in refs:
                for l in range(cfg["layers"]):
                    r.caches[2][l] = tuple(torch.zeros_like(c) for c in r.caches[2][l])
        for b in range(B):
            before = kv.stats()[1][b]
            kv.reserve(b, pos[b] + 1)  # the page of the position this launch appends
            crossed += kv.stats()[1][b] > before
        _write_table(st, info, kv)
        eng.bind_step(st)
        rep = eng.run()
        assert rep.status == 0, rep.message
        r64, r32 = (r.step(toks, pos) for r in refs)
        e = tr.errors(tens["logits"].view(B, -1), r64)
        floor = tr.errors(r32["logits"], r64)
        assert (e["rms"] <= 2e-2).all() and (e["max"] <= np.maximum(2e-2, 1.25 * floor["max"])).all(), (k, e, floor)
        agree += int(e["argmax_equal"].sum())
        total += B
        nxt = [int(x) for x in tens["next_token"].view(-1)[:B].tolist()]
        assert [int(x) for x in st[0:3 * B:3].tolist()] == nxt  # fed back on the device
        toks, pos = nxt, [p + 1 for p in pos]
    assert crossed >= B  # every request grew by at least one page during the run
    assert agree >= 0.99 * total, (agree, total)
    free, held = kv.stats()
    assert free + sum(held) == 24


def test_append_without_a_page_faults(cuda):
    torch, eng, tens, info, kv = _setup([100, 30], 4, pool_pages=8)
    kv.reserve(0, 100)
    kv.reserve(1, 30)
    st = torch.from_numpy(bc.step_block(info, [1, 2], [99, 64])).cuda()  # request 1 appends at 64: no page 1
    _write_table(st, info, kv)
    eng.bind_step(st)
    rep = eng.run()
    assert rep.status != 0 and "fault code 7" in rep.message, rep.message
