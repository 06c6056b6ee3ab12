"""Loop folding of the ring memory-core streams (ring_abi.h vdc_run; the
hot-path counterpart of the reference's fold.cpp:151-293):
every SM's LOAD stream of real programs folds into a few run words and
unfolds back to the same words, word for word."""
import numpy as np
import pytest

import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import fold_stream, unfold_stream

OP_LOAD, OP_HALT = 0x01, 0x45


def _vmc_streams(prog):
    n_cores = prog.cores()[0]
    out = []
    for i in range(0, n_cores, 2):  # 2 sm = memory core, 2 sm + 1 = compute core
        w = prog.words(i)
        if len(w) >= 16 and w[-16] == OP_HALT:
            w = w[:-16]
        out.append(w)
    return out


def _check(prog):
    total = folded = 0
    for w in _vmc_streams(prog):
        runs = fold_stream(w)
        n = len(w) // 16
        assert unfold_stream(runs, n) == w
        count, alt = runs["count_alt"] & 0xffffff, runs["count_alt"] >> 24
        assert int(count.sum()) == n and (count >= 1).all()
        assert ((alt == 1) | (alt == 2)).all()
        total += n
        folded += len(runs)
    return total, folded


def test_fold_c2_32_layers():
    total, folded = _check(Program.build(bench.model_request(32)))
    # about one run per job: 981,632 LOAD words -> 23,200 (~157 per SM)
    assert total > 900_000 and folded * 40 < total, (total, folded)


def test_fold_batched_c3_shapes():
    B = 32
    ctxs = bench.c3_contexts(B)
    pages = [(c + 63) // 64 for c in ctxs]
    req = {"engine": "ring", "model": {"preset": "llama3-8b", "layers": 2},
           "layout": {"batch": B, "req_pages": pages, "pages_per_job": 128, "gu_block": 128, "page_rows": 64},
           "profile": {"builtin": "b200"}}
    total, folded = _check(Program.build(req))
    assert folded * 10 < total, (total, folded)


def test_fold_tiny_and_edge_cases():
    _check(Program.build({"engine": "ring", "model": {"preset": "tiny"},
                          "layout": {"ctx_pages": 1, "max_ctx": 64, "job_rows": 16, "gu_block": 16},
                          "profile": {"builtin": "b200", "sm_count": 4}}))
    assert len(fold_stream(b"")) == 0
    # a single LOAD is a run of 1; non-affine coordinates split into runs
    prog = Program.build(bench.model_request(1))
    w = _vmc_streams(prog)[0]
    runs = fold_stream(w[:16])
    assert len(runs) == 1 and runs["count_alt"][0] == (1 | 1 << 24) and runs["base"][0].tobytes() == w[:16]
    shuffled = b"".join(w[16 * i: 16 * i + 16] for i in (0, 5, 1, 7, 2))
    runs = fold_stream(shuffled)
    assert unfold_stream(runs, 5) == shuffled and len(runs) >= 3
