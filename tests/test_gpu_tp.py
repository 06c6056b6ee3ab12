"""Tensor parallelism (§8e) on the ring engine, validated on one B200: the W
rank programs (column-parallel qkv / gate-up, row-parallel o / down with an
in-kernel ALLREDUCE_ADD over symmetric peer buffers, vocab-parallel lm_head)
run as W concurrent engine contexts on 148 // W SMs each, exchanging partial
sums through the same peer-store + system-scope counter protocol they use
across NVLink. The concatenated logits and the K/V rows must match the dense
reference of the assembled single-device model (bf16 tolerances of §8d)."""
import pytest

import ring_cases as rc
import tp_cases

pytestmark = pytest.mark.gpu


def assert_bf16_close(res):
    assert res["logits_max_abs"] <= 2e-2 * res["logits_rms"], res
    assert res["kv_rel"] <= 1e-2, res
    assert res["argmax_equal"], res


@pytest.mark.parametrize("world", [1, 2])
def test_tp_mid_matches_dense(cuda, world):
    results, _ = tp_cases.run_emulated(rc.MID, world, steps=((17, 300), (5, 301)))
    for res in results:
        assert_bf16_close(res)


def test_tp4_llama_shapes_match_dense(cuda):
    base = {"model": {"preset": "llama3-8b", "layers": 1, "vocab": 32000},
            "layout": {"ctx_pages": 8, "max_ctx": 512, "pages_per_job": 4, "gu_block": 4}}
    results, _ = tp_cases.run_emulated(base, 4, steps=((123, 400),))
    assert_bf16_close(results[0])
