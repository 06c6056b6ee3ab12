"""Probe: per-request, per-layer appended K/V errors of the batched Qwen3
QK-norm case (tests/test_gpu_batch.py::test_mid_qwen3_qk_norm_batch8)."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import batch_cases as bc
import decode_ref
import test_gpu_batch as t

model = dict(bc.MID_MODEL, qk_norm=True, eps=1e-6, theta=1e6)
rng = np.random.default_rng(5)
pages = [int(p) for p in rng.integers(1, 6, 8)]
pos0 = [int(rng.integers(0, 64 * p - 2)) for p in pages]
steps = [([int(x) for x in rng.integers(0, 4096, 8)], [p + s for p in pos0]) for s in range(2)]
orig = bc.check_batch


def check(info, state, host, tokens, pos, cfg=None):
    cfg = cfg or bc.model_cfg(info)
    for b in range(info["batch"]["nb"]):
        ref = decode_ref.decode_step(bc.request_view(info, state, b, cfg), cfg, int(tokens[b]), int(pos[b]))
        line = []
        for l in range(cfg["layers"]):
            k, v = bc.appended_rows(info, host, b, int(pos[b]), cfg, l)
            for nm, got, r in (("k", k, ref["k"][l]), ("v", v, ref["v"][l])):
                d = np.abs(got - r)
                line.append(f"L{l}{nm} {d.max() / np.abs(r).max():.2e}@{int(d.argmax())}(n>ulp {int((d > np.abs(r) * 2**-8 + 1e-30).sum())})")
        lg = host["logits"].reshape(info["batch"]["nb"], -1)[b]
        print(f"b={b} pos={pos[b]} logits {np.abs(lg - ref['logits']).max() / np.sqrt(np.mean(ref['logits']**2)):.2e} " + " ".join(line))
    return orig(info, state, host, tokens, pos, cfg)


bc.check_batch = check
for rs in t.run(model, pages, steps):
    print("---")
