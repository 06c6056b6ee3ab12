import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np
import test_gpu_batch as t
import batch_cases as bc
rng = np.random.default_rng(2)
pages = [int(p) for p in rng.integers(1, 7, 20)]
pos0 = [int(rng.integers(0, 64 * p - 3)) for p in pages]
steps = []
for s in range(3):
    steps.append(([int(x) for x in rng.integers(0, 4096, 20)], [p + s for p in pos0]))
for k, rs in enumerate(t.run(bc.MID_MODEL, pages, steps, argmax=True)):
    print("step", k, "max logits err/rms", max(r["logits_max_abs"]/r["logits_rms"] for r in rs), "kv_rel", max(r["kv_rel"] for r in rs), "argmax eq", sum(r["argmax_equal"] for r in rs))
