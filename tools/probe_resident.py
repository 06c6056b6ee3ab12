"""Probe: batched resident decode vs separate launches — where do the KV
caches differ (pool page, head, row, column)?"""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import torch
import batch_cases as bc
import test_gpu_decode_loop as t

pages = [2, 3, 1, 4, 2, 2]
pos0 = [60, 120, 10, 180, 70, 64]
tok0 = [5, 77, 901, 3, 1234, 42]
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
out = {}
for mode in ("launches", "resident", "launches2", "resident2"):
    req = bc.request(bc.MID_MODEL, pages, 4, None)
    req["layout"].update(argmax=True, feedback=True)
    eng, tens, info = t.engine(req)
    st = torch.from_numpy(bc.step_block(info, tok0, pos0)).cuda()
    eng.bind_step(st)
    if mode.startswith("resident"):
        eng.set_steps(steps)
        eng.run()
    else:
        for _ in range(steps):
            eng.run()
    out[mode] = {k: v.float().cpu().numpy() for k, v in tens.items() if not k.endswith(("sk", "part", "amax", "pad"))}
    shape = {d["name"]: d["shape"] for d in info["descriptors"]}
for m1, m2 in (("launches", "launches2"), ("resident", "resident2"), ("launches", "resident")):
  print("==", m1, "vs", m2)
  for k in out["launches"]:
    a, b = out[m1][k], out[m2][k]
    bad = np.nonzero(a != b)[0]
    if len(bad):
        sh = shape[k]
        print(k, sh, "differs at", len(bad), "elements; first:", [(int(i), float(a[i]), float(b[i])) for i in bad[:6]])
    else:
        pass
