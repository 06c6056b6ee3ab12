"""Precision-floor probe (diagnostic): engine logits vs the fp32 and fp64
torch checkers (same bf16 rounding points) as the model deepens.
  python tools/parity_probe.py [--batched]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import torch_ref as tr
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine


def stats(a, b):
    a, b = a.double(), b.double()
    rms = torch.sqrt((b * b).mean(dim=1))
    e = (a - b).abs()
    return (e.max(dim=1).values / rms).max().item(), (torch.sqrt((e * e).mean(dim=1)) / rms).max().item(), \
        float((a.argmax(1) == b.argmax(1)).float().mean())


def single(layers):
    import ring_cases as rc
    from bench import model_request
    req = model_request(layers, 4096)
    req["model"]["scaled_init"] = True
    prog = Program.build(req)
    info = prog.info()
    eng = Engine(prog, watchdog_ms=20000)
    tens = eng.synthesize(seed=0)
    cfg = dict(rc.model_cfg(info, req), vocab=128256, norm_scale_after=False)
    W = tr.weights_single(info, tens, cfg)
    st = torch.tensor([128000, 4000, 4001, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
    eng.bind_step(st)
    assert eng.run().status == 0
    out = {}
    for name, ct in (("f32", torch.float32), ("f64", torch.float64)):
        out[name] = tr.DenseDecoder(W, cfg, tr.caches_single(info, tens, cfg), ct).step([128000], [4000])["logits"]
    dev = tens["logits"].view(1, -1)[:, :128256]
    return out, dev


def batched(layers):
    import batch_cases as bc
    pages = [40, 20, 64, 9]
    req = bc.request({"preset": "llama3-8b", "layers": layers, "scaled_init": True}, pages, 64)
    prog = Program.build(req)
    info = prog.info()
    eng = Engine(prog, watchdog_ms=20000)
    tens = eng.synthesize(seed=3)
    cfg = dict(bc.model_cfg(info), vocab=tr.vocab_of(info))
    bi = info["batch"]
    pt = np.asarray(bi["page_table"], np.int64).reshape(bi["nb"], bi["maxp"])
    W = tr.weights_batched(info, tens, cfg)
    toks, pos = [1000, 2000, 3000, 4000], [p * 64 - 1 for p in pages]
    st = torch.from_numpy(bc.step_block(info, toks, pos)).cuda()
    eng.bind_step(st)
    assert eng.run().status == 0
    out = {}
    for name, ct in (("f32", torch.float32), ("f64", torch.float64)):
        out[name] = tr.DenseDecoder(W, cfg, tr.caches_batched(info, tens, cfg, pt, pages), ct).step(toks, pos)["logits"]
    return out, tens["logits"].view(4, -1)[:, : cfg["vocab"]]


if __name__ == "__main__":
    fn = batched if "--batched" in sys.argv else single
    for L in (1, 2, 4, 8, 16, 32):
        ref, dev = fn(L)
        print(f"layers {L:2d}: eng-vs-f64 max/rms-err {stats(dev, ref['f64'])}  f32-vs-f64 {stats(ref['f32'], ref['f64'])}  "
              f"eng-vs-f32 {stats(dev, ref['f32'])}", flush=True)
        torch.cuda.empty_cache()
