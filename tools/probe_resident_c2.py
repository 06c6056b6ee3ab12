"""C2 resident decode vs one launch per token on the SAME program (the
resident bench builds ctx_pages for the advanced positions, 67 pages at
ctx 4096 + 120 steps): separates the resident mechanism from the program
shape. Prints ms per step for each mode."""
import sys
sys.path.insert(0, '/root/repo')
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine


def timed(eng, launches, steps_per_launch):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(launches):
        eng.launch()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (launches * steps_per_launch)


def build(pages, feedback):
    req = bench.model_request(32)
    req["layout"].update(feedback=feedback, ctx_pages=pages, max_ctx=pages * 64)
    eng = Engine(Program.build(req), watchdog_ms=10000)
    bench.init_tensors(eng)
    step = torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
    eng.bind_step(step)
    return eng, step


for pages, fb in ((64, False), (67, False), (67, True)):
    eng, step = build(pages, fb)
    for _ in range(3):
        eng.run()
    step.copy_(torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0]))
    a = timed(eng, 20, 1)
    res = ""
    if fb:
        step.copy_(torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0]))
        eng.set_steps(20)
        eng.run()
        step.copy_(torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0]))
        b = timed(eng, 1, 20)
        eng.set_steps(1)
        res = f"  resident x20: {b:.4f} ms/step"
    print(f"pages {pages} feedback {fb}: one launch per step {a:.4f} ms/step{res}", flush=True)
    del eng
