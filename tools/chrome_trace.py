"""Device trace of one decode step as a Chrome trace (chrome://tracing /
Perfetto): every compute µop of every SM with its dependency wait and
execution, named by operator (SURVEY §8f observability).

  python tools/chrome_trace.py [layers] [out.json] [batch]

batch > 1 traces the batched (C3-shaped) program instead of the
single-request one."""
import sys
sys.path.insert(0, '/root/repo')
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/ring_trace.json"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if B > 1:
    ctxs = bench.c3_contexts(B)
    pages = [(c + 63) // 64 for c in ctxs]
    req = {"engine": "ring", "model": {"preset": "llama3-8b", "layers": layers},
           "layout": {"batch": B, "req_pages": pages, "pages_per_job": 64, "gu_block": 128, "page_rows": 64, "argmax": True},
           "profile": {"builtin": "b200"}}
    prog = Program.build(req)
else:
    prog = Program.build(bench.model_request(layers))
eng = Engine(prog, watchdog_ms=20000)
bench.init_tensors(eng)
info = eng.info
if B > 1:
    st = [0] * int(info["step_scalars"])
    for b in range(B):
        st[3 * b: 3 * b + 3] = [17 + b, ctxs[b] - 1, ctxs[b]]
    bi = info["batch"]
    st[bi["page_table_off"]: bi["page_table_off"] + len(bi["page_table"])] = bi["page_table"]
    eng.bind_step(torch.tensor(st, dtype=torch.int64, device="cuda"))
else:
    eng.bind_step(torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda"))
eng.enable_trace(1024)
for _ in range(3):
    rep = eng.run()
print(f"{eng.chrome_trace(out)} slices -> {out} (kernel {rep.elapsed_ms:.3f} ms)")
