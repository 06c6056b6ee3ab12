"""Device trace of one decode step as a Chrome trace (chrome://tracing /
Perfetto): every compute µop of every SM with its dependency wait and
execution, named by operator (SURVEY §8f observability).

  python tools/chrome_trace.py [layers] [out.json]"""
import sys
sys.path.insert(0, '/root/repo')
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/ring_trace.json"
prog = Program.build(bench.model_request(layers))
eng = Engine(prog, watchdog_ms=10000)
bench.init_tensors(eng)
eng.bind_step(torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda"))
eng.enable_trace(256)
for _ in range(3):
    rep = eng.run()
print(f"{eng.chrome_trace(out)} slices -> {out} (kernel {rep.elapsed_ms:.3f} ms)")
