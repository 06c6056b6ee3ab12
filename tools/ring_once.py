"""Minimal ring-engine launch sequence for ncu captures: N-layer Llama-3-8B
program, `launches` back-to-back launches (default 3)."""
import sys
sys.path.insert(0, '/root/repo')
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prog = Program.build(bench.model_request(layers))
eng = Engine(prog, watchdog_ms=20000)
bench.init_tensors(eng)
step = torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
eng.bind_step(step)
for _ in range(launches):
    rep = eng.run()
print("status", rep.status, "ms", rep.elapsed_ms)
