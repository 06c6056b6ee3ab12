"""Repeated launches of the Llama-3-8B ring program: hang/deadlock soak."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 12
n = int(sys.argv[3]) if len(sys.argv) > 3 else 200
prog = Program.build(bench.model_request(layers, ring_slots=slots))
eng = Engine(prog, watchdog_ms=2000)
bench.init_tensors(eng)
step = torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
eng.bind_step(step)
bad = 0
for i in range(n):
    rep = eng.run()
    if rep.status != 0:
        bad += 1
        print(i, rep.status, rep.message, flush=True)
print(f"slots={slots} launches={n} failures={bad} last_ms={rep.elapsed_ms:.3f}")
