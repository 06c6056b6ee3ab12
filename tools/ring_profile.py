"""Ring engine on the Llama-3-8B program (N layers): per-SM wait accounting."""
import sys, json
sys.path.insert(0, '/root/repo')
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ppj = int(sys.argv[3]) if len(sys.argv) > 3 else 4
prog = Program.build(bench.model_request(layers, ring_slots=slots, pages_per_job=ppj))
eng = Engine(prog, watchdog_ms=10000)
pf = int(sys.argv[4]) if len(sys.argv) > 4 else 0
eng.set_prefetch(pf)
tens = bench.init_tensors(eng)
nb = bench.algorithmic_bytes(eng.info, 4096)
step = torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
eng.bind_step(step)
for _ in range(3):
    rep = eng.run()
ms = []
for _ in range(10):
    rep = eng.run(); ms.append(rep.elapsed_ms)
ms.sort()
sms = eng.info["sm_count"]
clk = 1.965e9
t = ms[len(ms)//2]
print(f"layers={layers} slots={slots} ppj={ppj} pf={pf} status={rep.status} ms={t:.3f} (min {ms[0]:.3f}) GB/s={nb['total']/t/1e6:.1f} uops={rep.uops_executed} {rep.message}")
for k, v in rep.wait_cycles.items():
    if k == "jobs":
        print(f"  jobs/SM {v/sms:.1f}")
    else:
        print(f"  {k:16s} {v/sms/clk*1e3:8.3f} ms/SM ({v/sms/clk*1e3/t*100:5.1f}%)")
