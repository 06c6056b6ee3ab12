"""Run the Llama-3-8B decode program (N layers) and print engine wait-site
accounting (cycles per SM, as a fraction of the launch)."""
import sys, time, json
sys.path.insert(0, '/root/repo')
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
req = bench.model_request(layers)
if len(sys.argv) > 2:
    req["layout"].update(json.loads(sys.argv[2]))
prog = Program.build(req)
eng = Engine(prog, watchdog_ms=10000)
bench.init_tensors(eng)
step = torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
eng.bind_step(step)
for _ in range(3):
    rep = eng.run()
rep = eng.run()
sms = eng.info["sm_count"]
clk = 1.965e9
total = rep.elapsed_ms * 1e-3 * clk
print(rep.message); print(f"layers={layers} ms={rep.elapsed_ms:.3f} uops={rep.uops_executed} GB/s={rep.bytes_loaded/rep.elapsed_ms/1e6:.1f} status={rep.status}")
for k, v in rep.wait_cycles.items():
    if v:
        per = v / sms
        print(f"  {k:12s} {per/clk*1e3:9.3f} ms/SM  ({per/total*100:6.1f}% of launch)")
