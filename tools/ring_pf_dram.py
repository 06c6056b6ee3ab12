"""One 32-layer launch with a given L2 look-ahead (argv[1] rounds) for ncu dram-byte comparison."""
import sys
sys.path.insert(0, '/root/repo')
import torch, bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine
prog = Program.build(bench.model_request(32))
eng = Engine(prog, watchdog_ms=10000)
eng.set_prefetch(int(sys.argv[1]))
bench.init_tensors(eng)
eng.bind_step(torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda"))
for _ in range(4):
    rep = eng.run()
print("pf", sys.argv[1], "ms", rep.elapsed_ms)
