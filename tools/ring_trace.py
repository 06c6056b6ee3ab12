"""Per-job device trace of the ring engine (N-layer Llama-3-8B program):
per operator, the spread of SM start/ready/finish times."""
import sys, json
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prog = Program.build(bench.model_request(layers))
eng = Engine(prog, watchdog_ms=10000)
bench.init_tensors(eng)
step = torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
eng.bind_step(step)
eng.enable_trace(64)
for _ in range(3):
    rep = eng.run()
tr = eng.trace()
text = prog.text(False)
info = eng.info
# op ordinal of each (core, pc) from the stream text
ops = {}
for core_name, st in text["streams"].items():
    if ".vcc0" not in core_name:
        continue
    sm = int(core_name[2:].split(".")[0])
    pc = 0
    for line in st.splitlines():
        if line.startswith("#"):
            continue
        op = int(line.rsplit("op=", 1)[1]) if "op=" in line else -1
        ops[(2 * sm + 1, pc)] = (op, line.split()[0])
        pc += 1
t0 = min(r[2] for r in tr)
rows = {}
for core, pc, te, tr_, td in tr:
    op, name = ops.get((core, pc), (-1, "?"))
    rows.setdefault(op, []).append((core // 2, name, te - t0, tr_ - t0, td - t0))
print(f"layers={layers} kernel_ms={rep.elapsed_ms:.3f}")
prev_end = 0
for op in sorted(rows):
    r = rows[op]
    te = np.array([x[2] for x in r]); trd = np.array([x[3] for x in r]); td = np.array([x[4] for x in r])
    print(f"op {op:3d} {r[0][1]:13s} jobs={len(r):4d} ready[min {trd.min()/1e3:8.2f} med {np.median(trd)/1e3:8.2f} max {trd.max()/1e3:8.2f}] "
          f"done[min {td.min()/1e3:8.2f} med {np.median(td)/1e3:8.2f} max {td.max()/1e3:8.2f}] us  span {(td.max()-trd.min())/1e3:7.2f}")
