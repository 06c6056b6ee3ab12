"""Per-operator timeline of one decode step from the device trace."""
import sys, json, re, collections
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
req = bench.model_request(layers)
if len(sys.argv) > 2:
    req["layout"].update(json.loads(sys.argv[2]))
prog = Program.build(req)
txt = prog.text(False)
ops = [o["id"] for o in txt["graph"]["operators"]]
# (core name) -> pc -> op ordinal, for VCC streams
n, sms, vccs = prog.cores()
core_names = []
for sm in range(sms):
    core_names.append(f"sm{sm}.vmc")
    for v in range(vccs):
        core_names.append(f"sm{sm}.vcc{v}")
pc_op = {}
for ci, name in enumerate(core_names):
    if ".vcc" not in name or name not in txt["streams"]:
        continue
    lines = [l for l in txt["streams"][name].splitlines() if l and not l.startswith("#")]
    pc_op[ci] = [int(re.search(r"op=(\d+)", l).group(1)) for l in lines]
eng = Engine(prog, watchdog_ms=10000)
bench.init_tensors(eng)
step = torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
eng.bind_step(step)
eng.enable_trace(1024)
for _ in range(3):
    eng.run()
rep = eng.run()
tr = eng.trace()
t0 = min(r[2] for r in tr)
per = collections.defaultdict(list)
for core, pc, te, tp, td in tr:
    per[pc_op[core][pc]].append((te - t0, tp - t0, td - t0))
print(f"layers={layers} launch {rep.elapsed_ms:.3f} ms; per-op (us): first_enter  p50_pro  last_pro  first_done  p50_done  last_done  jobs")
for o in sorted(per):
    a = np.array(per[o]) / 1e3
    print(f"{o:3d} {ops[o]:10s} {a[:,0].min():9.1f} {np.median(a[:,1]):9.1f} {a[:,1].max():9.1f} {a[:,2].min():9.1f} {np.median(a[:,2]):9.1f} {a[:,2].max():9.1f} {len(a):5d}")
