"""Per-operator device trace of a batched (C3-shaped) program: for each
operator, when its jobs became ready and finished across the SMs, and the
busy time per SM (sum of job durations / SMs)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ppj = int(sys.argv[3]) if len(sys.argv) > 3 else 16
slots = int(sys.argv[4]) if len(sys.argv) > 4 else 8
ctxs = bench.c3_contexts(B)
pages = [(c + 63) // 64 for c in ctxs]
req = {"engine": "ring", "ring_slots": slots, "model": {"preset": "llama3-8b", "layers": layers},
       "layout": {"batch": B, "req_pages": pages, "pages_per_job": ppj, "gu_block": 128, "page_rows": 64},
       "profile": {"builtin": "b200"}}
prog = Program.build(req)
eng = Engine(prog, watchdog_ms=20000)
bench.init_tensors(eng)
info = eng.info
st = [0] * int(info["step_scalars"])
for b in range(B):
    st[3 * b: 3 * b + 3] = [17 + b, ctxs[b] - 1, ctxs[b]]
bi = info["batch"]
st[bi["page_table_off"]: bi["page_table_off"] + len(bi["page_table"])] = bi["page_table"]
eng.bind_step(torch.tensor(st, dtype=torch.int64, device="cuda"))
eng.enable_trace(2048)
for _ in range(3):
    rep = eng.run()
tr = eng.trace()
text = prog.text(False)
ops = {}
for core_name, s in text["streams"].items():
    if ".vcc0" not in core_name:
        continue
    sm = int(core_name[2:].split(".")[0])
    pc = 0
    for line in s.splitlines():
        if line.startswith("#"):
            continue
        op = int(line.rsplit("op=", 1)[1]) if "op=" in line else -1
        ops[(2 * sm + 1, pc)] = (op, line.split()[0])
        pc += 1
t0 = min(r[2] for r in tr)
rows = {}
for core, pc, te, trd, td in tr:
    op, name = ops.get((core, pc), (-1, "?"))
    rows.setdefault(op, []).append((core // 2, name, te - t0, trd - t0, td - t0))
print(f"layers={layers} B={B} ppj={ppj} kernel_ms={rep.elapsed_ms:.3f} waits={rep.wait_cycles}")
for op in sorted(rows):
    r = rows[op]
    te = np.array([x[2] for x in r]); trd = np.array([x[3] for x in r]); td = np.array([x[4] for x in r])
    busy = (td - te).sum() / 148 / 1e3
    wait = (trd - te).sum() / 148 / 1e3
    print(f"op {op:3d} {r[0][1]:13s} jobs={len(r):5d} start[min {te.min()/1e3:8.1f}] ready[med {np.median(trd)/1e3:8.1f}] "
          f"done[min {td.min()/1e3:8.1f} med {np.median(td)/1e3:8.1f} max {td.max()/1e3:8.1f}] us  busy/SM {busy:6.1f} (dep wait {wait:5.1f})")
# the latest SMs of each operator: their jobs (ready -> done, us)
if len(sys.argv) > 5 and sys.argv[5] == "late":
    for op in sorted(rows):
        r = rows[op]
        fin = {}
        for sm, name, te, trd, td in r:
            fin.setdefault(sm, []).append((te / 1e3, trd / 1e3, td / 1e3))
        late = sorted(fin, key=lambda s: max(x[2] for x in fin[s]))[-3:]
        print(f"op {op:3d} {r[0][1]:12s} latest SMs: " + "; ".join(
            f"sm{sm}: " + ", ".join(f"{a:.1f}/{b:.1f}->{c:.1f}" for a, b, c in fin[sm]) for sm in late))
