"""Per-SM lateness of the single-request ring kernel (C2 shapes, N layers):
for every GEMV operator, each SM's finish time minus the operator's median
finish, over several runs. Answers whether operator tails come from the same
SMs every time (a static per-SM rate difference a calibrated split could
remove) or move around (runtime noise that only dynamic balancing removes)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 6
prog = Program.build(bench.model_request(layers))
eng = Engine(prog, watchdog_ms=10000)
bench.init_tensors(eng)
eng.bind_step(torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda"))
eng.enable_trace(64)
text = prog.text(False)
ops = {}
for core_name, st in text["streams"].items():
    if ".vcc0" not in core_name:
        continue
    sm = int(core_name[2:].split(".")[0])
    pc = 0
    for line in st.splitlines():
        if line.startswith("#"):
            continue
        ops[(sm, pc)] = (int(line.rsplit("op=", 1)[1]) if "op=" in line else -1, line.split()[0])
        pc += 1
for _ in range(3):
    eng.run()
late = []  # runs x ops x sms
names = None
for r in range(runs):
    rep = eng.run()
    tr = eng.trace()
    done, ready = {}, {}
    for core, pc, te, trd, td in tr:
        op, name = ops.get((core // 2, pc), (-1, "?"))
        if "GEMV" not in name:
            continue
        k = (op, core // 2)
        done[k] = max(done.get(k, 0), td)
        ready[k] = min(ready.get(k, 1 << 62), trd)
    opl = sorted({k[0] for k in done})
    M = np.full((len(opl), 148), np.nan)
    for i, op in enumerate(opl):
        v = np.array([done.get((op, s), np.nan) for s in range(148)], dtype=float)
        M[i] = (v - np.nanmedian(v)) / 1e3
    late.append(M)
    names = opl
L = np.array(late)  # runs x ops x sms
print(f"layers={layers} runs={runs} kernel_ms={rep.elapsed_ms:.3f}")
mean_sm = np.nanmean(L, axis=(0, 1))
print("per-op tail (max - median finish, us), mean over runs:",
      " ".join(f"{np.nanmean(np.nanmax(L[:, i], axis=1)):.2f}" for i in range(len(names))))
# repeatability: correlation of per-SM lateness between runs and between ops
a = np.nanmean(L[: runs // 2], axis=1)
b = np.nanmean(L[runs // 2:], axis=1)
print("corr(run halves, per-SM lateness averaged over ops): %.3f" % np.corrcoef(a.mean(0), b.mean(0))[0, 1])
o1 = np.nanmean(L[:, ::2], axis=(0, 1)); o2 = np.nanmean(L[:, 1::2], axis=(0, 1))
print("corr(even ops, odd ops): %.3f" % np.corrcoef(o1, o2)[0, 1])
order = np.argsort(mean_sm)
print("earliest SMs:", [(int(s), round(float(mean_sm[s]), 2)) for s in order[:8]])
print("latest SMs:", [(int(s), round(float(mean_sm[s]), 2)) for s in order[-12:]])
print("per-SM mean lateness (us), sm 0..147:")
print(" ".join(f"{x:.2f}" for x in mean_sm))
# per-op lateness of the latest SMs
for s in order[-6:]:
    print(f"sm {s}: " + " ".join(f"{x:5.2f}" for x in np.nanmean(L[:, :, s], axis=0)))
