"""Batched attention cost model probe: per ATTN_DECODE job of a C3-shaped
2-layer program, (sm, pages, t_ready, t_done) from the device trace; fits
job duration = a + b * pages and prints the per-SM finish spread."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import bench
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import Engine

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ppj = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ctxs = bench.c3_contexts(B)
pages = [(c + 63) // 64 for c in ctxs]
req = {"engine": "ring", "model": {"preset": "llama3-8b", "layers": 2},
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
jobs = info["jobs"]
meta = {}
for core_name, s in text["streams"].items():
    if ".vcc0" not in core_name:
        continue
    sm = int(core_name[2:].split(".")[0])
    pc = 0
    for line in s.splitlines():
        if line.startswith("#"):
            continue
        op = int(line.rsplit("op=", 1)[1]) if "op=" in line else -1
        imm = None
        for f in line.split():
            if f.startswith("imm="):
                imm = int(f[4:])
        meta[(2 * sm + 1, pc)] = (op, line.split()[0], imm)
        pc += 1
t0 = min(r[2] for r in tr)
A = []
for core, pc, te, trd, td in tr:
    op, name, imm = meta.get((core, pc), (-1, "?", None))
    if name == "ATTN_DECODE" and op == 2 and imm is not None:
        j = jobs[imm]
        A.append((core // 2, j["r1"] - j["r0"], (te - t0) / 1e3, (trd - t0) / 1e3, (td - t0) / 1e3))
A = np.array(A)
dur = A[:, 4] - A[:, 3]
X = np.stack([np.ones(len(A)), A[:, 1]], 1)
coef, *_ = np.linalg.lstsq(X, dur, rcond=None)
print(f"B={B} ppj={ppj} kernel_ms={rep.elapsed_ms:.3f} jobs={len(A)}: duration = {coef[0]:.2f} us + {coef[1]:.3f} us/page "
      f"(pages min {A[:,1].min():.0f} max {A[:,1].max():.0f})")
fin = {}
tot = {}
for sm, pg, te, trd, td in A:
    fin[sm] = max(fin.get(sm, 0), td)
    tot[sm] = tot.get(sm, 0) + pg
f = np.array(list(fin.values()))
print(f"per-SM attention finish: min {f.min():.1f} med {np.median(f):.1f} max {f.max():.1f} us; pages/SM min {min(tot.values())} max {max(tot.values())}")
for sm in sorted(fin, key=lambda s: fin[s])[-5:]:
    js = A[A[:, 0] == sm]
    print(f"  sm {int(sm)} finish {fin[sm]:.1f}: jobs " + ", ".join(f"{int(p)}p {r:.0f}->{d:.0f}" for _, p, _, r, d in js))
