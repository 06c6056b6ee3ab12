"""Attention job phases on one SM of a C3-shaped batched program (debug tile
trace, VDC_RING_DEBUG = sm << 8 | 2): per ATTN_DECODE job entry, readiness,
page loop done, merge done (astamp events 0/1/3/4, first 8 jobs of the SM),
and the per-tile issue / landed / released times of the SM's ring."""
import os, sys, ctypes
SM = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ppj = int(sys.argv[2]) if len(sys.argv) > 2 else 64
os.environ["VDC_RING_DEBUG"] = str(SM << 8 | 2)
sys.path.insert(0, '/root/repo')
import numpy as np, torch, bench
from paper_2605_03190_b200 import Program, lib
from paper_2605_03190_b200.engine import Engine
B = 32
ctxs = bench.c3_contexts(B)
pages = [(c + 63) // 64 for c in ctxs]
req = {"engine": "ring", "model": {"preset": "llama3-8b", "layers": 1},
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
for _ in range(3):
    rep = eng.run()
buf = (ctypes.c_uint64 * (4 * 65536))()
L = lib(); L.vdc_debug_tile_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32]
assert L.vdc_debug_tile_trace(eng._h, buf, 4 * 65536) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
T = a[:3 * 20000].reshape(-1, 3)
n = int((T[:, 0] > 0).sum())
t0 = T[:n, 0].min()
S = a[60000:60064].reshape(8, 8)
text = prog.text(False)["streams"][f"sm{SM}.vcc0"].splitlines()
print(f"sm {SM} ppj {ppj} kernel_ms {rep.elapsed_ms:.3f}; stream: " + " | ".join(l.split()[0] + " " + " ".join(f for f in l.split() if f.startswith(("size=", "imm="))) for l in text if not l.startswith("#"))[:600])
for k in range(8):
    if S[k, 0] == 0:
        continue
    e = (S[k] - t0) / 1e3
    print(f"attn job {k}: entry {e[0]:8.2f} ready {e[1]:8.2f} q staged {e[2]:8.2f} pages done {e[3]:8.2f} merged {e[4]:8.2f} "
          f"arrived {e[5]:8.2f} end {e[6]:8.2f} us")
# tiles: issue, landed (seen by the consumer), released
R = (T[:n] - t0) / 1e3
lat = R[:, 1] - R[:, 0]
print("tiles", n, "issue->landed p10/50/90 (us)", np.percentile(lat[R[:, 1] > 0], [10, 50, 90]).round(2))
for g in range(0, n, max(1, n // 60)):
    print(f"tile {g:5d} issue {R[g,0]:8.2f} seen {R[g,1]:8.2f} released {R[g,2]:8.2f}")
