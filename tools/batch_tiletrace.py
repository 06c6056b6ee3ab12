"""Per-tile timeline of one SM of a batched (C3-shaped) program: VMC issue ->
MMA issuer sees the tile -> MMAs committed, for the BGEMM tiles."""
import os, sys, ctypes
os.environ["VDC_RING_DEBUG"] = str((int(sys.argv[2]) if len(sys.argv) > 2 else 7) << 8 | 2)
sys.path.insert(0, '/root/repo')
import numpy as np, torch, bench
from paper_2605_03190_b200 import Program, lib
from paper_2605_03190_b200.engine import Engine
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 1
B = 32
ctxs = bench.c3_contexts(B)
pages = [(c + 63) // 64 for c in ctxs]
req = {"engine": "ring", "model": {"preset": "llama3-8b", "layers": layers},
       "layout": {"batch": B, "req_pages": pages, "pages_per_job": 16, "gu_block": 128, "page_rows": 64},
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
XT = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)[100000:160000].reshape(-1, 2)
a = np.frombuffer(buf, dtype=np.uint64)[:3 * 60000].reshape(-1, 3).astype(np.int64)
n = int((a[:, 0] > 0).sum())
a = a[:n]
t0 = a[:, 0].min()
ok = (a[:, 1] > 0) & (a[:, 2] > 0)
print(f"tiles={n} with issuer stamps={int(ok.sum())} kernel_ms={rep.elapsed_ms:.3f}")
b = a[ok] - t0
lat = b[:, 1] - b[:, 0]; hold = b[:, 2] - b[:, 1]
print("issue -> issuer sees tile (ns): p10 %d p50 %d p90 %d" % tuple(np.percentile(lat, [10, 50, 90])))
print("issuer hold (ns):                p10 %d p50 %d p90 %d" % tuple(np.percentile(hold, [10, 50, 90])))
iss = np.sort(a[:, 0] - t0)
g = np.diff(iss)
print("issue gaps (ns): p50 %d p90 %d p99 %d" % tuple(np.percentile(g, [50, 90, 99])))
seen = np.sort(b[:, 1]); gs = np.diff(seen)
print("issuer tile-to-tile gaps (ns): p10 %d p50 %d p90 %d" % tuple(np.percentile(gs, [10, 50, 90])))
# BGEMM tiles: those with activation-chunk stamps (tile_trace[100000 + 2g])
A = a - t0
xt = XT[:len(A)]
bg = ok & (xt[:, 1] > 0)
ib = np.where(bg)[0]
print("BGEMM tiles", len(ib))
if len(ib):
    X = xt[ib] - t0
    print("  W issue -> W landed/seen      p10/p50/p90", np.percentile(A[ib, 1] - A[ib, 0], [10, 50, 90]).astype(int))
    print("  loop top -> X chunk ready     p10/p50/p90", np.percentile(X[:, 1] - X[:, 0], [10, 50, 90]).astype(int))
    print("  X ready -> W seen             p10/p50/p90", np.percentile(A[ib, 1] - X[:, 1], [10, 50, 90]).astype(int))
    print("  W seen -> MMAs committed      p10/p50/p90", np.percentile(A[ib, 2] - A[ib, 1], [10, 50, 90]).astype(int))
    turn = [A[g + 8, 0] - A[g, 2] for g in ib if g + 8 < len(A) and A[g + 8, 0] > 0]
    print("  commit -> next issue in slot  p10/p50/p90", np.percentile(turn, [10, 50, 90]).astype(int))
    step = int(os.environ.get("TT_STEP", max(1, len(ib) // 40)))
    for g in ib[: int(os.environ.get("TT_FIRST", len(ib)))][::step]:
        print(g, "issue", A[g, 0], "loop top", xt[g, 0] - t0, "x ready", xt[g, 1] - t0, "W seen", A[g, 1], "commit", A[g, 2])
# BGEMM µop phases on this SM: entry, ready, prologue done, issue loop done,
# MMAs complete, epilogue done (us, relative to the first tile issue)
B = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)[200000:200000 + 16 * 2048].reshape(-1, 16)
print("BGEMM µops, us after entry: ready prologue loop mma | tmem-read arrived | epilogue-done")
for k, row in enumerate(B):
    if row[0] == 0:
        continue
    r = [round((x - row[0]) / 1e3, 2) if x else None for x in row]
    print(k, "entry", round((row[0] - B[0][0]) / 1e3, 2), r[1:5], "|", r[6], r[7], "|", r[5], "| ssq start/loaded", r[9], r[8])
    if k > 60:
        break
