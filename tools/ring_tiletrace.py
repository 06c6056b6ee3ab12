"""Per-tile timeline of one SM (VMC issue -> compute sees full -> release)."""
import os, sys, ctypes
os.environ["VDC_RING_DEBUG"] = str((int(sys.argv[2]) if len(sys.argv) > 2 else 7) << 8 | 2 | (int(sys.argv[3]) if len(sys.argv) > 3 else 0))
sys.path.insert(0, '/root/repo')
import numpy as np, torch, bench
from paper_2605_03190_b200 import Program, lib
from paper_2605_03190_b200.engine import Engine
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prog = Program.build(bench.model_request(layers))
eng = Engine(prog, watchdog_ms=10000)
bench.init_tensors(eng)
step = torch.tensor([17, 4095, 4096, 0, 0, 0, 0, 0], dtype=torch.int64, device="cuda")
eng.bind_step(step)
for _ in range(3):
    rep = eng.run()
buf = (ctypes.c_uint64 * (3 * 65536))()
L = lib(); L.vdc_debug_tile_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32]
assert L.vdc_debug_tile_trace(eng._h, buf, 65536) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 3).astype(np.int64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
a = a - t0
iss, full, rel = a[:, 0], a[:, 1], a[:, 2]
ok = (full > 0) & (rel > 0)
lat = (full - iss)[ok]; hold = (rel - full)[ok]
print(f"tiles={len(a)} kernel_ms={rep.elapsed_ms:.3f}")
print("issue->compute-start (ns): p10 %d p50 %d p90 %d" % tuple(np.percentile(lat, [10, 50, 90])))
print("compute hold (ns):        p10 %d p50 %d p90 %d" % tuple(np.percentile(hold, [10, 50, 90])))
gaps = np.diff(np.sort(iss))
print("issue gaps (ns): p50 %d p90 %d p99 %d max %d" % tuple(np.percentile(gaps, [50, 90, 99, 100])))
for i in range(0, min(len(a), 400), 8):
    print(i, [(int(x[0]) // 100, int(x[1]) // 100, int(x[2]) // 100) for x in a[i:i + 8]])
ev = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 3).astype(np.int64).reshape(-1)[60000:60000 + 64].reshape(8, 8)
print("attention job stamps on this SM (us, rel. to tile0 issue): enter, ready, q staged, pages done, merged, arrived, [combined, published]")
for row in ev:
    if row[0]:
        print([round((x - t0) / 1e3, 2) if x else None for x in row])
# tiles consumed by the attention of layer 1 (between the stamps' ready and pages-done)
lo, hi = ev[1][1], ev[1][3]
sel = [(i, (int(x[0]) - 0) / 1e3, (int(x[1])) / 1e3, (int(x[2])) / 1e3) for i, x in enumerate(a) if x[1] > 0 and lo - t0 - 20000 <= x[1] <= hi - t0 + 2000]
print("tiles around layer-1 attention (idx, issue, full, release) us:")
for r in sel[:60]:
    print(r)
