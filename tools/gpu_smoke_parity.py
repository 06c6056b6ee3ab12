"""First GPU bring-up: every corpus program + tiny decode, device vs oracle."""
import sys, json, time, traceback
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import simulate
import corpus, harness

only = sys.argv[1:] 
results = []
cases = [(n, r) for n, r in corpus.cases() if not n.startswith('err_')]
cases.append(("tiny_decode_4sm", {"model": {"preset": "tiny"}, "layout": {"ctx_pages": 1, "max_ctx": 64, "job_rows": 16, "gu_block": 16}, "profile": {"builtin": "b200", "sm_count": 4}, "_step": [17, 16, 17]}))
cases.append(("tiny_decode_148sm", {"model": {"preset": "tiny"}, "layout": {"ctx_pages": 1, "max_ctx": 64, "job_rows": 16, "gu_block": 16}, "profile": {"builtin": "b200"}, "_step": [3, 40, 41]}))
for name, req in cases:
    if only and not any(o in name for o in only): continue
    step = req.pop('_step', None)
    try:
        prog = Program.build(req)
    except Exception as e:
        print(f"{name:28s} BUILD-FAIL {str(e)[:80]}"); continue
    t = prog.text(True)
    idx, ins, outs = harness.run_oracle(t, seed=5, step=step)
    if idx['returncode'] != 0:
        print(f"{name:28s} ORACLE {idx['stdout'][:80]}"); continue
    try:
        t0 = time.time()
        rep, host = simulate(prog, ins, step=step)
        bad = harness.compare(host, outs, 1e-4)
        print(f"{name:28s} status={rep.status} uops={rep.uops_executed}/{idx['uops']} ms={rep.elapsed_ms:.3f} bad={bad[:3]} {rep.message}", flush=True)
        results.append((name, rep.status == 0 and not bad))
    except Exception as e:
        print(f"{name:28s} EXC {e}", flush=True)
        results.append((name, 'shared memory' in str(e)))
print("PASS", sum(ok for _, ok in results), "/", len(results))
