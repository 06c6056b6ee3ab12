"""GPU bring-up of the ring engine: tiny (f32) and mid (bf16) decode vs the dense reference."""
import sys, time, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from paper_2605_03190_b200 import Program
from paper_2605_03190_b200.engine import simulate
import ring_cases as rc

for name, base, sms in [("tiny4", rc.TINY, 4), ("tiny", rc.TINY, None), ("mid", rc.MID, None)]:
    req = rc.request(base, sms)
    prog = Program.build(req)
    info = prog.info()
    ins = rc.synth_inputs(info)
    for token, pos in [(17, 40 if base is rc.TINY else 300), (3, 0)]:
        t0 = time.time()
        rep, host = simulate(prog, ins, step=[token, pos, pos + 1])
        print(name, token, pos, "status", rep.status, rep.message, "ms", round(rep.elapsed_ms, 3), flush=True)
        if rep.status == 0:
            print("   ", rc.check_against_dense(info, req, ins, host, token, pos), flush=True)
