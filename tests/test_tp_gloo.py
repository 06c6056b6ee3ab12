"""World-size-2 host-side tensor-parallel logic on CPU (gloo, 127.0.0.1):
each process builds its rank's ring program exactly as bench.py does under
torchrun, and the ranks agree on what the in-kernel allreduce needs: the
same symmetric tensors (name, shape), the same number of producer µops per
partial buffer (the readiness target every rank waits for is world x that),
disjoint weight shards whose union is the full model, and the max-over-ranks
timing reduction bench.py reports."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, batched=False):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2605_03190_b200 import Program
        if batched:  # batched decode (C4 / C5 shape), Qwen3 with QK-norm
            import batch_cases as bc
            req = bc.request({"preset": "qwen3-8b", "layers": 2, "vocab": 32768}, [3, 5, 2, 4, 1, 6, 2, 2], 4, None)
        else:
            req = bench.model_request(2)
        req["layout"]["tp_world"], req["layout"]["tp_rank"] = world, rank
        req["layout"]["argmax"] = True
        info = Program.build(req).info()
        sym = sorted((d["name"], tuple(d["shape"])) for d in info["descriptors"] if d.get("symmetric"))
        producers = {}
        for j in info["jobs"]:
            if j["flags"] & 0x100:
                producers[j["o"][0]] = producers.get(j["o"][0], 0) + 1
        ar_need = sorted({j["x"][2] for j in info["jobs"] if j["op"] == 0x2C})
        # fused sampling under TP: lm_head jobs exchange (max, global index) pairs;
        # their vocab base is the rank's first logit row
        vocab_rows = [d["shape"][0] for d in info["descriptors"] if d["name"] == "logits"] if not batched else \
            [d["shape"][1] for d in info["descriptors"] if d["name"] == "logits"]
        tpx = [j for j in info["jobs"] if j["flags"] & 0x10000]
        bases = sorted({j["o2"][1] for j in tpx}) if not batched else None
        mine = {"sym": sym, "producers": sorted(producers.values()), "ar_need": ar_need, "n_tpx": len(tpx),
                "bases": bases, "vocab_rows": vocab_rows,
                "slots": sorted({j["o"][1] for j in info["jobs"] if j["flags"] & 0x100})}
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        t = torch.tensor([float(rank + 1), 10.0 * (rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, allv, t.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batched", [False, True])
def test_two_rank_tp_programs_agree(batched):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, batched)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, allv, t in got:
        assert t == [2.0, 20.0]  # max over ranks (bench.py's timing reduction)
        r0, r1 = allv
        # o.part, d.part per layer + the sampling exchange head.amx
        assert r0["sym"] == r1["sym"] and len(r0["sym"]) == 2 * 2 + 1 and r0["sym"][-1][0] == "head.amx"
        assert r0["n_tpx"] == r1["n_tpx"] > 0
        if not batched:
            assert r0["bases"] == [0] and r1["bases"] == r0["vocab_rows"]
        assert r0["producers"] == r1["producers"]
        slot = 4096 * (16 if batched else 1)  # (npad x d) fp32 per rank slot when batched
        if not batched:
            assert r0["ar_need"] == r1["ar_need"] == [world * r0["producers"][0]]
        else:  # one publish per row block: d / 128 = 32 row blocks per producer
            assert r0["ar_need"] == r1["ar_need"] == [world * 32]
        assert r0["slots"] == [0] and r1["slots"] == [slot]  # each rank writes its own slot
