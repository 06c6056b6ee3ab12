#!/usr/bin/env python
"""Llama-3-8B bf16 decode on the B200 µop engine — the BASELINE.json metric.

One "step" = one decode step (B=1, 4K context) executed as one launch of the
persistent µop kernel over the full 32-layer program (2.06 M µops, 444
virtual cores). Prints ONE JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value      tokens/s with weights/KV/step block resident in HBM (K back-to-back launches)
e2e        tokens/s through the public API with host buffers: per step the step
           block (token id, position) is copied H2D from pinned memory, the engine
           is launched, the fp32 logits are copied D2H and the next token is picked
           on the host (greedy), i.e. a real serving loop
roofline   algorithmic bytes per step (bf16 weights once + KV read + KV append)
           / device time per step, against MEASURED_PEAKS.json hbm_gbs
N > 1      tensor parallel (Megatron split over the N GPUs, partial sums exchanged
           inside the persistent kernel over NVLink peer memory): value = tokens/s of
           the group (strong scaling), time = max over ranks; --parallel replicas
           runs N independent copies instead (weak scaling)
--impl reference   the CPU oracle (test-infrastructure restatement of the
           reference semantics, oracle/_ref/oracle_interp) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Llama-3-8B bf16 decode tokens/s (1/2/4/8 B200) + HBM GB/s fraction of peak"
CTX = 4096


def model_request(layers: int = 32, ctx: int = CTX, engine: str = "ring", ring_slots: int = 12,
                  pages_per_job: int = 4) -> dict:
    pages = (ctx + 63) // 64
    if engine == "ring":
        return {
            "engine": "ring", "ring_slots": ring_slots,
            "model": {"preset": "llama3-8b", "layers": layers},
            "layout": {"ctx_pages": pages, "max_ctx": pages * 64, "pages_per_job": pages_per_job, "gu_block": 4,
                       "argmax": True},
            "profile": {"builtin": "b200"},
        }
    return {
        "model": {"preset": "llama3-8b", "layers": layers},
        "layout": {"ctx_pages": pages, "max_ctx": pages * 64, "pages_per_job": 4, "job_rows": 16, "gu_block": 32,
                   "head_job_rows": 64},
        "profile": {"builtin": "b200"},
    }


def algorithmic_bytes(info: dict, ctx: int) -> dict:
    """bf16 weights read once + one embedding row + KV read over ctx + KV append."""
    w = kv_read = kv_write = 0
    for d in info["descriptors"]:
        if d["view_of"] >= 0:
            continue
        n = 1
        for s in d["shape"]:
            n *= s
        eb = {"f32": 4, "bf16": 2, "i64": 8}[d["dtype"]]
        name = d["name"]
        if name == "embed.table":
            w += d["shape"][-1] * eb
        elif name.endswith(".kc") or name.endswith(".vc"):
            hkv, _, hd = d["shape"]
            kv_read += hkv * ctx * hd * eb
            kv_write += hkv * hd * eb
        elif d["external"]:
            w += n * eb
    return {"weights": w, "kv_read": kv_read, "kv_write": kv_write, "total": w + kv_read + kv_write}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed regions."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.proc = None
        self.windows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        inside = [s for t, s in self.samples if any(a - 0.05 <= t <= b + 0.05 for a, b in self.windows)]
        use = inside or [s for _, s in self.samples]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in use:
            f = [x.strip() for x in s.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(use), "samples_in_timed_region": len(inside)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic():
    """dram read+write bytes per launch from the committed ncu capture, if any."""
    p = ROOT / "profiles" / "ncu_engine_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


# ---------------------------------------------------------------------------
# CPU oracle (reference arm and cpu_baseline)

def cpu_oracle_tokens_per_s(timeout_s: int = 240) -> dict:
    """Time the single-threaded CPU oracle on 1- and 2-layer programs of the
    same model and extrapolate to 32 layers: t = t1 + 31 * (t2 - t1)."""
    from paper_2605_03190_b200 import Program

    exe = ROOT / "oracle/_ref/oracle_interp"
    if not exe.exists():
        return {"value": None, "unavailable": "oracle/_ref/oracle_interp not built"}
    times = {}
    with tempfile.TemporaryDirectory() as d:
        for layers in (1, 2):
            prog = Program.build(model_request(layers, engine="reference"))
            pj = os.path.join(d, f"p{layers}.json")
            with open(pj, "w") as f:
                json.dump(prog.text(True), f)
            env = dict(os.environ, ORACLE_NO_DUMP="1")
            r = subprocess.run([str(exe), pj, d, "0", f"17,{CTX - 1},{CTX}"], capture_output=True, text=True,
                               env=env, timeout=timeout_s)
            idx = json.loads(Path(d, "index.json").read_text())
            if not idx.get("completed"):
                return {"value": None, "unavailable": "oracle did not complete: " + r.stdout[-200:]}
            times[layers] = float(idx["exec_seconds"])
    per_layer = max(times[2] - times[1], 1e-9)
    t_token = times[1] + 31 * per_layer
    return {"value": 1.0 / t_token, "unit": "tokens/s", "cores": 1, "kind": "port",
            "sample": (f"oracle_interp (scalar fp32 restatement, single thread) on the 1-layer ({times[1]:.2f} s) and "
                       f"2-layer ({times[2]:.2f} s) Llama-3-8B programs at ctx {CTX}; 32 layers extrapolated "
                       f"as t1 + 31*(t2-t1) = {t_token:.2f} s/token"),
            "cpu": _cpu_name(), "nproc": os.cpu_count()}


def dense_cpu_context(ctx: int, timeout_s: int = 120) -> dict:
    """BASELINE.md §3.2's optional context figure: a dense fp32 Llama-3-8B
    batch-1 decode step (32 layers + lm_head, ctx rows of KV) on every host
    core (oracle/_ref/dense_cpu, std::thread). Not the reference path and not
    the target; reported beside cpu_baseline only."""
    exe = ROOT / "oracle/_ref/dense_cpu"
    if not exe.exists():
        return {"value": None, "unavailable": "oracle/_ref/dense_cpu not built"}
    r = subprocess.run([str(exe), "32", str(ctx), "2"], capture_output=True, text=True, timeout=timeout_s)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    return {"value": out["tokens_per_s"], "unit": "tokens/s", "cores": out["threads"],
            "sample": (f"dense fp32 Llama-3-8B batch-1 decode, 32 layers + lm_head at ctx {ctx}, best of 2 steps, "
                       "one layer's weights reused for every layer (each step still streams 32 x 0.87 GB)")}


def _stream_stats(eng):
    try:  # (A/B runs may load an older library without the export)
        return eng.stream_stats()
    except Exception:
        return None


def _cpu_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------

def init_tensors(eng, rank: int = 0, tp: bool = False):
    """Synthetic inputs on the device from the reference synthesize_inputs
    stream (BASELINE §4: splitmix64 / unit_float keyed by seed ^ fnv1a(name),
    Engine.synthesize -> vdc_program_synthesize): weights scaled by
    1/sqrt(fan_in), norms ones, KV caches random, activations zero. Under TP
    the weight shards take per-rank seeds and the replicated tensors
    (embedding, norms) one seed; the symmetric exchange buffers are bound
    separately (bind_symmetric_tp)."""
    if not tp:
        return eng.synthesize(seed=0)
    rep = {d["name"]: 99 for d in eng.info["descriptors"] if d["name"] == "embed.table" or d["name"].endswith("norm")}
    return eng.synthesize(seed=100 + rank, skip_symmetric=True, seeds=rep)


def bind_symmetric_tp(eng, world: int, rank: int, local_rank: int):
    """TP exchange buffers: one symmetric allocation per symmetric tensor
    (128-byte counter header + W x D fp32 slots), peer-mapped over NVLink by
    torch symmetric memory; the engine stores partial sums into every rank's
    buffer and publishes on its header counter (in-kernel allreduce)."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    keep = []
    group = dist.group.WORLD.group_name
    if hasattr(symm_mem, "enable_symm_mem_for_group"):
        symm_mem.enable_symm_mem_for_group(group)
    for d in eng.info["descriptors"]:
        if not d.get("symmetric"):
            continue
        n = 32 + int(d["shape"][0]) * int(d["shape"][1])
        t = symm_mem.empty(n, dtype=torch.float32, device=f"cuda:{local_rank}")
        t.zero_()
        h = symm_mem.rendezvous(t, group)
        eng.bind_symmetric(d["name"], [int(p) for p in h.buffer_ptrs], world, rank)
        keep.append((t, h))
    torch.cuda.synchronize()
    dist.barrier()
    return keep


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    from paper_2605_03190_b200 import Program
    from paper_2605_03190_b200.engine import Engine

    torch.cuda.set_device(local_rank)
    tp = world > 1 and args.parallel == "tp"
    t_build = time.time()
    req = model_request(args.layers, args.ctx, args.engine, args.ring_slots, args.pages_per_job)
    R = max(1, args.resident)
    if R > 1:
        # resident decode: R steps per launch, the sampled token fed back on the
        # device; positions advance from ctx - 1 through warm-up and timed steps
        if args.steps % R:
            raise SystemExit("--steps must be a multiple of --resident")
        advance = args.warmup * R + args.steps
        pages = (args.ctx + advance + 63) // 64
        req["layout"].update(feedback=True, ctx_pages=pages, max_ctx=pages * 64)
    if tp:
        req["layout"]["tp_world"], req["layout"]["tp_rank"] = world, rank
        req["layout"]["tp_partials"] = args.tp_partials
    prog = Program.build(req)
    build_s = time.time() - t_build
    eng = Engine(prog, device=local_rank, watchdog_ms=10000)
    tens = init_tensors(eng, rank, tp)
    keep_sym = bind_symmetric_tp(eng, world, rank, local_rank) if tp else None
    info = eng.info
    # KV bytes at the mean context of the timed steps (resident decode advances it)
    ctx_mean = args.ctx + (args.warmup * R + (args.steps - 1) / 2.0 if R > 1 else 0)
    nbytes = algorithmic_bytes(info, int(round(ctx_mean)))
    step = torch.tensor([17, args.ctx - 1, args.ctx, 0, 0, 0, 0, 0], dtype=torch.int64, device=f"cuda:{local_rank}")
    eng.bind_step(step)
    stream = torch.cuda.Stream(device=local_rank)
    if R > 1:
        eng.set_steps(R)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            eng.launch(stream)
        rep = eng.wait()
    if not rep.completed:
        raise SystemExit(f"engine did not complete: {rep.message} stalled={rep.stalled}")
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)

    # ---- value: device-resident inputs, K back-to-back steps (resident: K / R
    # launches of R steps each)
    launches = args.steps // R
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(launches + 1)]
    barrier()
    w0 = time.time()
    with torch.cuda.stream(stream):
        ev[0].record(stream)
        for k in range(launches):
            eng.launch(stream)
            ev[k + 1].record(stream)
    stream.synchronize()
    w1 = time.time()
    barrier()
    sampler.mark(w0, w1)
    rep = eng.wait()
    per = [ev[k].elapsed_time(ev[k + 1]) / R for k in range(launches)]  # per decode step
    if R > 1:
        eng.set_steps(1)  # e2e: one step per launch, the host supplies every token
    total_ms = ev[0].elapsed_time(ev[-1])

    # ---- e2e: host loop through the public API (H2D step block; D2H of the
    # token sampled on the device: greedy argmax fused into lm_head, under TP
    # with the cross-rank (max, index) exchange inside the kernel)
    logits = tens["logits"]
    h_step = torch.zeros(8, dtype=torch.int64).pin_memory()
    n_logits = logits.numel()
    h_logits = torch.empty(n_logits, dtype=torch.float32).pin_memory()
    next_tok = tens.get("next_token")
    h_tok = torch.zeros(1, dtype=torch.int64).pin_memory()
    token = 17
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    w2 = time.time()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for k in range(args.steps):
            h_step[0], h_step[1], h_step[2] = token, args.ctx - 1, args.ctx
            step.copy_(h_step, non_blocking=True)
            eng.launch(stream)
            if next_tok is not None:  # (TP: the ranks exchanged their (max, index) pairs in the kernel)
                h_tok.copy_(next_tok, non_blocking=True)
                stream.synchronize()
                token = int(h_tok[0])
            else:
                h_logits.copy_(logits, non_blocking=True)
                stream.synchronize()
                token = int(torch.argmax(h_logits))
        e1.record(stream)
    stream.synchronize()
    w3 = time.time()
    barrier()
    sampler.mark(w2, w3)
    e2e_ms = e0.elapsed_time(e1)
    clocks = sampler.stop()

    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms, e2e_ms], device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0]), float(t[1])

    ms_per_step = total_ms / args.steps
    # TP: the group decodes one token per step; replicas: one token per GPU per step
    tokens_per_step = 1 if tp else world
    value = tokens_per_step * args.steps / (total_ms / 1e3)
    e2e_value = tokens_per_step * args.steps / (e2e_ms / 1e3)
    peak, peak_src = measured_peak()
    kernel_ms = sorted(per)[len(per) // 2]
    achieved = nbytes["total"] / (sum(per) / len(per) / 1e3) / 1e9  # this rank's bytes (its shard) per GPU
    parallelism = "1 GPU" if world == 1 else (f"tp{world} (Megatron split, in-kernel NVLink allreduce)" if tp
                                               else f"{world} independent replicas")
    result = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "strong" if tp else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: reference synthesize_inputs stream (splitmix64/unit_float, generated on the device) for the Llama-3-8B weights (scaled 1/sqrt(fan_in)) and the bf16 KV cache, greedy token feedback in e2e",
        "config": {"workload": f"C2 Llama-3-8B bf16 decode, batch 1, ctx {args.ctx}, {args.layers} layers + lm_head",
                   "model": "llama3-8b", "batch": 1, "ctx": args.ctx, "parallelism": parallelism,
                   "l2": "inputs larger than L2 (algorithmic %.2f GB per step vs 126 MB L2)" % (nbytes["total"] / 1e9),
                   "program_uops": info["total_uops"], "virtual_cores": prog.cores()[0], "build_seconds": round(build_s, 2),
                   "memory_core_streams": _stream_stats(eng),
                   "resident_steps_per_launch": R,
                   **({"ctx_mean_timed": round(ctx_mean, 1)} if R > 1 else {})},
        "e2e": {"value": round(e2e_value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 8 * 8,
                "d2h_bytes_per_step": 8 if next_tok is not None else n_logits * 4,
                "sampling": ("greedy argmax fused into the lm_head epilogue (device"
                             + (", cross-rank (max, index) exchange over NVLink)" if tp else ")"))
                            if next_tok is not None else "host argmax over D2H logits"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": committed_traffic() if world == 1 else None,
                     "peak_source": peak_src, "frac_of_8TBps_spec": round(achieved / 8000.0, 4),
                     "bytes_per_step": nbytes, "per_gpu": True,
                     "kernel": ("vdc_dev::ring::ring_kernel" if args.engine == "ring" else "vdc_dev::engine_kernel") + " (persistent, 1 CTA/SM)",
                     "kernel_ms_median": round(kernel_ms, 4)},
        "clocks": clocks,
        "engine_report": {"engine": args.engine, "uops_executed": rep.uops_executed, "bytes_loaded": rep.bytes_loaded,
                          "wait_cycles_sum_over_sms": rep.wait_cycles,
                          "bytes_stored": rep.bytes_stored},
    }
    del keep_sym
    return result


# ---------------------------------------------------------------------------
# C3: batched decode (B requests, per-request contexts, paged KV)

MASK64 = (1 << 64) - 1


def splitmix64_stream(seed: int):
    state = seed & MASK64
    while True:
        state = (state + 0x9E3779B97F4A7C15) & MASK64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        yield z ^ (z >> 31)


def c3_contexts(batch: int, lo: int = 128, hi: int = 8192, seed: int = 1) -> list:
    """ctx_r = splitmix64(seed 1) -> U[128, 8192]"""
    g = splitmix64_stream(seed)
    return [lo + next(g) % (hi - lo + 1) for _ in range(batch)]


def run_batched(args, rank: int = 0, world: int = 1, local_rank: int = 0):
    """C3 (1 GPU) / C4-C5 shaped (tensor parallel under torchrun) batched decode"""
    import torch
    from paper_2605_03190_b200 import Program
    from paper_2605_03190_b200.engine import Engine

    torch.cuda.set_device(local_rank)
    tp = world > 1
    B = args.batch
    if args.ctx_fixed:
        ctxs = [args.ctx_fixed] * B
    else:
        ctxs = c3_contexts(B)
    pages = [(c + 63) // 64 for c in ctxs]
    t_build = time.time()
    model = {"preset": args.model, "layers": args.layers}
    if args.no_qk_norm:  # ablation: the same shapes without Qwen3's QK-norm
        model["qk_norm"] = False
    req = {"engine": "ring", "model": model,
           "layout": {"batch": B, "req_pages": pages, "pages_per_job": args.pages_per_job, "gu_block": 128, "page_rows": 64,
                      **({"attn_job_cost": args.attn_job_cost} if args.attn_job_cost >= 0 else {}),
                      "argmax": True},
           "profile": {"builtin": "b200"}}
    if tp:
        req["layout"]["tp_world"], req["layout"]["tp_rank"] = world, rank
        req["layout"]["tp_partials"] = args.tp_partials
    prog = Program.build(req)
    build_s = time.time() - t_build
    eng = Engine(prog, device=local_rank, watchdog_ms=20000)
    tens = init_tensors(eng, rank, tp)
    keep_sym = bind_symmetric_tp(eng, world, rank, local_rank) if tp else None
    info = eng.info
    bi = info["batch"]
    st_host = [0] * int(info["step_scalars"])
    for b in range(B):
        st_host[3 * b: 3 * b + 3] = [17 + b, ctxs[b] - 1, ctxs[b]]
    st_host[bi["page_table_off"]: bi["page_table_off"] + len(bi["page_table"])] = bi["page_table"]
    step = torch.tensor(st_host, dtype=torch.int64, device=f"cuda:{local_rank}")
    eng.bind_step(step)
    stream = torch.cuda.Stream(device=local_rank)

    def barrier():
        if tp:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # algorithmic bytes: bf16 weights once + one embedding row per request + each
    # request's K/V rows over its context + the appended rows
    w = kvr = kvw = 0
    layers = args.layers
    for d in info["descriptors"]:
        if d["view_of"] >= 0 or not (d["external"] or d["state"]):
            continue
        n = 1
        for x in d["shape"]:
            n *= x
        if d["name"] == "embed.table":
            w += B * d["shape"][-1] * 2
        elif d["name"].endswith(".kc") or d["name"].endswith(".vc"):
            hkv, hd = d["shape"][1] // 64, d["shape"][2]
            kvr += sum(ctxs) * hkv * hd * 2
            kvw += B * hkv * hd * 2
        elif d["dtype"] == "bf16" and d["name"] != "ring.pad":
            w += n * 2
    nbytes = {"weights": w, "kv_read": kvr, "kv_write": kvw, "total": w + kvr + kvw}

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            eng.launch(stream)
        rep = eng.wait()
    if not rep.completed:
        raise SystemExit(f"engine did not complete: {rep.message} stalled={rep.stalled}")
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    w0 = time.time()
    with torch.cuda.stream(stream):
        ev[0].record(stream)
        for k in range(args.steps):
            eng.launch(stream)
            ev[k + 1].record(stream)
    stream.synchronize()
    sampler.mark(w0, time.time())
    rep = eng.wait()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])

    # e2e: per step the request triples (token, pos, ctx) go H2D from pinned
    # memory, the engine runs (greedy sampling fused into the lm_head GEMM)
    # and the B sampled tokens come back D2H; under TP the ranks exchanged
    # their (max, index) pairs in the kernel, so every rank holds the same tokens
    next_tok = tens["next_token"]
    h_trip = torch.tensor(st_host[: 3 * B], dtype=torch.int64).pin_memory()
    h_tok = torch.zeros(B, dtype=torch.int64).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    w2 = time.time()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for k in range(args.steps):
            step[: 3 * B].copy_(h_trip, non_blocking=True)
            eng.launch(stream)
            # greedy sampling fused into the lm_head GEMM (TP: cross-rank (max,
            # index) exchange in the kernel, every rank holds the same tokens)
            h_tok.copy_(next_tok.view(-1), non_blocking=True)
            stream.synchronize()
            h_trip.view(B, 3)[:, 0] = h_tok
        e1.record(stream)
    stream.synchronize()
    sampler.mark(w2, time.time())
    e2e_ms = e0.elapsed_time(e1)
    clocks = sampler.stop()
    if tp:
        import torch.distributed as dist
        t = torch.tensor([total_ms, e2e_ms], device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0]), float(t[1])
    del keep_sym
    value = B * args.steps / (total_ms / 1e3)
    peak, peak_src = measured_peak()
    achieved = nbytes["total"] / (sum(per) / len(per) / 1e3) / 1e9
    name = {"llama3-8b": "Llama-3-8B", "qwen3-8b": "Qwen3-8B", "llama3-70b": "Llama-3-70B"}.get(args.model, args.model)
    cfg_name = "C3" if (args.model == "llama3-8b" and not tp) else "C4" if args.model == "qwen3-8b" else "C5" if args.model == "llama3-70b" else "batched"
    return {
        "metric": f"{name} bf16 batched decode tokens/s ({cfg_name}: batch {B}, paged KV) + HBM GB/s fraction of peak",
        "value": round(value, 2), "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True, "scaling": "strong" if tp else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": f"synthetic: reference synthesize_inputs stream (splitmix64/unit_float, on the device) for the {name} weights and bf16 KV pages, contexts "
                + (f"fixed {args.ctx_fixed}" if args.ctx_fixed else "splitmix64(seed 1) -> U[128, 8192]"),
        "config": {"workload": f"{cfg_name} {name} bf16 decode, batch {B}, per-request contexts (sum {sum(ctxs)}), "
                               f"paged KV (64-row pages, {sum(pages)} pages), {layers} layers + lm_head",
                   "model": args.model, "batch": B, "contexts": ctxs,
                   "parallelism": f"tp{world} (Megatron split, in-kernel NVLink allreduce)" if tp else "1 GPU",
                   "l2": "inputs larger than L2 (algorithmic %.2f GB per step vs 126 MB L2)" % (nbytes["total"] / 1e9),
                   "program_uops": info["total_uops"], "build_seconds": round(build_s, 2),
                   "memory_core_streams": _stream_stats(eng)},
        "e2e": {"value": round(B * args.steps / (e2e_ms / 1e3), 2), "unit": "tokens/s", "h2d_bytes_per_step": 3 * B * 8,
                "d2h_bytes_per_step": B * 8,
                "sampling": "greedy argmax fused into the lm_head GEMM (device" + (
                    ", cross-rank (max, index) exchange over NVLink)" if tp else ")")},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                     "bytes_per_step": nbytes, "kernel": "vdc_dev::ring::ring_kernel<true> (persistent, 1 CTA/SM)",
                     "kernel_ms_median": round(sorted(per)[len(per) // 2], 4)},
        "clocks": clocks,
        "engine_report": {"uops_executed": rep.uops_executed, "bytes_loaded": rep.bytes_loaded,
                          "wait_cycles_sum_over_sms": rep.wait_cycles},
    }


def self_launch(n: int, impl: str) -> int:
    """Re-exec this command under torch.distributed.run with N ranks on this
    node (127.0.0.1 rendezvous, a free port); returns the launcher's exit code."""
    import socket

    if impl == "ours":  # (the reference arm: rank 0 works on the host, the others exit at once)
        import torch

        have = torch.cuda.device_count()
        if have < n:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {n} requested, {have} GPUs visible"}))
            return 1
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    print(f"bench.py: launching {n} ranks: {' '.join(cmd)}", file=sys.stderr)
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=CTX)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tp-partials", default="f32", choices=["f32", "bf16"],
                    help="TP exchange partials: bf16 halves the NVLink bytes of the in-kernel allreduce")
    ap.add_argument("--engine", default="ring", choices=["ring", "reference"])
    ap.add_argument("--ring-slots", type=int, default=12)
    ap.add_argument("--pages-per-job", type=int, default=None,
                    help="split-KV granularity (default 4 at batch 1, 128 for batched decode)")
    ap.add_argument("--model", default="llama3-8b", choices=["llama3-8b", "qwen3-8b", "llama3-70b"],
                    help="batched decode: model preset (C3 llama3-8b, C4 qwen3-8b, C5 llama3-70b)")
    ap.add_argument("--no-qk-norm", action="store_true", help="ablation: Qwen3 shapes without QK-norm")
    ap.add_argument("--ctx-fixed", type=int, default=0, help="batched decode: every request at this context (C4 4096, C5 8192)")
    ap.add_argument("--batch", type=int, default=1,
                    help="> 1: C3 batched decode (per-request contexts, paged KV, BGEMM on tcgen05); 1 GPU")
    ap.add_argument("--attn-job-cost", type=int, default=-1,
                    help="batched decode: fixed cost of a split-KV job in ring tiles for the attention load balance")
    ap.add_argument("--resident", type=int, default=1,
                    help="batch-1 decode: decode steps per launch of the persistent kernel (device-side "
                         "token feedback, vdc_set_steps); --steps must be a multiple")
    ap.add_argument("--parallel", default="tp", choices=["tp", "replicas"],
                    help="N>1: tensor parallel over the N GPUs (default) or N independent replicas")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` outside torchrun: re-launch as N ranks (one
        # process per GPU) exactly the way the driver does; rank 0 prints the line
        raise SystemExit(self_launch(args.gpus, args.impl))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    local_rank = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        if rank != 0:
            return
        t0 = time.time()
        cb = cpu_oracle_tokens_per_s()
        line = {"metric": METRIC, "impl": "reference", "value": cb.get("value"), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference RNG: splitmix64/unit_float)",
                "config": {"workload": f"C2 Llama-3-8B decode, batch 1, ctx {CTX} (sampled: 1- and 2-layer programs, extrapolated)",
                           "model": "llama3-8b", "batch": 1, "ctx": CTX},
                "cpu_baseline": cb, "wall_seconds": round(time.time() - t0, 1)}
        if cb.get("value") is None:
            line = {"impl": "reference", "unavailable": cb.get("unavailable", "oracle failed")}
        else:
            line["e2e"] = {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
        print(json.dumps(line))
        return

    if args.pages_per_job is None:
        # batched: one split-KV job per (request, kv head) up to 128 pages (8K
        # context); measured C3 3090 / 3115 / 3113 tok/s at 64 / 96 / 128
        args.pages_per_job = 128 if args.batch > 1 else 4
    if args.batch > 1:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        res = run_batched(args, rank, world, local_rank)
        if rank == 0:
            print(json.dumps(res))
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    result = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            try:
                result["cpu_baseline"] = cpu_oracle_tokens_per_s()
            except Exception as e:  # the baseline is reported, never the target
                result["cpu_baseline"] = {"value": None, "unavailable": str(e)[:200]}
            if args.batch == 1 and args.model == "llama3-8b":
                try:
                    result["cpu_baseline"]["dense_fp32_all_cores"] = dense_cpu_context(args.ctx)
                except Exception as e:
                    result["cpu_baseline"]["dense_fp32_all_cores"] = {"value": None, "unavailable": str(e)[:200]}
        print(json.dumps(result))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
