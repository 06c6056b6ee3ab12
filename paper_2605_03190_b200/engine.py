"""Device executor: the reference's `machine::Machine` shape over the C-ABI.

reference include/uopsim/machine.hpp:94-126      this module
  Machine(p, hw, inputs, opt)                     Engine(program, device) + bind()/bind_inputs()
  Machine::run(watchdog) -> ExecutionReport       Engine.run() -> Report (status, uops, bytes, ms)
  simulate(p, hw, opt, watchdog)                  simulate(program, inputs)
Deadlock is a report status (VDC_ERR_DEADLOCK), not an exception, exactly
like the reference's Termination::deadlock. Device memory is owned by the
caller (torch tensors); there is no CPU execution path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from ._native import (DTYPE, VDC_ERR_DEADLOCK, VDC_OK, Program, VdcError, check, lib, vdc_profile, vdc_report)


@dataclass
class Report:
    status: int
    uops_executed: int
    bytes_loaded: int
    bytes_stored: int
    elapsed_ms: float
    message: str
    stalled: list = field(default_factory=list)
    wait_cycles: dict = field(default_factory=dict)
    queues_drained: bool = True   # measured on the device at the end of the launch
    slots_all_free: bool = True

    @property
    def completed(self) -> bool:
        return self.status == VDC_OK


def _torch():
    import torch  # PyTorch is the device-memory/stream plumbing, not the compute path

    return torch


WAIT_SITES = ["cfu_alloc", "cfu_m2c", "cfu_unit", "ldu_idle", "ldu_dep", "stu_idle", "stu_c2m", "stu_dep",
              "vcc_ready", "vcc_barrier", "vcc_c2m", "vcc_compute", "cfu_total", "vcc_total", "ldu_issue", "cfu_resolve",
              "vcc_sync", "vcc_push", "vcc_prologue", "vcc_epilogue", "vcc_pop", "cfu_allocloop", "cfu_synckick", "cfu_dispatch"]

RING_SITES = ["vmc_empty_wait", "vcc_full_wait", "vcc_dep_wait", "vcc_epilogue", "vcc_total", "vmc_total", "jobs",
              "bgemm_xchunk_wait", "bgemm_xbuffer_wait", "bgemm_mma_wait", "bgemm_prologue"]

TORCH_DTYPE = {"f32": "float32", "bf16": "bfloat16", "i64": "int64"}


PACKED_SW128 = 0x80000000  # ring_abi.h VDC_DESC_PACKED_SW128
KPAGE_SWZ = 0x40000000     # ring_abi.h VDC_DESC_KPAGE_SWZ


def to_logical(d: dict, a: np.ndarray) -> np.ndarray:
    """device storage order -> row-major (packed weights and swizzled KV pages undone)"""
    if d.get("tma") == PACKED_SW128:
        return unpack_sw128(a, *d["shape"])
    if d.get("tma") == KPAGE_SWZ:
        return unswizzle_k(a.reshape(-1, 64, d["shape"][-1])).reshape(a.shape)
    return a


def to_storage(d: dict, a: np.ndarray) -> np.ndarray:
    """row-major host array -> the descriptor's device storage order"""
    if d.get("tma") == PACKED_SW128:
        return pack_sw128(a, *d["shape"])
    if d.get("tma") == KPAGE_SWZ:
        return swizzle_k(a.reshape(-1, 64, d["shape"][-1])).reshape(a.shape)
    return a


def _k_chunk_map(rows: int, hd: int) -> np.ndarray:
    """physical 16-byte chunk of logical chunk c in page row r: (c & 8) | ((c & 7) ^ (r & 7))"""
    r = np.arange(rows)[:, None]
    c = np.arange(hd // 8)[None, :]
    return (c & 8) | ((c & 7) ^ (r & 7))


def swizzle_k(pool: np.ndarray) -> np.ndarray:
    """(..., 64, hd) row-major K/V page rows -> the swizzled storage of batched
    KV pools (ring_abi.h VDC_DESC_KPAGE_SWZ)."""
    rows, hd = pool.shape[-2], pool.shape[-1]
    pc = _k_chunk_map(rows, hd)
    x = pool.reshape(pool.shape[:-1] + (hd // 8, 8))
    out = np.empty_like(x)
    out[..., np.arange(rows)[:, None], pc, :] = x
    return out.reshape(pool.shape)


def unswizzle_k(pool: np.ndarray) -> np.ndarray:
    """inverse of swizzle_k: swizzled K/V page rows -> logical order"""
    rows, hd = pool.shape[-2], pool.shape[-1]
    pc = _k_chunk_map(rows, hd)
    x = pool.reshape(pool.shape[:-1] + (hd // 8, 8))
    return np.ascontiguousarray(x[..., np.arange(rows)[:, None], pc, :]).reshape(pool.shape)


def pack_sw128(a: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """Row-major (rows, cols) -> packed 128 x 64 tiles, tile (rb, kt) at
    (rb * cols/64 + kt) * 8192 elements, 16-byte chunk c of tile row r stored
    at chunk c ^ (r % 8) (the 128-byte swizzle of the tcgen05 K-major operand)."""
    t = a.reshape(rows // 128, 128, cols // 64, 8, 8).transpose(0, 2, 1, 3, 4)  # rb, kt, r, c, e
    r = np.arange(128)[:, None]
    p = np.arange(8)[None, :]
    return np.ascontiguousarray(t[:, :, r, p ^ (r & 7), :]).reshape(-1)


def unpack_sw128(a: np.ndarray, rows: int, cols: int) -> np.ndarray:
    t = a.reshape(rows // 128, cols // 64, 128, 8, 8)  # rb, kt, r, p, e
    r = np.arange(128)[:, None]
    c = np.arange(8)[None, :]
    return np.ascontiguousarray(t[:, :, r, c ^ (r & 7), :].transpose(0, 2, 1, 3, 4)).reshape(-1)


# ring_abi.h vdc_run: one folded stretch of a memory-core stream
RUN_DTYPE = np.dtype([("base", "<u4", 4), ("count_alt", "<u4"), ("nin_talt", "<u4"), ("d_in", "i1", 3),
                      ("d_out", "i1", 3), ("rsv", "<u2")])
assert RUN_DTYPE.itemsize == 32


def fold_stream(words: bytes) -> np.ndarray:
    """fold a memory-core stream of LOAD words the way vdc_load_jobs does
    (vdc_fold_stream): the run entries, a RUN_DTYPE array"""
    import ctypes as c
    n = len(words) // 16
    runs = np.zeros(max(1, n), dtype=RUN_DTYPE)
    nr = c.c_uint32()
    check(lib().vdc_fold_stream(words, n, runs.ctypes.data, c.byref(nr)))
    return runs[:nr.value].copy()


def unfold_stream(runs: np.ndarray, capacity: int) -> bytes:
    """host expansion of run entries back to LOAD words (vdc_unfold_stream)"""
    import ctypes as c
    out = c.create_string_buffer(max(16, 16 * capacity))
    n = c.c_uint32()
    r = np.ascontiguousarray(runs, dtype=RUN_DTYPE)
    check(lib().vdc_unfold_stream(r.ctypes.data, len(r), out, capacity, c.byref(n)))
    return out.raw[:16 * n.value]


class Engine:
    """One vdc_ctx (one persistent-kernel configuration) with a loaded program."""

    def __init__(self, program: Program, device: int = 0, watchdog_ms: int = 2000):
        info = program.info()
        prof = vdc_profile(sm_count=info["sm_count"], vcc_per_sm=info["vcc_per_sm"], slot_size=info["slot_size"],
                           slot_budget=info["slot_budget"], ldu_count=info["ldu_count"], stu_count=info["stu_count"])
        self.program = program
        self.info = info
        self.device = device
        h = ctypes.c_void_p()
        check(lib().vdc_create(ctypes.byref(prof), device, ctypes.byref(h)))
        self._h = h
        check(lib().vdc_program_load(self._h, program.handle))
        check(lib().vdc_set_watchdog(self._h, watchdog_ms))
        self.tensors: dict[str, object] = {}
        self._step = None
        self.descs = {d["name"]: d for d in info["descriptors"]}

    # -- memory -------------------------------------------------------------
    def set_steps(self, steps: int) -> None:
        """Resident decode (vdc_set_steps): every following launch runs `steps`
        decode steps inside the persistent kernel (feedback programs only)."""
        check(lib().vdc_set_steps(self._h, steps))

    def stream_stats(self) -> dict:
        """Ring engine: memory-core LOAD words as built and as folded on the
        device (vdc_ring_stream_stats; ring_abi.h vdc_run)."""
        import ctypes as c
        a, b, r = c.c_uint64(), c.c_uint64(), c.c_uint64()
        check(lib().vdc_ring_stream_stats(self._h, c.byref(a), c.byref(b), c.byref(r)))
        return {"load_words": a.value, "run_entries": b.value, "multi_tile_runs": r.value}

    def set_prefetch(self, tiles: int) -> None:
        """Ring engine: the removed L2 look-ahead (only 0 is accepted)."""
        check(lib().vdc_set_prefetch(self._h, tiles))

    def storage_names(self):
        return [d["name"] for d in self.info["descriptors"] if d["view_of"] < 0]

    def bind(self, name: str, tensor) -> None:
        d = self.descs[name]
        torch = _torch()
        if not tensor.is_cuda or not tensor.is_contiguous():
            raise VdcError(2, f"{name}: expected a contiguous CUDA tensor")
        if str(tensor.dtype) != "torch." + TORCH_DTYPE[d["dtype"]]:
            raise VdcError(2, f"{name}: dtype {tensor.dtype} != {d['dtype']}")
        check(lib().vdc_bind_tensor(self._h, d["index"], ctypes.c_void_p(tensor.data_ptr()),
                                    tensor.numel() * tensor.element_size(), DTYPE[d["dtype"]]))
        self.tensors[name] = tensor
        del torch

    def bind_inputs(self, arrays: dict, skip_symmetric: bool = False) -> dict:
        """Allocate every storage tensor on the device from host arrays (float32
        values in logical row-major order; bf16 tensors are cast); missing names
        are zero-filled. Weights of batched programs are packed into pre-swizzled
        tiles (VDC_DESC_PACKED_SW128) and K/V page pools swizzled
        (VDC_DESC_KPAGE_SWZ) here, so callers never see the device layouts."""
        torch = _torch()
        out = {}
        for d in self.info["descriptors"]:
            if d["view_of"] >= 0 or (skip_symmetric and d.get("symmetric")):
                continue
            n = int(np.prod(d["shape"]))
            dt = getattr(torch, TORCH_DTYPE[d["dtype"]])
            if d["name"] in arrays:
                a = to_storage(d, np.ascontiguousarray(arrays[d["name"]], dtype=np.float32).reshape(-1))
                t = torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{self.device}").to(dt)
            else:
                t = torch.zeros(n, dtype=dt, device=f"cuda:{self.device}")
            self.bind(d["name"], t)
            out[d["name"]] = t
        return out

    def synthesize(self, seed: int = 0, skip_symmetric: bool = False, overrides: dict | None = None,
                   seeds: dict | None = None) -> dict:
        """Allocate every storage tensor and fill it ON THE DEVICE with the
        reference synthesize_inputs stream (vdc_program_synthesize: splitmix64 /
        unit_float keyed by seed ^ fnv1a(name), device storage layouts applied);
        `overrides` maps names to host arrays bound instead (bind_inputs rules);
        `seeds` maps names to their own seed (e.g. tensors replicated over TP
        ranks keep one seed while the shards get per-rank seeds)."""
        torch = _torch()
        out = {}
        stream = torch.cuda.current_stream(self.device)
        for d in self.info["descriptors"]:
            if d["view_of"] >= 0 or (skip_symmetric and d.get("symmetric")):
                continue
            dt = getattr(torch, TORCH_DTYPE[d["dtype"]])
            n = int(np.prod(d["shape"]))
            if overrides and d["name"] in overrides:
                a = to_storage(d, np.ascontiguousarray(overrides[d["name"]], dtype=np.float32).reshape(-1))
                t = torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{self.device}").to(dt)
            elif d["dtype"] in ("f32", "bf16"):
                t = torch.empty(n, dtype=dt, device=f"cuda:{self.device}")
                sd = (seeds or {}).get(d["name"], seed)
                check(lib().vdc_program_synthesize(self.program.handle, d["index"], sd, ctypes.c_void_p(t.data_ptr()),
                                                   n * t.element_size(), ctypes.c_void_p(stream.cuda_stream)))
            else:
                t = torch.zeros(n, dtype=dt, device=f"cuda:{self.device}")
            self.bind(d["name"], t)
            out[d["name"]] = t
        return out

    def bind_inputs_nonsym(self, arrays: dict) -> dict:
        """bind_inputs for every storage tensor except the symmetric (TP) buffers"""
        return self.bind_inputs(arrays, skip_symmetric=True)

    def bind_symmetric(self, name: str, peer_ptrs: list, world: int, rank: int) -> None:
        """TP exchange buffer: peer_ptrs[q] = rank q's buffer (128-byte header + data)"""
        d = self.descs[name]
        arr = (ctypes.c_void_p * len(peer_ptrs))(*peer_ptrs)
        check(lib().vdc_bind_symmetric(self._h, d["index"], arr, world, rank))

    def tp_alloc(self) -> bytes:
        """This rank's exchange buffers (vdc_tp_alloc): allocated and zeroed by
        the library; returns the IPC handle blob to hand to every rank."""
        n = ctypes.c_size_t(0)
        check(lib().vdc_tp_alloc(self._h, self.program.handle, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        check(lib().vdc_tp_alloc(self._h, self.program.handle, buf, n.value, ctypes.byref(n)))
        return buf.raw[: n.value]

    def tp_bind(self, blobs: list, rank: int) -> None:
        """Map and bind every rank's exchange buffers from their vdc_tp_alloc
        blobs (vdc_tp_bind: CUDA IPC across processes)."""
        keep = [ctypes.create_string_buffer(b, len(b)) for b in blobs]
        arr = (ctypes.c_void_p * len(keep))(*[ctypes.cast(k, ctypes.c_void_p) for k in keep])
        check(lib().vdc_tp_bind(self._h, arr, len(blobs), rank))

    def host_arrays(self, tensors: dict) -> dict:
        """bound device tensors -> host float32 arrays in logical row-major order"""
        return {k: to_logical(self.descs[k], v.float().cpu().numpy()) for k, v in tensors.items()}

    def bind_step(self, tensor) -> None:
        """Device-resident int64 step block (token, pos, ctx, ...)."""
        check(lib().vdc_bind_step(self._h, ctypes.c_void_p(tensor.data_ptr()), tensor.numel()))
        self._step = tensor

    def enable_trace(self, records_per_core: int = 512):
        """Device trace of every compute µop (see vdc_bind_trace)."""
        torch = _torch()
        n_cores = self.program.cores()[0]
        self._trace = torch.zeros(n_cores * records_per_core * 4, dtype=torch.int64, device=f"cuda:{self.device}")
        self._trace_cap = records_per_core
        check(lib().vdc_bind_trace(self._h, ctypes.c_void_p(self._trace.data_ptr()), records_per_core))

    def trace(self):
        """[(core, pc, t_enter, t_prologue, t_done)] of the last launch (ns)."""
        a = self._trace.view(-1, 4).cpu().numpy()
        a = a[a[:, 1] != 0]
        return [(int(r[0]) >> 32, int(r[0]) & 0xffffffff, int(r[1]), int(r[2]), int(r[3])) for r in a]

    def chrome_trace(self, path: str) -> int:
        """Write the last launch's per-µop device trace (vdc_bind_trace
        records) as a Chrome trace (chrome://tracing, Perfetto): one process
        per SM, one thread per core, a slice per compute µop split into its
        dependency wait ("wait") and its execution (opcode + operand block),
        named by the µop's operator. Returns the number of slices."""
        import json

        ops = {}
        text = self.program.text(False)
        for core_name, st in text["streams"].items():
            if ".vcc" not in core_name:
                continue
            sm = int(core_name[2:].split(".")[0])
            pc = 0
            for line in st.splitlines():
                if line.startswith("#"):
                    continue
                op = line.rsplit("op=", 1)[1] if "op=" in line else "?"
                imm = line.split("imm=")[1].split()[0] if "imm=" in line else "0"
                ops[(2 * sm + 1, pc)] = (line.split()[0], op, imm)
                pc += 1
        rows = self.trace()
        if not rows:
            return 0
        t0 = min(r[2] for r in rows)
        ev = []
        for core, pc, te, tr, td in rows:
            name, op, imm = ops.get((core, pc), ("?", "?", "0"))
            sm = core // 2
            if tr > te:
                ev.append({"name": "wait", "cat": "dep", "ph": "X", "pid": sm, "tid": 0, "ts": (te - t0) / 1e3,
                           "dur": (tr - te) / 1e3, "args": {"op": op}})
            ev.append({"name": f"{name} op{op}", "cat": "uop", "ph": "X", "pid": sm, "tid": 0, "ts": (tr - t0) / 1e3,
                       "dur": max(td - tr, 0) / 1e3, "args": {"pc": pc, "job": int(imm), "operator": op}})
        with open(path, "w") as f:
            json.dump({"traceEvents": ev, "displayTimeUnit": "ns"}, f)
        return len(ev)

    # -- execution ----------------------------------------------------------
    def launch(self, stream=None) -> None:
        s = ctypes.c_void_p(stream.cuda_stream if stream is not None else _torch().cuda.current_stream(self.device).cuda_stream)
        check(lib().vdc_launch(self._h, s))

    def wait(self) -> Report:
        r = vdc_report()
        rc = lib().vdc_wait(self._h, ctypes.byref(r))
        if rc not in (VDC_OK, VDC_ERR_DEADLOCK) and r.status == 0:
            check(rc)
        names = RING_SITES if self.info.get("ring_slots") else WAIT_SITES
        return Report(r.status, r.uops_executed, r.bytes_loaded, r.bytes_stored, r.elapsed_ms, r.message.decode(),
                      [(r.stalled_core[i], r.stalled_pc[i]) for i in range(min(16, r.n_stalled))],
                      {name: int(r.wait_cycles[i]) for i, name in enumerate(names)},
                      bool(r.queues_drained), bool(r.slots_all_free))

    def run(self, stream=None) -> Report:
        self.launch(stream)
        return self.wait()

    def __del__(self):
        if getattr(self, "_h", None):
            lib().vdc_destroy(self._h)
            self._h = None


def simulate(program: Program, inputs: dict, step=None, device: int = 0):
    """Build + bind + run once; returns (report, {name: host float32 array})."""
    torch = _torch()
    eng = Engine(program, device)
    tens = eng.bind_inputs(inputs)
    if step is not None:
        st = torch.tensor(list(step) + [0] * (8 - len(step)), dtype=torch.int64, device=f"cuda:{device}")
        eng.bind_step(st)
    rep = eng.run()
    host = eng.host_arrays(tens)
    return rep, host
