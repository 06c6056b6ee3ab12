"""ctypes binding of the C-ABI in include/vdc.h (libvdc.so, built in-tree).

The product path is native: every entry point below is a C function of
paper_2605_03190_b200/lib/libvdc.so. There is no Python fallback — if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import json
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("VDC_LIB", str(PKG / "lib" / "libvdc.so")))  # VDC_LIB: A/B experiments only

VDC_OK, VDC_ERR_INTERNAL, VDC_ERR_INPUT, VDC_ERR_DEADLOCK = 0, 1, 2, 3
DTYPE = {"f32": 0, "bf16": 1, "i64": 2}


class VdcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[vdc status {code}] {msg}")
        self.code = code


class vdc_profile(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("sm_count", "vcc_per_sm", "slot_size", "slot_budget", "ldu_count", "stu_count")]


class vdc_desc(ctypes.Structure):
    _fields_ = [
        ("base", ctypes.c_int64),
        ("shape", ctypes.c_int64 * 4),
        ("grid", ctypes.c_int64 * 4),
        ("tile_rows", ctypes.c_int64),
        ("tile_cols", ctypes.c_int64),
        ("rank", ctypes.c_uint32),
        ("dtype", ctypes.c_uint32),
        ("view_of", ctypes.c_int32),
        ("tma", ctypes.c_uint32),
    ]


class vdc_queue(ctypes.Structure):
    _fields_ = [
        ("dep_id", ctypes.c_uint16),
        ("depth", ctypes.c_uint16),
        ("producer_sm", ctypes.c_uint16),
        ("consumer_sm", ctypes.c_uint16),
        ("local", ctypes.c_uint32),
    ]


class vdc_report(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("n_stalled", ctypes.c_uint32),
        ("uops_executed", ctypes.c_uint64),
        ("bytes_loaded", ctypes.c_uint64),
        ("bytes_stored", ctypes.c_uint64),
        ("elapsed_ms", ctypes.c_double),
        ("stalled_core", ctypes.c_uint32 * 16),
        ("stalled_pc", ctypes.c_uint32 * 16),
        ("wait_cycles", ctypes.c_uint64 * 24),
        ("message", ctypes.c_char * 256),
        ("queues_drained", ctypes.c_uint32),
        ("slots_all_free", ctypes.c_uint32),
    ]


# every symbol include/vdc.h declares (the CPU suite checks they are exported)
EXPORTS = [
    "vdc_last_error", "vdc_version", "vdc_create", "vdc_destroy", "vdc_load_program", "vdc_load_jobs", "vdc_set_params",
    "vdc_bind_tensor", "vdc_bind_symmetric", "vdc_tp_alloc", "vdc_tp_bind", "vdc_bind_step", "vdc_bind_trace", "vdc_launch", "vdc_wait", "vdc_set_watchdog", "vdc_set_prefetch", "vdc_set_steps", "vdc_ring_stream_stats",
    "vdc_fold_stream", "vdc_unfold_stream", "vdc_program_build",
    "vdc_program_parse", "vdc_program_free", "vdc_program_text", "vdc_program_cores", "vdc_program_words",
    "vdc_program_load", "vdc_free_string", "vdc_program_synthesize",
    "vdc_kv_create", "vdc_kv_destroy", "vdc_kv_reserve", "vdc_kv_release", "vdc_kv_stats", "vdc_kv_table",
]

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(str(LIB_PATH))
    c = ctypes
    vp = c.c_void_p
    sig = {
        "vdc_last_error": ([], c.c_char_p),
        "vdc_version": ([], c.c_char_p),
        "vdc_create": ([c.POINTER(vdc_profile), c.c_int, c.POINTER(vp)], c.c_int),
        "vdc_destroy": ([vp], c.c_int),
        "vdc_load_program": ([vp, c.c_void_p, c.POINTER(c.c_uint32), c.c_uint32, c.POINTER(vdc_queue), c.c_uint32,
                              c.POINTER(vdc_desc), c.c_uint32, c.c_uint16, c.c_uint16], c.c_int),
        "vdc_load_jobs": ([vp, vp, c.c_uint32, c.c_uint32], c.c_int),
        "vdc_set_params": ([vp, c.POINTER(c.c_float), c.c_uint32], c.c_int),
        "vdc_bind_tensor": ([vp, c.c_uint16, vp, c.c_size_t, c.c_int], c.c_int),
        "vdc_bind_step": ([vp, vp, c.c_uint32], c.c_int),
        "vdc_bind_symmetric": ([vp, c.c_uint16, c.POINTER(c.c_void_p), c.c_uint32, c.c_uint32], c.c_int),
        "vdc_bind_trace": ([vp, vp, c.c_uint32], c.c_int),
        "vdc_launch": ([vp, vp], c.c_int),
        "vdc_wait": ([vp, c.POINTER(vdc_report)], c.c_int),
        "vdc_tp_alloc": ([vp, vp, vp, c.c_size_t, c.POINTER(c.c_size_t)], c.c_int),
        "vdc_tp_bind": ([vp, c.POINTER(c.c_void_p), c.c_uint32, c.c_uint32], c.c_int),
        "vdc_set_watchdog": ([vp, c.c_uint32], c.c_int),
        "vdc_set_prefetch": ([vp, c.c_uint32], c.c_int),
        "vdc_set_steps": ([vp, c.c_uint32], c.c_int),
        "vdc_ring_stream_stats": ([vp, c.POINTER(c.c_uint64), c.POINTER(c.c_uint64), c.POINTER(c.c_uint64)], c.c_int),
        "vdc_fold_stream": ([c.c_char_p, c.c_uint32, vp, c.POINTER(c.c_uint32)], c.c_int),
        "vdc_unfold_stream": ([vp, c.c_uint32, c.c_char_p, c.c_uint32, c.POINTER(c.c_uint32)], c.c_int),
        "vdc_program_build": ([c.c_char_p, c.POINTER(vp)], c.c_int),
        "vdc_program_parse": ([c.c_char_p, c.c_char_p, c.POINTER(vp)], c.c_int),
        "vdc_program_free": ([vp], None),
        "vdc_program_text": ([vp, c.c_int, c.POINTER(c.c_void_p)], c.c_int),
        "vdc_program_cores": ([vp, c.POINTER(c.c_uint32), c.POINTER(c.c_uint32), c.POINTER(c.c_uint32)], c.c_int),
        "vdc_program_words": ([vp, c.c_uint32, c.POINTER(c.c_void_p), c.POINTER(c.c_uint32)], c.c_int),
        "vdc_program_load": ([vp, vp], c.c_int),
        "vdc_free_string": ([c.c_void_p], None),
        "vdc_program_synthesize": ([vp, c.c_uint16, c.c_uint64, vp, c.c_size_t, vp], c.c_int),
        "vdc_kv_create": ([c.c_uint32, c.c_uint32, c.c_uint32, c.POINTER(vp)], c.c_int),
        "vdc_kv_destroy": ([vp], c.c_int),
        "vdc_kv_reserve": ([vp, c.c_uint32, c.c_uint64], c.c_int),
        "vdc_kv_release": ([vp, c.c_uint32], c.c_int),
        "vdc_kv_stats": ([vp, c.POINTER(c.c_uint32), c.POINTER(c.c_uint32)], c.c_int),
        "vdc_kv_table": ([vp, c.POINTER(c.c_int64)], c.c_int),
    }
    for name, (args, res) in sig.items():
        if "VDC_LIB" in os.environ and not hasattr(L, name):
            continue  # A/B runs against an older build: symbols it predates stay unbound
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(code: int) -> None:
    if code != VDC_OK:
        raise VdcError(code, lib().vdc_last_error().decode())


def take_string(ptr: ctypes.c_void_p) -> str:
    try:
        return ctypes.string_at(ptr).decode()
    finally:
        lib().vdc_free_string(ptr)


class Program:
    """Owns a vdc_program handle (generator::LoweredProgram + encoded words)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        self._info = None

    @classmethod
    def build(cls, request: dict) -> "Program":
        h = ctypes.c_void_p()
        check(lib().vdc_program_build(json.dumps(request).encode(), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def parse(cls, streams: dict, sidecar: str) -> "Program":
        h = ctypes.c_void_p()
        check(lib().vdc_program_parse(json.dumps(streams).encode(), sidecar.encode(), ctypes.byref(h)))
        return cls(h)

    @property
    def handle(self):
        return self._h

    def text(self, with_words: bool = False) -> dict:
        out = ctypes.c_void_p()
        check(lib().vdc_program_text(self._h, 1 if with_words else 0, ctypes.byref(out)))
        return json.loads(take_string(out))

    def unfolded_words(self) -> dict:
        """{core: hex} of every stream with its loops expanded (unfold_stream)."""
        out = ctypes.c_void_p()
        check(lib().vdc_program_text(self._h, 3, ctypes.byref(out)))
        return json.loads(take_string(out))["unfolded_words"]

    def info(self) -> dict:
        """Summary (descriptors, params, geometry) without stream text."""
        if self._info is None:
            out = ctypes.c_void_p()
            check(lib().vdc_program_text(self._h, 2, ctypes.byref(out)))
            self._info = json.loads(take_string(out))
        return self._info

    def cores(self):
        n, sms, vcc = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        check(lib().vdc_program_cores(self._h, ctypes.byref(n), ctypes.byref(sms), ctypes.byref(vcc)))
        return n.value, sms.value, vcc.value

    def words(self, core: int) -> bytes:
        p, n = ctypes.c_void_p(), ctypes.c_uint32()
        check(lib().vdc_program_words(self._h, core, ctypes.byref(p), ctypes.byref(n)))
        return ctypes.string_at(p, n.value * 16) if n.value else b""

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.vdc_program_free(self._h)
            self._h = None


class KvPages:
    """Paged-KV block allocator (vdc_kv_*): a pool of 64-row pages shared by
    the request rows of a batched program's page table."""

    def __init__(self, n_pages: int, n_requests: int, max_pages: int):
        self._h = ctypes.c_void_p()
        check(lib().vdc_kv_create(n_pages, n_requests, max_pages, ctypes.byref(self._h)))
        self.n_requests, self.max_pages = n_requests, max_pages

    def reserve(self, req: int, tokens: int) -> None:
        check(lib().vdc_kv_reserve(self._h, req, tokens))

    def release(self, req: int) -> None:
        check(lib().vdc_kv_release(self._h, req))

    def stats(self):
        free = ctypes.c_uint32()
        held = (ctypes.c_uint32 * self.n_requests)()
        check(lib().vdc_kv_stats(self._h, ctypes.byref(free), held))
        return free.value, list(held)

    def table(self):
        """n_requests x max_pages int64 (-1 = unallocated), request-major"""
        t = (ctypes.c_int64 * (self.n_requests * self.max_pages))()
        check(lib().vdc_kv_table(self._h, t))
        return list(t)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.vdc_kv_destroy(self._h)
            self._h = None
