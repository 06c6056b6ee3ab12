"""Vectorised numpy restatement of the reference input synthesis (TEST
INFRASTRUCTURE): reference src/workload.cpp:411-435 synthesize_inputs and
include/uopsim/util.hpp:15-33 splitmix64 / unit_float / fnv1a, plus the
`centered` extension of csrc/host/graph.cpp synthesize_tensor.

splitmix64 adds a constant per draw, so draw i (0-based) of a stream is
mix(state0 + (i + 1) * GOLDEN): computed for all i at once with wrapping
uint64 arithmetic. Pinned against the reference's own synthesize_inputs
(tests/golden/synth_golden.json, made by tests/golden/make_synth_golden.py
from oracle/_ref/ref_cli)."""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
INIT = {"random": 0, "zeros": 1, "ones": 2, "arange": 3, "centered": 4}


def fnv1a(s: str) -> int:
    h = 0xCBF29CE484222325
    for c in s.encode():
        h = ((h ^ c) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def draws(state0: int, n: int, start: int = 0) -> np.ndarray:
    """splitmix64 outputs start .. start + n - 1 of the stream seeded with state0"""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(state0) + i * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def unit_float(z: np.ndarray) -> np.ndarray:
    """reference arithmetic: float(double(z >> 40) * 2^-23) * 2 - 1, in [-1, 3)"""
    s = ((z >> np.uint64(40)).astype(np.float64) * (1.0 / 8388608.0)).astype(np.float32)
    return s * np.float32(2.0) - np.float32(1.0)


def bf16(x: np.ndarray) -> np.ndarray:
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def synthesize(name: str, n: int, init: int | str = 0, seed: int = 0, scale: float = 1.0, dtype: str = "f32",
               start: int = 0) -> np.ndarray:
    """logical elements start .. start + n - 1 of tensor `name`"""
    init = INIT[init] if isinstance(init, str) else init
    if init in (0, 4):
        u = unit_float(draws(seed ^ fnv1a(name), n, start))
        v = u if init == 0 else ((u - np.float32(1.0)) * np.float32(0.5)) * np.float32(scale)
    elif init == 2:
        v = np.ones(n, np.float32)
    elif init == 3:
        v = (np.arange(start, start + n) % 97).astype(np.float32)
    else:
        v = np.zeros(n, np.float32)
    return bf16(v) if dtype == "bf16" else v.astype(np.float32)


def bits_fnv1a(v: np.ndarray) -> int:
    """FNV-1a over the little-endian fp32 bit patterns (ref_cli's checksum)"""
    h = 0xCBF29CE484222325
    for b in np.asarray(v, np.float32).tobytes():
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h
