"""Packed weight layout of batched programs (ring_abi.h VDC_DESC_PACKED_SW128),
checked on the CPU: engine.pack_sw128 stores tile (rb, kt) of 128 x 64 bf16
contiguously with 16-byte chunk c of tile row r at chunk c ^ (r % 8) — the
K-major 128-byte-swizzle operand layout the tcgen05 descriptors in
ring_engine.cu (umma_sw128_desc) address — and unpack_sw128 inverts it."""
import numpy as np

from paper_2605_03190_b200.engine import pack_sw128, unpack_sw128, to_logical, PACKED_SW128


def test_roundtrip_and_layout():
    rows, cols = 256, 192
    a = np.random.default_rng(0).random(rows * cols).astype(np.float32)
    p = pack_sw128(a, rows, cols)
    assert p.shape == a.shape
    assert np.array_equal(unpack_sw128(p, rows, cols), a)
    W = a.reshape(rows, cols)
    for rb, kt, r, c in [(0, 0, 0, 0), (1, 2, 5, 3), (0, 1, 127, 7), (1, 0, 8, 1)]:
        off = (rb * (cols // 64) + kt) * 8192 + r * 64 + (c ^ (r & 7)) * 8
        assert np.array_equal(p[off:off + 8], W[rb * 128 + r, kt * 64 + c * 8: kt * 64 + c * 8 + 8])


def test_to_logical_only_unpacks_packed():
    a = np.arange(128 * 64, dtype=np.float32)
    assert np.array_equal(to_logical({"tma": PACKED_SW128, "shape": [128, 64]}, pack_sw128(a, 128, 64)), a)
    assert np.array_equal(to_logical({"tma": 16, "shape": [128, 64]}, a), a)
