"""Paged-KV block allocator (vdc_kv_*) and the paged
lowering on the CPU: allocation / growth / release semantics, error
behaviour, the step-block table layout, LOAD words addressed (request,
logical page, head) and pools past the old 4095-page cap."""
import numpy as np
import pytest

from paper_2605_03190_b200 import KvPages, Program, VdcError
import batch_cases as bc


def test_reserve_grows_in_whole_pages():
    kv = KvPages(10, 3, 4)
    kv.reserve(0, 1)
    kv.reserve(1, 64)
    kv.reserve(1, 65)
    kv.reserve(0, 64)  # still one page: no-op
    free, held = kv.stats()
    assert held == [1, 2, 0] and free == 7
    t = np.array(kv.table()).reshape(3, 4)
    assert t[0, 0] == 0 and list(t[1, :2]) == [1, 2]  # LIFO from page 0
    assert (t[0, 1:] == -1).all() and (t[2] == -1).all()


def test_release_returns_pages_and_reuses_first():
    kv = KvPages(4, 2, 4)
    kv.reserve(0, 128)
    kv.reserve(1, 64)
    kv.release(0)
    free, held = kv.stats()
    assert free == 3 and held == [0, 1]
    kv.reserve(1, 192)
    t = np.array(kv.table()).reshape(2, 4)
    assert list(t[1, :3]) == [2, 0, 1] and (t[0] == -1).all()


def test_errors_are_status_codes():
    kv = KvPages(2, 2, 3)
    with pytest.raises(VdcError, match="capacity"):
        kv.reserve(0, 4 * 64)
    kv.reserve(0, 2 * 64)
    with pytest.raises(VdcError, match="exhausted"):
        kv.reserve(1, 1)
    with pytest.raises(VdcError, match="out of range"):
        kv.reserve(5, 1)


def _words(prog, core):
    w = np.frombuffer(prog.words(core), np.uint8).reshape(-1, 16)
    return w


def test_paged_lowering_addresses_request_page_head():
    pages = [3, 1, 2]
    req = bc.request(bc.MID_MODEL, pages, 2)
    req["layout"]["pool_pages"] = 5  # shared pool smaller than sum(capacity) = 6
    prog = Program.build(req)
    info = prog.info()
    assert all(p == -1 for p in info["batch"]["page_table"])  # the host allocates
    kc = [d for d in info["descriptors"] if d["name"] == "L0.kc"][0]
    assert kc["shape"][0] == 5
    seen = set()
    n_cores = prog.cores()[0]
    for core in range(0, n_cores, 2):  # memory cores
        for w in _words(prog, core):
            if w[0] != 0x01:
                continue
            reg1 = w[7] & 0xF
            tensor = int(w[8]) | (int(w[9]) << 8)
            if tensor != kc["index"]:
                continue
            assert reg1 == 2  # VDC_LOAD_PAGED
            pl = int.from_bytes(bytes(w[10:16]), "little")
            seen.add((pl & 0xFFF, (pl >> 12) & 0xFFF, (pl >> 24) & 0xFFF))
    hkv = kc["shape"][1] // 64
    want = {(b, i, h) for b, n in enumerate(pages) for i in range(n) for h in range(hkv)}
    assert seen == want


def test_pool_beyond_4095_pages_builds():
    req = bc.request(bc.MID_MODEL, [128] * 40, 64)  # 5120 pages: past the old 12-bit pool cap
    prog = Program.build(req)
    kc = [d for d in prog.info()["descriptors"] if d["name"] == "L0.kc"][0]
    assert kc["shape"][0] == 5120
