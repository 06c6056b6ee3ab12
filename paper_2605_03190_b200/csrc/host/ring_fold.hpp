// Folding of ring memory-core streams (ring_abi.h vdc_run): the host side of
// the loop folding the device expands tile by tile (ring_engine.cu
// expand_run). PAPER.md:773 / reference fold.cpp:151-293 fold the µop
// streams of the reference form; here the folded object is the per-tile
// LOAD stream of the ring engine, the only per-tile stream it has.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

#include "uopsim/ring_abi.h"

namespace vdc_host {

using Word = std::array<uint32_t, 4>;

struct FoldedStream {
    std::vector<vdc_run> runs;  // in stream order; a lone tile is a run of 1
    uint64_t tiles = 0, multi = 0;
};

// fold one stream of LOAD words (no HALT)
FoldedStream fold_stream(const Word* w, size_t n);
inline uint32_t run_count(const vdc_run& r) { return r.count_alt & 0xffffffu; }
inline uint32_t run_alt(const vdc_run& r) { return r.count_alt >> 24; }
inline uint32_t run_nin(const vdc_run& r) { return r.nin_talt & 0xfffu; }
inline uint32_t run_talt(const vdc_run& r) { return r.nin_talt >> 12; }
// tile k of a run, as a LOAD word
Word expand_run(const vdc_run& r, uint32_t k);

}  // namespace vdc_host
