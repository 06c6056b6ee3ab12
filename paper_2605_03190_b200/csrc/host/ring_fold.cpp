// Folding of ring memory-core streams: see ring_fold.hpp and ring_abi.h
// (vdc_run). A LOAD word (uopsim::isa encoding, as resolve_load in
// ring_engine.cu reads it): x & 0xff opcode, z & 0xffff tensor, 36 bits of
// 12-bit tile coordinates from bit 16 of z (c0 | c1 << 12 | c2 << 24), the
// other bits are fields a run copies from its base word.
#include "ring_fold.hpp"

#include <algorithm>
#include <cstring>

#include "vdc.h"

namespace vdc_host {
namespace {

constexpr uint32_t kOpLoad = 0x01;

struct Parts {
    uint32_t x, y, hi;  // fields kept from the base word (hi: pl bits 36..47)
    uint16_t t;
    int32_t c[3];
};

uint64_t pl_of(const Word& w) { return uint64_t(w[2] >> 16) | (uint64_t(w[3]) << 16); }

Parts split(const Word& w) {
    const uint64_t pl = pl_of(w);
    return {w[0], w[1], uint32_t(pl >> 36), uint16_t(w[2] & 0xffff),
            {int32_t(pl & 0xfff), int32_t((pl >> 12) & 0xfff), int32_t((pl >> 24) & 0xfff)}};
}

Word join(const Parts& p) {
    const uint64_t pl = uint64_t(p.c[0] & 0xfff) | (uint64_t(p.c[1] & 0xfff) << 12) | (uint64_t(p.c[2] & 0xfff) << 24) |
                        (uint64_t(p.hi) << 36);
    return {p.x, p.y, uint32_t(p.t) | uint32_t((pl & 0xffff) << 16), uint32_t(pl >> 16)};
}

bool same_rest(const Parts& a, const Parts& b) { return a.x == b.x && a.y == b.y && a.hi == b.hi; }

bool fits8(int32_t v) { return v >= -128 && v <= 127; }

struct Cand {
    uint32_t count = 1, n_alt = 1, n_in = 1;
    uint16_t t_alt = 0;
    int32_t din[3] = {0, 0, 0}, dout[3] = {0, 0, 0};
};

// the longest run starting at w[i] with tensor alternation n_alt
Cand try_run(const Word* w, size_t n, size_t i, uint32_t n_alt) {
    Cand r;
    r.n_alt = n_alt;
    const Parts b = split(w[i]);
    auto is_load = [&](size_t k) { return k < n && (w[k][0] & 0xff) == kOpLoad; };
    // group g (n_alt tiles at w[i + g * n_alt]): same coordinates, tensors (t, t_alt)
    uint16_t t_alt = 0;
    auto group = [&](size_t g, int32_t (&c)[3]) -> bool {
        const size_t k = i + g * n_alt;
        if (!is_load(k) || (n_alt == 2 && !is_load(k + 1))) return false;
        const Parts p = split(w[k]);
        if (!same_rest(p, b) || p.t != b.t) return false;
        if (n_alt == 2) {
            const Parts q = split(w[k + 1]);
            if (!same_rest(q, b) || q.c[0] != p.c[0] || q.c[1] != p.c[1] || q.c[2] != p.c[2]) return false;
            if (g == 0) t_alt = q.t;
            if (q.t != t_alt || q.t == b.t) return false;
        }
        for (int d = 0; d < 3; ++d) c[d] = p.c[d];
        return true;
    };
    int32_t c0[3], cg[3];
    if (!group(0, c0)) {
        r.count = n_alt == 2 ? 0 : 1;
        return r;
    }
    r.t_alt = n_alt == 2 ? t_alt : 0;
    r.count = n_alt;
    const size_t ngroups_max = std::min<size_t>((n - i) / n_alt, (1u << 23) / n_alt);
    if (ngroups_max < 2 || !group(1, cg)) return r;
    int32_t din[3] = {cg[0] - c0[0], cg[1] - c0[1], cg[2] - c0[2]};
    if (!fits8(din[0]) || !fits8(din[1]) || !fits8(din[2])) return r;
    size_t nin = 2;
    for (; nin < ngroups_max && nin < 4095; ++nin) {
        if (!group(nin, cg)) break;
        if (cg[0] != c0[0] + int32_t(nin) * din[0] || cg[1] != c0[1] + int32_t(nin) * din[1] || cg[2] != c0[2] + int32_t(nin) * din[2])
            break;
    }
    // outer lines of nin groups, step d_out
    size_t nout = 1;
    int32_t dout[3] = {0, 0, 0};
    if (2 * nin <= ngroups_max && group(nin, cg)) {
        for (int d = 0; d < 3; ++d) dout[d] = cg[d] - c0[d];
        if (fits8(dout[0]) && fits8(dout[1]) && fits8(dout[2]))
            for (;; ++nout) {
                if ((nout + 1) * nin > ngroups_max) break;
                bool line = true;
                for (size_t j = 0; j < nin && line; ++j) {
                    line = group(nout * nin + j, cg);
                    for (int d = 0; d < 3 && line; ++d) line = cg[d] == c0[d] + int32_t(nout) * dout[d] + int32_t(j) * din[d];
                }
                if (!line) break;
            }
    }
    if (nout == 1) dout[0] = dout[1] = dout[2] = 0;
    for (int d = 0; d < 3; ++d) {
        r.din[d] = din[d];
        r.dout[d] = dout[d];
    }
    r.n_in = uint32_t(nin);
    r.count = uint32_t(n_alt * nin * nout);
    return r;
}

}  // namespace

Word expand_run(const vdc_run& r, uint32_t k) {
    Word base;
    std::memcpy(base.data(), r.base, 16);
    Parts p = split(base);
    const uint32_t n_alt = run_alt(r), n_in = run_nin(r);
    const uint32_t a = n_alt == 2 ? (k & 1u) : 0u, j = n_alt == 2 ? (k >> 1) : k;
    const uint32_t o = j / n_in, i = j % n_in;
    for (int d = 0; d < 3; ++d) p.c[d] += int32_t(i) * r.d_in[d] + int32_t(o) * r.d_out[d];
    if (a) p.t = uint16_t(run_talt(r));
    return join(p);
}

FoldedStream fold_stream(const Word* w, size_t n) {
    FoldedStream f;
    for (size_t i = 0; i < n;) {
        Cand best = try_run(w, n, i, 1);
        const Cand alt = try_run(w, n, i, 2);
        if (alt.count > best.count) best = alt;
        vdc_run r{};
        std::memcpy(r.base, w[i].data(), 16);
        if ((w[i][0] & 0xff) != kOpLoad || best.count < 2) best = Cand{};
        r.count_alt = best.count | (best.n_alt << 24);
        r.nin_talt = best.n_in | (uint32_t(best.t_alt) << 12);
        for (int d = 0; d < 3; ++d) {
            r.d_in[d] = int8_t(best.din[d]);
            r.d_out[d] = int8_t(best.dout[d]);
        }
        f.runs.push_back(r);
        f.multi += best.count > 1;
        i += best.count;
        f.tiles += best.count;
    }
    return f;
}

}  // namespace vdc_host

extern "C" int vdc_fold_stream(const uint8_t* words, uint32_t n, vdc_run* runs, uint32_t* n_runs) {
    if ((!words && n) || !runs || !n_runs) return VDC_ERR_INPUT;
    std::vector<vdc_host::Word> w(n);
    if (n) std::memcpy(w.data(), words, size_t(n) * 16);
    const vdc_host::FoldedStream f = vdc_host::fold_stream(w.data(), n);
    if (!f.runs.empty()) std::memcpy(runs, f.runs.data(), f.runs.size() * sizeof(vdc_run));
    *n_runs = uint32_t(f.runs.size());
    return VDC_OK;
}

extern "C" int vdc_unfold_stream(const vdc_run* runs, uint32_t n_runs, uint8_t* words, uint32_t capacity, uint32_t* n_words) {
    if ((!runs && n_runs) || !n_words) return VDC_ERR_INPUT;
    uint32_t k = 0;
    for (uint32_t i = 0; i < n_runs; ++i) {
        const uint32_t c = vdc_host::run_count(runs[i]), a = vdc_host::run_alt(runs[i]), nin = vdc_host::run_nin(runs[i]);
        if (c == 0 || (a != 1 && a != 2) || nin == 0 || c % (a * nin)) return VDC_ERR_INPUT;
        for (uint32_t t = 0; t < c; ++t, ++k) {
            if (k >= capacity) return VDC_ERR_INPUT;
            const vdc_host::Word e = vdc_host::expand_run(runs[i], t);
            std::memcpy(words + size_t(k) * 16, e.data(), 16);
        }
    }
    *n_words = k;
    return VDC_OK;
}
