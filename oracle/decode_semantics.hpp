// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// CPU restatement of the decode µop extension semantics (scalar fp32,
// sequential summation), written from the definitions in
// include/uopsim/decode_abi.h and DESIGN.md. The attention math restates the
// reference's online softmax (reference src/handlers.cpp:54-87: running max
// m, running sum l, rescale by exp(m_old - m_new), finalize acc / l) and its
// RMSNorm (handlers.cpp:101-113) with a configurable eps; SiLU follows
// handlers.cpp:27-33.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#include "uopsim/decode_abi.h"

namespace oracle {

inline float bf16_round(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return f;
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

struct Tile {  // one m2c message payload (values as float, already dtype-rounded)
    std::vector<float> v;
    int rows = 0, cols = 0, stride = 0, row0 = 0, col0 = 0;
    bool bf16 = false;
    uint16_t slots = 0;
    int64_t tensor = -1;
    float at(int r, int c) const { return v[size_t(r) * stride + c]; }
    void put(int64_t i, float x) { v[size_t(i)] = bf16 ? bf16_round(x) : x; }
};

inline float silu(float x) { return x / (1.0f + std::exp(-x)); }

// GEMV family: prologue [x (, norm_w | resid)], groups = W tiles, result.
inline void gemv(int op, int32_t imm, const float* hp, double pos, Tile& x, const Tile* third,
                 const std::vector<Tile*>& groups, Tile& res) {
    const int variant = imm & 0xff;
    const int K = x.rows * x.cols;
    if (op == 0x28) {  // RMS_GEMV: x <- round(x * 1/sqrt(mean(x^2)+eps) * w)
        float ss = 0.f;
        for (int i = 0; i < K; ++i) ss += x.v[size_t(i)] * x.v[size_t(i)];
        const float inv = 1.0f / std::sqrt(ss / float(K) + hp[VDC_GEMV_P_EPS]);
        for (int i = 0; i < K; ++i) x.put(i, x.v[size_t(i)] * inv * third->v[size_t(i)]);
    }
    std::vector<float> acc(4096, 0.f);
    int row0 = groups.empty() ? 0 : groups[0]->row0, raw = 0;
    for (const Tile* g : groups) {
        const int rb = g->row0 - row0;
        raw = std::max(raw, rb + g->rows);
        for (int r = 0; r < g->rows; ++r) {
            float s = 0.f;
            for (int c = 0; c < g->cols; ++c) s += g->at(r, c) * x.v[size_t(g->col0 + c)];
            acc[size_t(rb + r)] += s;
        }
    }
    const int nout = res.rows * res.cols;
    if (variant & VDC_GEMV_SWIGLU) {
        const int B = int(hp[VDC_GEMV_P_SWIGLU_BLOCK]);
        for (int o = 0; o < nout; ++o) {
            const int blk = o / (B / 2), j = o % (B / 2);
            res.put(o, silu(acc[size_t(blk * B + j)]) * acc[size_t(blk * B + B / 2 + j)]);
        }
    } else if (variant & VDC_GEMV_ROPE) {
        const double theta = hp[VDC_GEMV_P_THETA];
        const int hd = int(hp[VDC_GEMV_P_HEAD_DIM]);
        const int rope_rows = int(hp[VDC_GEMV_P_ROPE_ROWS]);
        for (int o = 0; o + 1 < nout; o += 2) {
            const int row = row0 + o;
            float a = acc[size_t(o)], b = acc[size_t(o + 1)];
            if (row < rope_rows) {
                const int d = row % hd;
                const double ang = pos * std::pow(theta, -double(d) / double(hd));
                const float cs = float(std::cos(ang)), sn = float(std::sin(ang));
                const float na = a * cs - b * sn, nb = a * sn + b * cs;
                a = na;
                b = nb;
            }
            res.put(o, a);
            res.put(o + 1, b);
        }
    } else if (op == 0x29) {
        for (int o = 0; o < nout; ++o) res.put(o, third->v[size_t(o)] + acc[size_t(o)]);
    } else {
        for (int o = 0; o < nout; ++o) res.put(o, acc[size_t(o)]);
    }
}

// split-KV partial: per q head h of the group, online softmax over the pages
inline void attn_decode(const float* hp, long long ctx, const Tile& q, const std::vector<std::pair<Tile*, Tile*>>& pages,
                        Tile& res) {
    const float scale = hp[VDC_ATTN_P_SCALE];
    const int hd = int(hp[VDC_ATTN_P_HEAD_DIM]), G = int(hp[VDC_ATTN_P_GROUP]);
    for (int h = 0; h < G; ++h) {
        float m = -std::numeric_limits<float>::infinity(), l = 0.f;
        std::vector<float> o(size_t(hd), 0.f);
        for (const auto& [kt, vt] : pages) {
            std::vector<float> s(size_t(kt->rows), -std::numeric_limits<float>::infinity());
            float pmax = -std::numeric_limits<float>::infinity();
            for (int r = 0; r < kt->rows; ++r) {
                if (kt->row0 + r >= ctx) continue;
                float a = 0.f;
                for (int d = 0; d < hd; ++d) a += q.v[size_t(h * hd + d)] * kt->at(r, d);
                s[size_t(r)] = a * scale;
                pmax = std::max(pmax, s[size_t(r)]);
            }
            if (pmax == -std::numeric_limits<float>::infinity()) continue;
            const float mn = std::max(m, pmax);
            const float corr = m == -std::numeric_limits<float>::infinity() ? 0.f : std::exp(m - mn);
            float psum = 0.f;
            std::vector<float> p(s.size(), 0.f);
            for (size_t r = 0; r < s.size(); ++r) {
                p[r] = s[r] == -std::numeric_limits<float>::infinity() ? 0.f : std::exp(s[r] - mn);
                psum += p[r];
            }
            l = l * corr + psum;
            for (int d = 0; d < hd; ++d) {
                float od = o[size_t(d)] * corr;
                for (int r = 0; r < vt->rows; ++r) od += p[size_t(r)] * vt->at(r, d);
                o[size_t(d)] = od;
            }
            m = mn;
        }
        for (int d = 0; d < hd; ++d) res.put(h * (hd + 2) + d, o[size_t(d)]);
        res.put(h * (hd + 2) + hd, m);
        res.put(h * (hd + 2) + hd + 1, l);
    }
}

inline void attn_combine(const float* hp, const std::vector<Tile*>& parts, Tile& res) {
    const int hd = int(hp[VDC_COMB_P_HEAD_DIM]), G = int(hp[VDC_COMB_P_GROUP]);
    for (int h = 0; h < G; ++h) {
        float M = -std::numeric_limits<float>::infinity(), L = 0.f;
        std::vector<float> O(size_t(hd), 0.f);
        for (const Tile* p : parts) {
            const float ms = p->v[size_t(h * (hd + 2) + hd)], ls = p->v[size_t(h * (hd + 2) + hd + 1)];
            if (ms == -std::numeric_limits<float>::infinity() || !(ls > 0.f)) continue;
            const float mn = std::max(M, ms);
            const float a = M == -std::numeric_limits<float>::infinity() ? 0.f : std::exp(M - mn), b = std::exp(ms - mn);
            for (int d = 0; d < hd; ++d) O[size_t(d)] = O[size_t(d)] * a + p->v[size_t(h * (hd + 2) + d)] * b;
            L = L * a + ls * b;
            M = mn;
        }
        for (int d = 0; d < hd; ++d) res.put(h * hd + d, L > 0.f ? O[size_t(d)] / L : 0.f);
    }
}

}  // namespace oracle
