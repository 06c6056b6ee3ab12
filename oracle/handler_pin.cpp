// TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Per-operator pin of the decode µops to the reference's own handler
// arithmetic: every decode operator of one layer is recomposed from
// uopsim::machine_detail::HandlerState (reference src/handlers.cpp, compiled
// unmodified into oracle/_ref/libuopsim_ref.a):
//
//   qkv      RMSNORM(x, attn_norm)        handlers.cpp:101-113
//            MATVEC(W_qkv, xn) by K tiles  handlers.cpp:40-52
//            ROPE on q and k row pairs     handlers.cpp:88-100
//   attn     ATTN per q head over the K/V   handlers.cpp:54-87, finalize :155-168
//            rows [0, ctx) in 64-row tiles (the device's split-KV + combine
//            must equal the reference's single online-softmax sweep)
//   o        MATVEC(W_o, attn) + ELEMWISE add (imm 2) of the residual   :114-134
//   gate/up  RMSNORM(x1, mlp_norm), MATVEC(W_gu), ELEMWISE silu (imm 1) on the
//            gate rows, ELEMWISE mul (imm 3) with the up rows
//   down     MATVEC(W_d, a) + ELEMWISE add of x1
//   head     RMSNORM(x_last, final_norm), MATVEC(lm_head)
//
// Each operator is evaluated on the DEVICE's own inputs to that operator (read
// back by the test), so the comparison isolates one µop's arithmetic. With
// "chain": true in the config every operator consumes the previous
// operator's pinned output instead (the appended K/V row written into copies
// of the caches): a full decode step in reference handler arithmetic, used on
// the CPU to pin the dense decode reference the GPU tests compare against.
//
// I/O: argv[1] = input file, argv[2] = output file, argv[3] = JSON config
// {"layers", "hidden", "heads", "kv_heads", "head_dim", "ffn", "vocab",
//  "theta", "pos", "gu_block"}. Files: repeated records {u32 name length,
// name, u64 count, count float32}.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "handlers.hpp"
#include "nlohmann/json.hpp"

using uopsim::isa::Opcode;
using uopsim::machine_detail::GroupInput;
using uopsim::machine_detail::HandlerState;
using Vec = std::vector<float>;

namespace {

std::map<std::string, Vec> read_all(const char* path) {
    std::map<std::string, Vec> out;
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    for (;;) {
        uint32_t nl = 0;
        if (std::fread(&nl, 4, 1, f) != 1) break;
        std::string name(nl, '\0');
        uint64_t n = 0;
        if (std::fread(name.data(), 1, nl, f) != nl || std::fread(&n, 8, 1, f) != 1) throw std::runtime_error("bad input file");
        Vec v(n);
        if (n && std::fread(v.data(), 4, n, f) != n) throw std::runtime_error("bad input file");
        out.emplace(std::move(name), std::move(v));
    }
    std::fclose(f);
    return out;
}

void write_all(const char* path, const std::map<std::string, Vec>& m) {
    FILE* f = std::fopen(path, "wb");
    for (const auto& [name, v] : m) {
        const uint32_t nl = uint32_t(name.size());
        const uint64_t n = v.size();
        std::fwrite(&nl, 4, 1, f);
        std::fwrite(name.data(), 1, nl, f);
        std::fwrite(&n, 8, 1, f);
        std::fwrite(v.data(), 4, n, f);
    }
    std::fclose(f);
}

GroupInput gin(const float* p, int64_t rows, int64_t cols, int64_t stride, int64_t row0 = 0) {
    GroupInput g;
    g.dims = {rows, cols};
    g.data = std::span<const float>(p, size_t((rows - 1) * stride + cols));
    g.stride = stride;
    g.row0 = row0;
    return g;
}

// RMSNORM handler over a column vector (rows x 1)
Vec rmsnorm(const Vec& x, const Vec& w) {
    HandlerState st;
    st.op = Opcode::RMSNORM;
    st.size = 1;
    st.out = {int64_t(x.size()), 1};
    st.out_stride = 1;
    st.begin();
    const GroupInput in[2] = {gin(x.data(), int64_t(x.size()), 1, 1), gin(w.data(), int64_t(w.size()), 1, 1)};
    st.group(0, in);
    Vec out(x.size());
    st.finalize(out);
    return out;
}

// MATVEC handler: y = W x, W (M x K) row-major, swept in K tiles of `kt` columns
Vec matvec(const float* W, int64_t M, int64_t K, const Vec& x, int64_t kt = 64) {
    HandlerState st;
    st.op = Opcode::MATVEC;
    st.out = {M, 1};
    st.out_stride = 1;
    const int64_t groups = (K + kt - 1) / kt;
    st.size = uint16_t(groups);
    st.begin();
    for (int64_t g = 0; g < groups; ++g) {
        const int64_t k0 = g * kt, kc = std::min(kt, K - k0);
        const GroupInput in[2] = {gin(x.data() + k0, kc, 1, 1), gin(W + k0, M, kc, K)};
        st.group(size_t(g), in);
    }
    Vec out(static_cast<size_t>(M));
    st.finalize(out);
    return out;
}

// ELEMWISE handler: unary (imm 0 relu / 1 silu) or binary (imm 3 mul, else add)
Vec elemwise(const Vec& a, const Vec* b, int32_t imm) {
    HandlerState st;
    st.op = Opcode::ELEMWISE;
    st.imm = imm;
    st.size = b ? 2 : 1;
    st.out = {int64_t(a.size()), 1};
    st.out_stride = 1;
    st.begin();
    const GroupInput ia[1] = {gin(a.data(), int64_t(a.size()), 1, 1)};
    st.group(0, ia);
    if (b) {
        const GroupInput ib[1] = {gin(b->data(), int64_t(b->size()), 1, 1)};
        st.group(1, ib);
    }
    Vec out(a.size());
    st.finalize(out);
    return out;
}

// ROPE handler on consecutive row pairs of x with per-row angles
Vec rope(const Vec& x, const Vec& ang) {
    HandlerState st;
    st.op = Opcode::ROPE;
    st.size = 1;
    st.out = {int64_t(x.size()), 1};
    st.out_stride = 1;
    st.begin();
    const GroupInput in[2] = {gin(x.data(), int64_t(x.size()), 1, 1), gin(ang.data(), int64_t(ang.size()), 1, 1)};
    st.group(0, in);
    Vec out(x.size());
    st.finalize(out);
    return out;
}

// ATTN handler: one q row against K / V rows [0, ctx) in 64-row tiles
Vec attention(const float* q, const float* K, const float* V, int64_t ctx, int64_t hd) {
    HandlerState st;
    st.op = Opcode::ATTN;
    st.out = {1, hd};
    st.out_stride = hd;
    st.prologue = gin(q, 1, hd, hd);
    const int64_t tiles = (ctx + 63) / 64;
    st.size = uint16_t(tiles);
    st.begin();
    for (int64_t t = 0; t < tiles; ++t) {
        const int64_t r0 = t * 64, rows = std::min<int64_t>(64, ctx - r0);
        const GroupInput in[2] = {gin(K + r0 * hd, rows, hd, hd, r0), gin(V + r0 * hd, rows, hd, hd, r0)};
        st.group(size_t(t), in);
    }
    Vec out(static_cast<size_t>(hd));
    st.finalize(out);
    return out;
}

const Vec& need(const std::map<std::string, Vec>& m, const std::string& k) {
    const auto it = m.find(k);
    if (it == m.end()) throw std::runtime_error("missing input " + k);
    return it->second;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: handler_pin in.bin out.bin config.json\n");
        return 2;
    }
    try {
        const auto T = read_all(argv[1]);
        const auto cfg = nlohmann::json::parse(std::string(argv[3]));
        const int64_t L = cfg.at("layers"), d = cfg.at("hidden"), hq = cfg.at("heads"), hkv = cfg.at("kv_heads"),
                      hd = cfg.at("head_dim"), ffn = cfg.at("ffn"), V = cfg.at("vocab"), pos = cfg.at("pos"),
                      gub = cfg.at("gu_block");
        const double theta = cfg.at("theta");
        const bool chain = cfg.value("chain", false);
        std::map<std::string, Vec> own;  // chain mode: this program's own intermediates
        auto src = [&](const std::string& k) -> const Vec& {
            const auto it = own.find(k);
            return chain && it != own.end() ? it->second : need(T, k);
        };
        const int64_t qr = hq * hd, kvr = hkv * hd, T_ctx = pos + 1, G = hq / hkv;
        std::map<std::string, Vec> out;
        Vec x = need(T, "x.in");  // hidden input of layer 0 (the embedding row)
        // rotary angles of the position (per row pair within a head), computed in double like the device
        Vec ang_q(static_cast<size_t>(qr)), ang_k(static_cast<size_t>(kvr));
        for (int64_t r = 0; r < qr; r += 2) ang_q[size_t(r)] = float(double(pos) * std::pow(theta, -double(r % hd) / double(hd)));
        for (int64_t r = 0; r < kvr; r += 2) ang_k[size_t(r)] = float(double(pos) * std::pow(theta, -double(r % hd) / double(hd)));
        for (int64_t l = 0; l < L; ++l) {
            const std::string P = "L" + std::to_string(l) + ".";
            const Vec& xin = l == 0 ? x : src("L" + std::to_string(l - 1) + ".x2");
            // qkv: RMSNORM -> MATVEC -> ROPE (q, k); v as is
            const Vec xn = rmsnorm(xin, need(T, P + "attn_norm"));
            const Vec y = matvec(need(T, P + "wqkv").data(), qr + 2 * kvr, d, xn);
            const Vec q = rope(Vec(y.begin(), y.begin() + qr), ang_q);
            const Vec k = rope(Vec(y.begin() + qr, y.begin() + qr + kvr), ang_k);
            out[P + "q"] = q;
            out[P + "k_row"] = k;
            out[P + "v_row"] = Vec(y.begin() + qr + kvr, y.end());
            if (chain) {  // the caches with this step's row appended at pos
                Vec kc2 = need(T, P + "kc"), vc2 = need(T, P + "vc");
                const int64_t Tc = int64_t(kc2.size()) / (hkv * hd);
                for (int64_t h = 0; h < hkv; ++h)
                    for (int64_t e = 0; e < hd; ++e) {
                        kc2[size_t((h * Tc + pos) * hd + e)] = k[size_t(h * hd + e)];
                        vc2[size_t((h * Tc + pos) * hd + e)] = y[size_t(qr + kvr + h * hd + e)];
                    }
                own[P + "q"] = q;
                own[P + "kc"] = std::move(kc2);
                own[P + "vc"] = std::move(vc2);
            }
            // attention over the device's caches (the appended row included), q from the device
            const Vec& qd = src(P + "q");
            const Vec& kc = src(P + "kc");
            const Vec& vc = src(P + "vc");
            const int64_t Tcap = int64_t(kc.size()) / (hkv * hd);
            Vec att(static_cast<size_t>(qr));
            for (int64_t h = 0; h < hq; ++h) {
                const int64_t kh = h / G;
                const Vec o = attention(qd.data() + h * hd, kc.data() + kh * Tcap * hd, vc.data() + kh * Tcap * hd, T_ctx, hd);
                std::copy(o.begin(), o.end(), att.begin() + h * hd);
            }
            out[P + "attn"] = att;
            own[P + "attn"] = att;
            // o-proj + residual, on the device's attention output
            const Vec ov = matvec(need(T, P + "wo").data(), d, qr, src(P + "attn"));
            out[P + "x1"] = elemwise(ov, &xin, 2);
            own[P + "x1"] = out[P + "x1"];
            // gate/up: RMSNORM -> MATVEC -> silu(gate) * up (rows in blocks [gate x gub/2 | up x gub/2])
            const Vec& x1 = src(P + "x1");
            const Vec x1n = rmsnorm(x1, need(T, P + "mlp_norm"));
            const Vec gu = matvec(need(T, P + "wgu").data(), 2 * ffn, d, x1n);
            Vec gate(static_cast<size_t>(ffn)), up(static_cast<size_t>(ffn));
            const int64_t hb = gub / 2;
            for (int64_t j = 0; j < ffn; ++j) {
                const int64_t blk = j / hb, jj = j % hb;
                gate[size_t(j)] = gu[size_t(blk * gub + jj)];
                up[size_t(j)] = gu[size_t(blk * gub + hb + jj)];
            }
            const Vec sg = elemwise(gate, nullptr, 1);
            out[P + "a"] = elemwise(sg, &up, 3);
            own[P + "a"] = out[P + "a"];
            // down + residual, on the device's activations
            const Vec dv = matvec(need(T, P + "wd").data(), d, ffn, src(P + "a"));
            out[P + "x2"] = elemwise(dv, &x1, 2);
            own[P + "x2"] = out[P + "x2"];
        }
        const Vec& xl = src("L" + std::to_string(L - 1) + ".x2");
        out["logits"] = matvec(need(T, "lm_head").data(), V, d, rmsnorm(xl, need(T, "final_norm")));
        write_all(argv[2], out);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "handler_pin: %s\n", e.what());
        return 1;
    }
    return 0;
}
