// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Restated functional µop interpreter (the reference's machine.cpp is absent
// from the tree). It follows:
//   - reference include/uopsim/machine.hpp:17-136 (types, run/termination),
//   - SPEC.md:301-427 (queues, slot allocator, in-order allocation),
//   - reference src/elaborate.cpp:108-344 (µop effects: which µops allocate,
//     SEND/RECV pops and pushes, STORE_LOCAL slot handoff, FREE size),
//   - reference src/fold.cpp:278-365 (control flow + DYNAMIC addressing),
// executing cores in the elaborator's round-robin certificate order with real
// tile data. Reference compute opcodes call the reference's own
// machine_detail::HandlerState (src/handlers.cpp, linked from oracle/_ref);
// decode extension opcodes use oracle/decode_semantics.hpp.
#include "interp.hpp"

#include <algorithm>
#include <array>
#include <cstring>
#include <deque>
#include <map>
#include <stdexcept>

#include "decode_semantics.hpp"
#include "handlers.hpp"  // reference src/handlers.hpp (HandlerState)
#include "uopsim/util.hpp"

namespace oracle {

namespace {

enum : uint32_t {
    LOAD = 0x01, STORE = 0x02, LOAD_DEP = 0x03, STORE_DEP = 0x04, LOAD_LOCAL = 0x05, STORE_LOCAL = 0x06, ALLOC = 0x07,
    FREE = 0x08, LOAD_WAIT = 0x09, MATVEC = 0x20, GEMM_TILE = 0x21, ATTN = 0x22, ROPE = 0x23, RMSNORM = 0x24,
    ELEMWISE = 0x25, EMBED = 0x26, GEMV = 0x27, RMS_GEMV = 0x28, GEMV_ADD = 0x29, ATTN_DECODE = 0x2A,
    ATTN_COMBINE = 0x2B, LOOP = 0x40, REPEAT = 0x41, CONTINUE_IF = 0x42, SET_ACC = 0x43, ADD_ACC = 0x44, HALT = 0x45,
    SET_ACC_MEM = 0x46,
};

// 16-byte word layout (reference include/uopsim/isa.hpp:126-130)
struct W {
    uint32_t op, flags, kind, rank, dep, flow, size, reg0, reg1;
    int32_t imm;
    uint32_t tensor;
    uint64_t payload;
};
W decode(const uint8_t* b) {
    W w{};
    w.op = b[0];
    w.flags = b[1] & 0xf;
    w.kind = (b[1] >> 4) & 3;
    w.rank = (b[1] >> 6) + 1;
    w.dep = uint32_t(b[2]) | (uint32_t(b[3]) << 8);
    w.flow = b[4];
    w.size = uint32_t(b[5]) | (uint32_t(b[6]) << 8);
    w.reg0 = b[7] >> 4;
    w.reg1 = b[7] & 0xf;
    uint32_t imm = 0;
    for (int i = 0; i < 4; ++i) imm |= uint32_t(b[8 + i]) << (8 * i);
    w.imm = int32_t(imm);
    w.tensor = uint32_t(b[8]) | (uint32_t(b[9]) << 8);
    w.payload = 0;
    for (int i = 0; i < 6; ++i) w.payload |= uint64_t(b[10 + i]) << (8 * i);
    return w;
}

struct HandlerShape {
    int pro, iter_pop, iter_push, res_pop, epi_push, res_push;
    bool streaming;
};
HandlerShape shape_of(uint32_t op) {  // reference isa.cpp:511-526 + decode extension
    switch (op) {
        case MATVEC: case GEMM_TILE: case ROPE: case RMSNORM: return {0, 2, 2, 1, 0, 1, false};
        case ATTN: return {1, 2, 2, 1, 1, 1, false};
        case ELEMWISE: return {0, 1, 1, 1, 0, 1, false};
        case EMBED: return {1, 1, 1, 1, 1, 1, false};
        case GEMV: return {1, 1, 1, 1, 1, 1, true};
        case RMS_GEMV: case GEMV_ADD: return {2, 1, 1, 1, 2, 1, true};
        case ATTN_DECODE: return {1, 2, 2, 1, 1, 1, true};
        case ATTN_COMBINE: return {0, 1, 1, 1, 0, 1, true};
        default: throw std::runtime_error("oracle: unknown compute opcode");
    }
}

struct Fifo {
    std::deque<Tile> q;
    size_t depth = 4;
};

struct Core {
    int sm = 0, vcc = -1;  // vcc < 0: VMC
    std::vector<W> s;
    size_t pc = 0;
    std::vector<std::pair<size_t, uint32_t>> loops;
    std::array<int64_t, 16> acc{};
    uint32_t phase = 0;
    std::vector<Tile> held;  // streaming job: prologue + group copies
    bool done() const { return pc >= s.size(); }
};

}  // namespace

struct Interp::Impl {
    const Program& p;
    std::map<int, std::vector<float>>& mem;  // storage descriptor -> values
    std::vector<Core> cores;
    std::map<int, uint32_t> used;
    std::map<uint32_t, Fifo> deps;
    std::map<std::pair<int, int>, Fifo> m2c, c2m;
    std::map<int, uint64_t> counters;
    uint64_t uops = 0;
    std::string stall;

    Impl(const Program& prog, std::map<int, std::vector<float>>& m) : p(prog), mem(m) {}

    const Desc& D(int i) const { return p.descs.at(size_t(i)); }
    int storage(int i) const { return D(i).view_of >= 0 ? D(i).view_of : i; }

    struct Addr {
        int desc = -1;
        int64_t off = 0;  // element offset of the tile origin in storage
        int rows_at = 0, cols_at = 0, row0 = 0, col0 = 0, tile_rows = 0, tile_cols = 0;
    };

    Addr tile_addr(int di, int64_t lin) const {
        const Desc& d = D(di);
        std::vector<int64_t> c(d.grid.size());
        for (size_t i = d.grid.size(); i-- > 0; lin /= d.grid[i]) c[i] = lin % d.grid[i];
        const size_t n = d.grid.size();
        const int64_t rows = d.shape.size() >= 2 ? d.shape[d.shape.size() - 2] : 1, cols = d.shape.back();
        const int64_t rt = c[n - 2], ct = c[n - 1];
        int64_t off = rt * d.tile_rows * cols + ct * d.tile_cols;
        int64_t plane = rows * cols;
        for (size_t i = n - 2; i-- > 0;) {  // leading dims, innermost first
            off += c[i] * plane;
            plane *= d.shape[i];
        }
        Addr a;
        a.desc = di;
        a.off = off;
        a.rows_at = int(std::min<int64_t>(d.tile_rows, rows - rt * d.tile_rows));
        a.cols_at = int(std::min<int64_t>(d.tile_cols, cols - ct * d.tile_cols));
        a.row0 = int(rt * d.tile_rows);
        a.col0 = int(ct * d.tile_cols);
        a.tile_rows = int(d.tile_rows);
        a.tile_cols = int(d.tile_cols);
        return a;
    }

    Addr resolve(const W& w, const Core& c) const {
        if (w.kind == 2) {
            const Desc& d = D(int(w.tensor));
            int64_t lin = 0;
            for (size_t i = 0; i < d.grid.size(); ++i) {
                const int64_t ci = i < w.rank ? int64_t((w.payload >> (12 * i)) & 0xfff) : 0;
                lin = lin * d.grid[i] + ci;
            }
            int di = int(w.tensor);
            if (w.flags & 4) {  // DYNAMIC: global tile index + acc, re-resolved (fold.cpp:278-293)
                const int64_t g = d.base + lin + c.acc[w.reg0];
                di = -1;
                for (size_t i = 0; i < p.descs.size(); ++i)
                    if (g >= p.descs[i].base && g < p.descs[i].base + p.descs[i].tile_count()) {
                        di = int(i);
                        break;
                    }
                if (di < 0) throw std::runtime_error("oracle: dynamic address outside every tensor");
                lin = g - D(di).base;
            }
            return tile_addr(di, lin);
        }
        if (w.kind == 1) {
            const Desc& d = D(int(w.tensor));
            int64_t off = int64_t(w.payload) + ((w.flags & 4) ? c.acc[w.reg0] : 0);
            const int64_t n = std::min<int64_t>(int64_t(std::max<uint32_t>(1, w.size)) * p.slot_size / d.elem_bytes(),
                                                d.elem_count() - off);
            Addr a;
            a.desc = int(w.tensor);
            a.off = off;
            a.rows_at = int(n);
            a.cols_at = 1;
            a.row0 = int(off);
            a.tile_rows = int(n);
            a.tile_cols = 1;
            return a;
        }
        return {};
    }

    Tile read_tile(const Addr& a) const {
        Tile t;
        t.rows = a.rows_at;
        t.cols = a.cols_at;
        t.stride = a.tile_cols;
        t.row0 = a.row0;
        t.col0 = a.col0;
        t.tensor = a.desc;
        t.bf16 = D(a.desc).dtype == 1;
        t.v.assign(size_t(a.tile_rows) * size_t(a.tile_cols), 0.f);
        const Desc& d = D(a.desc);
        const auto& src = mem.at(storage(a.desc));
        const int64_t cols = d.shape.back();
        for (int r = 0; r < a.rows_at; ++r)
            for (int c = 0; c < a.cols_at; ++c) t.v[size_t(r) * a.tile_cols + c] = src[size_t(a.off + r * cols + c)];
        return t;
    }

    // slot -> global: the payload is read with the target tile's row pitch,
    // exactly like the device store unit (engine.cu copy_out)
    void write_tile(const Addr& a, const Tile& t) {
        const Desc& d = D(a.desc);
        auto& dst = mem.at(storage(a.desc));
        const int64_t cols = d.shape.back();
        const bool bf = d.dtype == 1;
        for (int r = 0; r < a.rows_at; ++r)
            for (int c = 0; c < a.cols_at; ++c) {
                const size_t si = size_t(r) * size_t(a.tile_cols) + size_t(c);
                const float v = si < t.v.size() ? t.v[si] : 0.f;
                dst[size_t(a.off + r * cols + c)] = bf ? bf16_round(v) : v;
            }
    }

    bool block(const Core& c, const std::string& why) {
        stall = "sm" + std::to_string(c.sm) + (c.vcc < 0 ? ".vmc" : ".vcc" + std::to_string(c.vcc)) + ": " + why;
        return false;
    }

    bool step(Core& c) {
        const W& w = c.s[c.pc];
        switch (w.op) {
            case LOOP:
                if (w.size == 0) c.pc += size_t(w.imm) + 2;
                else {
                    c.loops.push_back({c.pc + 1, w.size});
                    ++c.pc;
                }
                ++uops;
                return true;
            case REPEAT:
                if (--c.loops.back().second > 0) c.pc = c.loops.back().first;
                else {
                    c.loops.pop_back();
                    ++c.pc;
                }
                ++uops;
                return true;
            case SET_ACC: c.acc[w.reg0] = w.imm; ++c.pc; ++uops; return true;
            case ADD_ACC: c.acc[w.reg0] += w.imm; ++c.pc; ++uops; return true;
            case SET_ACC_MEM: {
                const int idx = w.imm & 0xff;
                const int64_t mult = (w.imm >> 8) ? (w.imm >> 8) : 1;
                c.acc[w.reg0] = (idx < int(p.step.size()) ? p.step[size_t(idx)] : 0) * mult;
                ++c.pc;
                ++uops;
                return true;
            }
            case CONTINUE_IF:
                if (!c.loops.empty() && c.acc[w.reg0] == w.imm) {
                    size_t q = c.pc + 1;
                    for (int nest = 0; q < c.s.size(); ++q) {
                        if (c.s[q].op == LOOP) ++nest;
                        if (c.s[q].op == REPEAT && nest-- == 0) break;
                    }
                    c.pc = q;
                } else ++c.pc;
                ++uops;
                return true;
            case HALT: c.pc = c.s.size(); return true;
            default: break;
        }
        return c.vcc < 0 ? memory(c, w) : compute(c, w);
    }

    bool memory(Core& c, const W& w) {
        const Addr a = resolve(w, c);
        const auto key = std::make_pair(c.sm, int(w.reg1));
        uint32_t& u = used[c.sm];
        const bool allocates = (w.op == LOAD || w.op == LOAD_DEP || w.op == ALLOC || w.op == LOAD_WAIT) && w.size > 0;
        if (allocates && u + w.size > p.slot_budget) return block(c, "slot budget");
        if ((w.op == LOAD_DEP || w.op == LOAD_LOCAL) && deps[w.dep].q.empty()) return block(c, "dep empty");
        if ((w.op == STORE_DEP || w.op == STORE_LOCAL) && deps[w.dep].q.size() >= deps[w.dep].depth) return block(c, "dep full");
        if (w.op == LOAD_WAIT && counters[storage(a.desc)] < w.dep) return block(c, "counter");
        if ((w.flags & 1) && m2c[key].q.size() >= m2c[key].depth) return block(c, "m2c full");
        const size_t need = w.op == FREE ? w.size : 1;
        if ((w.flags & 2) && c2m[key].q.size() < need) return block(c, "c2m short");

        Tile carried;
        if (w.op == LOAD_DEP || w.op == LOAD_LOCAL) {
            carried = std::move(deps[w.dep].q.front());
            deps[w.dep].q.pop_front();
        }
        std::vector<Tile> popped;
        if (w.flags & 2)
            for (size_t i = 0; i < need; ++i) {
                popped.push_back(std::move(c2m[key].q.front()));
                c2m[key].q.pop_front();
            }
        if (allocates) u += w.size;
        Tile out;
        switch (w.op) {
            case LOAD:
            case LOAD_DEP:
            case LOAD_WAIT:
                out = read_tile(a);
                out.slots = uint16_t(w.size);
                break;
            case ALLOC:
                out.rows = a.rows_at;
                out.cols = a.cols_at;
                out.stride = a.tile_cols;
                out.row0 = a.row0;
                out.col0 = a.col0;
                out.tensor = a.desc;
                out.bf16 = a.desc >= 0 && D(a.desc).dtype == 1;
                out.v.assign(size_t(std::max(1, a.tile_rows)) * size_t(std::max(1, a.tile_cols)), 0.f);
                out.slots = uint16_t(w.size);
                break;
            case LOAD_LOCAL:
                out = std::move(carried);
                break;
            default:
                break;
        }
        if (w.flags & 1) m2c[key].q.push_back(std::move(out));
        if (w.op == FREE)
            for (const Tile& t : popped) u -= t.slots;
        if ((w.op == STORE || w.op == STORE_DEP) && (w.flags & 2)) {
            if (w.size > 0) {
                write_tile(a, popped.front());
                ++counters[storage(a.desc)];
            }
            u -= popped.front().slots;
        }
        if (w.op == STORE_DEP) deps[w.dep].q.push_back(Tile{});
        if (w.op == STORE_LOCAL) deps[w.dep].q.push_back(std::move(popped.front()));  // ownership moves, no free
        ++c.pc;
        ++uops;
        return true;
    }

    void run_reference(const W& w, std::vector<Tile>& in, Tile& res, const HandlerShape& hs) {
        using uopsim::machine_detail::GroupInput;
        uopsim::machine_detail::HandlerState st;
        st.op = static_cast<uopsim::isa::Opcode>(w.op);
        st.size = uint16_t(w.size);
        st.imm = w.imm;
        st.out = {res.rows, res.cols};
        st.out_stride = res.stride;
        auto gi_of = [](const Tile& t) {
            return GroupInput{{t.rows, t.cols}, std::span<const float>(t.v), t.stride, t.row0};
        };
        if (hs.pro) st.prologue = gi_of(in[0]);
        st.begin();
        for (uint32_t g = 0; g < w.size; ++g) {
            std::vector<GroupInput> grp;
            for (int i = 0; i < hs.iter_pop; ++i) grp.push_back(gi_of(in[size_t(hs.pro + g * hs.iter_pop + i)]));
            st.group(g, grp);
        }
        st.finalize(std::span<float>(res.v));
        if (res.bf16)
            for (float& x : res.v) x = bf16_round(x);
    }

    void run_decode(const Core& c, const W& w, std::vector<Tile>& in, Tile& res) {
        const float* hp = p.params.data() + (w.imm >> 8);
        if (w.op == GEMV || w.op == RMS_GEMV || w.op == GEMV_ADD) {
            const int pro = w.op == GEMV ? 1 : 2;
            std::vector<Tile*> groups;
            for (size_t i = size_t(pro); i < in.size(); ++i) groups.push_back(&in[i]);
            gemv(int(w.op), w.imm, hp, double(c.acc[w.reg0]), in[0], pro > 1 ? &in[1] : nullptr, groups, res);
        } else if (w.op == ATTN_DECODE) {
            std::vector<std::pair<Tile*, Tile*>> pages;
            for (size_t i = 1; i + 1 < in.size(); i += 2) pages.push_back({&in[i], &in[i + 1]});
            attn_decode(hp, c.acc[w.reg0], in[0], pages, res);
        } else {
            std::vector<Tile*> parts;
            for (auto& t : in) parts.push_back(&t);
            attn_combine(hp, parts, res);
        }
    }

    bool compute(Core& c, const W& w) {
        const HandlerShape hs = shape_of(w.op);
        auto& in = m2c[{c.sm, c.vcc}].q;
        auto& back = c2m[{c.sm, c.vcc}];
        if (!hs.streaming) {
            const size_t pops = size_t(hs.pro + hs.iter_pop * int(w.size) + hs.res_pop);
            const size_t pushes = size_t(hs.iter_push * int(w.size) + hs.epi_push + hs.res_push);
            if (in.size() < pops) return block(c, "m2c short");
            if (back.q.size() + pushes > back.depth) return block(c, "c2m full");
            std::vector<Tile> got;
            for (size_t i = 0; i < pops; ++i) {
                got.push_back(std::move(in.front()));
                in.pop_front();
            }
            Tile res = std::move(got.back());
            got.pop_back();
            run_reference(w, got, res, hs);
            for (uint32_t g = 0; g < w.size; ++g)
                for (int i = 0; i < hs.iter_push; ++i) back.q.push_back(got[size_t(hs.pro + int(g) * hs.iter_pop + i)]);
            for (int i = 0; i < hs.epi_push; ++i) back.q.push_back(got[size_t(i)]);
            back.q.push_back(std::move(res));
            ++c.pc;
            ++uops;
            return true;
        }
        // streaming: prologue, then one group at a time (released right away), then result
        if (c.phase == 0) {
            if (in.size() < size_t(hs.pro)) return block(c, "m2c short");
            c.held.clear();
            for (int i = 0; i < hs.pro; ++i) {
                c.held.push_back(std::move(in.front()));
                in.pop_front();
            }
            c.phase = 1;
            return true;
        }
        if (c.phase - 1 < w.size) {
            if (in.size() < size_t(hs.iter_pop)) return block(c, "m2c short");
            if (back.q.size() + size_t(hs.iter_push) > back.depth) return block(c, "c2m full");
            for (int i = 0; i < hs.iter_pop; ++i) {
                c.held.push_back(in.front());  // keep a copy for the arithmetic
                back.q.push_back(std::move(in.front()));
                in.pop_front();
            }
            ++c.phase;
            return true;
        }
        if (in.size() < size_t(hs.res_pop)) return block(c, "m2c short");
        if (back.q.size() + size_t(hs.epi_push + hs.res_push) > back.depth) return block(c, "c2m full");
        Tile res = std::move(in.front());
        in.pop_front();
        run_decode(c, w, c.held, res);
        for (int i = 0; i < hs.epi_push; ++i) back.q.push_back(c.held[size_t(i)]);
        back.q.push_back(std::move(res));
        c.held.clear();
        c.phase = 0;
        ++c.pc;
        ++uops;
        return true;
    }
};

Interp::Interp(const Program& p, std::map<int, std::vector<float>>& mem) : impl_(std::make_unique<Impl>(p, mem)) {
    for (const auto& cs : p.cores) {
        Core c;
        c.sm = cs.sm;
        c.vcc = cs.vcc;
        for (size_t i = 0; i + 16 <= cs.words.size(); i += 16) c.s.push_back(decode(cs.words.data() + i));
        for (const W& w : c.s)
            if (c.vcc < 0 && ((w.flags & 1) || (w.flags & 2))) {
                impl_->m2c[{c.sm, int(w.reg1)}].depth = p.local_depth;
                impl_->c2m[{c.sm, int(w.reg1)}].depth = p.local_depth;
            }
        if (c.vcc >= 0) {
            impl_->m2c[{c.sm, c.vcc}].depth = p.local_depth;
            impl_->c2m[{c.sm, c.vcc}].depth = p.local_depth;
        }
        impl_->cores.push_back(std::move(c));
    }
    for (const auto& q : p.queues) impl_->deps[q.dep].depth = q.depth;
}

Interp::~Interp() = default;

RunResult Interp::run() {
    auto& I = *impl_;
    for (bool moved = true; moved;) {
        moved = false;
        for (auto& c : I.cores)
            while (!c.done() && I.step(c)) moved = true;
    }
    RunResult r;
    r.completed = std::all_of(I.cores.begin(), I.cores.end(), [](const Core& c) { return c.done(); });
    r.uops = I.uops;
    r.stall = I.stall;
    for (const auto& kv : I.used) r.slots_all_free = r.slots_all_free && kv.second == 0;
    for (const auto& kv : I.m2c) r.queues_drained = r.queues_drained && kv.second.q.empty();
    for (const auto& kv : I.c2m) r.queues_drained = r.queues_drained && kv.second.q.empty();
    return r;
}

// synthetic contents (reference workload.cpp:411-435 + the `centered` extension)
std::vector<float> synthesize(const Desc& d, uint64_t seed) {
    std::vector<float> v(size_t(d.elem_count()), 0.f);
    uint64_t state = seed ^ uopsim::fnv1a(d.name);
    switch (d.init) {
        case 0: for (auto& x : v) x = uopsim::unit_float(state); break;
        case 1: break;
        case 2: std::fill(v.begin(), v.end(), 1.0f); break;
        case 3: for (size_t i = 0; i < v.size(); ++i) v[i] = float(i % 97); break;
        case 4: for (auto& x : v) x = (uopsim::unit_float(state) - 1.0f) * 0.5f * d.init_scale; break;
        default: break;
    }
    if (d.dtype == 1)
        for (auto& x : v) x = bf16_round(x);
    return v;
}

}  // namespace oracle
