// Decode lowering (ext): decode-kind graphs -> per-core µop streams.
//
// Differences from the reference lowering (emit.cpp), and why:
//  * Dependencies are per-tensor readiness counters, not per-consumer dep
//    ids: a load of a produced tensor becomes LOAD_WAIT with dep_id = the
//    number of tile stores that tensor receives in one launch. Broadcast
//    reads (every GEMV job reads the whole input vector) cost no ids, which
//    removes the 16-bit dep-id exhaustion the reference hits at 2 Llama-8B
//    layers (SURVEY finding 3).
//  * Handlers stream (HandlerIo::streaming): FREE µops are interleaved with
//    the weight loads with a per-job lag window, so a job's slot demand is
//    bounded by its window instead of its whole K sweep (finding 6).
//  * Jobs are placed by a global bytes-balanced greedy (least-loaded SM, then
//    least-loaded VCC on it) instead of `chunk % pairs`, because at decode
//    every SM streams weights and the per-SM byte total sets the step time.
//  * Unit routing by flow: dependency-gated loads (flow 2 -> LDU0), plain
//    loads/ALLOC (flow 1 -> LDU1), releases/stores of VCC v (flow 3+v ->
//    STU (3+v) mod 2), so weight prefetch never queues behind a dependency.
// The result is verified by the same elaborator (fix_deadlocks) and carries
// a baseline allocation certificate like every other program.
#include <algorithm>
#include <cmath>
#include <queue>

#include "jobs.hpp"
#include "uopsim/decode_abi.h"
#include "uopsim/util.hpp"

namespace uopsim::generator {

using isa::Opcode;
using isa::UopWord;
using workload::OpKind;

void refresh_certificate(LoweredProgram& p);

namespace {

struct DFetch {
    uint16_t tensor = 0;
    std::vector<uint16_t> coord;
    int8_t dyn_reg = -1;  // DYNAMIC accumulator register, -1 = static
};

struct DJob {
    Opcode compute{};
    int32_t imm = 0;
    uint8_t reg0 = 0;
    std::vector<DFetch> prologue;
    std::vector<std::vector<DFetch>> groups;
    DFetch out;
    uint64_t bytes = 0;
    uint32_t ordinal = 0;
    uint16_t sm = 0;
    uint8_t vcc = 0;
};

constexpr uint8_t kAccToken = 0;  // VMC: token id (embedding row)
constexpr uint8_t kAccPosSeg = 1; // VMC: pos * (head_dim / job_rows) (KV append)
constexpr uint8_t kAccPos = 1;    // VCC: position (rope)
constexpr uint8_t kAccCtx = 2;    // VCC: valid KV length (attention mask)

int64_t attr_int(const workload::OperatorNode& n, const char* key, int64_t dflt) {
    const auto it = n.attrs.find(key);
    return it == n.attrs.end() ? dflt : std::stoll(it->second);
}
double attr_num(const workload::OperatorNode& n, const char* key, double dflt) {
    const auto it = n.attrs.find(key);
    return it == n.attrs.end() ? dflt : std::stod(it->second);
}

class DecodeLowering {
  public:
    DecodeLowering(const workload::OperatorGraph& g, const costmodel::HardwareProfile& hw)
        : g_(g), hw_(hw), desc_(build_descriptors(g)) {}

    LoweredProgram run(const GenOptions& opt) {
        if (hw_.vmc_per_sm != 1) throw GeneratorError("decode lowering assumes one VMC per SM");
        const auto order = detail::topo_nodes(g_);
        uint32_t ordinal = 0;
        for (const auto* n : order) plan(*n, ordinal++);
        place();
        LoweredProgram p;
        p.descriptors = desc_;
        p.slot_budget = static_cast<uint16_t>(hw_.slot_budget());
        p.operator_count = ordinal;
        p.workload_hash = g_.content_hash();
        p.profile_name = hw_.name;
        p.input_seed = opt.input_seed;
        p.params = params_;
        p.step_scalars = VDC_STEP_MAX;
        p.slot_size = hw_.slot_size;
        p.vcc_per_sm = static_cast<uint16_t>(hw_.vcc_per_sm);
        p.sm_count = static_cast<uint16_t>(hw_.sm_count);
        p.local_queue_depth = 64;
        emit(p);
        p = fix_deadlocks(std::move(p));
        refresh_certificate(p);
        for (auto& [core, s] : p.streams)
            if (!s.empty()) s.back().flags |= isa::kFlagLast;
        const auto v = p.validate();
        if (!v.empty()) throw GeneratorError("decode program invalid: " + v.front().message);
        return p;
    }

  private:
    const workload::OperatorGraph& g_;
    const costmodel::HardwareProfile& hw_;
    std::vector<TileDescriptor> desc_;
    std::vector<DJob> jobs_;
    std::vector<float> params_;
    std::map<int32_t, uint32_t> stores_;  // storage tensor -> stores per launch
    std::map<int32_t, bool> produced_;

    int32_t storage(uint16_t t) const { return desc_[t].view_of >= 0 ? desc_[t].view_of : int32_t(t); }
    uint16_t idx(const std::string& name) const { return g_.tensor_index(name); }
    uint16_t slots(uint16_t t) const {
        return static_cast<uint16_t>(std::max<uint64_t>(1, ceil_div<uint64_t>(desc_[t].tile_bytes(), hw_.slot_size)));
    }
    DFetch at(uint16_t t, std::vector<uint16_t> c, int8_t dyn = -1) const { return {t, std::move(c), dyn}; }
    int32_t param_block(std::initializer_list<float> v) {
        const auto base = int32_t(params_.size());
        params_.insert(params_.end(), v);
        return base;
    }
    DJob& job(Opcode op, uint32_t ordinal) {
        DJob& j = jobs_.emplace_back();
        j.compute = op;
        j.ordinal = ordinal;
        return j;
    }

    void plan(const workload::OperatorNode& n, uint32_t ordinal) {
        for (const auto& o : n.outputs) produced_[storage(idx(o))] = true;
        switch (n.kind) {
            case OpKind::GEMV:
            case OpKind::RMS_GEMV:
            case OpKind::GEMV_ADD:
                plan_gemv(n, ordinal);
                break;
            case OpKind::ATTN_DECODE:
                plan_attention(n, ordinal);
                break;
            case OpKind::ATTN_COMBINE:
                plan_combine(n, ordinal);
                break;
            case OpKind::EMBED_ROW: {
                DJob& j = job(Opcode::ELEMWISE, ordinal);
                j.imm = 2;  // size-1 non-unary ELEMWISE = copy of group 0 (reference handlers.cpp:118-126)
                j.groups.push_back({at(idx(n.inputs[0]), {0, 0}, int8_t(kAccToken))});
                j.out = at(idx(n.outputs[0]), {0, 0});
                break;
            }
            default:
                throw GeneratorError("node " + n.id + ": reference kinds cannot be mixed into a decode program");
        }
    }

    void plan_gemv(const workload::OperatorNode& n, uint32_t ordinal) {
        const uint16_t w = idx(n.inputs[0]);
        const TileDescriptor& wd = desc_[w];
        // W is (M,K) or (P, M/P, K) planes of the same row-major storage
        const int64_t plane_rows = wd.rows(), M = wd.elem_count() / wd.cols(), R = attr_int(n, "job_rows", 16);
        const bool planar = wd.shape.size() == 3;
        if (plane_rows % R) throw GeneratorError("node " + n.id + ": job_rows must divide the rows of a weight plane");
        const int64_t swiglu = attr_int(n, "swiglu", 0);
        const bool rope = attr_int(n, "rope", 0) != 0;
        if (R % wd.tile_rows) throw GeneratorError("node " + n.id + ": job_rows must be a multiple of the weight tile rows");
        if (M % R) throw GeneratorError("node " + n.id + ": rows must be a multiple of job_rows");
        const int64_t ktiles = wd.grid.back();
        const Opcode op = n.kind == OpKind::GEMV ? Opcode::GEMV : n.kind == OpKind::RMS_GEMV ? Opcode::RMS_GEMV : Opcode::GEMV_ADD;

        // qkv split: outputs [q, kcache.seg, vcache.seg] with rows [q | k | v]
        int64_t qrows = M, kvrows = 0, head_dim = 0;
        if (n.outputs.size() == 3) {
            const TileDescriptor& kc = desc_[idx(n.outputs[1])];
            head_dim = kc.shape.back();
            kvrows = kc.shape[0] * head_dim;
            qrows = desc_[idx(n.outputs[0])].rows();
            if (qrows + 2 * kvrows != M) throw GeneratorError("node " + n.id + ": q/k/v rows do not add up to W rows");
            if (head_dim % R) throw GeneratorError("node " + n.id + ": job_rows must divide head_dim");
        }
        const int32_t pbase = param_block({float(attr_num(n, "eps", 1e-5)), float(attr_num(n, "theta", 10000.0)),
                                           float(head_dim), float(rope ? qrows + kvrows : 0), float(swiglu)});
        const int32_t variant = (rope ? VDC_GEMV_ROPE : 0) | (swiglu ? VDC_GEMV_SWIGLU : 0);
        for (int64_t j = 0; j < M / R; ++j) {
            DJob& jb = job(op, ordinal);
            jb.imm = (pbase << 8) | variant;
            jb.reg0 = kAccPos;
            jb.prologue.push_back(at(idx(n.inputs[1]), {0, 0}));
            if (n.kind != OpKind::GEMV) {
                const uint16_t third = idx(n.inputs[2]);
                jb.prologue.push_back(n.kind == OpKind::RMS_GEMV ? at(third, {0, 0}) : at(third, {uint16_t(j), 0}));
            }
            const int64_t plane = (j * R) / plane_rows, prow = (j * R) % plane_rows;
            for (int64_t rt = prow / wd.tile_rows; rt < (prow + R) / wd.tile_rows; ++rt)
                for (int64_t kt = 0; kt < ktiles; ++kt)
                    jb.groups.push_back({planar ? at(w, {uint16_t(plane), uint16_t(rt), uint16_t(kt)})
                                                : at(w, {uint16_t(rt), uint16_t(kt)})});
            const int64_t r0 = j * R;
            if (n.outputs.size() == 3 && r0 >= qrows) {
                const bool is_k = r0 < qrows + kvrows;
                const int64_t local = r0 - qrows - (is_k ? 0 : kvrows);
                const uint16_t cache = idx(n.outputs[is_k ? 1 : 2]);
                jb.out = at(cache, {uint16_t(local / head_dim), 0, uint16_t((local % head_dim) / R)}, int8_t(kAccPosSeg));
                pos_seg_mult_ = int32_t(head_dim / R);
            } else {
                // output tile j holds rows [j*out_rows, (j+1)*out_rows), out_rows = R (R/2 for swiglu)
                const TileDescriptor& od = desc_[idx(n.outputs[0])];
                if (od.tile_rows != (swiglu ? R / 2 : R))
                    throw GeneratorError("node " + n.id + ": output tile rows must equal the job's output rows");
                jb.out = at(idx(n.outputs[0]), {uint16_t(j), 0});
            }
        }
    }

    void plan_attention(const workload::OperatorNode& n, uint32_t ordinal) {
        const uint16_t q = idx(n.inputs[0]), kc = idx(n.inputs[1]), vc = idx(n.inputs[2]), part = idx(n.outputs[0]);
        const TileDescriptor& kd = desc_[kc];
        const int64_t hkv = kd.shape[0], hd = kd.shape[2], page_rows = kd.tile_rows;
        const int64_t grp = desc_[q].tile_rows / hd;
        const int64_t pages = attr_int(n, "ctx_pages", 1), per = attr_int(n, "pages_per_job", 1);
        const int64_t splits = ceil_div(pages, per);
        const int32_t pbase = param_block({float(1.0 / std::sqrt(double(hd))), float(hd), float(grp), float(page_rows)});
        for (int64_t h = 0; h < hkv; ++h)
            for (int64_t s = 0; s < splits; ++s) {
                DJob& jb = job(Opcode::ATTN_DECODE, ordinal);
                jb.imm = pbase << 8;
                jb.reg0 = kAccCtx;
                jb.prologue.push_back(at(q, {uint16_t(h), 0}));
                for (int64_t pg = s * per; pg < std::min(pages, (s + 1) * per); ++pg)
                    jb.groups.push_back({at(kc, {uint16_t(h), uint16_t(pg), 0}), at(vc, {uint16_t(h), uint16_t(pg), 0})});
                jb.out = at(part, {uint16_t(h * splits + s), 0});
            }
        attn_splits_[part] = splits;
    }

    void plan_combine(const workload::OperatorNode& n, uint32_t ordinal) {
        const uint16_t part = idx(n.inputs[0]), out = idx(n.outputs[0]);
        const int64_t splits = attn_splits_.at(uint16_t(storage(part)));
        const TileDescriptor& pd = desc_[part];
        const int64_t hd = pd.tile_cols - 2;
        const int64_t per_tile = pd.tile_rows;  // partial rows per tile (splits * G when viewed per head)
        const int64_t grp = desc_[storage(part)].tile_rows;
        const int64_t hkv = pd.rows() / (splits * grp);
        const int64_t tiles_per_head = (splits * grp) / per_tile;
        const int32_t pbase = param_block({float(hd), float(grp)});
        for (int64_t h = 0; h < hkv; ++h) {
            DJob& jb = job(Opcode::ATTN_COMBINE, ordinal);
            jb.imm = pbase << 8;
            for (int64_t s = 0; s < tiles_per_head; ++s) jb.groups.push_back({at(part, {uint16_t(h * tiles_per_head + s), 0})});
            jb.out = at(out, {uint16_t(h), 0});
        }
    }

    // bytes-balanced placement: least-loaded SM, then least-loaded VCC on it
    void place() {
        const uint32_t sms = hw_.sm_count, vccs = hw_.vcc_per_sm;
        std::vector<uint64_t> sm_bytes(sms, 0), vcc_bytes(size_t(sms) * vccs, 0);
        using Entry = std::pair<uint64_t, uint32_t>;
        std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
        for (uint32_t s = 0; s < sms; ++s) heap.push({0, s});
        for (DJob& j : jobs_) {
            j.bytes = 0;
            for (const auto& f : j.prologue) j.bytes += desc_[f.tensor].tile_bytes();
            for (const auto& grp : j.groups)
                for (const auto& f : grp) j.bytes += desc_[f.tensor].tile_bytes();
            const auto [load, sm] = heap.top();
            heap.pop();
            uint32_t best = 0;
            for (uint32_t v = 1; v < vccs; ++v)
                if (vcc_bytes[sm * vccs + v] < vcc_bytes[sm * vccs + best]) best = v;
            j.sm = uint16_t(sm);
            j.vcc = uint8_t(best);
            vcc_bytes[sm * vccs + best] += j.bytes + 1;
            sm_bytes[sm] = load + j.bytes + 1;
            heap.push({sm_bytes[sm], sm});
        }
        for (const DJob& j : jobs_) ++stores_[storage(j.out.tensor)];
    }

    UopWord fetch_word(const DFetch& f, uint8_t vcc) const {
        UopWord u;
        const int32_t st = storage(f.tensor);
        const bool gated = produced_.count(st) && stores_.count(st);
        u.opcode = gated ? Opcode::LOAD_WAIT : Opcode::LOAD;
        if (gated) u.dep_id = static_cast<uint16_t>(stores_.at(st));
        u.flags = isa::kFlagSend;
        u.flow = gated ? 2 : 1;
        u.reg1 = vcc;
        u.size = slots(f.tensor);
        u.addr = isa::AddressSpec::tile(f.tensor, f.coord);
        if (f.dyn_reg >= 0) {
            u.flags |= isa::kFlagDynamic;
            u.reg0 = uint8_t(f.dyn_reg);
        }
        return u;
    }

    // per-VCC job stream (VMC side) with the streaming FREE lag window
    void job_stream(const DJob& j, int32_t task, std::vector<std::pair<UopWord, UopMeta>>& out) const {
        static const isa::HandlerTable table = isa::default_handler_table();
        const isa::HandlerIo& io = table.handler(j.compute).io;
        const UopMeta meta{j.ordinal, task, -1};
        const uint8_t stu_flow = uint8_t(3 + j.vcc);
        auto release = [&](int n) {
            UopWord fr;
            fr.opcode = Opcode::FREE;
            fr.flags = isa::kFlagRecv;
            fr.flow = stu_flow;
            fr.reg1 = j.vcc;
            fr.size = uint16_t(n);
            out.push_back({fr, meta});
        };
        int pro_slots = 0, grp_slots = 0;
        for (const auto& f : j.prologue) pro_slots += slots(f.tensor);
        for (const auto& grp : j.groups) {
            int s = 0;
            for (const auto& f : grp) s += slots(f.tensor);
            grp_slots = std::max(grp_slots, s);
        }
        const int res_slots = slots(j.out.tensor);
        const int half = int(hw_.slot_budget() / std::max<uint32_t>(1, hw_.vcc_per_sm));
        int window = io.streaming ? std::max(1, (half - pro_slots - res_slots) / std::max(1, grp_slots)) : int(j.groups.size());
        if (io.streaming && pro_slots + res_slots + grp_slots > half)
            throw GeneratorError("decode job does not fit half the slot budget");

        for (const auto& f : j.prologue) out.push_back({fetch_word(f, j.vcc), meta});
        const int n = int(j.groups.size());
        for (int gi = 0; gi < n; ++gi) {
            // release group gi-window before loading group gi: the job never
            // holds more than prologue + window groups (+ result at the end)
            if (io.streaming && gi >= window) release(io.iter_pushes_c2m);
            for (const auto& f : j.groups[size_t(gi)]) out.push_back({fetch_word(f, j.vcc), meta});
        }
        UopWord alloc;
        alloc.opcode = Opcode::ALLOC;
        alloc.flags = isa::kFlagSend;
        alloc.flow = 1;
        alloc.reg1 = j.vcc;
        alloc.size = uint16_t(res_slots);
        alloc.addr = isa::AddressSpec::tile(j.out.tensor, j.out.coord);
        out.push_back({alloc, meta});
        if (io.streaming) {
            const int pending = std::min(n, window) * io.iter_pushes_c2m;
            if (pending) release(pending);
            if (io.epilogue_pushes_c2m) release(io.epilogue_pushes_c2m);
        } else {
            release(io.release_pushes_c2m(n));
        }
        UopWord st;
        st.opcode = Opcode::STORE;
        st.flags = isa::kFlagRecv;
        st.flow = stu_flow;
        st.reg1 = j.vcc;
        st.size = uint16_t(res_slots);
        st.addr = isa::AddressSpec::tile(j.out.tensor, j.out.coord);
        if (j.out.dyn_reg >= 0) {
            st.flags |= isa::kFlagDynamic;
            st.reg0 = uint8_t(j.out.dyn_reg);
        }
        out.push_back({st, meta});
    }

    void emit(LoweredProgram& p) {
        const uint32_t sms = hw_.sm_count, vccs = hw_.vcc_per_sm;
        // per (sm, vcc) job lists in program order
        std::vector<std::vector<size_t>> lists(size_t(sms) * vccs);
        for (size_t i = 0; i < jobs_.size(); ++i) lists[size_t(jobs_[i].sm) * vccs + jobs_[i].vcc].push_back(i);
        int32_t task = 0;
        std::vector<int32_t> task_of(jobs_.size());
        for (size_t i = 0; i < jobs_.size(); ++i) task_of[i] = task++;

        auto ctl = [](Opcode op, uint8_t reg, int32_t imm) {
            UopWord c;
            c.opcode = op;
            c.reg0 = reg;
            c.imm = imm;
            return c;
        };
        for (uint32_t sm = 0; sm < sms; ++sm) {
            const CoreId vmc = CoreId::vmc(uint16_t(sm));
            auto& vs = p.streams[vmc];
            auto& vm = p.meta[vmc];
            vs.push_back(ctl(Opcode::SET_ACC_MEM, kAccToken, VDC_STEP_TOKEN));
            vm.push_back({0, -1, -1});
            vs.push_back(ctl(Opcode::SET_ACC_MEM, kAccPosSeg, VDC_STEP_POS | (pos_seg_mult_ << 8)));
            vm.push_back({0, -1, -1});
            // merge the per-VCC job streams by cumulative bytes (keeps both fed)
            std::vector<std::vector<std::pair<UopWord, UopMeta>>> parts(vccs);
            std::vector<size_t> cursor(vccs, 0);
            std::vector<uint64_t> fed(vccs, 0);
            for (uint32_t v = 0; v < vccs; ++v) {
                for (size_t ji : lists[size_t(sm) * vccs + v]) job_stream(jobs_[ji], task_of[ji], parts[v]);
                const CoreId vcc = CoreId::vcc_id(uint16_t(sm), uint8_t(v));
                auto& cs = p.streams[vcc];
                auto& cm = p.meta[vcc];
                cs.push_back(ctl(Opcode::SET_ACC_MEM, kAccPos, VDC_STEP_POS));
                cm.push_back({0, -1, -1});
                cs.push_back(ctl(Opcode::SET_ACC_MEM, kAccCtx, VDC_STEP_CTX));
                cm.push_back({0, -1, -1});
                for (size_t ji : lists[size_t(sm) * vccs + v]) {
                    const DJob& j = jobs_[ji];
                    UopWord cu;
                    cu.opcode = j.compute;
                    cu.size = uint16_t(j.groups.size());
                    cu.imm = j.imm;
                    cu.reg0 = j.reg0;
                    cu.flow = 1;
                    cs.push_back(cu);
                    cm.push_back({j.ordinal, task_of[ji], -1});
                }
            }
            // A dependency-gated load of operator o may not precede any µop of an
            // earlier operator on this VMC: in the sequential (certificate) model
            // the VMC would block on a counter whose producer store sits later in
            // its own stream.
            auto next_op = [&](uint32_t v) {
                return cursor[v] < parts[v].size() ? parts[v][cursor[v]].second.op : UINT32_MAX;
            };
            for (;;) {
                int pick = -1;
                for (uint32_t v = 0; v < vccs; ++v)
                    if (cursor[v] < parts[v].size() && (pick < 0 || fed[v] < fed[size_t(pick)])) pick = int(v);
                if (pick < 0) break;
                const auto& cand = parts[size_t(pick)][cursor[size_t(pick)]];
                if (cand.first.opcode == Opcode::LOAD_WAIT)
                    for (uint32_t v = 0; v < vccs; ++v)
                        if (int(v) != pick && next_op(v) < cand.second.op) {
                            pick = int(v);
                            break;
                        }
                const auto& [u, m] = parts[size_t(pick)][cursor[size_t(pick)]++];
                if (isa::is_load_class(u.opcode) && u.opcode != Opcode::ALLOC) fed[size_t(pick)] += desc_[u.addr.tensor].tile_bytes();
                vs.push_back(u);
                vm.push_back(m);
            }
        }
    }

    std::map<uint16_t, int64_t> attn_splits_;
    int32_t pos_seg_mult_ = 1;
};

}  // namespace

LoweredProgram lower_decode(const workload::OperatorGraph& g, const costmodel::HardwareProfile& hw, const GenOptions& opt) {
    return DecodeLowering(g, hw).run(opt);
}

}  // namespace uopsim::generator
