// C-ABI over the host builder (include/vdc.h, "host program builder").
// No exception crosses the boundary: every entry point returns a VDC_* code
// and leaves the message in vdc_last_error().
#include <cstring>
#include <sstream>

#include <nlohmann/json.hpp>

#include "capi_common.hpp"
#include "uopsim/decode.hpp"
#include "uopsim/generator.hpp"
#include "uopsim/ring_abi.h"
#include "uopsim/util.hpp"
#include "vdc.h"

namespace vdc_dev {
int synthesize_launch(void* out, uint64_t n, int bf16, int init, float scale, uint64_t state0, uint32_t layout, int64_t rows,
                      int64_t cols, void* stream);
}

using json = nlohmann::ordered_json;
using namespace uopsim;

namespace vdc_impl {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
    set_error(msg);
    return code;
}

int classify(const std::exception& e) {
    if (dynamic_cast<const generator::DeadlockError*>(&e)) return VDC_ERR_DEADLOCK;
    if (dynamic_cast<const workload::WorkloadError*>(&e) || dynamic_cast<const costmodel::ProfileError*>(&e) ||
        dynamic_cast<const isa::EncodeError*>(&e) || dynamic_cast<const isa::DecodeError*>(&e) ||
        dynamic_cast<const generator::GeneratorError*>(&e) || dynamic_cast<const json::exception*>(&e) ||
        dynamic_cast<const std::invalid_argument*>(&e) || dynamic_cast<const std::out_of_range*>(&e))
        return VDC_ERR_INPUT;
    return VDC_ERR_INTERNAL;
}

namespace {

costmodel::HardwareProfile profile_from(const json& j) {
    if (j.contains("builtin")) {
        auto p = costmodel::builtin_profile(j.at("builtin").get<std::string>());
        if (!p) throw costmodel::ProfileError("unknown builtin profile");
        auto hw = *p;
        if (j.contains("sm_count")) hw.sm_count = j.at("sm_count").get<uint32_t>();
        if (j.contains("stu_count")) hw.stu_count = j.at("stu_count").get<uint32_t>();
        hw.validate();
        return hw;
    }
    if (j.contains("test")) {
        const auto& t = j.at("test");
        return costmodel::make_test_profile(t.at(0).get<std::string>(), t.at(1).get<uint32_t>(), t.at(2).get<double>(),
                                            t.at(3).get<double>(), t.size() > 4 ? t.at(4).get<uint32_t>() : 32u);
    }
    return costmodel::parse_profile(j.dump());
}

workload::SplitAxis axis_from(const std::string& s) {
    for (auto a : {workload::SplitAxis::M, workload::SplitAxis::N, workload::SplitAxis::K,
                   workload::SplitAxis::token_block, workload::SplitAxis::head_block})
        if (workload::axis_name(a) == s) return a;
    throw std::invalid_argument("bad axis " + s);
}

decode::ModelConfig model_from(const json& j) {
    const std::string preset = j.value("preset", std::string("tiny"));
    decode::ModelConfig m = preset == "llama3-8b"    ? decode::llama3_8b()
                            : preset == "qwen3-8b"   ? decode::qwen3_8b()
                            : preset == "llama3-70b" ? decode::llama3_70b()
                            : preset == "tiny"       ? decode::tiny_llama()
                                                     : throw std::invalid_argument("unknown model preset " + preset);
    m.layers = j.value("layers", m.layers);
    m.hidden = j.value("hidden", m.hidden);
    m.heads = j.value("heads", m.heads);
    m.kv_heads = j.value("kv_heads", m.kv_heads);
    m.head_dim = j.value("head_dim", m.head_dim);
    m.ffn = j.value("ffn", m.ffn);
    m.vocab = j.value("vocab", m.vocab);
    m.eps = j.value("eps", m.eps);
    m.theta = j.value("theta", m.theta);
    m.scaled_init = j.value("scaled_init", m.scaled_init);
    m.qk_norm = j.value("qk_norm", m.qk_norm);
    if (j.contains("dtype")) {
        auto e = workload::elem_from_name(j.at("dtype").get<std::string>());
        if (!e) throw std::invalid_argument("bad dtype");
        m.dtype = *e;
    }
    return m;
}

decode::LayoutConfig layout_from(const json& j) {
    decode::LayoutConfig l;
    l.ctx_pages = j.value("ctx_pages", l.ctx_pages);
    l.page_rows = j.value("page_rows", l.page_rows);
    l.max_ctx = j.value("max_ctx", std::max(l.max_ctx, l.ctx_pages * l.page_rows));
    l.pages_per_job = j.value("pages_per_job", l.pages_per_job);
    l.job_rows = j.value("job_rows", l.job_rows);
    l.head_job_rows = j.value("head_job_rows", l.head_job_rows);
    l.gu_block = j.value("gu_block", l.gu_block);
    l.wtile_bytes = j.value("wtile_bytes", l.wtile_bytes);
    l.ring = j.value("ring", l.ring);
    l.tp_world = j.value("tp_world", l.tp_world);
    l.tp_rank = j.value("tp_rank", l.tp_rank);
    if (j.contains("tp_partials")) {
        const std::string tpp = j.at("tp_partials").get<std::string>();
        if (tpp != "bf16" && tpp != "f32") throw std::invalid_argument("layout.tp_partials must be \"bf16\" or \"f32\"");
        l.tp_bf16_partials = tpp == "bf16";
    }
    l.batch = j.value("batch", l.batch);
    l.argmax = j.value("argmax", l.argmax);
    l.feedback = j.value("feedback", l.feedback);
    l.prefill = j.value("prefill", l.prefill);
    l.req_pages = j.value("req_pages", l.req_pages);
    l.pool_pages = j.value("pool_pages", l.pool_pages);
    l.attn_job_cost = j.value("attn_job_cost", l.attn_job_cost);
    return l;
}

}  // namespace

ProgramBox* build(const std::string& request) {
    const json req = json::parse(request);
    auto box = std::make_unique<ProgramBox>();
    const auto hw = profile_from(req.value("profile", json{{"builtin", "b200"}}));
    generator::GenOptions opt;
    const json jo = req.value("options", json::object());
    opt.theta = jo.value("theta", 1.2);
    opt.flows = jo.value("flows", true);
    opt.fusion = jo.value("fusion", true);
    opt.fold = jo.value("fold", true);
    opt.input_seed = jo.value("seed", uint64_t(0));

    workload::OperatorGraph g;
    const bool ring = req.value("engine", std::string("reference")) == "ring";
    if (req.contains("model")) {
        auto layout = layout_from(req.value("layout", json::object()));
        layout.ring = layout.ring || ring;
        g = decode::build_decode_graph(model_from(req.at("model")), layout);
    } else {
        g = workload::parse_workload(req.at("workload").dump());
    }
    box->graph_json = workload::serialize_workload(g);

    bool decode_graph = false;
    for (const auto& n : g.nodes) decode_graph = decode_graph || workload::is_decode_kind(n.kind);
    std::map<std::string, workload::TilingChoice> tilings;
    if (decode_graph && ring) {
        const bool batched = req.value("layout", json::object()).value("batch", 0) >= 1;
        box->program = generator::lower_decode_ring(g, hw, opt, req.value("ring_slots", batched ? 8 : 12));
        const auto v = generator::validate_ring_program(box->program);
        if (!v.empty()) throw generator::GeneratorError("ring program invalid: " + v.front().message);
    } else if (decode_graph) {
        box->program = generator::generate(g, hw, opt);
    } else if (req.contains("tilings") || req.contains("passes")) {
        if (req.contains("tilings")) {
            for (const auto& n : g.nodes) tilings[n.id] = workload::TilingChoice{n.id, {}};
            for (const auto& [node, parts] : req.at("tilings").items()) {
                workload::TilingChoice c{node, {}};
                for (const auto& [ax, v] : parts.items()) c.parts[axis_from(ax)] = v.get<int>();
                tilings[node] = c;
            }
        } else {
            tilings = generator::select_tilings(g, hw, opt.theta);
        }
        const auto passes = req.value("passes", std::vector<std::string>{"flows", "fusion", "fold", "deadlock", "redundancy", "last"});
        auto p = generator::lower(g, tilings, hw);
        p.input_seed = opt.input_seed;
        for (const auto& ps : passes) {
            if (ps == "flows") p = generator::assign_virtual_flows(std::move(p));
            else if (ps == "flows_off") {
                for (auto& [core, s] : p.streams)
                    for (auto& u : s)
                        if (u.klass() != isa::OpClass::control) u.flow = 1;
            } else if (ps == "fusion") p = generator::apply_dynamic_fusion(std::move(p));
            else if (ps == "fold") p = generator::fold_loops(std::move(p));
            else if (ps == "deadlock") p = generator::fix_deadlocks(std::move(p));
            else if (ps == "redundancy") {
                p = generator::eliminate_redundant_dependencies(std::move(p));
                p = generator::fix_deadlocks(std::move(p));
            } else if (ps == "last") {
                for (auto& [core, s] : p.streams)
                    if (!s.empty()) s.back().flags |= isa::kFlagLast;
            } else throw std::invalid_argument("unknown pass " + ps);
        }
        box->program = std::move(p);
    } else {
        tilings = generator::select_tilings(g, hw, opt.theta);
        box->program = generator::generate(g, hw, opt);
    }
    json jt = json::object();
    for (const auto& [node, c] : tilings) {
        json parts = json::object();
        for (const auto& [ax, v] : c.parts) parts[std::string(workload::axis_name(ax))] = v;
        jt[node] = parts;
    }
    box->tilings_json = jt.dump();
    box->hw = hw;
    box->finish();
    return box.release();
}

void ProgramBox::finish() {
    generator::LoweredProgram& p = program;
    if (!p.ring_slots) p.slot_size = hw.slot_size;
    p.vcc_per_sm = p.ring_slots ? uint16_t(1) : uint16_t(hw.vcc_per_sm);
    p.sm_count = uint16_t(hw.sm_count);
    uint32_t sms = hw.sm_count;
    for (const auto& kv : p.streams) sms = std::max<uint32_t>(sms, uint32_t(kv.first.sm) + 1);
    sm_count = sms;
    vcc_per_sm = p.vcc_per_sm;
    cores.clear();
    words.clear();
    for (uint32_t sm = 0; sm < sms; ++sm) {
        cores.push_back(generator::CoreId::vmc(uint16_t(sm)));
        for (uint32_t v = 0; v < vcc_per_sm; ++v) cores.push_back(generator::CoreId::vcc_id(uint16_t(sm), uint8_t(v)));
    }
    for (const auto& c : cores) {
        const auto it = p.streams.find(c);
        words.push_back(it == p.streams.end() ? std::vector<uint8_t>{} : isa::encode_stream(it->second));
    }
}

std::string ProgramBox::text(int mode) const {
    if (mode == 3) {  // every core's stream unfolded (LOOP/REPEAT expanded), encoded words as hex
        static const char* hexd = "0123456789abcdef";
        json out, hex = json::object();
        out["ok"] = true;
        for (const auto& c : cores) {
            if (!program.streams.count(c)) continue;
            const auto enc = isa::encode_stream(generator::unfold_stream(program, c));
            std::string h;
            h.reserve(enc.size() * 2);
            for (uint8_t b : enc) {
                h.push_back(hexd[b >> 4]);
                h.push_back(hexd[b & 15]);
            }
            hex[c.name()] = h;
        }
        out["unfolded_words"] = hex;
        return out.dump();
    }
    const bool with_words = mode == 1, summary = mode == 2;
    json out;
    out["ok"] = true;
    out["tilings"] = json::parse(tilings_json.empty() ? "{}" : tilings_json);
    json streams = json::object(), hex = json::object();
    static const char* digits = "0123456789abcdef";
    for (size_t i = 0; i < cores.size() && !summary; ++i) {
        const auto it = program.streams.find(cores[i]);
        if (it == program.streams.end()) continue;
        streams[cores[i].name()] = generator::serialize_stream(program, cores[i]);
        if (with_words) {
            std::string h;
            h.reserve(words[i].size() * 2);
            for (uint8_t b : words[i]) {
                h.push_back(digits[b >> 4]);
                h.push_back(digits[b & 15]);
            }
            hex[cores[i].name()] = h;
        }
    }
    out["streams"] = streams;
    if (with_words) out["words"] = hex;
    out["total_uops"] = program.total_uops();
    if (!summary) {
        out["sidecar"] = generator::serialize_sidecar(program);
        out["certificate_ok"] = program.ring_slots ? generator::validate_ring_program(program).empty()
                                                   : generator::replay_certificate(program);
        try {
            out["makespan_estimate"] = program.ring_slots ? json(nullptr) : json(generator::estimate_makespan(program, hw));
        } catch (const std::exception&) {
            out["makespan_estimate"] = nullptr;
        }
    }
    json descs = json::array();
    for (const auto& d : program.descriptors)
        descs.push_back({{"name", d.tensor}, {"index", d.index}, {"base", d.base}, {"shape", d.shape},
                         {"grid", d.grid}, {"tile", {d.tile_rows, d.tile_cols}}, {"dtype", std::string(workload::elem_name(d.elem))},
                         {"view_of", d.view_of}, {"external", d.external}, {"state", d.state},
                         {"init", int(d.init)}, {"init_scale", d.init_scale},
                         {"symmetric", d.symmetric}, {"tma", d.tma}});
    out["descriptors"] = descs;
    out["params"] = program.params;
    out["ring_slots"] = program.ring_slots;
    json jobs = json::array();
    for (const auto& jb : program.jobs)
        jobs.push_back({{"op", jb.op}, {"flags", jb.flags}, {"r0", jb.r0}, {"r1", jb.r1}, {"k", jb.k},
                        {"tile", {jb.tile_rows, jb.tile_cols}}, {"x", {jb.x_t, jb.x_off, jb.x_need}},
                        {"a", {jb.a_t, jb.a_off, jb.a_need}}, {"b", {jb.b_t, jb.b_off, jb.b_need}},
                        {"o", {jb.o_t, jb.o_off}}, {"o2", {jb.o2_t, jb.o2_off}}, {"out_row0", jb.out_row0}, {"head_dim", jb.head_dim},
                        {"split", jb.split}, {"arrive", {jb.arrive_ctr, jb.arrive_need}},
                        {"group", jb.group}, {"block", jb.block}, {"cache_rows", jb.cache_rows},
                        {"eps", jb.eps}, {"theta", jb.theta}, {"scale", jb.scale}, {"kt", {jb.kt0, jb.kt1}},
                        {"req", jb.req}, {"part", {jb.part_t, jb.part_off}}, {"x2", {jb.x2_t, jb.x2_need}},
                        {"o3", {jb.o3_t, jb.w3_t}}, {"lead_pad", jb.lead_pad}});
    out["jobs"] = jobs;
    if (program.batch)
        out["batch"] = {{"nb", program.batch}, {"npad", program.npad}, {"maxp", program.maxp},
                        {"page_table_off", program.page_table_off}, {"page_table", program.page_table}};
    json queues = json::array();
    for (const auto& q : program.queues)
        queues.push_back({{"dep", q.dep_id}, {"depth", q.depth}, {"local", q.local}, {"producer_sm", q.producer.sm},
                          {"consumer_sm", q.consumer.sm}});
    out["queues"] = queues;
    out["slot_size"] = program.slot_size;
    out["ldu_count"] = hw.ldu_count;
    out["stu_count"] = hw.stu_count;
    out["step_scalars"] = program.step_scalars;
    out["slot_budget"] = program.slot_budget;
    out["local_queue_depth"] = program.local_queue_depth;
    out["sm_count"] = sm_count;
    out["vcc_per_sm"] = vcc_per_sm;
    out["graph"] = json::parse(graph_json.empty() ? "{}" : graph_json);
    return out.dump();
}

}  // namespace vdc_impl

using namespace vdc_impl;

extern "C" {

const char* vdc_last_error(void) { return g_last_error.c_str(); }
const char* vdc_version(void) { return "vdc-b200 0.1 (sm_100a)"; }

int vdc_program_build(const char* request_json, vdc_program** out) {
    if (!request_json || !out) return fail(VDC_ERR_INPUT, "null argument");
    try {
        *out = reinterpret_cast<vdc_program*>(build(request_json));
        return VDC_OK;
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

int vdc_program_parse(const char* streams_json, const char* sidecar, vdc_program** out) {
    if (!streams_json || !sidecar || !out) return fail(VDC_ERR_INPUT, "null argument");
    try {
        const json js = json::parse(streams_json);
        std::vector<std::pair<std::string, std::string>> cs;
        for (const auto& [k, v] : js.items()) cs.emplace_back(k, v.get<std::string>());
        auto box = std::make_unique<ProgramBox>();
        box->program = generator::parse_program(cs, sidecar);
        box->hw = *costmodel::builtin_profile("b200");
        box->hw.sm_count = box->program.sm_count;
        box->hw.vcc_per_sm = box->program.vcc_per_sm;
        uint32_t max_vcc = 0;
        for (const auto& kv : box->program.streams)
            if (kv.first.kind == isa::CoreKind::vcc) max_vcc = std::max<uint32_t>(max_vcc, kv.first.vcc + 1u);
        box->hw.vcc_per_sm = std::max<uint32_t>(box->hw.vcc_per_sm, max_vcc);
        box->finish();
        *out = reinterpret_cast<vdc_program*>(box.release());
        return VDC_OK;
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

void vdc_program_free(vdc_program* prog) { delete reinterpret_cast<ProgramBox*>(prog); }

int vdc_program_text(const vdc_program* prog, int with_words, char** out_json) {
    if (!prog || !out_json) return fail(VDC_ERR_INPUT, "null argument");
    try {
        const std::string s = reinterpret_cast<const ProgramBox*>(prog)->text(with_words);
        *out_json = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(*out_json, s.c_str(), s.size() + 1);
        return VDC_OK;
    } catch (const std::exception& e) {
        return fail(classify(e), e.what());
    }
}

int vdc_program_cores(const vdc_program* prog, uint32_t* n_cores, uint32_t* sm_count, uint32_t* vcc_per_sm) {
    if (!prog) return fail(VDC_ERR_INPUT, "null program");
    const auto* b = reinterpret_cast<const ProgramBox*>(prog);
    if (n_cores) *n_cores = uint32_t(b->cores.size());
    if (sm_count) *sm_count = b->sm_count;
    if (vcc_per_sm) *vcc_per_sm = b->vcc_per_sm;
    return VDC_OK;
}

int vdc_program_words(const vdc_program* prog, uint32_t core, const uint8_t** words, uint32_t* n_words) {
    if (!prog || !words || !n_words) return fail(VDC_ERR_INPUT, "null argument");
    const auto* b = reinterpret_cast<const ProgramBox*>(prog);
    if (core >= b->words.size()) return fail(VDC_ERR_INPUT, "core index out of range");
    *words = b->words[core].data();
    *n_words = uint32_t(b->words[core].size() / 16);
    return VDC_OK;
}

int vdc_program_synthesize(const vdc_program* prog, uint16_t tensor, uint64_t seed, void* dptr, size_t bytes, void* stream) {
    if (!prog || !dptr) return fail(VDC_ERR_INPUT, "null argument");
    const auto* b = reinterpret_cast<const ProgramBox*>(prog);
    const auto& ds = b->program.descriptors;
    if (tensor >= ds.size()) return fail(VDC_ERR_INPUT, "tensor index out of range");
    const auto& d = ds[tensor];
    if (d.view_of >= 0) return fail(VDC_ERR_INPUT, d.tensor + " is a view: synthesize its storage owner");
    if (d.elem != workload::ElemType::f32 && d.elem != workload::ElemType::bf16)
        return fail(VDC_ERR_INPUT, d.tensor + ": only f32 / bf16 tensors are synthesised");
    const uint64_t n = uint64_t(d.elem_count());
    const int bf = d.elem == workload::ElemType::bf16 ? 1 : 0;
    if (bytes != n * (bf ? 2u : 4u)) return fail(VDC_ERR_INPUT, d.tensor + ": buffer size does not match the descriptor");
    // reference synthesize_inputs: only external tensors (and, ext, KV state) carry contents
    const int init = (d.external || d.state) && !d.symmetric ? int(d.init) : int(workload::InitKind::zeros);
    const uint32_t layout = (d.tma == VDC_DESC_PACKED_SW128 || d.tma == VDC_DESC_KPAGE_SWZ) ? d.tma : 0u;
    if (layout == VDC_DESC_PACKED_SW128 && (d.shape.size() != 2 || d.shape[0] % 128 || d.shape[1] % 64))
        return fail(VDC_ERR_INPUT, d.tensor + ": packed weights are (rows % 128, cols % 64)");
    if (layout && n % (bf ? 8u : 4u)) return fail(VDC_ERR_INPUT, d.tensor + ": swizzled layouts need whole 16-byte chunks");
    const int rc = vdc_dev::synthesize_launch(dptr, n, bf, init, d.init_scale, seed ^ fnv1a(d.tensor), layout, d.rows(), d.cols(),
                                              stream);
    if (rc != 0) return fail(VDC_ERR_INTERNAL, "synthesis kernel launch failed (cuda error " + std::to_string(rc) + ")");
    return VDC_OK;
}

void vdc_free_string(char* s) { std::free(s); }

}  // extern "C"
