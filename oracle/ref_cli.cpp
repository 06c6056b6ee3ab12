// ORACLE / TEST INFRASTRUCTURE ONLY. Drives the *reference* generator
// (/root/reference/proj/src, compiled by oracle/Makefile) so the parity tests
// can diff our host library's output against it byte for byte.
//
// Input (stdin): one JSON request
//   { "workload": <workload document, reference schema workload.cpp:333-380>,
//     "profile":  {"builtin": "h100"} | {"test": [name, pairs, bw, flops, slots]} | <profile json>,
//     "options":  {"theta":1.2,"flows":true,"fusion":true,"fold":true,"seed":0},
//     "tilings":  {"node": {"M":4,...}}            (optional: bypass select_tilings)
//     "passes":   ["flows","fusion","fold","deadlock","redundancy","last"] (optional;
//                  default = the full generate() pipeline, elaborate.cpp:492-520) }
// Output (stdout): JSON {ok, error, tilings, streams:{core:text}, sidecar, words:{core:hex},
//                        makespan_estimate, certificate_ok}
#include <cstring>
#include <iostream>
#include <iterator>
#include <sstream>

#include <nlohmann/json.hpp>

#include "uopsim/costmodel.hpp"
#include "uopsim/generator.hpp"
#include "uopsim/isa.hpp"
#include "uopsim/workload.hpp"

using nlohmann::ordered_json;
using namespace uopsim;

static costmodel::HardwareProfile profile_from(const ordered_json& j) {
    if (j.contains("builtin")) {
        auto p = costmodel::builtin_profile(j.at("builtin").get<std::string>());
        if (!p) throw std::runtime_error("unknown builtin profile");
        return *p;
    }
    if (j.contains("test")) {
        const auto& t = j.at("test");
        return costmodel::make_test_profile(t.at(0).get<std::string>(), t.at(1).get<uint32_t>(),
                                            t.at(2).get<double>(), t.at(3).get<double>(),
                                            t.size() > 4 ? t.at(4).get<uint32_t>() : 32u);
    }
    return costmodel::parse_profile(j.dump());
}

static workload::SplitAxis axis_from(const std::string& s) {
    if (s == "M") return workload::SplitAxis::M;
    if (s == "N") return workload::SplitAxis::N;
    if (s == "K") return workload::SplitAxis::K;
    if (s == "token") return workload::SplitAxis::token_block;
    if (s == "head") return workload::SplitAxis::head_block;
    throw std::runtime_error("bad axis " + s);
}

int main() {
    std::string text((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
    ordered_json out;
    try {
        auto req = ordered_json::parse(text);
        auto g = workload::parse_workload(req.at("workload").dump());
        if (req.contains("synthesize")) {
            // golden vectors of the reference synthesize_inputs (workload.cpp:411-435):
            // per tensor the first `head` values' fp32 bits and an FNV-1a of all bits
            const auto& sj = req.at("synthesize");
            const size_t head = sj.value("head", size_t(16));
            auto arrays = workload::synthesize_inputs(g, sj.value("seed", 0ull));
            ordered_json ts = ordered_json::array();
            for (auto& [name, v] : arrays) {
                uint64_t h = 0xcbf29ce484222325ULL;
                ordered_json first = ordered_json::array();
                for (size_t i = 0; i < v.size(); ++i) {
                    uint32_t u;
                    std::memcpy(&u, &v[i], 4);
                    for (int k = 0; k < 4; ++k) h = (h ^ ((u >> (8 * k)) & 0xff)) * 0x100000001b3ULL;
                    if (i < head) first.push_back(u);
                }
                ts.push_back({{"name", name}, {"n", v.size()}, {"head_bits", first}, {"fnv1a_bits", std::to_string(h)}});
            }
            out["synthesized"] = ts;
            out["ok"] = true;
            std::cout << out.dump() << "\n";
            return 0;
        }
        auto hw = profile_from(req.value("profile", ordered_json{{"builtin", "h100"}}));
        generator::GenOptions opt;
        auto jo = req.value("options", ordered_json::object());
        opt.theta = jo.value("theta", 1.2);
        opt.flows = jo.value("flows", true);
        opt.fusion = jo.value("fusion", true);
        opt.fold = jo.value("fold", true);
        opt.input_seed = jo.value("seed", 0ull);

        std::map<std::string, workload::TilingChoice> tilings;
        if (req.contains("tilings")) {
            for (const auto& n : g.nodes) tilings[n.id] = workload::TilingChoice{n.id, {}};
            for (auto& [node, parts] : req.at("tilings").items()) {
                workload::TilingChoice c{node, {}};
                for (auto& [ax, v] : parts.items()) c.parts[axis_from(ax)] = v.get<int>();
                tilings[node] = c;
            }
        } else {
            tilings = generator::select_tilings(g, hw, opt.theta);
        }
        ordered_json jt = ordered_json::object();
        for (auto& [node, c] : tilings) {
            ordered_json parts = ordered_json::object();
            for (auto& [ax, v] : c.parts) parts[std::string(workload::axis_name(ax))] = v;
            jt[node] = parts;
        }
        out["tilings"] = jt;

        generator::LoweredProgram p;
        if (req.contains("passes") || req.contains("tilings")) {
            std::vector<std::string> passes = req.value(
                "passes", std::vector<std::string>{"flows", "fusion", "fold", "deadlock", "redundancy", "last"});
            p = generator::lower(g, tilings, hw);
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
                    // refresh the certificate exactly like generate() (elaborate.cpp:508-513)
                    p = generator::fix_deadlocks(std::move(p));
                } else if (ps == "last") {
                    for (auto& [core, s] : p.streams)
                        if (!s.empty()) s.back().flags |= isa::kFlagLast;
                } else throw std::runtime_error("unknown pass " + ps);
            }
        } else {
            p = generator::generate(g, hw, opt);
        }
        ordered_json streams = ordered_json::object(), words = ordered_json::object();
        for (auto& [core, s] : p.streams) {
            streams[core.name()] = generator::serialize_stream(p, core);
            auto bytes = isa::encode_stream(s);
            std::ostringstream hex;
            static const char* d = "0123456789abcdef";
            for (uint8_t b : bytes) hex << d[b >> 4] << d[b & 15];
            words[core.name()] = hex.str();
        }
        out["streams"] = streams;
        out["words"] = words;
        out["sidecar"] = generator::serialize_sidecar(p);
        out["total_uops"] = p.total_uops();
        out["certificate_ok"] = generator::replay_certificate(p);
        try {
            out["makespan_estimate"] = generator::estimate_makespan(p, hw);
        } catch (const std::exception& e) {
            out["makespan_estimate"] = nullptr;
        }
        out["ok"] = true;
    } catch (const std::exception& e) {
        out["ok"] = false;
        out["error"] = e.what();
    }
    std::cout << out.dump() << "\n";
    return 0;
}
