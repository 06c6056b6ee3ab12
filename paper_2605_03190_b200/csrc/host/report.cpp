// ExecutionReport serialisation. The reference declares these four members
// (proj/include/uopsim/machine.hpp:84-87) without bodies in its tree; SPEC.md
// fixes only the contents (makespan, per-resource busy
// intervals, traffic bytes, event trace, final tensors, termination status
// with the wait-for cycle) and the Chrome trace event format.
//
//   to_json      one JSON object with every field; from_json is its inverse
//                (round trip is exact: floats are written with 9 significant
//                digits, integers as integers)
//   to_kv_text   one `key=value` line per scalar, a summary line per busy
//                resource, tensor and wait-for edge (diff-friendly)
//   chrome_trace Chrome Trace Event JSON array: one complete ("X") event per
//                traced µop, pid = SM, tid = core name, times in µs
#include <cstdio>
#include <sstream>

#include "nlohmann/json.hpp"
#include "uopsim/machine.hpp"

namespace uopsim::machine {

using nlohmann::json;

namespace {

json core_json(const generator::CoreId& c) { return c.name(); }
generator::CoreId core_from(const json& j) { return generator::CoreId::parse(j.get<std::string>()); }

}  // namespace

std::string ExecutionReport::to_json() const {
    json j;
    j["status"] = status == Termination::completed ? "completed" : "deadlock";
    j["deadlock_cycle"] = json::array();
    for (const auto& c : deadlock_cycle) j["deadlock_cycle"].push_back(core_json(c));
    j["wait_edges"] = json::array();
    for (const auto& e : wait_edges) j["wait_edges"].push_back({{"from", core_json(e.from)}, {"to", core_json(e.to)}, {"reason", e.reason}});
    j["makespan"] = makespan;
    j["traffic_bytes"] = traffic_bytes;
    j["busy"] = json::object();
    for (const auto& [res, iv] : busy) {
        json a = json::array();
        for (const auto& [s, e] : iv) a.push_back({s, e});
        j["busy"][res] = a;
    }
    j["trace"] = json::array();
    for (const auto& t : trace)
        j["trace"].push_back({{"ts", t.ts}, {"dur", t.dur}, {"resource", t.resource}, {"core", core_json(t.core)}, {"name", t.name},
                              {"stream_index", t.stream_index}, {"instance", t.instance}, {"flow", t.flow}, {"unit_seq", t.unit_seq}});
    j["tensors"] = json::object();
    for (const auto& [name, v] : tensors) j["tensors"][name] = v;
    j["queues_drained"] = queues_drained;
    j["slots_all_free"] = slots_all_free;
    j["uops_executed"] = uops_executed;
    j["barrier_times"] = barrier_times;
    j["workload_name"] = workload_name;
    j["workload_hash"] = workload_hash;
    j["profile_name"] = profile_name;
    j["dram_bw"] = dram_bw;
    j["dram_busy_ns"] = dram_busy_ns;
    return j.dump();
}

ExecutionReport ExecutionReport::from_json(const std::string& text) {
    json j;
    try {
        j = json::parse(text);
    } catch (const std::exception& e) {
        throw MachineError(std::string("report json: ") + e.what());
    }
    ExecutionReport r;
    try {
        const std::string st = j.at("status").get<std::string>();
        if (st != "completed" && st != "deadlock") throw MachineError("report json: bad status '" + st + "'");
        r.status = st == "completed" ? Termination::completed : Termination::deadlock;
        for (const auto& c : j.at("deadlock_cycle")) r.deadlock_cycle.push_back(core_from(c));
        for (const auto& e : j.at("wait_edges"))
            r.wait_edges.push_back({core_from(e.at("from")), core_from(e.at("to")), e.at("reason").get<std::string>()});
        r.makespan = j.at("makespan").get<int64_t>();
        r.traffic_bytes = j.at("traffic_bytes").get<uint64_t>();
        for (const auto& [res, iv] : j.at("busy").items())
            for (const auto& p : iv) r.busy[res].push_back({p.at(0).get<int64_t>(), p.at(1).get<int64_t>()});
        for (const auto& t : j.at("trace")) {
            TraceEvent e;
            e.ts = t.at("ts").get<int64_t>();
            e.dur = t.at("dur").get<int64_t>();
            e.resource = t.at("resource").get<std::string>();
            e.core = core_from(t.at("core"));
            e.name = t.at("name").get<std::string>();
            e.stream_index = t.at("stream_index").get<uint32_t>();
            e.instance = t.at("instance").get<uint64_t>();
            e.flow = t.at("flow").get<uint8_t>();
            e.unit_seq = t.at("unit_seq").get<uint64_t>();
            r.trace.push_back(std::move(e));
        }
        for (const auto& [name, v] : j.at("tensors").items()) r.tensors[name] = v.get<std::vector<float>>();
        r.queues_drained = j.at("queues_drained").get<bool>();
        r.slots_all_free = j.at("slots_all_free").get<bool>();
        r.uops_executed = j.at("uops_executed").get<uint64_t>();
        r.barrier_times = j.at("barrier_times").get<std::vector<int64_t>>();
        r.workload_name = j.at("workload_name").get<std::string>();
        r.workload_hash = j.at("workload_hash").get<uint64_t>();
        r.profile_name = j.at("profile_name").get<std::string>();
        r.dram_bw = j.at("dram_bw").get<double>();
        r.dram_busy_ns = j.at("dram_busy_ns").get<int64_t>();
    } catch (const MachineError&) {
        throw;
    } catch (const std::exception& e) {
        throw MachineError(std::string("report json: ") + e.what());
    }
    return r;
}

std::string ExecutionReport::to_kv_text() const {
    std::ostringstream o;
    o << "status=" << (status == Termination::completed ? "completed" : "deadlock") << "\n";
    o << "makespan=" << makespan << "\n";
    o << "traffic_bytes=" << traffic_bytes << "\n";
    o << "uops_executed=" << uops_executed << "\n";
    o << "queues_drained=" << (queues_drained ? 1 : 0) << "\n";
    o << "slots_all_free=" << (slots_all_free ? 1 : 0) << "\n";
    o << "workload_name=" << workload_name << "\n";
    o << "workload_hash=" << workload_hash << "\n";
    o << "profile_name=" << profile_name << "\n";
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.9g", dram_bw);
    o << "dram_bw=" << buf << "\n";
    o << "dram_busy_ns=" << dram_busy_ns << "\n";
    o << "deadlock_cycle=";
    for (size_t i = 0; i < deadlock_cycle.size(); ++i) o << (i ? "," : "") << deadlock_cycle[i].name();
    o << "\n";
    for (const auto& e : wait_edges) o << "wait_edge=" << e.from.name() << "->" << e.to.name() << ":" << e.reason << "\n";
    for (const auto& [res, iv] : busy) {
        int64_t tot = 0;
        for (const auto& [s, e] : iv) tot += e - s;
        o << "busy." << res << "=" << iv.size() << "," << tot << "\n";
    }
    o << "trace_events=" << trace.size() << "\n";
    for (const auto& [name, v] : tensors) {
        double sum = 0;
        for (float x : v) sum += double(x);
        std::snprintf(buf, sizeof buf, "%.9g", sum);
        o << "tensor." << name << "=" << v.size() << "," << buf << "\n";
    }
    return o.str();
}

std::string ExecutionReport::chrome_trace() const {
    json a = json::array();
    for (const auto& t : trace)
        a.push_back({{"name", t.name},
                     {"cat", t.core.kind == isa::CoreKind::vmc ? "vmc" : "vcc"},
                     {"ph", "X"},
                     {"ts", double(t.ts) / 1e3},
                     {"dur", double(t.dur) / 1e3},
                     {"pid", t.core.sm},
                     {"tid", t.resource},
                     {"args", {{"pc", t.stream_index}, {"instance", t.instance}, {"flow", t.flow}}}});
    return a.dump();
}

}  // namespace uopsim::machine
