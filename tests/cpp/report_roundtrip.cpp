// CPU check of ExecutionReport's serialisations (csrc/host/report.cpp; the
// reference declares them at proj/include/uopsim/machine.hpp:84-87): a report
// with every field populated survives to_json -> from_json exactly, to_kv_text
// and chrome_trace carry its contents, malformed JSON raises MachineError.
#include <cstdio>
#include <string>

#include "uopsim/machine.hpp"

using namespace uopsim;

int main() {
    machine::ExecutionReport r;
    r.status = machine::Termination::deadlock;
    r.deadlock_cycle = {generator::CoreId::vmc(0), generator::CoreId::vcc_id(1, 1)};
    r.wait_edges = {{generator::CoreId::vmc(0), generator::CoreId::vmc(1), "dep 9 empty"}};
    r.makespan = 123456;
    r.traffic_bytes = 1ull << 40;
    r.busy["sm0.vcc0"] = {{0, 10}, {20, 35}};
    machine::TraceEvent e;
    e.ts = 20;
    e.dur = 15;
    e.resource = "sm0.vcc0";
    e.core = generator::CoreId::vcc_id(0, 0);
    e.name = "MATVEC";
    e.stream_index = 3;
    e.instance = 1;
    e.flow = 2;
    r.trace = {e};
    r.tensors["R"] = {1.5f, -2.25f, 3.0e-7f};
    r.queues_drained = false;
    r.slots_all_free = true;
    r.uops_executed = 42;
    r.barrier_times = {5, 9};
    r.workload_name = "fig4";
    r.workload_hash = 0xfedcba9876543210ull;
    r.profile_name = "b200";
    r.dram_bw = 6.5e12;
    r.dram_busy_ns = 777;
    const std::string j = r.to_json();
    const auto back = machine::ExecutionReport::from_json(j);
    if (back.to_json() != j) {
        std::printf("FAIL: json round trip\n%s\n%s\n", j.c_str(), back.to_json().c_str());
        return 1;
    }
    if (back.tensors.at("R")[2] != 3.0e-7f || back.workload_hash != r.workload_hash || back.wait_edges.size() != 1 ||
        back.status != machine::Termination::deadlock || back.deadlock_cycle[1] != generator::CoreId::vcc_id(1, 1)) {
        std::printf("FAIL: fields\n");
        return 1;
    }
    const std::string kv = r.to_kv_text();
    for (const char* want : {"status=deadlock\n", "makespan=123456\n", "queues_drained=0\n", "wait_edge=sm0.vmc->sm1.vmc:dep 9 empty\n",
                             "busy.sm0.vcc0=2,25\n", "deadlock_cycle=sm0.vmc,sm1.vcc1\n", "tensor.R=3,"})
        if (kv.find(want) == std::string::npos) {
            std::printf("FAIL: kv text lacks %s\n%s", want, kv.c_str());
            return 1;
        }
    const std::string ct = r.chrome_trace();
    if (ct.find("\"ph\":\"X\"") == std::string::npos || ct.find("\"name\":\"MATVEC\"") == std::string::npos) {
        std::printf("FAIL: chrome trace %s\n", ct.c_str());
        return 1;
    }
    try {
        machine::ExecutionReport::from_json("{\"status\": \"completed\"}");
        std::printf("FAIL: incomplete json accepted\n");
        return 1;
    } catch (const machine::MachineError&) {
    }
    std::printf("report round trip ok (%zu json bytes, %zu kv bytes)\n", j.size(), kv.size());
    return 0;
}
