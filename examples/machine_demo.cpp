// C++ drop-in demo: the reference's `uopsim::machine::simulate(p, hw)` call
// site, unchanged, running on the B200 engine through include/uopsim/machine.hpp.
//   1. the SPEC Fig. 4 program (matvec -> rope) built with generator::generate
//   2. the tiny decode model lowered in ring mode, one decode step
// Prints one line per program; exit code 0 when both completed.
#include <cstdio>

#include "uopsim/decode.hpp"
#include "uopsim/machine.hpp"

using namespace uopsim;

int main() {
    auto hw = *costmodel::builtin_profile("b200");
    hw.sm_count = 2;
    hw.shmem_per_sm = 16 * 8192;  // 16 slots: fits a B200 CTA next to the control block
    hw.stu_count = 1;             // one store unit per VMC: each VCC release ring has one consumer
    workload::OperatorGraph g = workload::parse_workload(R"({
      "tensors": [{"name": "M", "shape": [64, 64], "tile": [16, 64]}, {"name": "N", "shape": [64, 1], "tile": [64, 1]},
                  {"name": "O", "shape": [64, 1], "tile": [16, 1], "init": "zeros"},
                  {"name": "T", "shape": [64, 1], "tile": [16, 1]},
                  {"name": "R", "shape": [64, 1], "tile": [16, 1], "init": "zeros"}],
      "operators": [{"id": "mv", "kind": "matvec", "inputs": ["M", "N"], "outputs": ["O"]},
                    {"id": "rope", "kind": "rope", "inputs": ["O", "T"], "outputs": ["R"]}]})");
    const auto p = generator::generate(g, hw);
    const auto rep = machine::simulate(p, hw);
    double cs = 0;
    for (float v : rep.tensors.at("R")) cs += v;
    std::printf("fig4: status=%s uops=%llu makespan_ns=%lld checksum(R)=%.6f\n",
                rep.status == machine::Termination::completed ? "completed" : "deadlock",
                (unsigned long long)rep.uops_executed, (long long)rep.makespan, cs);

    // the report's serialisations (reference machine.hpp:84-87): JSON round
    // trip, key=value text, Chrome trace; conservation measured on the device
    const std::string js = rep.to_json();
    const auto back = machine::ExecutionReport::from_json(js);
    const std::string kv = rep.to_kv_text(), ct = rep.chrome_trace();
    size_t kv_lines = 0;
    for (char ch : kv) kv_lines += ch == '\n';
    std::printf("fig4 report: json_roundtrip=%s trace_events=%zu busy_resources=%zu kv_lines=%zu chrome_bytes=%zu "
                "queues_drained=%d slots_all_free=%d\n",
                back.to_json() == js ? "exact" : "MISMATCH", rep.trace.size(), rep.busy.size(), kv_lines, ct.size(),
                int(rep.queues_drained), int(rep.slots_all_free));

    // a wait that can never be satisfied: sm0.vmc first waits on dep queue 9,
    // whose declared producer (sm1.vmc) never stores to it -> the device
    // watchdog reports a deadlock and wait_for_edges() names the wait
    auto stuck = p;
    generator::QueueInfo q9;
    q9.dep_id = 9;
    q9.producer = generator::CoreId::vmc(1);
    q9.consumer = generator::CoreId::vmc(0);
    q9.depth = 2;
    stuck.queues.push_back(q9);
    isa::UopWord w;
    w.opcode = isa::Opcode::LOAD_DEP;
    w.dep_id = 9;
    w.flow = 1;
    w.addr = isa::AddressSpec::tile2(0, 0, 0);  // size 0: a token wait, no data
    auto& s0 = stuck.streams.at(generator::CoreId::vmc(0));
    s0.insert(s0.begin(), w);
    auto& m0 = stuck.meta.at(generator::CoreId::vmc(0));
    m0.insert(m0.begin(), generator::UopMeta{});
    machine::MachineOptions so;
    so.watchdog_ms = 200;
    machine::Machine sm(stuck, hw, machine::synthesize_program_inputs(stuck), so);
    const auto dr = sm.run();
    const auto edges = sm.wait_for_edges();
    bool named = false;
    for (const auto& e : edges) {
        std::printf("wait edge: %s -> %s (%s)\n", e.from.name().c_str(), e.to.name().c_str(), e.reason.c_str());
        named = named || (e.from == generator::CoreId::vmc(0) && e.to == generator::CoreId::vmc(1) && e.reason == "dep 9 empty");
    }
    std::printf("stuck program: status=%s edges=%zu named=%s\n",
                dr.status == machine::Termination::deadlock ? "deadlock" : "completed", edges.size(), named ? "yes" : "no");

    decode::LayoutConfig lay;
    lay.ring = true;
    lay.gu_block = 16;
    const auto dg = decode::build_decode_graph(decode::tiny_llama(), lay);
    auto hw2 = *costmodel::builtin_profile("b200");
    const auto rp = generator::lower_decode_ring(dg, hw2);
    machine::Machine m(rp, hw2, machine::synthesize_program_inputs(rp));
    m.set_step({17, 40, 41});
    const auto r2 = m.run();
    double lg = 0;
    for (float v : r2.tensors.at("logits")) lg += v;
    std::printf("tiny decode (ring): status=%s tile_loads=%llu makespan_ns=%lld checksum(logits)=%.6f\n",
                r2.status == machine::Termination::completed ? "completed" : "deadlock",
                (unsigned long long)r2.uops_executed, (long long)r2.makespan, lg);
    return rep.status == machine::Termination::completed && r2.status == machine::Termination::completed &&
                   back.to_json() == js && rep.queues_drained && rep.slots_all_free &&
                   dr.status == machine::Termination::deadlock && named
               ? 0
               : 1;
}
