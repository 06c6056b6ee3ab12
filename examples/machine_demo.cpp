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
    return rep.status == machine::Termination::completed && r2.status == machine::Termination::completed ? 0 : 1;
}
