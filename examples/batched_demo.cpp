// C++ host driving a batched decode program through the drop-in Machine
// (include/uopsim/machine.hpp): 4 requests of a small bf16 Llama-style model,
// paged KV in a shared 16-page pool managed by the vdc_kv_* block allocator,
// greedy sampling fused into the lm_head GEMM. Each step the host reserves
// pages for the new positions, writes (token, position, context) per request
// and the page table into the step block (sized by the program:
// LoweredProgram::step_scalars), runs the engine and feeds the sampled tokens
// back. Prints one line per step; exit code 0 when every step completed.
#include <cstdio>

#include "uopsim/decode.hpp"
#include "uopsim/machine.hpp"

using namespace uopsim;

int main() {
    decode::ModelConfig m = decode::llama3_8b();
    m.layers = 2;
    m.hidden = 1024;
    m.heads = 8;
    m.kv_heads = 2;
    m.ffn = 2816;
    m.vocab = 4096;
    decode::LayoutConfig lay;
    lay.ring = true;
    lay.batch = 4;
    lay.req_pages = {2, 3, 1, 2};  // per-request capacity (pages of 64 positions)
    lay.pool_pages = 16;           // shared pool: pages are handed out by the block allocator
    lay.pages_per_job = 4;
    lay.gu_block = 128;
    lay.argmax = true;
    const auto g = decode::build_decode_graph(m, lay);
    const auto hw = *costmodel::builtin_profile("b200");
    const auto p = generator::lower_decode_ring(g, hw, {}, 8);
    machine::MachineOptions opt;
    opt.record_trace = false;
    machine::Machine mach(p, hw, machine::synthesize_program_inputs(p), opt);

    vdc_kv_pages* kv = nullptr;
    if (vdc_kv_create(uint32_t(lay.pool_pages), uint32_t(lay.batch), uint32_t(p.maxp), &kv) != VDC_OK) return 2;
    std::vector<int64_t> pos = {70, 150, 20, 100}, tok = {17, 18, 19, 20};
    bool ok = true;
    for (int step = 0; step < 4; ++step) {
        std::vector<int64_t> st(mach.step_scalars(), 0);
        for (int b = 0; b < lay.batch; ++b) {
            if (vdc_kv_reserve(kv, uint32_t(b), uint64_t(pos[b] + 1)) != VDC_OK) return 3;
            st[3 * b] = tok[b];
            st[3 * b + 1] = pos[b];
            st[3 * b + 2] = pos[b] + 1;
        }
        vdc_kv_table(kv, st.data() + p.page_table_off);
        mach.set_step(st);
        const auto r = mach.run();
        ok = ok && r.status == machine::Termination::completed && r.queues_drained && r.slots_all_free;
        const auto& nt = r.tensors.at("next_token");
        std::printf("batched step %d: status=%s tokens=", step, r.status == machine::Termination::completed ? "completed" : "deadlock");
        for (int b = 0; b < lay.batch; ++b) {
            tok[b] = int64_t(nt[size_t(b)]);
            pos[b] += 1;
            std::printf("%s%lld", b ? "," : "", (long long)tok[b]);
        }
        uint32_t free_pages = 0;
        vdc_kv_stats(kv, &free_pages, nullptr);
        std::printf(" free_pages=%u\n", free_pages);
    }
    vdc_kv_destroy(kv);
    return ok ? 0 : 1;
}
