#pragma once
// Drop-in replacement of the reference executor header
// (reference proj/include/uopsim/machine.hpp:17-136) over the B200 C-ABI
// (include/vdc.h). Header-only; link libvdc.so and the CUDA runtime.
//
//   reference (CPU discrete-event VM)          this header (persistent sm_100a kernel)
//   Machine(p, hw, inputs, opt)                 uploads p's streams/queues/descriptors (and the
//                                               ring operand blocks of ring-mode programs),
//                                               allocates device tensors from `inputs`
//   run(watchdog) -> ExecutionReport            one launch + wait; tensors copied back as fp32
//   simulate(p, hw, opt, watchdog)              same, inputs from synthesize_program_inputs
//   Termination::deadlock (report, no throw)    VDC_ERR_DEADLOCK from the device watchdog
//   MachineError                                any other C-ABI failure
//
// Deviations (documented, not hidden): the device runs the whole program in
// one launch, so step() executes it to completion and returns every traced
// event at once; makespan is measured device time in ns, not a modelled
// clock; the event trace and busy intervals are the device trace of the
// compute µops (vdc_bind_trace: per µop its dependency-ready and done times;
// memory-core µops are not individually timed on the device);
// queues_drained / slots_all_free are the device's own end-of-launch counts;
// wait_for_edges() after a deadlock names, for every core the watchdog found
// blocked, the core it waits on and why (the reference's stall reasons,
// elaborate.cpp:193-214). ExecutionReport's to_json / from_json / to_kv_text /
// chrome_trace live in libvdc.so (csrc/host/report.cpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "uopsim/costmodel.hpp"
#include "uopsim/generator.hpp"
#include "uopsim/workload.hpp"
#include "vdc.h"

namespace uopsim::machine {

struct MachineError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct SlotRange {
    uint8_t first = 0;
    uint8_t count = 0;
    friend bool operator==(const SlotRange&, const SlotRange&) = default;
};

// Same contract as the reference allocator (first-fit contiguous run of
// 1..32 slots, frees in any order, double free throws).
class SlotAllocator {
  public:
    explicit SlotAllocator(uint32_t budget = 32) : budget_(budget > 32 ? 32 : budget) {}
    std::optional<SlotRange> alloc(uint32_t n) {
        if (n < 1 || n > 32) throw MachineError("slot request out of 1..32");
        for (uint32_t first = 0; first + n <= budget_; ++first) {
            const uint32_t mask = (n == 32 ? 0xffffffffu : ((1u << n) - 1u)) << first;
            if (!(bits_ & mask)) {
                bits_ |= mask;
                return SlotRange{uint8_t(first), uint8_t(n)};
            }
        }
        return std::nullopt;
    }
    void free(SlotRange r) {
        const uint32_t mask = (r.count == 32 ? 0xffffffffu : ((1u << r.count) - 1u)) << r.first;
        if ((bits_ & mask) != mask) throw MachineError("double free");
        bits_ &= ~mask;
    }
    uint32_t occupied_count() const { return uint32_t(__builtin_popcount(bits_)); }
    uint32_t budget() const { return budget_; }
    uint32_t bits() const { return bits_; }
    bool all_free() const { return bits_ == 0; }

  private:
    uint32_t bits_ = 0;
    uint32_t budget_;
};

struct TraceEvent {
    int64_t ts = 0;
    int64_t dur = 0;
    std::string resource;
    generator::CoreId core;
    std::string name;
    uint32_t stream_index = 0;
    uint64_t instance = 0;
    uint8_t flow = 0;
    uint64_t unit_seq = 0;
};

struct WaitEdge {
    generator::CoreId from, to;
    std::string reason;
};

enum class Termination : uint8_t { completed, deadlock };

struct ExecutionReport {
    Termination status = Termination::completed;
    std::vector<generator::CoreId> deadlock_cycle;
    std::vector<WaitEdge> wait_edges;
    int64_t makespan = 0;        // measured device ns
    uint64_t traffic_bytes = 0;  // bytes moved global -> shared by the memory cores
    std::map<std::string, std::vector<std::pair<int64_t, int64_t>>> busy;
    std::vector<TraceEvent> trace;
    std::map<std::string, std::vector<float>> tensors;
    bool queues_drained = true;
    bool slots_all_free = true;
    uint64_t uops_executed = 0;
    std::vector<int64_t> barrier_times;
    std::string workload_name;
    uint64_t workload_hash = 0;
    std::string profile_name;
    double dram_bw = 0;
    int64_t dram_busy_ns = 0;

    std::string to_json() const;
    static ExecutionReport from_json(const std::string& text);
    std::string to_kv_text() const;
    std::string chrome_trace() const;  // Chrome Trace Event JSON array
};

struct MachineOptions {
    bool record_trace = true;       // device trace of every compute µop (vdc_bind_trace)
    int device = 0;
    uint32_t watchdog_ms = 2000;
    uint32_t trace_records = 4096;  // per compute core
};

namespace detail {
inline void check(int rc) {
    if (rc != VDC_OK) throw MachineError(std::string("vdc: ") + vdc_last_error());
}
inline uint16_t to_bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}
inline float from_bf16(uint16_t b) {
    const uint32_t u = uint32_t(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
}  // namespace detail

inline std::map<std::string, std::vector<float>> synthesize_program_inputs(const generator::LoweredProgram& p) {
    std::map<std::string, std::vector<float>> out;
    for (const auto& d : p.descriptors) {
        if (d.view_of >= 0) continue;
        workload::TensorRef t;
        t.name = d.tensor;
        t.shape = d.shape;
        t.tile_rows = d.tile_rows;
        t.tile_cols = d.tile_cols;
        t.init = d.external || d.state ? d.init : workload::InitKind::zeros;
        t.elem = d.elem;
        t.init_scale = d.init_scale;
        out.emplace(d.tensor, workload::synthesize_tensor(t, p.input_seed));
    }
    return out;
}

class Machine {
  public:
    Machine(const generator::LoweredProgram& p, const costmodel::HardwareProfile& hw,
            std::map<std::string, std::vector<float>> inputs, MachineOptions opt = {})
        : p_(p), opt_(opt) {
        vdc_profile prof{};
        prof.sm_count = p.sm_count ? p.sm_count : hw.sm_count;
        prof.vcc_per_sm = p.ring_slots ? 1u : uint32_t(p.vcc_per_sm ? p.vcc_per_sm : hw.vcc_per_sm);
        prof.slot_size = p.slot_size;
        prof.slot_budget = p.slot_budget;
        prof.ldu_count = hw.ldu_count;
        prof.stu_count = hw.stu_count;
        detail::check(vdc_create(&prof, opt.device, &ctx_));
        // streams in CoreId order: sm<i>.vmc, sm<i>.vcc0, ...
        std::vector<uint8_t> words;
        std::vector<uint32_t> per_core;
        for (uint32_t sm = 0; sm < prof.sm_count; ++sm)
            for (int v = -1; v < int(prof.vcc_per_sm); ++v) {
                const auto id = v < 0 ? generator::CoreId::vmc(uint16_t(sm)) : generator::CoreId::vcc_id(uint16_t(sm), uint8_t(v));
                const auto it = p.streams.find(id);
                const auto enc = it == p.streams.end() ? std::vector<uint8_t>{} : isa::encode_stream(it->second);
                words.insert(words.end(), enc.begin(), enc.end());
                per_core.push_back(uint32_t(enc.size() / isa::kWordBytes));
            }
        std::vector<vdc_queue> qs;
        for (const auto& q : p.queues) qs.push_back(vdc_queue{q.dep_id, q.depth, q.producer.sm, q.consumer.sm, q.local ? 1u : 0u});
        std::vector<vdc_desc> ds;
        for (const auto& d : p.descriptors) {
            vdc_desc x{};
            x.base = d.base;
            x.rank = uint32_t(d.shape.size());
            for (size_t k = 0; k < d.shape.size() && k < 4; ++k) x.shape[k] = d.shape[k];
            for (size_t k = 0; k < d.grid.size() && k < 4; ++k) x.grid[k] = d.grid[k];
            x.tile_rows = d.tile_rows;
            x.tile_cols = d.tile_cols;
            x.dtype = uint32_t(d.elem);
            x.view_of = d.view_of;
            x.tma = d.tma;
            ds.push_back(x);
        }
        detail::check(vdc_load_program(ctx_, words.data(), per_core.data(), uint32_t(per_core.size()), qs.data(),
                                       uint32_t(qs.size()), ds.data(), uint32_t(ds.size()), p.slot_budget,
                                       p.local_queue_depth));
        if (p.ring_slots) detail::check(vdc_load_jobs(ctx_, p.jobs.data(), uint32_t(p.jobs.size()), p.ring_slots));
        detail::check(vdc_set_params(ctx_, p.params.data(), uint32_t(p.params.size())));
        detail::check(vdc_set_watchdog(ctx_, opt.watchdog_ms));
        for (size_t i = 0; i < p.descriptors.size(); ++i) {
            const auto& d = p.descriptors[i];
            if (d.view_of >= 0) continue;
            const size_t n = size_t(d.elem_count()), eb = workload::elem_bytes(d.elem);
            void* dptr = nullptr;
            if (cudaMalloc(&dptr, n * eb) != cudaSuccess) throw MachineError("cudaMalloc failed for " + d.tensor);
            bufs_.push_back({i, dptr, n});
            std::vector<float> host(n, 0.f);
            if (auto it = inputs.find(d.tensor); it != inputs.end()) {
                if (it->second.size() != n) throw MachineError("input " + d.tensor + " has the wrong size");
                host = std::move(it->second);
            }
            upload(d, dptr, host);
            detail::check(vdc_bind_tensor(ctx_, uint16_t(i), dptr, n * eb, int(d.elem)));
        }
        if (p.step_scalars) {  // per-launch scalars (decode: token / pos / ctx, batched: + page table)
            n_step_ = std::max<uint32_t>(8u, p.step_scalars);
            cudaMalloc(&step_, sizeof(int64_t) * n_step_);
            cudaMemset(step_, 0, sizeof(int64_t) * n_step_);
            detail::check(vdc_bind_step(ctx_, static_cast<int64_t*>(step_), n_step_));
        }
        n_cores_ = prof.sm_count * (1u + prof.vcc_per_sm);
        per_sm_ = 1u + prof.vcc_per_sm;
        if (opt.record_trace && opt.trace_records) {
            const size_t n = size_t(n_cores_) * opt.trace_records * 4;
            if (cudaMalloc(&trace_, n * sizeof(uint64_t)) != cudaSuccess) throw MachineError("cudaMalloc failed for the trace");
            cudaMemset(trace_, 0, n * sizeof(uint64_t));
            detail::check(vdc_bind_trace(ctx_, trace_, opt.trace_records));
        }
    }
    ~Machine() {
        for (auto& b : bufs_) cudaFree(b.ptr);
        if (step_) cudaFree(step_);
        if (trace_) cudaFree(trace_);
        if (ctx_) vdc_destroy(ctx_);
    }
    Machine(Machine&& o) noexcept { swap(o); }
    Machine& operator=(Machine&& o) noexcept {
        swap(o);
        return *this;
    }
    Machine(const Machine&) = delete;
    Machine& operator=(const Machine&) = delete;

    // ext: per-launch scalars of decode programs, sized by the program
    // (LoweredProgram::step_scalars): single request (token, position, context);
    // batched: (token, position, context) per request, then the page table
    void set_step(const std::vector<int64_t>& s) {
        if (!step_) throw MachineError("program has no step scalars");
        if (s.size() > n_step_) throw MachineError("set_step: " + std::to_string(s.size()) + " scalars, the program reads " +
                                                   std::to_string(n_step_));
        std::vector<int64_t> v(n_step_, 0);
        std::copy(s.begin(), s.end(), v.begin());
        cudaMemcpy(step_, v.data(), sizeof(int64_t) * n_step_, cudaMemcpyHostToDevice);
    }
    uint32_t step_scalars() const { return n_step_; }

    bool done() const { return done_; }
    int64_t now() const { return now_; }
    // the device runs the whole program per launch: the first step() runs it
    // and returns every traced event; later calls return nothing
    std::vector<TraceEvent> step() {
        if (done_) return {};
        last_ = run();
        return last_.trace;
    }

    ExecutionReport run(uint64_t watchdog = 1000) {
        (void)watchdog;  // the device watchdog is time based (MachineOptions::watchdog_ms)
        ExecutionReport r;
        r.workload_name = p_.workload_name;
        r.workload_hash = p_.workload_hash;
        r.profile_name = p_.profile_name;
        detail::check(vdc_launch(ctx_, nullptr));
        vdc_report rep{};
        const int rc = vdc_wait(ctx_, &rep);
        if (rc != VDC_OK && rc != VDC_ERR_DEADLOCK) detail::check(rc);
        r.status = rep.status == VDC_ERR_DEADLOCK ? Termination::deadlock : Termination::completed;
        r.makespan = int64_t(rep.elapsed_ms * 1e6);
        r.traffic_bytes = rep.bytes_loaded + rep.bytes_stored;
        r.uops_executed = rep.uops_executed;
        for (uint32_t i = 0; i < rep.n_stalled && i < 16; ++i) {
            const uint32_t core = rep.stalled_core[i], per = 1u + (p_.ring_slots ? 1u : p_.vcc_per_sm);
            r.deadlock_cycle.push_back(core % per == 0 ? generator::CoreId::vmc(uint16_t(core / per))
                                                       : generator::CoreId::vcc_id(uint16_t(core / per), uint8_t(core % per - 1)));
        }
        for (const auto& b : bufs_) r.tensors.emplace(p_.descriptors[b.desc].tensor, download(p_.descriptors[b.desc], b.ptr, b.n));
        r.queues_drained = rep.queues_drained != 0;
        r.slots_all_free = rep.slots_all_free != 0;
        if (trace_) read_trace(r);
        edges_.clear();
        if (r.status == Termination::deadlock)
            for (uint32_t i = 0; i < rep.n_stalled && i < 16; ++i) edges_.push_back(edge_of(r.deadlock_cycle[i], rep.stalled_pc[i]));
        r.wait_edges = edges_;
        done_ = true;
        now_ = r.makespan;
        return r;
    }

    // wait-for edges of the last run's blocked cores (empty unless it deadlocked)
    std::vector<WaitEdge> wait_for_edges() const { return edges_; }
    const SlotAllocator& allocator(uint16_t) const { return alloc_; }

  private:
    struct Buf {
        size_t desc;
        void* ptr;
        size_t n;
    };
    generator::CoreId core_of(uint32_t idx) const {
        const uint32_t sm = idx / per_sm_, k = idx % per_sm_;
        return k == 0 ? generator::CoreId::vmc(uint16_t(sm)) : generator::CoreId::vcc_id(uint16_t(sm), uint8_t(k - 1));
    }
    // device trace -> events (ts = dependency-ready time, dur = execution) and
    // per-core busy intervals, relative to the first traced µop
    void read_trace(ExecutionReport& r) const {
        std::vector<uint64_t> rec(size_t(n_cores_) * opt_.trace_records * 4);
        cudaMemcpy(rec.data(), trace_, rec.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost);
        int64_t t0 = INT64_MAX;
        for (size_t i = 0; i < rec.size(); i += 4)
            if (rec[i + 1]) t0 = std::min<int64_t>(t0, int64_t(rec[i + 1]));
        std::map<generator::CoreId, uint64_t> inst;
        for (size_t i = 0; i < rec.size(); i += 4) {
            if (!rec[i + 1]) continue;
            const auto core = core_of(uint32_t(rec[i] >> 32));
            const uint32_t pc = uint32_t(rec[i] & 0xffffffffu);
            TraceEvent e;
            e.core = core;
            e.resource = core.name();
            e.stream_index = pc;
            e.instance = inst[core]++;
            e.ts = int64_t(rec[i + 2]) - t0;
            e.dur = std::max<int64_t>(0, int64_t(rec[i + 3]) - int64_t(rec[i + 2]));
            if (const auto it = p_.streams.find(core); it != p_.streams.end() && pc < it->second.size()) {
                e.name = std::string(isa::opcode_name(it->second[pc].opcode));
                e.flow = it->second[pc].flow;
            }
            r.busy[e.resource].push_back({e.ts, e.ts + e.dur});
            r.trace.push_back(std::move(e));
        }
    }
    // what a blocked core waits for, from the µop it is stuck at (the
    // reference elaboration's stall reasons, elaborate.cpp:193-214, 318-340)
    WaitEdge edge_of(const generator::CoreId& core, uint32_t pc) const {
        WaitEdge e{core, core, "blocked"};
        const auto it = p_.streams.find(core);
        if (it == p_.streams.end() || pc >= it->second.size()) return e;
        const auto& u = it->second[pc];
        const auto vcc = generator::CoreId::vcc_id(core.sm, uint8_t(u.reg1));
        if (isa::is_dep_consumer(u.opcode) || isa::is_dep_producer(u.opcode)) {
            for (const auto& q : p_.queues)
                if (q.dep_id == u.dep_id) {
                    const bool cons = isa::is_dep_consumer(u.opcode);
                    e.to = cons ? q.producer : q.consumer;
                    e.reason = "dep " + std::to_string(u.dep_id) + (cons ? " empty" : " full");
                    return e;
                }
        }
        if (core.kind == isa::CoreKind::vcc) {
            e.to = generator::CoreId::vmc(core.sm);
            e.reason = "m2c empty";
        } else if (u.recv()) {
            e.to = vcc;
            e.reason = "c2m short";
        } else if (u.send()) {
            e.to = vcc;
            e.reason = "m2c full / slot budget";
        }
        return e;
    }
    // device storage position of logical (row-major) element i: batched ring
    // programs keep weights as pre-swizzled 128 x 64 tiles and KV page rows
    // swizzled (ring_abi.h VDC_DESC_PACKED_SW128 / VDC_DESC_KPAGE_SWZ)
    static size_t storage_index(const generator::TileDescriptor& d, size_t i) {
        const size_t cols = size_t(d.shape.back());
        const size_t r = i / cols, c = i % cols;
        if (d.tma == VDC_DESC_PACKED_SW128) {
            const size_t kt = cols / 64, rb = r / 128, rr = r % 128, t = c / 64, ch = (c % 64) / 8;
            return ((rb * kt + t) * 128 + rr) * 64 + ((ch ^ (rr % 8)) * 8) + c % 8;
        }
        if (d.tma == VDC_DESC_KPAGE_SWZ) {
            const size_t ch = c / 8;
            return r * cols + (((ch & 8) | ((ch & 7) ^ (r & 7))) * 8) + c % 8;
        }
        return i;
    }
    static bool permuted(const generator::TileDescriptor& d) {
        return d.tma == VDC_DESC_PACKED_SW128 || d.tma == VDC_DESC_KPAGE_SWZ;
    }
    static void upload(const generator::TileDescriptor& d, void* dptr, const std::vector<float>& host) {
        if (d.elem == workload::ElemType::bf16) {
            std::vector<uint16_t> b(host.size());
            for (size_t i = 0; i < host.size(); ++i) b[permuted(d) ? storage_index(d, i) : i] = detail::to_bf16(host[i]);
            cudaMemcpy(dptr, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
        } else if (d.elem == workload::ElemType::i64) {
            std::vector<int64_t> b(host.size());
            for (size_t i = 0; i < host.size(); ++i) b[i] = int64_t(host[i]);
            cudaMemcpy(dptr, b.data(), b.size() * 8, cudaMemcpyHostToDevice);
        } else {
            cudaMemcpy(dptr, host.data(), host.size() * 4, cudaMemcpyHostToDevice);
        }
    }
    static std::vector<float> download(const generator::TileDescriptor& d, const void* dptr, size_t n) {
        std::vector<float> out(n);
        if (d.elem == workload::ElemType::bf16) {
            std::vector<uint16_t> b(n);
            cudaMemcpy(b.data(), dptr, n * 2, cudaMemcpyDeviceToHost);
            for (size_t i = 0; i < n; ++i) out[i] = detail::from_bf16(b[permuted(d) ? storage_index(d, i) : i]);
        } else if (d.elem == workload::ElemType::i64) {
            std::vector<int64_t> b(n);
            cudaMemcpy(b.data(), dptr, n * 8, cudaMemcpyDeviceToHost);
            for (size_t i = 0; i < n; ++i) out[i] = float(b[i]);
        } else {
            cudaMemcpy(out.data(), dptr, n * 4, cudaMemcpyDeviceToHost);
        }
        return out;
    }
    void swap(Machine& o) {
        std::swap(p_, o.p_);
        std::swap(opt_, o.opt_);
        std::swap(ctx_, o.ctx_);
        std::swap(bufs_, o.bufs_);
        std::swap(step_, o.step_);
        std::swap(done_, o.done_);
        std::swap(now_, o.now_);
        std::swap(alloc_, o.alloc_);
        std::swap(trace_, o.trace_);
        std::swap(n_step_, o.n_step_);
        std::swap(n_cores_, o.n_cores_);
        std::swap(per_sm_, o.per_sm_);
        std::swap(edges_, o.edges_);
        std::swap(last_, o.last_);
    }

    generator::LoweredProgram p_;
    MachineOptions opt_;
    vdc_ctx* ctx_ = nullptr;
    std::vector<Buf> bufs_;
    void* step_ = nullptr;
    bool done_ = false;
    int64_t now_ = 0;
    SlotAllocator alloc_;
    ExecutionReport last_;
    void* trace_ = nullptr;
    uint32_t n_step_ = 0, n_cores_ = 0, per_sm_ = 1;
    std::vector<WaitEdge> edges_;
};

inline ExecutionReport simulate(const generator::LoweredProgram& p, const costmodel::HardwareProfile& hw,
                                MachineOptions opt = {}, uint64_t watchdog = 1000) {
    Machine m(p, hw, synthesize_program_inputs(p), opt);
    return m.run(watchdog);
}

}  // namespace uopsim::machine
