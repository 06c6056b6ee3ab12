// Ring-mode decode lowering (ext): decode-kind graphs -> per-SM memory and
// compute µop streams for the sm_100a ring engine (include/uopsim/ring_abi.h).
//
// Relation to the reference-form decode lowering (decode_lower.cpp) and to
// the reference's lower() (reference src/lower.cpp:48-260):
//  * Same operator -> job decomposition idea (one compute µop per output row
//    range, groups = per-tile fetches in pop order, generator.cpp:156-289),
//    but each operator's rows are split into one contiguous, tile-aligned
//    range per SM (equal tile counts +-1) instead of `chunk % pairs`: at
//    batch 1 every SM streams weights and the slowest SM sets the step time.
//  * Weight / KV-page tiles are the only memory µops: LOAD [send] size=1 in
//    exactly the order the SM's compute µops consume them, so the memory
//    core can run ahead across operator boundaries (the paper's decoupling,
//    PAPER.md:588-626) — its only back-pressure is the ring's slot release.
//  * Activation dependencies are per-tensor readiness counters (the
//    broadcast dependency the reference lacks, SURVEY finding 3), carried in
//    the compute µop's operand block (vdc_job) as (tensor, target).
//  * Operators appear in every SM's streams in topological order, so every
//    counter wait targets jobs that precede it on every SM: the program is
//    deadlock-free by construction (checked by validate_ring_program).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <set>

#include "jobs.hpp"
#include "uopsim/decode.hpp"
#include "uopsim/decode_abi.h"
#include "uopsim/ring_abi.h"
#include "uopsim/util.hpp"

namespace uopsim::generator {

using isa::Opcode;
using isa::UopWord;
using workload::OpKind;

namespace {

int64_t attr_int(const workload::OperatorNode& n, const char* key, int64_t dflt) {
    const auto it = n.attrs.find(key);
    return it == n.attrs.end() ? dflt : std::stoll(it->second);
}
double attr_num(const workload::OperatorNode& n, const char* key, double dflt) {
    const auto it = n.attrs.find(key);
    return it == n.attrs.end() ? dflt : std::stod(it->second);
}

struct Tile {
    uint16_t tensor;
    std::vector<uint16_t> coord;
    uint8_t mode = 0;  // LOAD reg1: 0 plain, VDC_LOAD_PAGED (request, logical page, head), VDC_LOAD_CTX (ctx-bounded page)
};

struct RJob {
    vdc_job j{};
    std::vector<int32_t> publishes;  // counters bumped when the µop completes (default: o_t)
    int32_t head = -1;        // attention: kv head
    std::vector<Tile> tiles;  // ring tiles in consumption order
    uint32_t ordinal = 0;
    uint32_t sm = 0;
    bool counts = true;       // counted in the readiness targets of its outputs (stream-K: one piece per row block)
};

class RingLowering {
  public:
    RingLowering(const workload::OperatorGraph& g, const costmodel::HardwareProfile& hw, int ring_slots)
        : g_(g), hw_(hw), desc_(build_descriptors(g)), ring_slots_(ring_slots) {}

    LoweredProgram run(const GenOptions& opt) {
        if (hw_.vmc_per_sm != 1) throw GeneratorError("ring lowering assumes one VMC per SM");
        sms_ = hw_.sm_count;
        const auto order = detail::topo_nodes(g_);
        uint32_t ordinal = 0;
        for (const auto* n : order) plan(*n, ordinal++);
        // readiness targets: jobs writing each storage tensor per launch
        std::map<int32_t, int32_t> writers;
        std::set<std::pair<int32_t, int32_t>> combined;
        for (const auto& r : jobs_) {
            if (!r.counts) continue;
            if (r.publishes.empty()) ++writers[r.j.o_t];
            for (int32_t t : r.publishes) ++writers[t];
            if (r.j.op == int32_t(Opcode::ATTN_DECODE) && r.j.o2_t >= 0 && combined.insert({r.j.o2_t, r.j.o2_off}).second)
                ++writers[r.j.o2_t];  // one combiner per kv head
        }
        for (auto& r : jobs_) {
            auto need = [&](int32_t t) { return t >= 0 && writers.count(storage(uint16_t(t))) ? writers.at(storage(uint16_t(t))) : 0; };
            if (!(r.j.flags & VDC_JOB_SYM_IN)) r.j.x_need = need(r.j.x_t);
            r.j.a_need = need(r.j.a_t);
            r.j.b_need = need(r.j.b_t);
            r.j.x2_need = need(r.j.x2_t);
            if (r.j.flags & VDC_JOB_BATCH) r.j.maxp = maxp_;
        }
        LoweredProgram p;
        p.descriptors = desc_;
        p.slot_budget = uint16_t(ring_slots_);
        p.ring_slots = uint16_t(ring_slots_);
        p.slot_size = VDC_RING_SLOT_BYTES;
        p.operator_count = ordinal;
        p.workload_hash = g_.content_hash();
        p.profile_name = hw_.name;
        p.input_seed = opt.input_seed;
        p.step_scalars = VDC_STEP_MAX;
        p.vcc_per_sm = 1;
        p.sm_count = uint16_t(sms_);
        p.local_queue_depth = uint16_t(ring_slots_);
        if (batched_) {
            if (ring_slots_ != VDC_RING_COMPUTE_WARPS)
                throw GeneratorError("batched ring programs use 8 ring slots (attention pages map to warp pairs by slot)");
            p.batch = nb_;
            p.npad = npad_;
            p.maxp = maxp_;
            p.page_table_off = 3 * nb_;
            // default page table: the contiguous allocation (shared pools:
            // every entry unallocated, -1, until the host's block allocator
            // fills it); entries past a request's capacity stay -1
            p.page_table.assign(size_t(nb_) * size_t(maxp_), -1);
            if (!shared_pool_)
                for (size_t b = 0; b < pages_.size(); ++b)
                    for (size_t i = 0; i < pages_[b].size(); ++i) p.page_table[b * size_t(maxp_) + i] = pages_[b][i];
            p.step_scalars = uint16_t(3 * nb_ + nb_ * maxp_);
        }
        emit(p);
        return p;
    }

  private:
    const workload::OperatorGraph& g_;
    const costmodel::HardwareProfile& hw_;
    std::vector<TileDescriptor> desc_;
    int ring_slots_;
    uint32_t sms_ = 1;
    std::vector<RJob> jobs_;

    int32_t storage(uint16_t t) const { return desc_[t].view_of >= 0 ? desc_[t].view_of : int32_t(t); }
    uint16_t idx(const std::string& name) const { return g_.tensor_index(name); }

    static vdc_job blank(Opcode op) {
        vdc_job j{};
        j.op = int32_t(op);
        j.x_t = j.a_t = j.b_t = j.o_t = j.o2_t = -1;
        j.x2_t = j.o3_t = j.w3_t = j.part_t = -1;
        j.arrive_ctr = -1;
        j.ssq_t = -1;
        return j;
    }
    // the sums-of-squares companion of a batched activation (decode_graph.cpp), or -1
    int32_t ssq_of(const std::string& x) const {
        return g_.find_tensor(x + ".ssq") ? storage(idx(x + ".ssq")) : -1;
    }

    // contiguous, unit-aligned share of `units` for SM s
    std::pair<int64_t, int64_t> share(int64_t units, uint32_t s) const {
        return {units * s / sms_, units * (s + 1) / sms_};
    }

    void plan(const workload::OperatorNode& n, uint32_t ordinal) {
        if (n.attrs.count("batch")) {
            plan_batched(n, ordinal);
            return;
        }
        switch (n.kind) {
            case OpKind::GEMV:
            case OpKind::RMS_GEMV:
            case OpKind::GEMV_ADD: {
                const size_t first = jobs_.size();
                plan_gemv(n, ordinal);
                if (attr_int(n, "argmax", 0)) {  // greedy sampling fused into the lm_head jobs
                    // one slot per SM: the SM's last job of the node posts (block = 1)
                    const int32_t ctr = int32_t(desc_.size()) + n_arrive_++;
                    std::map<uint32_t, size_t> last;
                    for (size_t i = first; i < jobs_.size(); ++i) last[jobs_[i].sm] = i;
                    std::map<uint32_t, int32_t> slot;
                    for (const auto& [sm, i] : last) slot[sm] = int32_t(slot.size());
                    for (size_t i = first; i < jobs_.size(); ++i) {
                        vdc_job& j = jobs_[i].j;
                        j.flags |= VDC_JOB_ARGMAX | (attr_int(n, "feedback", 0) ? VDC_JOB_FEEDBACK : 0);
                        j.b_t = storage(idx("head.amax"));
                        j.o2_t = storage(idx("next_token"));
                        j.arrive_ctr = ctr;
                        j.arrive_need = int32_t(last.size());
                        j.split = slot[jobs_[i].sm];
                        j.block = last[jobs_[i].sm] == i ? 1 : 0;
                        if (n.attrs.count("tp_argmax")) {  // vocab-parallel: cross-rank (max, index) exchange
                            j.flags |= VDC_JOB_TP_ARGMAX;
                            j.group = storage(idx(n.attrs.at("tp_argmax")));
                            j.o2_off = int32_t(attr_int(n, "vocab_base", 0));
                        }
                    }
                }
                break;
            }
            case OpKind::ATTN_DECODE:
                plan_attention(n, ordinal);
                break;
            case OpKind::ATTN_COMBINE:
                plan_combine(n, ordinal);
                break;
            case OpKind::ALLREDUCE_ADD:
                plan_allreduce(n, ordinal);
                break;
            case OpKind::EMBED_ROW: {
                // no µop: consumers read the embedding row in place (TOKEN_ROW /
                // TOKEN_AUX operands), which removes one global dependency hop
                const uint16_t tab = idx(n.inputs[0]);
                embed_out_ = storage(idx(n.outputs[0]));
                embed_tab_ = storage(tab);
                embed_len_ = int32_t(desc_[tab].cols());
                break;
            }
            default:
                throw GeneratorError("node " + n.id + ": reference kinds cannot be lowered in ring mode");
        }
    }

    void plan_gemv(const workload::OperatorNode& n, uint32_t ordinal) {
        const uint16_t w = idx(n.inputs[0]);
        const TileDescriptor& wd = desc_[w];
        if (wd.view_of >= 0) throw GeneratorError("node " + n.id + ": weight must own its storage");
        const int64_t K = wd.cols(), plane_rows = wd.rows(), M = wd.elem_count() / K;
        const int64_t tr = wd.tile_rows, tc = wd.tile_cols, tpr = K / tc;
        const int64_t eb = workload::elem_bytes(wd.elem);
        if (K % tc || 8 % tr || uint64_t(tr * tc * eb) > VDC_RING_SLOT_BYTES)
            throw GeneratorError("node " + n.id + ": weight tiles are not ring tiles (build the graph with layout.ring)");
        if (K * eb > 2 * VDC_RING_MAX_K || (K * eb) % 16 || (tc * eb) % 16)
            throw GeneratorError("node " + n.id + ": reduction length unsupported by the ring engine");
        if (wd.elem == workload::ElemType::bf16) {  // tensor-core tiles: 2/4/8 rows, whole k-steps of 16 * (16 / rows) chunks
            const int64_t nc = 16 / std::max<int64_t>(1, tr), cpt = tc / 8;
            if ((tr != 2 && tr != 4 && tr != 8) || cpt % (2 * nc))
                throw GeneratorError("node " + n.id + ": bf16 weight tile shape unsupported by the tensor-core GEMV");
        }
        const bool rope = attr_int(n, "rope", 0) != 0;
        const int64_t swiglu = attr_int(n, "swiglu", 0);
        int64_t unit = tr;
        if (rope) unit = std::lcm(unit, int64_t(2));
        if (swiglu) unit = std::lcm(unit, swiglu);
        if (M % unit) throw GeneratorError("node " + n.id + ": rows not a multiple of the job alignment");
        // output regions (qkv: q | k | v), each a separate job family
        struct Region {
            int64_t r0, r1;
            uint16_t out;
            bool kv;
        };
        std::vector<Region> regions;
        int64_t head_dim = 0, qrows = M, kvrows = 0;
        const bool qkv = n.outputs.size() == 3;
        if (qkv) {
            // one job per SM share even across the q | k | v boundaries (the
            // engine routes each row: VDC_JOB_QKV), so no SM pays two epilogues
            const TileDescriptor& kc = desc_[idx(n.outputs[1])];
            head_dim = kc.shape.back();
            kvrows = kc.shape[0] * head_dim;
            qrows = desc_[idx(n.outputs[0])].rows();
            if (qrows + 2 * kvrows != M) throw GeneratorError("node " + n.id + ": q/k/v rows do not add up to W rows");
            if (qrows % unit || kvrows % unit || !rope)
                throw GeneratorError("node " + n.id + ": q/k/v boundaries must be tile aligned and rotary enabled");
            regions = {{0, M, idx(n.outputs[0]), false}};
        } else {
            regions = {{0, M, idx(n.outputs[0]), false}};
        }
        if (tpr > VDC_RING_MAX_COL_TILES) throw GeneratorError("node " + n.id + ": more column tiles per row than the engine keeps");
        const int64_t max_rows = (VDC_RING_MAX_JOB_ROWS / unit) * unit;
        const int64_t units = M / unit;
        const TileDescriptor& xd = desc_[idx(n.inputs[1])];
        for (uint32_t s = 0; s < sms_; ++s) {
            const auto [u0, u1] = share(units, s);
            for (const auto& reg : regions) {
                int64_t a = std::max(u0 * unit, reg.r0), b = std::min(u1 * unit, reg.r1);
                for (int64_t c0 = a; c0 < b; c0 += max_rows) {
                    const int64_t c1 = std::min(b, c0 + max_rows);
                    RJob r;
                    r.ordinal = ordinal;
                    r.sm = s;
                    vdc_job& j = r.j;
                    j = blank(n.kind == OpKind::GEMV ? Opcode::GEMV : n.kind == OpKind::RMS_GEMV ? Opcode::RMS_GEMV : Opcode::GEMV_ADD);
                    j.r0 = int32_t(c0);
                    j.r1 = int32_t(c1);
                    j.k = int32_t(K);
                    j.tile_rows = int32_t(tr);
                    j.tile_cols = int32_t(tc);
                    j.x_t = storage(idx(n.inputs[1]));
                    j.x_off = 0;
                    if (j.x_t == embed_out_) {
                        j.x_t = embed_tab_;
                        j.flags |= VDC_JOB_TOKEN_ROW;
                    }
                    if (xd.elem_count() != K) throw GeneratorError("node " + n.id + ": input length != reduction length");
                    if (n.kind == OpKind::RMS_GEMV) {
                        j.flags |= VDC_JOB_RMS;
                        j.a_t = storage(idx(n.inputs[2]));
                        j.eps = float(attr_num(n, "eps", 1e-5));
                    } else if (n.kind == OpKind::GEMV_ADD) {
                        j.flags |= VDC_JOB_RESID;
                        j.a_t = storage(idx(n.inputs[2]));
                        j.a_off = 0;
                        if (j.a_t == embed_out_) {
                            j.a_t = embed_tab_;
                            j.flags |= VDC_JOB_TOKEN_AUX;
                            j.cache_rows = embed_len_;
                        }
                    }
                    j.o_t = storage(reg.out);
                    j.out_row0 = int32_t(reg.r0);
                    j.head_dim = int32_t(head_dim);
                    if (qkv) {
                        j.flags |= VDC_JOB_QKV;
                        if (attr_int(n, "qk_norm", 0)) j.flags |= VDC_JOB_QKNORM;  // q / k stored un-rotated
                        j.theta = float(attr_num(n, "theta", 10000.0));
                        j.block = int32_t(qrows);
                        j.split = int32_t(kvrows);
                        j.b_t = storage(idx(n.outputs[1]));
                        j.o2_t = storage(idx(n.outputs[2]));
                        j.cache_rows = int32_t(desc_[idx(n.outputs[1])].shape[1]);
                        if (desc_[uint16_t(j.b_t)].tma == VDC_DESC_KPAGE_SWZ) j.flags |= VDC_JOB_KVSWZ;
                        if (c0 < qrows) r.publishes.push_back(j.o_t);
                        if (c0 < qrows + kvrows && c1 > qrows) r.publishes.push_back(j.b_t);
                        if (c1 > qrows + kvrows) r.publishes.push_back(j.o2_t);
                    } else {
                        r.publishes.push_back(j.o_t);
                    }
                    if (desc_[reg.out].symmetric) {  // TP partial sums: this rank's slot of every rank's buffer
                        j.flags |= VDC_JOB_SYM_OUT;
                        j.o_off = int32_t(attr_int(n, "tp_rank", 0) * M);
                        j.group = int32_t(attr_int(n, "tp_world", 1));
                    }
                    if (swiglu) {
                        j.flags |= VDC_JOB_SWIGLU;
                        j.block = int32_t(swiglu);
                    }
                    // consumption order of the ring engine: row groups outer,
                    // column tiles inner (tile t -> compute warp t mod 8)
                    for (int64_t row = c0; row < c1; row += tr)
                        for (int64_t ct = 0; ct < tpr; ++ct) {
                            const int64_t plane = row / plane_rows, prow = row % plane_rows;
                            if (wd.shape.size() == 3)
                                r.tiles.push_back({w, {uint16_t(plane), uint16_t(prow / tr), uint16_t(ct)}});
                            else
                                r.tiles.push_back({w, {uint16_t(prow / tr), uint16_t(ct)}});
                        }
                    jobs_.push_back(std::move(r));
                }
            }
        }
    }

    // Qwen3 QK-norm: the attention µop normalises q and the appended k row
    // (weights in out_row0 / block), then applies the rotary
    void qk_norm_fields(const workload::OperatorNode& n, vdc_job& j) const {
        if (!n.attrs.count("q_norm")) return;
        j.flags |= VDC_JOB_QKNORM;
        j.out_row0 = storage(idx(n.attrs.at("q_norm")));
        j.block = storage(idx(n.attrs.at("k_norm")));
        j.eps = float(attr_num(n, "eps", 1e-6));
        j.theta = float(attr_num(n, "theta", 10000.0));
    }

    void plan_attention(const workload::OperatorNode& n, uint32_t ordinal) {
        const uint16_t q = idx(n.inputs[0]), kc = idx(n.inputs[1]), vc = idx(n.inputs[2]), part = idx(n.outputs[0]);
        const TileDescriptor& kd = desc_[kc];
        const int64_t hkv = kd.shape[0], T = kd.shape[1], hd = kd.shape[2], page_rows = kd.tile_rows;
        const int64_t grp = desc_[q].tile_rows / hd;
        if (kd.tile_cols != hd || uint64_t(page_rows * hd * workload::elem_bytes(kd.elem)) > VDC_RING_SLOT_BYTES)
            throw GeneratorError("node " + n.id + ": KV pages do not fit a ring slot");
        const bool bf = kd.elem == workload::ElemType::bf16;
        if (!(bf ? (hd == 128 && (grp == 4 || grp == 8)) : (hd == 64 && grp == 1)))
            throw GeneratorError("node " + n.id + ": ring attention is built for bf16 head_dim 128 with GQA group 4/8 "
                                 "and fp32 head_dim 64 with group 1");
        if (page_rows != 64) throw GeneratorError("node " + n.id + ": ring attention pages are 64 rows");
        const int64_t pages = attr_int(n, "ctx_pages", 1), per = attr_int(n, "pages_per_job", 1);
        // all of a job's K/V tiles must fit the ring at once: the engine lets
        // any warp wait on them (the page -> warp-pair map ignores slot owners)
        if (2 * std::min(pages, per) > ring_slots_)
            throw GeneratorError("node " + n.id + ": 2 * pages_per_job must not exceed ring_slots");
        const int64_t splits = ceil_div(pages, per);
        int64_t k = 0;
        for (int64_t h = 0; h < hkv; ++h) {
            const int32_t ctr = int32_t(desc_.size()) + n_arrive_++;  // per-kv-head arrival counter
            for (int64_t s = 0; s < splits; ++s, ++k) {
                RJob r;
                r.ordinal = ordinal;
                r.sm = uint32_t(k % sms_);
                r.head = int32_t(h);
                vdc_job& j = r.j;
                j = blank(Opcode::ATTN_DECODE);
                j.r0 = int32_t(s * per);
                j.r1 = int32_t(std::min(pages, (s + 1) * per));
                j.k = int32_t(hd);
                j.head_dim = int32_t(hd);
                j.group = int32_t(grp);
                j.tile_rows = int32_t(page_rows);
                j.tile_cols = int32_t(hd);
                j.cache_rows = int32_t(T);
                j.scale = float(1.0 / std::sqrt(double(hd)));
                j.x_t = storage(q);
                j.x_off = int32_t(h * grp * hd);
                j.a_t = storage(kc);
                j.a_off = int32_t(h * T * hd);
                j.b_t = storage(vc);
                j.b_off = int32_t(h * T * hd);
                j.o_t = storage(part);
                j.o_off = int32_t((h * splits + s) * grp * (hd + 2));
                j.split = int32_t(s);
                j.arrive_ctr = ctr;
                j.arrive_need = int32_t(splits);
                if (kd.tma == VDC_DESC_KPAGE_SWZ) j.flags |= VDC_JOB_KVSWZ;
                qk_norm_fields(n, j);
                // ctx-bounded: pages past the step's context are not loaded
                for (int64_t pg = j.r0; pg < j.r1; ++pg) {
                    r.tiles.push_back({kc, {uint16_t(h), uint16_t(pg), 0}, VDC_LOAD_CTX});
                    r.tiles.push_back({vc, {uint16_t(h), uint16_t(pg), 0}, VDC_LOAD_CTX});
                }
                jobs_.push_back(std::move(r));
            }
        }
        attn_ = {hkv, splits, grp, hd, k};
    }

    // ALLREDUCE_ADD: x_next = residual + sum of the W rank slots of the
    // symmetric partial buffer (fixed rank order), rows split over the SMs
    // like a GEMV share; no ring tiles. The readiness target of the partials
    // is world x (this rank's producer µops): every rank runs the same split.
    void plan_allreduce(const workload::OperatorNode& n, uint32_t ordinal) {
        const int32_t part = storage(idx(n.inputs[0])), res = storage(idx(n.inputs[1])), out = storage(idx(n.outputs[0]));
        const int64_t d = desc_[uint16_t(out)].rows(), W = attr_int(n, "tp_world", 1);
        int32_t producers = 0;
        for (const auto& r : jobs_)
            for (int32_t t : r.publishes) producers += t == part;
        const int64_t unit = 8, units = ceil_div<int64_t>(d, unit);
        for (uint32_t s = 0; s < sms_; ++s) {
            const auto [u0, u1] = share(units, s);
            if (u0 == u1) continue;
            RJob r;
            r.ordinal = ordinal;
            r.sm = s;
            vdc_job& j = r.j;
            j = blank(Opcode::ALLREDUCE_ADD);
            j.flags = VDC_JOB_SYM_IN | VDC_JOB_RESID;
            j.r0 = int32_t(u0 * unit);
            j.r1 = int32_t(std::min(d, u1 * unit));
            j.k = int32_t(d);
            j.group = int32_t(W);
            j.x_t = part;
            j.x_need = int32_t(W) * producers;  // fixed here: the symmetric counter collects every rank
            j.a_t = res;
            if (j.a_t == embed_out_) {
                j.a_t = embed_tab_;
                j.flags |= VDC_JOB_TOKEN_AUX;
                j.cache_rows = embed_len_;
            }
            j.o_t = out;
            r.publishes.push_back(out);
            jobs_.push_back(std::move(r));
        }
    }

    // ring mode fuses the combine into the attention jobs (the last split of
    // each kv head to arrive merges, saving one dependency hop); the node
    // names the output the combiner writes. Combine µops use the same
    // operand layout (o_t/o_off = partials of the head, o2 = output).
    void plan_combine(const workload::OperatorNode& n, uint32_t ordinal) {
        (void)ordinal;
        const int32_t part = storage(idx(n.inputs[0])), out = storage(idx(n.outputs[0]));
        for (auto& r : jobs_)
            if (r.j.op == int32_t(Opcode::ATTN_DECODE) && r.j.o_t == part) {
                r.j.o2_t = out;
                r.j.o2_off = r.head * r.j.group * r.j.head_dim;
            }
    }

    void emit(LoweredProgram& p) {
        std::vector<std::vector<size_t>> per_sm(sms_);
        for (size_t i = 0; i < jobs_.size(); ++i) per_sm[jobs_[i].sm].push_back(i);
        for (uint32_t s = 0; s < sms_; ++s) {
            std::stable_sort(per_sm[s].begin(), per_sm[s].end(),
                             [&](size_t a, size_t b) { return jobs_[a].ordinal < jobs_[b].ordinal; });
            auto& vs = p.streams[CoreId::vmc(uint16_t(s))];
            auto& vm = p.meta[CoreId::vmc(uint16_t(s))];
            auto& cs = p.streams[CoreId::vcc_id(uint16_t(s), 0)];
            auto& cm = p.meta[CoreId::vcc_id(uint16_t(s), 0)];
            size_t tiles_so_far = 0;
            for (size_t ji : per_sm[s]) {
                RJob r = jobs_[ji];
                if ((r.j.flags & VDC_JOB_BATCH) && r.j.op == int32_t(Opcode::ATTN_DECODE) && (tiles_so_far & 1)) {
                    // K tiles on even ring indices: pages map to warp pairs by slot
                    r.j.lead_pad = 1;
                    r.tiles.insert(r.tiles.begin(), Tile{pad_t_, {0, 0}});
                }
                tiles_so_far += r.tiles.size();
                const int32_t slot = int32_t(p.jobs.size());
                p.jobs.push_back(r.j);
                for (const Tile& t : r.tiles) {
                    UopWord u;
                    u.opcode = Opcode::LOAD;
                    u.flags = isa::kFlagSend;
                    u.flow = 1;
                    u.size = 1;
                    u.addr = isa::AddressSpec::tile(t.tensor, t.coord);
                    u.reg1 = desc_[t.tensor].tma == VDC_DESC_PACKED_SW128 ? 1 : t.mode;  // packed 16 KB weight tile / KV page mode
                    vs.push_back(u);
                    vm.push_back({r.ordinal, slot, -1});
                }
                UopWord c;
                c.opcode = Opcode(r.j.op);
                c.size = uint16_t(r.tiles.size());
                c.imm = slot;
                c.flow = 1;
                cs.push_back(c);
                cm.push_back({r.ordinal, slot, -1});
            }
            for (auto* st : {&vs, &cs}) {
                UopWord h;
                h.opcode = Opcode::HALT;
                h.flags = isa::kFlagLast;
                st->push_back(h);
            }
            vm.push_back({0, -1, -1});
            cm.push_back({0, -1, -1});
        }
    }

    // ---------------------------------------------------------------- batched
    // Batched programs (decode.hpp LayoutConfig::batch): BGEMM µops on the
    // tensor cores, split-KV attention per (request, kv head), paged pools.
    bool batched_ = false;
    int32_t nb_ = 0, npad_ = 0, maxp_ = 0;
    bool shared_pool_ = false;  // layout.pool_pages > 0: the host allocates pages (page table starts unallocated)
    std::vector<std::vector<int64_t>> pages_;  // request -> physical page of each logical page
    uint16_t pad_t_ = 0;

    void plan_batched(const workload::OperatorNode& n, uint32_t ordinal) {
        batched_ = true;
        nb_ = int32_t(attr_int(n, "batch", 1));
        npad_ = decode::batch_npad(nb_);
        pad_t_ = idx("ring.pad");
        switch (n.kind) {
            case OpKind::EMBED_ROW:  // one job per request, spread over the SMs
                for (int32_t rq = 0; rq < nb_; ++rq) {
                RJob r;
                r.ordinal = ordinal;
                r.sm = uint32_t(rq) % sms_;
                vdc_job& j = r.j;
                j = blank(Opcode::ELEMWISE);
                j.flags = VDC_JOB_BATCH;
                j.r0 = rq;
                j.r1 = rq + 1;
                j.nb = nb_;
                j.npad = npad_;
                j.x_t = storage(idx(n.inputs[0]));
                j.w3_t = storage(idx(n.inputs[1]));
                j.k = int32_t(desc_[uint16_t(j.x_t)].cols());
                j.o_t = storage(idx(n.outputs[0]));
                j.o3_t = storage(idx(n.outputs[1]));
                j.ssq_t = ssq_of(n.outputs[0]);
                r.publishes = {j.o_t, j.o3_t};
                jobs_.push_back(std::move(r));
                }
                break;
            case OpKind::RMS_GEMV:
            case OpKind::GEMV_ADD:
            case OpKind::GEMV:
                plan_bgemm(n, ordinal);
                break;
            case OpKind::ALLREDUCE_ADD:
                plan_ballreduce(n, ordinal);
                break;
            case OpKind::ATTN_DECODE:
                plan_battention(n, ordinal);
                break;
            case OpKind::ATTN_COMBINE: {
                const int32_t part = storage(idx(n.inputs[0])), out = storage(idx(n.outputs[0]));
                const int64_t width = desc_[uint16_t(out)].cols();
                for (auto& r : jobs_)
                    if (r.j.op == int32_t(Opcode::ATTN_DECODE) && r.j.o_t == part) {
                        r.j.o2_t = out;
                        r.j.o2_off = int32_t(r.j.req * width + r.head * r.j.group * r.j.head_dim);
                    }
                break;
            }
            default:
                throw GeneratorError("node " + n.id + ": kind has no batched lowering");
        }
    }

    // stream-K: the op's (row block, k tile) grid in row-block-major order is
    // cut into one contiguous range per SM; each maximal run inside a row
    // block is a piece (one µop). Pieces of a split block write fp32
    // partials; the last to arrive adds them in piece order and runs the
    // epilogue, so every SM streams the same number of weight tiles (+-1).
    void plan_bgemm(const workload::OperatorNode& n, uint32_t ordinal) {
        const uint16_t w = idx(n.inputs[0]);
        const TileDescriptor& wd = desc_[w];
        const int64_t M = wd.rows(), K = wd.cols();
        if (wd.tile_rows != VDC_RING_BGEMM_ROWS || wd.tile_cols != VDC_RING_BGEMM_KT || wd.tma != VDC_DESC_PACKED_SW128 ||
            M % VDC_RING_BGEMM_ROWS || K % VDC_RING_BGEMM_KT)
            throw GeneratorError("node " + n.id + ": batched weights need packed 128 x 64 tiles");
        const int64_t rb = M / VDC_RING_BGEMM_ROWS, kts = K / VDC_RING_BGEMM_KT, T = rb * kts;
        const bool qkv = n.outputs.size() == 3, resid = n.kind == OpKind::GEMV_ADD, swiglu = attr_int(n, "swiglu", 0) != 0;
        const std::string op = n.id.substr(n.id.find('.') == std::string::npos ? 0 : n.id.find('.') + 1);
        const uint16_t skt = idx(op + ".sk");
        if (desc_[skt].elem_count() < (rb + int64_t(sms_)) * npad_ * VDC_RING_BGEMM_ROWS)
            throw GeneratorError("node " + n.id + ": stream-K partial buffer too small for " + std::to_string(sms_) + " SMs");
        struct Piece {
            uint32_t sm;
            int64_t kt0, kt1;
        };
        std::vector<std::vector<Piece>> blocks;
        blocks.resize(size_t(rb));
        for (uint32_t s = 0; s < sms_; ++s) {
            const auto [t0, t1] = share(T, s);
            for (int64_t t = t0; t < t1;) {
                const int64_t b = t / kts, e = std::min(t1, (b + 1) * kts);
                blocks[size_t(b)].push_back({s, t - b * kts, e - b * kts});
                t = e;
            }
        }
        int32_t slot = 0;
        const size_t first_job = jobs_.size();
        for (int64_t b = 0; b < rb; ++b) {
            const auto& ps = blocks[size_t(b)];
            const int32_t ctr = ps.size() > 1 ? int32_t(desc_.size()) + n_arrive_++ : -1;
            for (size_t i = 0; i < ps.size(); ++i) {
                RJob r;
                r.ordinal = ordinal;
                r.sm = ps[i].sm;
                r.counts = i == 0;  // one publisher per row block (whichever piece arrives last)
                vdc_job& j = r.j;
                j = blank(Opcode::BGEMM);
                j.flags = VDC_JOB_BATCH;
                j.r0 = int32_t(b * VDC_RING_BGEMM_ROWS);
                j.r1 = j.r0 + VDC_RING_BGEMM_ROWS;
                j.k = int32_t(K);
                j.tile_rows = VDC_RING_BGEMM_ROWS;
                j.tile_cols = VDC_RING_BGEMM_KT;
                j.kt0 = int32_t(ps[i].kt0);
                j.kt1 = int32_t(ps[i].kt1);
                j.nb = nb_;
                j.npad = npad_;
                j.x_t = storage(idx(n.inputs[1]));
                if (desc_[uint16_t(j.x_t)].tma != uint32_t(npad_) || desc_[uint16_t(j.x_t)].cols() != K)
                    throw GeneratorError("node " + n.id + ": activations must be an (npad, K) TMA tensor");
                j.part_t = storage(skt);
                j.part_off = slot++;
                j.split = int32_t(i);
                j.arrive_ctr = ctr;
                j.arrive_need = int32_t(ps.size());
                j.o_t = storage(idx(n.outputs[0]));
                j.cache_rows = int32_t(M);
                if (n.kind == OpKind::RMS_GEMV) {
                    j.flags |= VDC_JOB_RMS;
                    j.x2_t = storage(idx(n.inputs[2]));
                    j.eps = float(attr_num(n, "eps", 1e-5));
                    j.ssq_t = ssq_of(n.inputs[2]);
                }
                if (resid) {
                    j.flags |= VDC_JOB_RESID;
                    j.a_t = storage(idx(n.inputs[2]));
                    j.w3_t = storage(idx(n.inputs[3]));
                    j.o3_t = storage(idx(n.outputs[1]));
                    j.ssq_t = ssq_of(n.outputs[0]);
                    r.publishes = {j.o_t, j.o3_t};
                } else if (qkv) {
                    const TileDescriptor& kc = desc_[idx(n.outputs[1])];
                    j.flags |= VDC_JOB_QKV;
                    if (attr_int(n, "qk_norm", 0)) j.flags |= VDC_JOB_QKNORM;
                    j.head_dim = int32_t(kc.shape[2]);
                    j.kvrows = int32_t(kc.shape[1] / 64 * kc.shape[2]);
                    j.block = int32_t(M - 2 * j.kvrows);
                    j.cache_rows = j.block;  // q row stride
                    j.theta = float(attr_num(n, "theta", 10000.0));
                    j.b_t = storage(idx(n.outputs[1]));
                    j.o2_t = storage(idx(n.outputs[2]));
                    j.ptab = 3 * nb_;
                    r.publishes = {j.o_t, j.b_t, j.o2_t};
                } else {
                    if (swiglu) {
                        j.flags |= VDC_JOB_SWIGLU;
                        j.cache_rows = int32_t(M / 2);
                    }
                    if (desc_[uint16_t(j.o_t)].symmetric) {  // TP partial sums -> slot tp_rank of every rank's buffer
                        j.flags |= VDC_JOB_SYM_OUT;
                        j.o_off = int32_t(attr_int(n, "tp_rank", 0) * npad_ * M);
                        j.group = int32_t(attr_int(n, "tp_world", 1));
                    }
                    r.publishes = {j.o_t};
                }
                for (int64_t kt = ps[i].kt0; kt < ps[i].kt1; ++kt) r.tiles.push_back({w, {uint16_t(b), uint16_t(kt)}});
                jobs_.push_back(std::move(r));
            }
        }
        if (attr_int(n, "argmax", 0)) {
            // greedy sampling: each SM merges its finished row blocks per request;
            // its last piece (block = 1) posts slot `req`; arrival counter am_ctr,
            // am_need SMs; the last SM writes the tokens
            const int32_t ctr = int32_t(desc_.size()) + n_arrive_++;
            std::map<uint32_t, size_t> last;
            for (size_t i = first_job; i < jobs_.size(); ++i) last[jobs_[i].sm] = i;
            std::map<uint32_t, int32_t> slot_of;
            for (const auto& [sm, i] : last) slot_of[sm] = int32_t(slot_of.size());
            if (slot_of.size() > 256) throw GeneratorError("node " + n.id + ": argmax slots exceed 256 SMs");
            for (size_t i = first_job; i < jobs_.size(); ++i) {
                vdc_job& j = jobs_[i].j;
                j.flags |= VDC_JOB_ARGMAX | (attr_int(n, "feedback", 0) ? VDC_JOB_FEEDBACK : 0);
                j.b_t = storage(idx("head.amax"));
                j.o2_t = storage(idx("next_token"));
                j.req = slot_of[jobs_[i].sm];
                j.block = last[jobs_[i].sm] == i ? 1 : 0;
                j.am_ctr = ctr;
                j.am_need = int32_t(slot_of.size());
                if (n.attrs.count("tp_argmax")) {  // vocab-parallel: cross-rank (max, index) exchange
                    j.flags |= VDC_JOB_TP_ARGMAX;
                    j.am_sym = storage(idx(n.attrs.at("tp_argmax")));
                    j.am_base = int32_t(attr_int(n, "vocab_base", 0));
                    j.am_valid = int32_t(attr_int(n, "vocab_valid", 1 << 30));
                }
            }
        }
    }

    // batched ALLREDUCE_ADD (TP): rows split over the SMs (8-row units); per
    // row and request x = residual + sum of the W rank slots (rank order),
    // plus the next RMSNorm's operand x * w. The partials' readiness target
    // is W x (row blocks of the producer) on the local header counter.
    void plan_ballreduce(const workload::OperatorNode& n, uint32_t ordinal) {
        const int32_t part = storage(idx(n.inputs[0])), res = storage(idx(n.inputs[1])), nw = storage(idx(n.inputs[2]));
        const int32_t out = storage(idx(n.outputs[0])), outn = storage(idx(n.outputs[1]));
        const int64_t d = desc_[uint16_t(out)].cols(), W = attr_int(n, "tp_world", 1);
        int32_t producers = 0;
        for (const auto& r : jobs_)
            for (int32_t t : r.publishes)
                if (t == part) producers += r.counts ? 1 : 0;
        const int64_t unit = 8, units = ceil_div<int64_t>(d, unit);
        for (uint32_t s = 0; s < sms_; ++s) {
            const auto [u0, u1] = share(units, s);
            if (u0 == u1) continue;
            RJob r;
            r.ordinal = ordinal;
            r.sm = s;
            vdc_job& j = r.j;
            j = blank(Opcode::ALLREDUCE_ADD);
            j.flags = VDC_JOB_SYM_IN | VDC_JOB_RESID | VDC_JOB_BATCH;
            j.r0 = int32_t(u0 * unit);
            j.r1 = int32_t(std::min(d, u1 * unit));
            j.k = int32_t(d);
            j.group = int32_t(W);
            j.nb = nb_;
            j.npad = npad_;
            j.x_t = part;
            j.x_need = int32_t(W) * producers;
            j.a_t = res;
            j.w3_t = nw;
            j.o_t = out;
            j.o3_t = outn;
            r.publishes = {out, outn};
            jobs_.push_back(std::move(r));
        }
    }

    // split-KV jobs of (request, kv head, page range), balanced over the SMs
    // by page count (longest first onto the least loaded SM)
    void plan_battention(const workload::OperatorNode& n, uint32_t ordinal) {
        const uint16_t q = idx(n.inputs[0]), kc = idx(n.inputs[1]), vc = idx(n.inputs[2]), part = idx(n.outputs[0]);
        const TileDescriptor& kd = desc_[kc];
        const int64_t hd = kd.shape[2], hkv = kd.shape[1] / 64, qrows = desc_[q].cols(), grp = qrows / hd / hkv;
        if (!(grp == 4 || grp == 8) || hd != 128) throw GeneratorError("node " + n.id + ": batched attention needs hd 128, group 4/8");
        const int64_t per = attr_int(n, "pages_per_job", 4);
        if (pages_.empty()) {  // contiguous page allocation in the pool, request-major
            std::vector<int64_t> rp;
            std::string s = n.attrs.at("req_pages");
            for (size_t p0 = 0; p0 < s.size();) {
                const size_t p1 = s.find(',', p0);
                rp.push_back(std::stoll(s.substr(p0, p1 == std::string::npos ? std::string::npos : p1 - p0)));
                p0 = p1 == std::string::npos ? s.size() : p1 + 1;
            }
            int64_t next = 0;
            const bool shared = attr_int(n, "prefill", 0) != 0;  // prefill chunk: one sequence's pages
            for (int64_t c : rp) {
                pages_.emplace_back();
                if (shared) next = 0;
                for (int64_t i = 0; i < c; ++i) pages_.back().push_back(next++);
                maxp_ = std::max<int32_t>(maxp_, int32_t(c));
            }
            if (int64_t(pages_.size()) != nb_) throw GeneratorError("req_pages does not match the batch");
            shared_pool_ = attr_int(n, "pool_pages", 0) > 0;
        }
        struct AJ {
            int64_t b, h, s, p0, p1;
        };
        std::vector<AJ> all;
        for (int64_t b = 0; b < nb_; ++b) {
            const int64_t np = int64_t(pages_[size_t(b)].size()), splits = ceil_div(np, per);
            for (int64_t h = 0; h < hkv; ++h)
                for (int64_t s = 0; s < splits; ++s) all.push_back({b, h, s, s * per, std::min(np, (s + 1) * per)});
        }
        // partial slots: (b, h) blocks contiguous in split order (the combiner walks them)
        std::vector<int64_t> order(all.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t c) {
            return all[size_t(a)].p1 - all[size_t(a)].p0 > all[size_t(c)].p1 - all[size_t(c)].p0;
        });
        // cost model (in ring tiles): 2 per page plus a fixed per-job cost
        // (q staging, warp merge, arrival, the last split's combine; measured
        // ~8 us = ~22 tiles at a 0.35 us tile, tools/attn_cost.py);
        // layout.attn_job_cost overrides it
        const int64_t fixed = attr_int(n, "job_cost", 22);
        std::vector<int64_t> load(sms_, 0);
        std::vector<uint32_t> sm_of(all.size());
        for (int64_t i : order) {
            const uint32_t s = uint32_t(std::min_element(load.begin(), load.end()) - load.begin());
            sm_of[size_t(i)] = s;
            load[s] += 2 * (all[size_t(i)].p1 - all[size_t(i)].p0) + fixed;
        }
        std::map<std::pair<int64_t, int64_t>, int32_t> ctr;
        for (size_t i = 0; i < all.size(); ++i) {
            const AJ& a = all[i];
            if (!ctr.count({a.b, a.h})) ctr[{a.b, a.h}] = int32_t(desc_.size()) + n_arrive_++;
            RJob r;
            r.ordinal = ordinal;
            r.sm = sm_of[i];
            r.head = int32_t(a.h);
            vdc_job& j = r.j;
            j = blank(Opcode::ATTN_DECODE);
            j.flags = VDC_JOB_BATCH | (attr_int(n, "prefill", 0) ? VDC_JOB_PREFILL : 0);
            j.r0 = int32_t(a.p0);
            j.r1 = int32_t(a.p1);
            j.k = int32_t(hd);
            j.head_dim = int32_t(hd);
            j.group = int32_t(grp);
            j.tile_rows = 64;
            j.tile_cols = int32_t(hd);
            j.cache_rows = int32_t(hkv * 64);
            j.scale = float(1.0 / std::sqrt(double(hd)));
            j.nb = nb_;
            j.npad = npad_;
            j.req = int32_t(a.b);
            j.ptab = 3 * nb_;
            j.x_t = storage(q);
            j.x_off = int32_t(a.b * qrows + a.h * grp * hd);
            j.a_t = storage(kc);
            j.a_off = int32_t(a.h * 64 * hd);
            j.b_t = storage(vc);
            j.b_off = j.a_off;
            j.o_t = storage(part);
            j.o_off = int32_t(i) * int32_t(grp * (hd + 2));
            j.split = int32_t(a.s);
            j.arrive_ctr = ctr[{a.b, a.h}];
            qk_norm_fields(n, j);
            j.arrive_need = int32_t(ceil_div<int64_t>(int64_t(pages_[size_t(a.b)].size()), per));
            // (request, logical page, head): the memory core resolves the
            // physical page through the step block's page table at run time
            // and skips pages past the request's context (no DRAM traffic)
            for (int64_t pg = a.p0; pg < a.p1; ++pg) {
                r.tiles.push_back({kc, {uint16_t(a.b), uint16_t(pg), uint16_t(a.h)}, VDC_LOAD_PAGED});
                r.tiles.push_back({vc, {uint16_t(a.b), uint16_t(pg), uint16_t(a.h)}, VDC_LOAD_PAGED});
            }
            jobs_.push_back(std::move(r));
        }
    }

    int32_t n_arrive_ = 0;
    int32_t embed_out_ = -2, embed_tab_ = -1, embed_len_ = 0;
    struct AttnInfo {
        int64_t hkv = 0, splits = 1, grp = 1, hd = 0, jobs = 0;
    } attn_;
};

}  // namespace

LoweredProgram lower_decode_ring(const workload::OperatorGraph& g, const costmodel::HardwareProfile& hw, const GenOptions& opt,
                                 int ring_slots) {
    // ring tile g lives in slot g % R and is consumed by compute warp
    // (g % R) % 8: every slot has a single consumer warp (a slot shared by
    // two warps could be waited on one phase ahead, which mbarrier parity
    // waits cannot distinguish); R = 9 would give an attention page's K and
    // V slots the same owner
    if (ring_slots < VDC_RING_COMPUTE_WARPS || ring_slots > VDC_RING_MAX_SLOTS || ring_slots == VDC_RING_COMPUTE_WARPS + 1)
        throw GeneratorError("ring_slots must be 8, 10, 11 or 12");
    return RingLowering(g, hw, ring_slots).run(opt);
}

// Ring-program invariants (the ring analogue of validate + the certificate):
// per SM, compute µops consume exactly the LOADs of its memory stream in
// order, and every readiness wait targets an operator that precedes the
// waiting µop on every SM (topological per-SM order => no cyclic waits).
std::vector<isa::Violation> validate_ring_program(const LoweredProgram& p) {
    std::vector<isa::Violation> v;
    std::map<int32_t, uint32_t> writer_op;  // storage -> operator ordinal
    for (const auto& [core, m] : p.meta) {
        if (core.kind != isa::CoreKind::vcc) continue;
        const auto& s = p.streams.at(core);
        for (size_t i = 0; i < s.size(); ++i)
            if (s[i].klass() == isa::OpClass::compute) {
                const vdc_job& j = p.jobs.at(size_t(s[i].imm));
                writer_op[j.o_t] = m[i].op;
                if (j.flags & VDC_JOB_QKV) writer_op[j.b_t] = writer_op[j.o2_t] = m[i].op;
                if (j.o3_t >= 0 && (j.flags & VDC_JOB_BATCH)) writer_op[j.o3_t] = m[i].op;
            }
    }
    for (const auto& [core, s] : p.streams) {
        if (core.kind != isa::CoreKind::vcc) continue;
        const auto& vmc = p.streams.at(CoreId::vmc(core.sm));
        size_t loads = 0;
        for (const auto& u : vmc) loads += u.opcode == Opcode::LOAD;
        size_t consumed = 0;
        uint32_t last_op = 0;
        const auto& m = p.meta.at(core);
        for (size_t i = 0; i < s.size(); ++i) {
            if (s[i].klass() != isa::OpClass::compute) continue;
            consumed += s[i].size;
            if (m[i].op < last_op) v.push_back({i, core.name() + ": operators out of topological order"});
            last_op = m[i].op;
            const vdc_job& j = p.jobs.at(size_t(s[i].imm));
            const int32_t b_in = (j.flags & VDC_JOB_QKV) ? -1 : j.b_t;  // QKV: b_t is an output (K cache)
            const int32_t x2 = (j.flags & VDC_JOB_BATCH) ? j.x2_t : -1;
            for (int32_t t : {j.x_t, j.a_t, b_in, x2}) {
                const auto it = writer_op.find(t);
                if (it != writer_op.end() && it->second >= m[i].op)
                    v.push_back({i, core.name() + ": waits on an operator that does not precede it"});
            }
        }
        if (consumed != loads) v.push_back({0, core.name() + ": compute µops consume " + std::to_string(consumed) +
                                                   " ring tiles, memory stream loads " + std::to_string(loads)});
    }
    return v;
}

}  // namespace uopsim::generator
