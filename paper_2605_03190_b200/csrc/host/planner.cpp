// Core ids, descriptor/program bookkeeping, job planning and the
// critical-path tiling search. Reference behaviour: src/generator.cpp
// (CoreId :14-37, descriptors :39-58, program helpers :60-104, split/topo
// :111-137, plan_node :156-289, plan_graph :293-312, flops :314-333,
// descriptors :335-354, tiling search :365-516) and src/tilemath.hpp:18-44.
#include <algorithm>
#include <functional>
#include <set>

#include "jobs.hpp"
#include "uopsim/util.hpp"

namespace uopsim::generator {

using workload::OpKind;
using workload::SplitAxis;

std::string CoreId::name() const {
    return "sm" + std::to_string(sm) + (kind == isa::CoreKind::vmc ? ".vmc" : ".vcc" + std::to_string(vcc));
}

CoreId CoreId::parse(const std::string& text) {
    auto bad = [&]() -> CoreId { throw GeneratorError("bad core name '" + text + "'"); };
    const size_t dot = text.find('.');
    if (text.rfind("sm", 0) != 0 || dot == std::string::npos) return bad();
    CoreId c;
    c.sm = static_cast<uint16_t>(std::stoul(text.substr(2, dot - 2)));
    const std::string unit = text.substr(dot + 1);
    if (unit == "vmc") {
        c.kind = isa::CoreKind::vmc;
    } else if (unit.rfind("vcc", 0) == 0) {
        c.kind = isa::CoreKind::vcc;
        c.vcc = static_cast<uint8_t>(std::stoul(unit.substr(3)));
    } else {
        return bad();
    }
    return c;
}

int64_t TileDescriptor::tile_count() const {
    int64_t n = 1;
    for (int64_t e : grid) n *= e;
    return n;
}
int64_t TileDescriptor::elem_count() const {
    int64_t n = 1;
    for (int64_t e : shape) n *= e;
    return n;
}
int64_t TileDescriptor::linear_tile(std::span<const uint16_t> coord) const {
    int64_t lin = 0;
    for (size_t i = 0; i < grid.size(); ++i) lin = lin * grid[i] + (i < coord.size() ? coord[i] : 0);
    return lin;
}
std::vector<uint16_t> TileDescriptor::coord_of(int64_t linear) const {
    std::vector<uint16_t> c(grid.size());
    for (size_t i = grid.size(); i-- > 0; linear /= grid[i]) c[i] = static_cast<uint16_t>(linear % grid[i]);
    return c;
}

const QueueInfo* LoweredProgram::queue(uint16_t dep) const {
    for (const auto& q : queues)
        if (q.dep_id == dep) return &q;
    return nullptr;
}
QueueInfo* LoweredProgram::queue(uint16_t dep) {
    for (auto& q : queues)
        if (q.dep_id == dep) return &q;
    return nullptr;
}
const TileDescriptor* LoweredProgram::descriptor_for_global_tile(int64_t global) const {
    for (const auto& d : descriptors)
        if (global >= d.base && global < d.base + d.tile_count()) return &d;
    return nullptr;
}
size_t LoweredProgram::total_uops() const {
    size_t n = 0;
    for (const auto& kv : streams) n += kv.second.size();
    return n;
}

std::vector<isa::Violation> LoweredProgram::validate() const {
    std::vector<isa::Violation> out;
    std::vector<std::pair<isa::CoreKind, std::span<const isa::UopWord>>> views;
    std::set<uint16_t> deps;
    for (const auto& [core, s] : streams) {
        for (auto& v : isa::validate_stream(s, core.kind)) out.push_back({v.index, core.name() + ": " + v.message});
        views.emplace_back(core.kind, std::span<const isa::UopWord>(s));
        for (const auto& u : s)
            if (u.dep_id && !isa::waits_on_counter(u.opcode)) deps.insert(u.dep_id);
    }
    for (auto& v : isa::validate_dep_pairing(views)) out.push_back(v);
    for (uint16_t dep : deps)
        if (!queue(dep)) out.push_back({size_t(-1), "dep " + std::to_string(dep) + " missing from queue table"});
    for (const auto& q : queues)
        if (!deps.count(q.dep_id))
            out.push_back({size_t(-1), "queue table entry " + std::to_string(q.dep_id) + " unused by any stream"});
    return out;
}

std::vector<TileDescriptor> build_descriptors(const workload::OperatorGraph& g) {
    std::vector<TileDescriptor> out;
    int64_t base = 0;
    for (size_t i = 0; i < g.tensors.size(); ++i) {
        const workload::TensorRef& t = g.tensors[i];
        TileDescriptor d;
        d.tensor = t.name;
        d.index = static_cast<uint16_t>(i);
        d.base = base;
        d.shape = t.shape;
        d.grid = t.grid();
        d.tile_rows = t.tile_rows;
        d.tile_cols = t.tile_cols;
        d.init = t.init;
        d.external = g.is_external(t.name);
        d.elem = t.elem;
        d.view_of = t.view_of.empty() ? -1 : int32_t(g.tensor_index(g.storage_of(t.name).name));
        d.state = t.state;
        d.init_scale = t.init_scale;
        d.symmetric = t.symmetric;
        d.tma = t.tma;
        base += d.tile_count();
        out.push_back(std::move(d));
    }
    return out;
}

namespace detail {

std::vector<std::pair<int64_t, int64_t>> split_range(int64_t extent, int parts) {
    std::vector<std::pair<int64_t, int64_t>> chunks;
    chunks.reserve(parts);
    const int64_t q = extent / parts, r = extent % parts;
    for (int64_t i = 0, at = 0; i < parts; ++i) {
        const int64_t len = q + (i < r ? 1 : 0);
        chunks.emplace_back(at, len);
        at += len;
    }
    return chunks;
}

std::vector<const workload::OperatorNode*> topo_nodes(const workload::OperatorGraph& g) {
    std::map<std::string, const workload::OperatorNode*> maker;
    for (const auto& n : g.nodes)
        for (const auto& t : n.outputs) maker[t] = &n;
    std::vector<const workload::OperatorNode*> order;
    std::set<std::string> seen;
    std::function<void(const workload::OperatorNode&)> post = [&](const workload::OperatorNode& n) {
        if (!seen.insert(n.id).second) return;
        for (const auto& t : n.inputs)
            if (auto it = maker.find(t); it != maker.end()) post(*it->second);
        order.push_back(&n);
    };
    for (const auto& n : g.nodes) post(n);
    return order;
}

namespace {

int parts_on(const workload::TilingChoice& c, SplitAxis a) {
    const auto it = c.parts.find(a);
    return it == c.parts.end() ? 1 : it->second;
}
Fetch at2(uint16_t t, int64_t r, int64_t c) { return {t, {uint16_t(r), uint16_t(c)}}; }
Fetch at3(uint16_t t, int64_t h, int64_t r, int64_t c) { return {t, {uint16_t(h), uint16_t(r), uint16_t(c)}}; }

int32_t elemwise_func(const workload::OperatorNode& node) {
    int32_t f = node.inputs.size() == 2 ? 2 : 0;
    if (const auto it = node.attrs.find("func"); it != node.attrs.end()) {
        static const std::pair<const char*, int32_t> names[] = {{"relu", 0}, {"silu", 1}, {"add", 2}, {"mul", 3}};
        auto m = std::find_if(std::begin(names), std::end(names), [&](auto& p) { return it->second == p.first; });
        if (m == std::end(names)) throw GeneratorError("node " + node.id + ": unknown elemwise func " + it->second);
        f = m->second;
    }
    return f;
}

}  // namespace

std::vector<Job> plan_node(const workload::OperatorNode& node, const workload::TilingChoice& choice,
                           const workload::OperatorGraph& g, const costmodel::HardwareProfile& hw) {
    const uint32_t pairs = hw.pair_count();
    auto idx = [&](const std::string& name) { return g.tensor_index(name); };
    auto row_grid = [&](const std::string& name) {
        const auto gr = g.tensor(name).grid();
        return gr[gr.size() - 2];
    };
    std::vector<Job> jobs;
    auto start = [&](uint32_t chunk, isa::Opcode op) -> Job& {
        Job& j = jobs.emplace_back();
        j.pair = chunk % pairs;
        j.compute = op;
        return j;
    };

    switch (node.kind) {
        case OpKind::MATVEC:
        case OpKind::GEMM: {
            const bool vec = node.kind == OpKind::MATVEC;
            const workload::TensorRef& a = g.tensor(node.inputs[0]);
            const auto og = g.tensor(node.outputs[0]).grid();
            const int64_t ktiles = ceil_div(a.cols(), a.tile_cols);
            const int pm = parts_on(choice, SplitAxis::M), pn = parts_on(choice, SplitAxis::N);
            const auto mchunks = split_range(og[og.size() - 2], pm);
            const auto nchunks = split_range(og.back(), pn);
            for (int i = 0; i < pm; ++i)
                for (int j = 0; j < pn; ++j)
                    for (int64_t r = mchunks[i].first; r < mchunks[i].first + mchunks[i].second; ++r)
                        for (int64_t c = nchunks[j].first; c < nchunks[j].first + nchunks[j].second; ++c) {
                            Job& job = start(uint32_t(i * pn + j), vec ? isa::Opcode::MATVEC : isa::Opcode::GEMM_TILE);
                            job.out = at2(idx(node.outputs[0]), r, c);
                            for (int64_t k = 0; k < ktiles; ++k)
                                job.groups.push_back({at2(idx(node.inputs[1]), k, vec ? 0 : c), at2(idx(node.inputs[0]), r, k)});
                        }
            break;
        }
        case OpKind::ATTENTION: {
            const workload::TensorRef& q = g.tensor(node.inputs[0]);
            const int64_t token_tiles = ceil_div(q.shape[1], q.tile_rows);
            const int ph = parts_on(choice, SplitAxis::head_block), pt = parts_on(choice, SplitAxis::token_block);
            const auto hchunks = split_range(q.shape[0], ph);
            const auto tchunks = split_range(token_tiles, pt);
            for (int i = 0; i < ph; ++i)
                for (int j = 0; j < pt; ++j)
                    for (int64_t h = hchunks[i].first; h < hchunks[i].first + hchunks[i].second; ++h)
                        for (int64_t t = tchunks[j].first; t < tchunks[j].first + tchunks[j].second; ++t) {
                            Job& job = start(uint32_t(i * pt + j), isa::Opcode::ATTN);
                            job.prologue = at3(idx(node.inputs[0]), h, t, 0);
                            for (int64_t k = 0; k < token_tiles; ++k)
                                job.groups.push_back({at3(idx(node.inputs[1]), h, k, 0), at3(idx(node.inputs[2]), h, k, 0)});
                            job.out = at3(idx(node.outputs[0]), h, t, 0);
                        }
            break;
        }
        case OpKind::ROPE:
        case OpKind::RMSNORM: {
            const auto chunks = split_range(row_grid(node.outputs[0]), std::max(parts_on(choice, SplitAxis::M), 1));
            for (size_t i = 0; i < chunks.size(); ++i)
                for (int64_t r = chunks[i].first; r < chunks[i].first + chunks[i].second; ++r) {
                    Job& job = start(uint32_t(i), node.kind == OpKind::ROPE ? isa::Opcode::ROPE : isa::Opcode::RMSNORM);
                    job.groups.push_back({at2(idx(node.inputs[0]), r, 0), at2(idx(node.inputs[1]), r, 0)});
                    job.out = at2(idx(node.outputs[0]), r, 0);
                }
            break;
        }
        case OpKind::ELEMWISE: {
            const auto og = g.tensor(node.outputs[0]).grid();
            const int pm = parts_on(choice, SplitAxis::M);
            const auto chunks = split_range(og[og.size() - 2], pm);
            const int32_t func = elemwise_func(node);
            for (int i = 0; i < pm; ++i)
                for (int64_t r = chunks[i].first; r < chunks[i].first + chunks[i].second; ++r)
                    for (int64_t c = 0; c < og.back(); ++c) {
                        Job& job = start(uint32_t(i), isa::Opcode::ELEMWISE);
                        job.imm = func;
                        for (const auto& in : node.inputs) job.groups.push_back({at2(idx(in), r, c)});
                        job.out = at2(idx(node.outputs[0]), r, c);
                    }
            break;
        }
        case OpKind::EMBED: {
            const workload::TensorRef& table = g.tensor(node.inputs[0]);
            const int64_t vocab_tiles = ceil_div(table.rows(), table.tile_rows);
            const int pm = parts_on(choice, SplitAxis::M);
            const auto chunks = split_range(row_grid(node.outputs[0]), pm);
            for (int i = 0; i < pm; ++i)
                for (int64_t r = chunks[i].first; r < chunks[i].first + chunks[i].second; ++r) {
                    Job& job = start(uint32_t(i), isa::Opcode::EMBED);
                    job.prologue = at2(idx(node.inputs[1]), r, 0);
                    for (int64_t v = 0; v < vocab_tiles; ++v) job.groups.push_back({at2(idx(node.inputs[0]), v, 0)});
                    job.out = at2(idx(node.outputs[0]), r, 0);
                }
            break;
        }
        case OpKind::MLP:
            throw GeneratorError("mlp nodes are expanded at parse time");
        default:
            throw GeneratorError("node " + node.id + ": decode kinds are planned by the decode lowering");
    }
    return jobs;
}

std::vector<OpPlan> plan_graph(const workload::OperatorGraph& g,
                               const std::map<std::string, workload::TilingChoice>& tilings,
                               const costmodel::HardwareProfile& hw) {
    if (hw.vmc_per_sm != 1)
        throw GeneratorError("lowering assumes one VMC per SM (profile has " + std::to_string(hw.vmc_per_sm) + ")");
    std::vector<OpPlan> plans;
    for (const workload::OperatorNode* node : topo_nodes(g)) {
        const auto it = tilings.find(node->id);
        if (it == tilings.end()) throw GeneratorError("no tiling chosen for node " + node->id);
        OpPlan& p = plans.emplace_back();
        p.node = node;
        p.ordinal = static_cast<uint32_t>(plans.size() - 1);
        p.parts = it->second.total_parts();
        p.jobs = plan_node(*node, it->second, g, hw);
    }
    return plans;
}

uint64_t compute_group_flops(isa::Opcode op, std::span<const TileDims> group, const TileDims& prologue,
                             const TileDims& out, size_t gi, size_t ngroups) {
    using isa::Opcode;
    switch (op) {
        case Opcode::MATVEC:
        case Opcode::GEMM_TILE:
            return 2ull * group[1].rows * group[1].cols * group[0].cols;
        case Opcode::ATTN:
            return uint64_t(prologue.rows) * group[0].rows * (4ull * prologue.cols + 8ull);
        case Opcode::ROPE:
            return 3ull * group[0].rows * group[0].cols;
        case Opcode::RMSNORM:
            return 4ull * group[0].rows * group[0].cols;
        case Opcode::ELEMWISE:
            if (ngroups == 1) return 4ull * group[0].rows * group[0].cols;
            return gi + 1 == ngroups ? uint64_t(group[0].rows) * group[0].cols : 0;
        case Opcode::EMBED:
            return uint64_t(out.rows) * out.cols / (ngroups ? ngroups : 1) + 1;
        case Opcode::GEMV:
        case Opcode::RMS_GEMV:
        case Opcode::GEMV_ADD:
            return 2ull * group[0].rows * group[0].cols;
        case Opcode::ATTN_DECODE:
            return 4ull * group[0].rows * group[0].cols;
        case Opcode::ATTN_COMBINE:
            return 4ull * group[0].rows * group[0].cols;
        default:
            return 0;
    }
}

namespace {
TileDims fetch_dims(const Fetch& f, const workload::OperatorGraph& g) {
    const workload::TensorRef& t = g.tensors[f.tensor];
    const size_t n = t.grid().size();
    return {t.tile_rows_at(f.coord[n - 2]), t.tile_cols_at(f.coord[n - 1])};
}
}  // namespace

uint64_t group_flops(const Job& job, size_t gi, const workload::OperatorGraph& g) {
    std::vector<TileDims> dims;
    for (const Fetch& f : job.groups[gi]) dims.push_back(fetch_dims(f, g));
    const TileDims pro = job.prologue ? fetch_dims(*job.prologue, g) : TileDims{};
    return compute_group_flops(job.compute, dims, pro, fetch_dims(job.out, g), gi, job.groups.size());
}

uint64_t job_flops(const Job& job, const workload::OperatorGraph& g) {
    uint64_t total = 0;
    for (size_t i = 0; i < job.groups.size(); ++i) total += group_flops(job, i, g);
    return total;
}

}  // namespace detail

// ---------------------------------------------------------------------------
// adaptive tiling (reference generator.cpp:365-516)

namespace {

// Worst per-pair cost of one operator under `choice`: issue + transfer +
// compute + queue ops summed per pair.
int64_t node_cost_under(const workload::OperatorNode& node, const workload::TilingChoice& choice,
                        const workload::OperatorGraph& g, const costmodel::HardwareProfile& hw) {
    if (hw.vmc_per_sm != 1)
        throw GeneratorError("lowering assumes one VMC per SM (profile has " + std::to_string(hw.vmc_per_sm) + ")");
    const auto jobs = detail::plan_node(node, choice, g, hw);
    std::map<uint32_t, int64_t> per_pair;
    for (const detail::Job& job : jobs) {
        uint64_t bytes = 0;
        int uops = 4;  // alloc + free + store + compute
        if (job.prologue) {
            bytes += g.tensors[job.prologue->tensor].tile_bytes();
            ++uops;
        }
        for (const auto& grp : job.groups)
            for (const auto& f : grp) {
                bytes += g.tensors[f.tensor].tile_bytes();
                ++uops;
            }
        bytes += 2ull * g.tensors[job.out.tensor].tile_bytes();  // store + consumer reload
        per_pair[job.pair] += int64_t(uops) * hw.issue_cost_ns + costmodel::transfer_ns(bytes, hw) +
                              costmodel::compute_ns(detail::job_flops(job, g), hw) +
                              int64_t(2 + job.groups.size()) * hw.queue_op_cost_ns;
    }
    int64_t worst = 0;
    for (const auto& kv : per_pair) worst = std::max(worst, kv.second);
    return worst;
}

struct PathScan {
    int64_t crit = 0;
    std::string end;
    std::map<std::string, std::string> prev;
};

PathScan longest_path(const workload::OperatorGraph& g, const std::map<std::string, int64_t>& cost,
                      const costmodel::HardwareProfile& hw) {
    PathScan s;
    std::map<std::string, int64_t> finish;
    for (const workload::OperatorNode* n : detail::topo_nodes(g)) {
        int64_t ready = 0;
        std::string via;
        for (const auto& in : n->inputs)
            if (const auto* p = g.producer_of(in)) {
                const int64_t t = finish[p->id] + int64_t(hw.queue_op_cost_ns);
                if (t > ready) {
                    ready = t;
                    via = p->id;
                }
            }
        finish[n->id] = ready + cost.at(n->id);
        s.prev[n->id] = via;
        if (finish[n->id] > s.crit) {
            s.crit = finish[n->id];
            s.end = n->id;
        }
    }
    return s;
}

int64_t spread_total(const workload::OperatorGraph& g, const std::map<std::string, int64_t>& cost,
                     const std::map<std::string, workload::TilingChoice>& tilings) {
    int64_t total = 0;
    for (const auto& n : g.nodes) total += cost.at(n.id) * tilings.at(n.id).total_parts();
    return total;
}

int64_t makespan_of(const workload::OperatorGraph& g, const std::map<std::string, int64_t>& cost,
                    const std::map<std::string, workload::TilingChoice>& tilings, const costmodel::HardwareProfile& hw) {
    const int64_t total = spread_total(g, cost, tilings);
    return std::max(longest_path(g, cost, hw).crit, total / std::max<int64_t>(1, hw.pair_count()));
}

}  // namespace

int64_t estimate_tiling_makespan(const workload::OperatorGraph& g,
                                 const std::map<std::string, workload::TilingChoice>& tilings,
                                 const costmodel::HardwareProfile& hw) {
    std::map<std::string, int64_t> cost;
    for (const auto& n : g.nodes) cost[n.id] = node_cost_under(n, tilings.at(n.id), g, hw);
    return makespan_of(g, cost, tilings, hw);
}

std::map<std::string, workload::TilingChoice> select_tilings(const workload::OperatorGraph& g,
                                                            const costmodel::HardwareProfile& hw, double theta) {
    if (theta <= 1.0) throw GeneratorError("theta must exceed 1");
    std::map<std::string, std::vector<workload::TilingChoice>> catalog;
    std::map<std::string, size_t> level;  // index into catalog (back = coarsest)
    for (const auto& n : g.nodes) {
        catalog[n.id] = workload::decompositions(n, g, hw);
        level[n.id] = catalog[n.id].size() - 1;
    }
    auto choose = [&](const std::map<std::string, size_t>& at) {
        std::map<std::string, workload::TilingChoice> t;
        for (const auto& n : g.nodes) t.emplace(n.id, catalog[n.id][at.at(n.id)]);
        return t;
    };
    auto tilings = choose(level);
    std::map<std::string, int64_t> cost;
    for (const auto& n : g.nodes) cost[n.id] = node_cost_under(n, tilings.at(n.id), g, hw);
    int64_t makespan = makespan_of(g, cost, tilings, hw);

    const size_t max_iter = 64 * g.nodes.size() + 64;
    for (size_t iter = 0; iter < max_iter; ++iter) {
        const int64_t avg = std::max<int64_t>(1, spread_total(g, cost, tilings) / std::max<int64_t>(1, hw.pair_count()));
        const PathScan path = longest_path(g, cost, hw);
        if (path.end.empty() || double(path.crit) <= theta * double(avg)) break;

        // costliest refinable node on the dominant path (lowest id on ties)
        std::string pickn;
        int64_t pickc = -1;
        for (std::string at = path.end; !at.empty();) {
            if (level[at] > 0 && (cost[at] > pickc || (cost[at] == pickc && (pickn.empty() || at < pickn)))) {
                pickc = cost[at];
                pickn = at;
            }
            const auto pv = path.prev.find(at);
            if (pv == path.prev.end()) break;
            at = pv->second;
        }
        if (pickn.empty()) break;

        auto trial_level = level;
        --trial_level[pickn];
        auto trial = choose(trial_level);
        auto trial_cost = cost;
        trial_cost[pickn] = node_cost_under(*g.find_node(pickn), trial.at(pickn), g, hw);
        const int64_t trial_span = makespan_of(g, trial_cost, trial, hw);
        if (double(trial_span) > double(makespan) * 0.99) break;  // marginal benefit
        level = std::move(trial_level);
        tilings = std::move(trial);
        cost = std::move(trial_cost);
        makespan = trial_span;
    }
    return tilings;
}

}  // namespace uopsim::generator
