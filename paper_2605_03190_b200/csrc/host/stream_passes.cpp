// Stream transformations: virtual-flow assignment (greedy chain cover of the
// intra-core dependency relation), dynamic fusion (one-to-one same-VMC
// STORE_DEP/LOAD_DEP -> *_LOCAL slot handoff) and same-flow redundant
// dependency elimination. Reference behaviour: src/passes.cpp:47-194.
#include <algorithm>
#include <map>
#include <set>

#include "uopsim/generator.hpp"

namespace uopsim::generator {

using isa::Opcode;
using isa::UopWord;

namespace {

struct SiteRef {
    CoreId core;
    size_t index;
};

// dep id -> producer / consumer stream position (one of each per valid program)
struct DepSites {
    std::map<uint16_t, SiteRef> made, used;
    explicit DepSites(const LoweredProgram& p) {
        for (const auto& [core, s] : p.streams)
            for (size_t i = 0; i < s.size(); ++i) {
                if (!s[i].dep_id) continue;
                if (isa::is_dep_producer(s[i].opcode)) made[s[i].dep_id] = {core, i};
                if (isa::is_dep_consumer(s[i].opcode)) used[s[i].dep_id] = {core, i};
            }
    }
};

}  // namespace

LoweredProgram assign_virtual_flows(LoweredProgram p) {
    const DepSites sites(p);
    for (auto& [core, s] : p.streams) {
        if (core.kind == isa::CoreKind::vcc) {
            // compute µops never depend on each other directly: one chain per job
            uint32_t n = 0;
            for (auto& u : s)
                if (u.klass() != isa::OpClass::control) u.flow = static_cast<uint8_t>((n++ % 255) + 1);
            continue;
        }
        const auto& meta = p.meta.at(core);
        // task -> load-class positions seen so far (predecessors of the task's stores)
        std::map<int32_t, std::vector<size_t>> task_loads;
        std::vector<uint32_t> chain(s.size(), 0);
        std::map<uint32_t, size_t> chain_end;
        uint32_t chains = 0;
        for (size_t i = 0; i < s.size(); ++i) {
            const UopWord& u = s[i];
            if (u.klass() == isa::OpClass::control) continue;
            std::vector<size_t> preds;
            if (isa::is_dep_consumer(u.opcode)) {
                const auto it = sites.made.find(u.dep_id);
                if (it != sites.made.end() && it->second.core == core && it->second.index < i) preds.push_back(it->second.index);
            }
            if (isa::is_store_class(u.opcode) && meta[i].task >= 0) {
                const auto it = task_loads.find(meta[i].task);
                if (it != task_loads.end()) preds.insert(preds.end(), it->second.begin(), it->second.end());
            }
            if (meta[i].store_group >= 0 && size_t(meta[i].store_group) != i) preds.push_back(size_t(meta[i].store_group));
            std::sort(preds.begin(), preds.end());

            uint32_t pick = 0;
            for (size_t pr : preds) {
                const uint32_t c = chain[pr];
                if (!c) continue;
                const auto e = chain_end.find(c);
                if (e != chain_end.end() && e->second == pr && (!pick || c < pick)) pick = c;
            }
            if (!pick) pick = ++chains;
            chain[i] = pick;
            chain_end[pick] = i;
            if (isa::is_load_class(u.opcode)) task_loads[meta[i].task].push_back(i);
        }
        for (size_t i = 0; i < s.size(); ++i)
            if (s[i].klass() != isa::OpClass::control) s[i].flow = static_cast<uint8_t>(((chain[i] - 1) % 255) + 1);
        // fan-out tokens stay on their data store's flow
        for (size_t i = 0; i < s.size(); ++i)
            if (meta[i].store_group >= 0 && size_t(meta[i].store_group) != i) s[i].flow = s[size_t(meta[i].store_group)].flow;
    }
    return p;
}

LoweredProgram apply_dynamic_fusion(LoweredProgram p) {
    const DepSites sites(p);
    // (core, store_group) -> number of stream positions in the group
    std::map<std::pair<CoreId, int32_t>, int> group_size;
    for (const auto& [core, m] : p.meta)
        for (const auto& mm : m)
            if (mm.store_group >= 0) ++group_size[{core, mm.store_group}];
    for (auto& q : p.queues) {
        if (q.local) continue;
        const auto w = sites.made.find(q.dep_id);
        const auto r = sites.used.find(q.dep_id);
        if (w == sites.made.end() || r == sites.used.end()) continue;
        if (!(w->second.core == r->second.core)) continue;  // same VMC only
        UopWord& store = p.streams.at(w->second.core)[w->second.index];
        UopWord& load = p.streams.at(r->second.core)[r->second.index];
        if (store.opcode != Opcode::STORE_DEP || load.opcode != Opcode::LOAD_DEP) continue;
        if (store.size == 0) continue;  // a fan-out token moves no data
        const int32_t grp = p.meta.at(w->second.core)[w->second.index].store_group;
        if (grp >= 0 && group_size[{w->second.core, grp}] > 1) continue;  // tile forwarded elsewhere too
        store.opcode = Opcode::STORE_LOCAL;
        load.opcode = Opcode::LOAD_LOCAL;
        q.local = true;
    }
    return p;
}

LoweredProgram eliminate_redundant_dependencies(LoweredProgram p) {
    const DepSites sites(p);
    std::set<uint16_t> dropped;
    std::map<CoreId, std::set<size_t>> erase_at;
    for (const auto& q : p.queues) {
        if (q.local) continue;  // slot handoff must stay
        const auto w = sites.made.find(q.dep_id);
        const auto r = sites.used.find(q.dep_id);
        if (w == sites.made.end() || r == sites.used.end()) continue;
        if (!(w->second.core == r->second.core)) continue;
        auto& s = p.streams.at(w->second.core);
        UopWord& store = s[w->second.index];
        UopWord& load = s[r->second.index];
        if (!store.flow || store.flow != load.flow) continue;
        if (w->second.index >= r->second.index) continue;
        if (store.size == 0) {
            erase_at[w->second.core].insert(w->second.index);
        } else {
            store.opcode = Opcode::STORE;
            store.dep_id = 0;
        }
        load.opcode = Opcode::LOAD;
        load.dep_id = 0;
        dropped.insert(q.dep_id);
    }
    if (dropped.empty()) return p;
    std::erase_if(p.queues, [&](const QueueInfo& q) { return dropped.count(q.dep_id) > 0; });
    for (auto& [core, idx] : erase_at) {
        auto& s = p.streams.at(core);
        auto& m = p.meta.at(core);
        std::vector<UopWord> ns;
        std::vector<UopMeta> nm;
        for (size_t i = 0; i < s.size(); ++i)
            if (!idx.count(i)) {
                ns.push_back(s[i]);
                nm.push_back(m[i]);
            }
        s.swap(ns);
        m.swap(nm);
    }
    return p;
}

}  // namespace uopsim::generator
