// Paged-KV block allocator: the host side of batched
// programs' page pools. A pool of `n_pages` physical 64-row pages is shared
// by `n_requests` request rows of the program's page table (`max_pages`
// logical pages each, the request's capacity in the program). Pages are
// handed out from a LIFO free list (a freed page is reused first: its lines
// are the likeliest to still sit in L2), grown per request as its context
// advances, and returned when a request finishes. The table is exported in
// the step-block layout (int64, request-major, -1 = unallocated) the device
// resolves VDC_LOAD_PAGED tiles and KV appends through, so growing a context
// is a table update between launches, never a program rebuild.
//
// Reference anchor: the reference addresses tiles through descriptors
// (TileDescriptor, generator.hpp:50-65) re-resolved per access
// (resolve_address, fold.cpp:278-293); the page table is that indirection
// made dynamic.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "capi_common.hpp"
#include "vdc.h"

struct vdc_kv_pages {
    uint32_t n_pages = 0, n_requests = 0, max_pages = 0;
    std::vector<int64_t> table;  // n_requests x max_pages, -1 = unallocated
    std::vector<uint32_t> held;  // pages per request (a prefix of its row)
    std::vector<int64_t> free_list;
};

using vdc_impl::fail;

extern "C" {

int vdc_kv_create(uint32_t n_pages, uint32_t n_requests, uint32_t max_pages, vdc_kv_pages** out) {
    if (!out) return fail(VDC_ERR_INPUT, "null argument");
    if (!n_pages || !n_requests || !max_pages) return fail(VDC_ERR_INPUT, "pool, request count and capacity must be > 0");
    auto* kv = new vdc_kv_pages;
    kv->n_pages = n_pages;
    kv->n_requests = n_requests;
    kv->max_pages = max_pages;
    kv->table.assign(size_t(n_requests) * max_pages, -1);
    kv->held.assign(n_requests, 0);
    kv->free_list.reserve(n_pages);
    for (int64_t p = int64_t(n_pages) - 1; p >= 0; --p) kv->free_list.push_back(p);  // page 0 first
    *out = kv;
    return VDC_OK;
}

int vdc_kv_destroy(vdc_kv_pages* kv) {
    delete kv;
    return VDC_OK;
}

int vdc_kv_reserve(vdc_kv_pages* kv, uint32_t req, uint64_t tokens) {
    if (!kv) return fail(VDC_ERR_INPUT, "null pool");
    if (req >= kv->n_requests) return fail(VDC_ERR_INPUT, "request index out of range");
    const uint64_t need = (tokens + 63) / 64;
    if (need > kv->max_pages)
        return fail(VDC_ERR_INPUT, "request " + std::to_string(req) + " needs " + std::to_string(need) +
                                       " pages, the program's capacity is " + std::to_string(kv->max_pages));
    const uint32_t have = kv->held[req];
    if (need <= have) return VDC_OK;
    if (need - have > kv->free_list.size())
        return fail(VDC_ERR_INPUT, "KV pool exhausted: " + std::to_string(need - have) + " pages wanted, " +
                                       std::to_string(kv->free_list.size()) + " free");
    int64_t* row = kv->table.data() + size_t(req) * kv->max_pages;
    for (uint64_t i = have; i < need; ++i) {
        row[i] = kv->free_list.back();
        kv->free_list.pop_back();
    }
    kv->held[req] = uint32_t(need);
    return VDC_OK;
}

int vdc_kv_release(vdc_kv_pages* kv, uint32_t req) {
    if (!kv) return fail(VDC_ERR_INPUT, "null pool");
    if (req >= kv->n_requests) return fail(VDC_ERR_INPUT, "request index out of range");
    int64_t* row = kv->table.data() + size_t(req) * kv->max_pages;
    for (uint32_t i = kv->held[req]; i-- > 0;) {  // reverse: the request's first page is reused first
        kv->free_list.push_back(row[i]);
        row[i] = -1;
    }
    kv->held[req] = 0;
    return VDC_OK;
}

int vdc_kv_stats(const vdc_kv_pages* kv, uint32_t* free_pages, uint32_t* held_by_req) {
    if (!kv) return fail(VDC_ERR_INPUT, "null pool");
    if (free_pages) *free_pages = uint32_t(kv->free_list.size());
    if (held_by_req) std::copy(kv->held.begin(), kv->held.end(), held_by_req);
    return VDC_OK;
}

int vdc_kv_table(const vdc_kv_pages* kv, int64_t* table) {
    if (!kv || !table) return fail(VDC_ERR_INPUT, "null argument");
    std::memcpy(table, kv->table.data(), kv->table.size() * sizeof(int64_t));
    return VDC_OK;
}

}  // extern "C"
