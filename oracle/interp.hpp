// ORACLE / TEST INFRASTRUCTURE ONLY — see interp.cpp.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace oracle {

struct Desc {
    std::string name;
    int64_t base = 0;
    std::vector<int64_t> shape, grid;
    int64_t tile_rows = 0, tile_cols = 0;
    int dtype = 0;  // 0 f32, 1 bf16, 2 i64
    int view_of = -1;
    bool external = true, state = false;
    int init = 0;   // 0 random 1 zeros 2 ones 3 arange 4 centered
    float init_scale = 1.f;
    int64_t tile_count() const {
        int64_t n = 1;
        for (auto g : grid) n *= g;
        return n;
    }
    int64_t elem_count() const {
        int64_t n = 1;
        for (auto s : shape) n *= s;
        return n;
    }
    int elem_bytes() const { return dtype == 1 ? 2 : dtype == 2 ? 8 : 4; }
};

struct CoreStream {
    int sm = 0, vcc = -1;
    std::vector<uint8_t> words;
};

struct QueueDesc {
    uint32_t dep = 0;
    size_t depth = 4;
};

struct Program {
    std::vector<Desc> descs;
    std::vector<CoreStream> cores;  // CoreId order
    std::vector<QueueDesc> queues;
    std::vector<float> params;
    std::vector<int64_t> step;
    uint32_t slot_budget = 32, slot_size = 8192;
    size_t local_depth = 8;
};

struct RunResult {
    bool completed = false;
    bool queues_drained = true;
    bool slots_all_free = true;
    uint64_t uops = 0;
    std::string stall;
};

class Interp {
  public:
    Interp(const Program& p, std::map<int, std::vector<float>>& mem);
    ~Interp();
    RunResult run();

  private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

std::vector<float> synthesize(const Desc& d, uint64_t seed);

}  // namespace oracle
