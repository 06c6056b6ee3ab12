// ORACLE / TEST INFRASTRUCTURE ONLY.
// oracle_interp <program.json> <out_dir> [seed] [step csv] [inputs.bin]
//   program.json : vdc_program_text(with_words=1) output of the program under test
//   out_dir      : receives index.json, inputs.bin (initial storage tensors) and
//                  outputs.bin (storage tensors after execution), float32 LE
//   inputs.bin   : optional override of the initial contents (same layout)
#include <chrono>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>

#include <nlohmann/json.hpp>

#include "interp.hpp"

using json = nlohmann::json;

static std::vector<uint8_t> unhex(const std::string& h) {
    std::vector<uint8_t> v(h.size() / 2);
    auto d = [](char c) { return uint8_t(c <= '9' ? c - '0' : c - 'a' + 10); };
    for (size_t i = 0; i < v.size(); ++i) v[i] = uint8_t(d(h[2 * i]) << 4 | d(h[2 * i + 1]));
    return v;
}

int main(int argc, char** argv) {
    if (argc < 3) {
        std::cerr << "usage: oracle_interp program.json out_dir [seed] [step csv] [inputs.bin]\n";
        return 2;
    }
    std::ifstream f(argv[1]);
    const json j = json::parse(f);
    oracle::Program p;
    for (const auto& d : j.at("descriptors")) {
        oracle::Desc x;
        x.name = d.at("name");
        x.base = d.at("base");
        x.shape = d.at("shape").get<std::vector<int64_t>>();
        x.grid = d.at("grid").get<std::vector<int64_t>>();
        x.tile_rows = d.at("tile").at(0);
        x.tile_cols = d.at("tile").at(1);
        const std::string dt = d.at("dtype");
        x.dtype = dt == "bf16" ? 1 : dt == "i64" ? 2 : 0;
        x.view_of = d.at("view_of");
        x.external = d.at("external");
        x.state = d.at("state");
        x.init = d.at("init");
        x.init_scale = d.at("init_scale");
        p.descs.push_back(x);
    }
    const int sms = j.at("sm_count"), vccs = j.at("vcc_per_sm");
    for (int sm = 0; sm < sms; ++sm)
        for (int v = -1; v < vccs; ++v) {
            oracle::CoreStream c;
            c.sm = sm;
            c.vcc = v;
            const std::string name = "sm" + std::to_string(sm) + (v < 0 ? ".vmc" : ".vcc" + std::to_string(v));
            if (j.at("words").contains(name)) c.words = unhex(j.at("words").at(name));
            p.cores.push_back(std::move(c));
        }
    for (const auto& q : j.value("queues", json::array())) p.queues.push_back({q.at("dep"), q.at("depth")});
    p.params = j.at("params").get<std::vector<float>>();
    p.slot_budget = j.at("slot_budget");
    p.local_depth = j.at("local_queue_depth");
    p.slot_size = j.value("slot_size", 8192u);
    const uint64_t seed = argc > 3 ? std::stoull(argv[3]) : 0;
    if (argc > 4) {
        std::stringstream ss(argv[4]);
        for (std::string t; std::getline(ss, t, ',');) p.step.push_back(std::stoll(t));
    }
    std::map<int, std::vector<float>> mem;
    json index = json::array();
    size_t off = 0;
    for (size_t i = 0; i < p.descs.size(); ++i) {
        const auto& d = p.descs[i];
        if (d.view_of >= 0) continue;
        mem[int(i)] = (d.external || d.state) ? oracle::synthesize(d, seed) : std::vector<float>(size_t(d.elem_count()), 0.f);
        index.push_back({{"name", d.name}, {"index", i}, {"offset", off}, {"count", d.elem_count()}});
        off += size_t(d.elem_count());
    }
    if (argc > 5) {  // caller-provided initial contents
        std::ifstream in(argv[5], std::ios::binary);
        for (auto& [i, v] : mem) in.read(reinterpret_cast<char*>(v.data()), std::streamsize(v.size() * 4));
    }
    const std::string out = argv[2];
    const bool dump = !std::getenv("ORACLE_NO_DUMP");
    if (dump) {
        std::ofstream o(out + "/inputs.bin", std::ios::binary);
        for (auto& [i, v] : mem) o.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * 4));
    }
    oracle::Interp interp(p, mem);
    const auto t0 = std::chrono::steady_clock::now();
    const auto r = interp.run();
    const double exec_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (dump) {
        std::ofstream o(out + "/outputs.bin", std::ios::binary);
        for (auto& [i, v] : mem) o.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * 4));
    }
    std::ofstream(out + "/index.json") << json{{"tensors", index}, {"completed", r.completed}, {"uops", r.uops},
                                               {"stall", r.stall}, {"queues_drained", r.queues_drained},
                                               {"slots_all_free", r.slots_all_free}, {"exec_seconds", exec_s}}.dump(1);
    std::cout << (r.completed ? "completed" : "DEADLOCK " + r.stall) << " uops=" << r.uops << " exec_s=" << exec_s << "\n";
    return r.completed ? 0 : 3;
}
