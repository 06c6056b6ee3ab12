#pragma once
// internal: state shared by the host and device halves of the C-ABI.
#include <memory>
#include <string>
#include <vector>

#include "uopsim/costmodel.hpp"
#include "uopsim/generator.hpp"

namespace vdc_impl {

extern thread_local std::string g_last_error;
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int classify(const std::exception& e);

// what a vdc_program handle points to
struct ProgramBox {
    uopsim::generator::LoweredProgram program;
    uopsim::costmodel::HardwareProfile hw;
    std::string tilings_json;
    std::string graph_json;
    uint32_t sm_count = 0;
    uint32_t vcc_per_sm = 1;
    std::vector<uopsim::generator::CoreId> cores;  // CoreId order, every core of every SM
    std::vector<std::vector<uint8_t>> words;       // encode_stream per core

    void finish();
    std::string text(int mode) const;  // 0 streams, 1 streams + words, 2 summary
};

ProgramBox* build(const std::string& request);

}  // namespace vdc_impl
