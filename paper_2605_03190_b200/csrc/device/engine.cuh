// Device-side data structures of the persistent µop engine.
//
// One CTA per SM, warp-specialised into the paper's virtual cores:
//   warp 0                 VMC control-flow unit (CFU): fetches the VMC
//                          stream, runs control µops, resolves addresses,
//                          allocates slots in stream order (the in-order
//                          allocation that the generator's certificate
//                          proves deadlock-free), dispatches to units
//   warps 1..ldu           load units (LDU): dependency waits + bulk copies
//                          global -> shared slot (cp.async.bulk / mbarrier)
//   next stu warps         store units (STU): FREE / STORE / dep tokens
//   4 warps per VCC        compute virtual cores executing the handlers
// Shared memory: `slot_budget` slots of `slot_size` bytes, then the control
// block below (rings between the cores, slot barriers, allocator mask).
#pragma once
#include <cstdint>

#include "uopsim/ring_abi.h"

namespace vdc_dev {

constexpr int kMaxVcc = 2;
constexpr int kMaxLdu = 2;
constexpr int kMaxStu = 2;
constexpr int kVccWarps = 4;
constexpr int kM2cDepth = 64;   // >= any program's local_queue_depth (checked at load)
constexpr int kC2mDepth = 64;
constexpr int kUnitDepth = 16;
constexpr int kCfuChunk = 64;   // words per stream prefetch chunk (1 KB)
constexpr int kAccRows = 256;   // per-VCC fp32 accumulator scratch (streaming GEMV rows)
constexpr int kMaxSlots = 32;

// Resolved-tile view of a descriptor, prepared on the host at load/bind.
struct DevDesc {
    int64_t base;         // first global tile index
    int64_t grid[4];
    int64_t lead_stride[2];  // element stride of the leading (plane) grid dims
    int64_t rows, cols;   // trailing two extents
    int64_t tile_rows, tile_cols;
    int64_t tile_count;
    int64_t elem_count;
    char* ptr;            // storage base (view -> owner's pointer)
    int32_t grid_rank;
    int32_t elem;         // bytes per element
    int32_t dtype;        // VDC_DTYPE_*
    int32_t storage;      // counter index (owner descriptor)
};

struct DepQueue {          // global FIFO per dep id (single producer / consumer site)
    uint32_t produced;
    uint32_t consumed;
    uint32_t depth;
    uint32_t local;
    uint32_t payload[6];   // STORE_LOCAL slot handoff: slots lo, hi, count ; rows ; cols ; stride
};

// wait-site accounting (cycles spent blocked, per SM, summed over roles)
enum WaitSite : int {
    W_CFU_ALLOC = 0, W_CFU_M2C, W_CFU_UNIT, W_LDU_IDLE, W_LDU_DEP, W_STU_IDLE, W_STU_C2M, W_STU_DEP,
    W_VCC_READY, W_VCC_BAR, W_VCC_C2M, W_VCC_COMPUTE, W_CFU_TOTAL, W_VCC_TOTAL, W_LDU_ISSUE, W_CFU_RESOLVE,
    W_VCC_SYNC, W_VCC_PUSH, W_VCC_PROLOGUE, W_VCC_EPILOGUE, W_VCC_POP, W_CFU_ALLOCLOOP, W_CFU_SYNCK, W_CFU_DISPATCH, W_NSITES
};

struct SmStats {
    unsigned long long uops;
    unsigned long long bytes_loaded;
    unsigned long long bytes_stored;
    unsigned long long cfu_stall_cycles;
    unsigned long long wait[24];
    unsigned long long cfu_phase[4];  // refill, resolve, m2c, unit push
    // end-of-launch conservation: reference-form engine: rings
    // (m2c / c2m / unit queues) still holding entries and the slot mask; ring
    // engine: tiles issued by the memory core and consumed by the compute core
    unsigned long long rings_pending, slot_mask, tiles_issued, tiles_consumed;
};

struct Status {
    int32_t abort;          // 1 = deadlock watchdog fired, 2 = fault
    int32_t n_stalled;
    uint32_t stalled_core[16];
    uint32_t stalled_pc[16];
    uint32_t fault_code;
    uint32_t fault_info;
};

struct EngineParams {
    const uint4* words;
    const uint32_t* core_off;  // n_cores + 1 word offsets (CoreId order)
    DevDesc* descs;
    int32_t n_desc;
    DepQueue* deps;
    uint32_t* counters;        // per descriptor (storage) store counts
    const float* hparams;
    const int64_t* step;
    int32_t n_step;
    uint32_t sm_count, vcc_per_sm, ldu_count, stu_count;
    uint32_t slot_size, slot_shift, slot_budget, local_depth;
    SmStats* stats;
    Status* status;
    unsigned long long watchdog_ns;
    // optional device trace: per VCC core, `trace_cap` records of
    // {core << 32 | pc, t_enter, t_prologue_ready, t_done} (%globaltimer ns)
    unsigned long long* trace;
    uint32_t trace_cap;
};

// Parameters of the ring engine (ring_engine.cu; ring-mode programs, see
// include/uopsim/ring_abi.h). Cores in CoreId order: 2*sm = vmc, 2*sm+1 = vcc0.
struct RingParams {
    const uint4* words;
    const uint32_t* core_off;
    const DevDesc* descs;
    const ::vdc_job* jobs;
    const char* jobs_core;     // the first 128 bytes of every operand block, packed (single-request programs)
    uint32_t* counters;        // per storage descriptor, monotonic across launches
    const int64_t* step;
    int32_t n_step;
    uint32_t epoch;            // 1-based launch ordinal since the counters were zeroed
    uint32_t ring_slots;
    // memory-core streams, folded (ring_abi.h vdc_run): run entries of SM s
    // at runs[voff[s] .. voff[s + 1]), vtiles[s] ring tiles once expanded
    const uint32_t* voff;
    const uint32_t* vtiles;
    const ::vdc_run* runs;
    uint32_t debug;            // bit 0: GEMV tiles are released without computing (bandwidth experiments)
    unsigned long long* tile_trace;  // debug: per ring tile of SM `debug >> 8`: {t_issue, t_full, t_release}
    char* const* sym;          // [n_desc][VDC_RING_MAX_TP] peer buffer bases of symmetric tensors (null: not symmetric)
    uint32_t tp_rank, tp_world;
    uint32_t tile_trace_cap;
    SmStats* stats;            // written (not accumulated) by each SM
    Status* status;
    unsigned long long watchdog_ns;
    unsigned long long* trace;  // optional: per VCC core trace_cap records {core<<32|pc, t_enter, t_ready, t_done}
    uint32_t trace_cap;
    uint32_t batched;           // batched program: TMEM accumulator + X ring for BGEMM µops
    const void* tmaps;          // CUtensorMap[n_desc] (128 bytes each), indexed by descriptor (vdc_desc.tma > 0 only)
    int32_t ptab, maxp;         // batched programs: page table at step[ptab + b * maxp + logical page] (VDC_LOAD_PAGED)
    // resident decode: the launch runs n_epochs decode steps back to back
    // (epochs epoch .. epoch + n_epochs - 1); step e > 0 starts once the
    // sampled-token counter fb_ctr shows step e - 1 fed its token back
    uint32_t n_epochs;
    int32_t fb_ctr;
};
size_t ring_smem_bytes(uint32_t ring_slots, bool batched = false);
const void* ring_kernel_entry(bool batched, bool qknorm = false);
// 8 compute warps (two warpgroups) + a third warpgroup whose first warp is
// the memory core: with 9 warps one SM sub-partition holds 3 warps anyway
// (168 registers each); with 12, the third warpgroup hands its registers to
// the compute warpgroups at start (setmaxnreg), which then run at 224
constexpr uint32_t kRingThreads = 32 * 12;

// A region of `count` slots, not necessarily contiguous (indices packed 8
// bits each): the allocator prefers a contiguous run but falls back to any
// free slots, so admission is exactly "free slots >= count" — the condition
// the generator's certificate is computed with (contiguity-only allocation
// can starve on fragmentation). Reference programs only use 1-slot tiles.
struct SlotList {
    uint32_t lo, hi;  // slot indices 0..3 / 4..7
    uint32_t count;
    __host__ __device__ uint32_t at(uint32_t i) const { return ((i < 4 ? lo >> (8 * i) : hi >> (8 * (i - 4))) & 0xff); }
};

// m2c message: one slot region handed from the VMC to a VCC.
struct M2C {
    SlotList slots;
    int32_t rows, cols; // payload extents (edge-trimmed)
    int32_t stride;     // padded row stride in elements (tile_cols)
    int32_t row0, col0; // global first row / col of the tile (trailing dims)
    uint32_t meta;      // dtype | (parity << 8) | (wait << 9) | (barrier slot << 16)
    volatile uint32_t ready;  // entry index + 1 once the LDU has issued the data movement
};

// c2m message: a region released (or produced) by a VCC.
struct C2M {
    SlotList slots;
    int32_t rows, cols, stride;
};

// CFU -> unit work item (written with four 16-byte stores).
struct alignas(16) UnitOp {
    uint8_t op, flags, reg1, dtype;
    uint16_t dep_id, size;
    SlotList slots;       // allocated region
    uint32_t m2c;         // m2c entry index (send)
    int32_t storage;      // counter index of the resolved tensor (-1 none)
    uint32_t bytes;       // tile payload bytes (0 = no data movement)
    int32_t rows_at, cols_at;
    int32_t elem;         // bytes per element
    int32_t tile_cols;    // slot row stride in elements
    char* gptr;           // first element of the tile in global memory
    int64_t gpitch;       // global row pitch in bytes
    uint32_t core_pc;
    uint32_t raw;         // loads: data stores of this SM to the tile's bucket that must complete first (mod 2^16)
};

// Same-SM store -> load ordering (reference elaborate.cpp:175-279: a memory
// core executes its µops one at a time in stream order, so a LOAD sees every
// earlier STORE of its stream): data stores are counted per tensor bucket
// (storage % kRawBuckets) when the CFU dispatches them and when the STU has
// written them; a LOAD of that bucket issues once the written count reaches
// the dispatched count it saw (loads and stores run on different units).
constexpr int kRawBuckets = 64;

struct Ring {
    volatile uint32_t head;
    volatile uint32_t tail;
};

// per-batch scratch of the warp-parallel CFU
struct CfuScratch {
    uint32_t info[32];    // per lane: count | send << 8 | vcc << 9 | (unit + 1) << 12
    SlotList lists[32];   // slot lists chosen by lane 0's in-order allocation
};

struct alignas(16) Control {
    uint64_t full_bar[kMaxSlots];
    uint32_t bar_uses[kMaxSlots];
    volatile uint32_t alloc_mask;
    uint32_t pad0[3];
    Ring m2c_ring[kMaxVcc];
    Ring c2m_ring[kMaxVcc];
    Ring ldu_ring[kMaxLdu];
    Ring stu_ring[kMaxStu];
    M2C m2c[kMaxVcc][kM2cDepth];
    C2M c2m[kMaxVcc][kC2mDepth];
    UnitOp ldu_q[kMaxLdu][kUnitDepth];
    UnitOp stu_q[kMaxStu][kUnitDepth];
    CfuScratch cfu;
    // per-role wait-site counters (cycles >> 6) and per-core accumulator
    // registers live in shared memory: run-time indexed per-thread arrays
    // would sit in local memory, which misses L1 after every gpu-scope fence
    uint32_t stat[1 + kMaxLdu + kMaxStu + kMaxVcc][24];
    long long acc_regs[1 + kMaxVcc][16];
    uint4 vcc_word[kMaxVcc];
    float acc[kMaxVcc][kAccRows];
    float red[kMaxVcc][32];
    volatile int32_t done_roles;
    uint32_t raw_disp[kRawBuckets];           // CFU: data stores dispatched per bucket
    volatile uint32_t raw_done[kRawBuckets];  // STU: data stores written per bucket
};

}  // namespace vdc_dev
