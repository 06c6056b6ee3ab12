/*
 * vdc.h — C-ABI of the B200 µop decode engine (drop-in boundary).
 *
 * The reference (arxiv 2605.03190 "VDCores", /root/reference/proj) exposes its
 * executor only as C++ (`uopsim::machine::Machine` / `simulate`,
 * include/uopsim/machine.hpp:94-126, bodies absent from the tree) and its
 * builder as `uopsim::generator::generate` (include/uopsim/generator.hpp:132).
 * This header is the C-level replacement: plain pointers and sizes, no C++ or
 * torch types, `int` status codes, no exceptions across the boundary.
 *
 *   reference                                  replaced by
 *   ---------------------------------------    -----------------------------------------
 *   Machine(p, hw, inputs, opt)  machine.hpp:96 vdc_create + vdc_load_program + vdc_bind_tensor
 *   Machine::run(watchdog)       machine.hpp:112 vdc_launch + vdc_wait (report.status, deadlock)
 *   ExecutionReport              machine.hpp:65  vdc_report
 *   MachineError / Termination   machine.hpp:19,58 VDC_ERR_* / vdc_report.status
 *   simulate(p, hw, opt, wd)     machine.hpp:124 vdc_program_build + vdc_program_load + launch/wait
 *   generator::generate(g,hw,o)  generator.hpp:132 vdc_program_build (request JSON)
 *   serialize_stream/_sidecar    generator.hpp:154 vdc_program_text
 *   isa::encode_stream           isa.hpp:134      vdc_program_words
 *
 * Status codes mirror the reference CLI's exit codes:
 * 0 ok, 1 internal, 2 input, 3 deadlock. The last error message of the
 * calling thread is available from vdc_last_error().
 */
#ifndef VDC_H
#define VDC_H

#include <stddef.h>
#include <stdint.h>

#include "uopsim/ring_abi.h"

#ifdef __cplusplus
extern "C" {
#endif

#define VDC_OK 0
#define VDC_ERR_INTERNAL 1
#define VDC_ERR_INPUT 2
#define VDC_ERR_DEADLOCK 3

#define VDC_DTYPE_F32 0
#define VDC_DTYPE_BF16 1
#define VDC_DTYPE_I64 2

/* Virtual-core declaration of the device (costmodel::HardwareProfile subset). */
typedef struct vdc_profile {
    uint32_t sm_count;    /* persistent CTAs (<= multiprocessor count) */
    uint32_t vcc_per_sm;  /* compute virtual cores per SM (1 or 2)     */
    uint32_t slot_size;   /* bytes per shared-memory slot              */
    uint32_t slot_budget; /* slots per SM                              */
    uint32_t ldu_count;   /* load units per VMC (1 or 2)               */
    uint32_t stu_count;   /* store units per VMC (1 or 2)              */
} vdc_profile;

/* One tile descriptor (generator::TileDescriptor). Tensors are row-major in
 * device memory; tiles are the 2-d boxes over the trailing two dims. */
typedef struct vdc_desc {
    int64_t base;       /* first global tile index                       */
    int64_t shape[4];
    int64_t grid[4];
    int64_t tile_rows;
    int64_t tile_cols;
    uint32_t rank;      /* rank of shape == rank of grid                  */
    uint32_t dtype;     /* VDC_DTYPE_*                                    */
    int32_t view_of;    /* storage owner descriptor, -1 = owns storage    */
    uint32_t tma;       /* ext: >0 = TMA tensor map with a {64 x tma} box, 128-byte swizzle
                           (batched ring programs: weights tma=128, activations tma=npad) */
} vdc_desc;

/* Dependency queue wiring (generator::QueueInfo). */
typedef struct vdc_queue {
    uint16_t dep_id;
    uint16_t depth;
    uint16_t producer_sm;
    uint16_t consumer_sm;
    uint32_t local; /* slot handoff (STORE_LOCAL -> LOAD_LOCAL) */
} vdc_queue;

typedef struct vdc_report {
    int32_t status;            /* VDC_OK or VDC_ERR_DEADLOCK / VDC_ERR_INTERNAL */
    uint32_t n_stalled;        /* cores still blocked when the watchdog fired    */
    uint64_t uops_executed;
    uint64_t bytes_loaded;     /* global -> shared (DRAM/L2) bytes               */
    uint64_t bytes_stored;     /* shared -> global bytes                         */
    double elapsed_ms;         /* device time of the last launch                 */
    uint32_t stalled_core[16]; /* core index (CoreId order) of blocked cores     */
    uint32_t stalled_pc[16];
    /* cycles spent at each engine wait site, summed over SMs (see
     * engine.cuh WaitSite: cfu alloc/m2c/unit, ldu idle/dep, stu idle/c2m/dep,
     * vcc ready/barrier/c2m, vcc compute, cfu total, vcc total, ldu issue) */
    uint64_t wait_cycles[24];
    char message[256];
    /* end-of-launch conservation (reference SPEC.md:402, machine.hpp
     * ExecutionReport): every m2c / c2m / unit / dep queue empty (ring engine:
     * every issued tile consumed), every slot free (ring engine: every ring
     * slot handed back). Measured on the device, not assumed. */
    uint32_t queues_drained;
    uint32_t slots_all_free;
} vdc_report;

typedef struct vdc_ctx vdc_ctx;
typedef struct vdc_program vdc_program;

const char* vdc_last_error(void);
const char* vdc_version(void);

/* ---- device executor ------------------------------------------------- */
int vdc_create(const vdc_profile* profile, int device, vdc_ctx** out);
int vdc_destroy(vdc_ctx* ctx);

/* words: concatenated isa::encode_stream bytes of every core in CoreId order
 * (sm0.vmc, sm0.vcc0, sm0.vcc1, sm1.vmc, ...), words_per_core[i] 16-byte words. */
int vdc_load_program(vdc_ctx* ctx, const uint8_t* words, const uint32_t* words_per_core, uint32_t n_cores,
                     const vdc_queue* queues, uint32_t n_queues, const vdc_desc* descs, uint32_t n_desc,
                     uint16_t slot_budget, uint16_t local_depth);
/* ring-mode programs (uopsim/ring_abi.h): compute-µop operand blocks and the
 * shared-memory ring depth; switches the context to the ring engine and
 * zeroes its readiness counters. The context must have been created with
 * slot_size = VDC_RING_SLOT_BYTES and vcc_per_sm = 1. */
int vdc_load_jobs(vdc_ctx* ctx, const vdc_job* jobs, uint32_t n_jobs, uint32_t ring_slots);
/* extension handler parameter table (LoweredProgram::params) */
int vdc_set_params(vdc_ctx* ctx, const float* params, uint32_t n);
/* device memory (row-major) backing descriptor `tensor`; the caller owns it */
int vdc_bind_tensor(vdc_ctx* ctx, uint16_t tensor, void* dptr, size_t bytes, int dtype);
/* tensor parallelism (ring programs): bind symmetric tensor `tensor` of rank
 * `rank` of `world` (<= VDC_RING_MAX_TP). peer_bases[q] is rank q's buffer as
 * mapped in this process (NVLink peer / IPC / same device); every buffer is
 * VDC_SYM_HEADER_BYTES of header (u32 readiness counter at offset 0, zeroed
 * by the caller before the first launch) followed by the tensor's data.
 * Replaces the reference-side `vdc_tp_init` + host allreduce: the partial
 * sums move by peer stores inside the persistent kernel. */
int vdc_bind_symmetric(vdc_ctx* ctx, uint16_t tensor, void* const* peer_bases, uint32_t world, uint32_t rank);
/* Tensor-parallel setup without torch (the reference-side `vdc_tp_init` of
 * SURVEY §8b): vdc_tp_alloc allocates and zeroes this rank's exchange buffer
 * for every symmetric tensor of `prog` and writes an IPC handle blob to `out`
 * (out = NULL: *len = the blob size); the host exchanges the W blobs between
 * its rank processes (any channel: MPI, sockets, files) and vdc_tp_bind maps
 * the peers' buffers (CUDA IPC over NVLink) and binds them
 * (vdc_bind_symmetric). Contexts of several ranks in one process (single-GPU
 * emulation) bind each other's buffers directly. The context owns the
 * buffers and mappings (released by vdc_destroy). */
int vdc_tp_alloc(vdc_ctx* ctx, const vdc_program* prog, void* out, size_t cap, size_t* len);
int vdc_tp_bind(vdc_ctx* ctx, const void* const* blobs, uint32_t world, uint32_t rank);
/* step block: device-resident int64 scalars read by SET_ACC_MEM */
int vdc_bind_step(vdc_ctx* ctx, int64_t* dptr, uint32_t n);
/* one execution of the loaded program on `stream` (a cudaStream_t, NULL =
 * default stream); readiness counters and queues are reset on the stream. */
int vdc_launch(vdc_ctx* ctx, void* stream);
/* synchronise with the last launch and fill the report */
int vdc_wait(vdc_ctx* ctx, vdc_report* report);
/* device trace (optional): per VCC core `records_per_core` records of four
 * uint64 {core << 32 | pc, t_enter, t_prologue_ready, t_done} in %globaltimer
 * ns, written for each compute µop; dptr = NULL disables tracing */
int vdc_bind_trace(vdc_ctx* ctx, void* dptr, uint32_t records_per_core);
/* ring engine: formerly the L2 prefetch look-ahead of the memory core. The
 * look-ahead measured slower at every depth and was removed: only 0 is
 * accepted */
int vdc_set_prefetch(vdc_ctx* ctx, uint32_t tiles);
/* ring engine: the memory-core streams as loaded (one LOAD word per ring
 * tile) and as folded on the device (ring_abi.h vdc_run): total LOAD words,
 * run entries, entries covering more than one tile. Valid after vdc_load_jobs */
int vdc_ring_stream_stats(vdc_ctx* ctx, uint64_t* load_words, uint64_t* entries, uint64_t* multi_tile_runs);
/* fold one memory-core stream of LOAD words (16 bytes each, no HALT) the way
 * vdc_load_jobs does into run entries (`runs`, capacity n); vdc_unfold_stream
 * expands entries back to LOAD words (the host reference of the device
 * expansion). Test / tooling entry points */
int vdc_fold_stream(const uint8_t* words, uint32_t n, vdc_run* runs, uint32_t* n_runs);
int vdc_unfold_stream(const vdc_run* runs, uint32_t n_runs, uint8_t* words, uint32_t capacity, uint32_t* n_words);
/* resident decode: every following launch runs `steps`
 * decode steps inside the persistent kernel. Needs a program that samples on
 * the device and feeds the token back (layout.argmax + layout.feedback): step
 * e + 1 starts on each SM once step e's token is in the step block, while the
 * memory cores keep streaming the next step's weights across the boundary
 * (KV pages wait for the token, they may hold step e's appended rows). */
int vdc_set_steps(vdc_ctx* ctx, uint32_t steps);
/* watchdog: abort a launch whose cores make no progress for `ms` (0 = off) */
int vdc_set_watchdog(vdc_ctx* ctx, uint32_t ms);

/* ---- host program builder (uopsim C++ library) ------------------------ */
/* request_json: {"workload": {...} | "model": {...}, "profile": {...},
 *                "options": {...}, "tilings": {...}, "passes": [...]}      */
int vdc_program_build(const char* request_json, vdc_program** out);
int vdc_program_parse(const char* streams_json, const char* sidecar, vdc_program** out);
void vdc_program_free(vdc_program* prog);
/* JSON: {"streams":{core:text}, "sidecar":..., "words":{core:hex}?, "tilings":..., ...}
 * mode 0: streams + sidecar, 1: also encoded words, 2: summary (descriptors, params, geometry),
 * 3: {"unfolded_words": {core: hex}} every stream with its loops expanded (generator::unfold_stream) */
int vdc_program_text(const vdc_program* prog, int mode, char** out_json);
int vdc_program_cores(const vdc_program* prog, uint32_t* n_cores, uint32_t* sm_count, uint32_t* vcc_per_sm);
/* encoded stream of core i (CoreId order over sm_count x (1 + vcc_per_sm)) */
int vdc_program_words(const vdc_program* prog, uint32_t core, const uint8_t** words, uint32_t* n_words);
int vdc_program_load(vdc_ctx* ctx, const vdc_program* prog);
void vdc_free_string(char* s);
/* a26 input synthesis on the device (reference workload.cpp:411-435
 * synthesize_inputs, util.hpp:15-33 splitmix64/unit_float): fills dptr
 * (`bytes` = the descriptor's element count x its element size) with tensor
 * `tensor`'s synthetic contents, stream state = seed ^ fnv1a(name), element i
 * of the logical row-major tensor = the reference stream's draw i, written
 * in the tensor's device storage order (packed / swizzled layouts applied).
 * Non-external tensors are zero-filled, like the reference. Asynchronous on
 * `stream` (a cudaStream_t). */
int vdc_program_synthesize(const vdc_program* prog, uint16_t tensor, uint64_t seed, void* dptr, size_t bytes, void* stream);

/* ---- paged-KV block allocator (batched programs) ---------------------- */
/* A pool of n_pages 64-row pages shared by the n_requests rows of a batched
 * program's page table (max_pages = the program's pages per request,
 * vdc_program_text summary "batch.maxp"). The table is exported in the step
 * block's layout (int64 request-major, -1 = unallocated): copy it to
 * step[page_table_off ...] before a launch. KV tiles and appends resolve
 * through it at run time (ring_abi.h VDC_LOAD_PAGED), so contexts grow by
 * reserving pages between launches. A launch that appends at a position
 * without a page fails with fault 7. Replaces the reference's static
 * TileDescriptor addressing (generator.hpp:50-65, fold.cpp:278-293). */
typedef struct vdc_kv_pages vdc_kv_pages;
int vdc_kv_create(uint32_t n_pages, uint32_t n_requests, uint32_t max_pages, vdc_kv_pages** out);
int vdc_kv_destroy(vdc_kv_pages* kv);
/* request `req` holds pages for `tokens` positions (grows only; VDC_ERR_INPUT
 * when the pool is exhausted or the program's capacity is exceeded) */
int vdc_kv_reserve(vdc_kv_pages* kv, uint32_t req, uint64_t tokens);
/* return every page of request `req` to the pool */
int vdc_kv_release(vdc_kv_pages* kv, uint32_t req);
/* free pages; held_by_req (optional): n_requests page counts */
int vdc_kv_stats(const vdc_kv_pages* kv, uint32_t* free_pages, uint32_t* held_by_req);
/* the n_requests x max_pages table (int64, -1 = unallocated) */
int vdc_kv_table(const vdc_kv_pages* kv, int64_t* table);

#ifdef __cplusplus
}
#endif
#endif /* VDC_H */
