// Ring engine: the persistent sm_100a executor of ring-mode µop programs
// (include/uopsim/ring_abi.h; lowering in host/ring_lower.cpp).
//
// One CTA per SM, 12 warps (three warpgroups):
//   warps 0..7  compute virtual core (VCC), 224 registers (setmaxnreg.inc).
//               Walks sm<i>.vcc0; each compute µop reads its operand block
//               (vdc_job), waits for the readiness counters of its
//               activation inputs, consumes `size` ring tiles (full mbarrier
//               -> compute -> empty mbarrier arrive = the c2m release),
//               writes its output rows and publishes them with a release
//               increment of the output tensor's counter.
//   warp 8      memory virtual core (VMC), 56 registers (setmaxnreg.dec).
//               Walks the SM's folded LOAD stream (ring_abi.h vdc_run);
//               lane s issues ring tiles s, s + R, s + 2R, ... into slot s
//               (one cp.async.bulk / TMA per tile) once the slot's previous
//               tenant was released. Never waits on data dependencies, so
//               weight prefetch crosses operator boundaries (the paper's
//               decoupled memory core, §4.1), bounded only by the
//               ring depth.
//   warps 9..11 only donate their registers to the compute warpgroups.
//
// Arithmetic follows the reference handlers (reference src/handlers.cpp):
// fp32 accumulation of bf16/f32 products, RMSNorm x*rsqrt(mean(x^2)+eps)*w
// (handlers.cpp:101-113, multi-tile), interleaved-pair RoPE (:88-100) with
// double-precision angles, online softmax with running max/sum (:54-87)
// split over KV pages and merged like the reference finalize (:155-168),
// SwiGLU silu(g)*u (:27-33), residual add; bf16 round-to-nearest-even at
// every stored activation (decode_abi.h conventions shared with the oracle).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.cuh"
#include "ptx.cuh"
#include "uopsim/decode_abi.h"
#include "uopsim/ring_abi.h"
#include "vdc.h"

namespace vdc_dev {
namespace ring {

constexpr int CW = VDC_RING_COMPUTE_WARPS;
constexpr int NCT = CW * 32;
constexpr int XBUF = VDC_RING_MAX_K * 2;  // bytes of the staged GEMV input vector
constexpr int XPT = (XBUF / 16 + CW * 32 - 1) / (CW * 32);  // 16-byte chunks of x per compute thread
constexpr int RMAX = VDC_RING_MAX_JOB_ROWS;
constexpr int MAX_TPR = VDC_RING_MAX_COL_TILES;
constexpr uint32_t SLOT = VDC_RING_SLOT_BYTES;
constexpr int BAR_VCC = 1;
constexpr int MAX_HD = 128;
constexpr int MAX_DPL = MAX_HD / 32;

enum : uint32_t {
    OP_LOAD = 0x01, OP_ELEMWISE = 0x25, OP_GEMV = 0x27, OP_RMS_GEMV = 0x28, OP_GEMV_ADD = 0x29, OP_ATTN_DECODE = 0x2A,
    OP_ATTN_COMBINE = 0x2B, OP_ALLREDUCE_ADD = 0x2C, OP_BGEMM = 0x2D, OP_HALT = 0x45,
};
constexpr int NXMAX = 16;  // activation-chunk groups of batched GEMMs
// batched kernel: activation-chunk ring after the control block. Its loads
// queue behind the in-flight weight tiles of the SM's copy engine, so the
// MMA issuer keeps more than a ring's worth of chunks in flight.
constexpr uint32_t XRING_BYTES = 64 * 1024;
constexpr uint32_t TMEM_COLS = 512;  // one fp32 accumulator (npad columns) per compute warp

// stat slots (SmStats::wait)
enum : int { S_VMC_EMPTY = 0, S_VCC_FULL = 1, S_VCC_DEP = 2, S_VCC_EPI = 3, S_VCC_TOTAL = 4, S_VMC_TOTAL = 5, S_NJOBS = 6,
             S_X_FULL = 7, S_X_EMPTY = 8, S_MMA_DONE = 9, S_BG_PRO = 10 };

struct alignas(16) Shared {
    uint64_t full[VDC_RING_MAX_SLOTS];
    uint64_t empty[VDC_RING_MAX_SLOTS];
    float red[MAX_TPR][RMAX];  // GEMV row partials, one plane per column tile (fixed summation order)
    float bc[2 * CW];
    float rope_cs[MAX_HD / 2], rope_sn[MAX_HD / 2];  // rotary table of the launch's position
    int32_t flag;
    alignas(16) uint4 x[XBUF / 16];  // GEMV input vector (normalised, model dtype), reused across jobs;
                                       // batched programs: activation-chunk ring (128-byte swizzle, from the first 1 KB boundary)
    // batched programs: activation-chunk barriers, MMA completion, TMEM base, rms scales
    uint64_t xfull[NXMAX], xempty[NXMAX], mma_bar;
    uint64_t lbar;  // batched programs: bulk copy of the RMS sums of squares
    uint32_t tmem_base;
    float binv[VDC_RING_MAX_BATCH];
    // batched programs: each request's position and the physical page of its
    // appended KV row (-1: none), read from the step block once per launch
    // (constant within a launch) instead of per epilogue element
    int32_t bpos[VDC_RING_MAX_BATCH];
    int32_t bpage[VDC_RING_MAX_BATCH];
    int32_t btok[VDC_RING_MAX_BATCH], bctx[VDC_RING_MAX_BATCH];
    // single-request programs: token, position, context of the running step
    int64_t sstep[3];
    // compute-core wait-site cycles and the trace's readiness stamp, updated by
    // thread 0 only: in shared memory, not in registers that every compute
    // thread would carry through the whole µop loop
    unsigned long long vstat[8];
    unsigned long long t_ready;
    float am_v[VDC_RING_MAX_BATCH];  // batched greedy sampling: this SM's best logit per request
    int32_t am_i[VDC_RING_MAX_BATCH];
};

// both kernel instances must fit one B200 CTA (227 KB of dynamic shared memory)
static_assert(VDC_RING_MAX_SLOTS * SLOT + ((sizeof(Shared) + 127) & ~size_t(127)) <= 232448,
              "single-request ring + control block exceed the B200 shared memory per CTA");
static_assert(8 * SLOT + ((sizeof(Shared) + 1023) & ~size_t(1023)) + XRING_BYTES <= 232448,
              "batched ring + control block + activation ring exceed the B200 shared memory per CTA");
size_t smem_bytes(uint32_t slots, bool batched) {
    return size_t(slots) * SLOT + (batched ? ((sizeof(Shared) + 1023) & ~size_t(1023)) + XRING_BYTES
                                           : ((sizeof(Shared) + 127) & ~size_t(127)));
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}
__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }
__device__ __forceinline__ uint16_t f2bf(float v) { return __bfloat16_as_ushort(__float2bfloat16_rn(v)); }
__device__ __forceinline__ uint32_t pack2(float lo, float hi) { return uint32_t(f2bf(lo)) | (uint32_t(f2bf(hi)) << 16); }
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
// step-block scalar: an L2 (coherent) load. The device writes the step block
// during a launch (fed-back token, positions) and resident decode reads the
// new values in the next step, so no L1 / non-coherent copy may be used.
__device__ __forceinline__ int64_t ldstep(const int64_t* p) {
    int64_t v;
    asm volatile("ld.global.cg.s64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ldcg64(const void* p) {
    uint2 v;
    asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

// 16-byte chunk dot product: 8 bf16 or 4 f32 lanes
template <bool BF>
__device__ __forceinline__ float dot16(uint4 a, uint4 b) {
    if constexpr (BF) {
        float s = bf_lo(a.x) * bf_lo(b.x);
        s = fmaf(bf_hi(a.x), bf_hi(b.x), s);
        s = fmaf(bf_lo(a.y), bf_lo(b.y), s);
        s = fmaf(bf_hi(a.y), bf_hi(b.y), s);
        s = fmaf(bf_lo(a.z), bf_lo(b.z), s);
        s = fmaf(bf_hi(a.z), bf_hi(b.z), s);
        s = fmaf(bf_lo(a.w), bf_lo(b.w), s);
        s = fmaf(bf_hi(a.w), bf_hi(b.w), s);
        return s;
    } else {
        float s = __uint_as_float(a.x) * __uint_as_float(b.x);
        s = fmaf(__uint_as_float(a.y), __uint_as_float(b.y), s);
        s = fmaf(__uint_as_float(a.z), __uint_as_float(b.z), s);
        s = fmaf(__uint_as_float(a.w), __uint_as_float(b.w), s);
        return s;
    }
}

// Qwen3 QK-norm on one 128-dim head held 4 dims per lane (bf16x4 in u):
// x = bf16(x * rsqrt(mean(x^2) + eps) * w), then the interleaved-pair rotary
// from the job's rotary table (double-precision angles), rounded to bf16. Not inlined: its
// double-precision registers stay out of the kernel's allocation.
__device__ __forceinline__ uint2 qk_norm_rope4(uint2 u, uint2 wv, int head_dim, float eps, float2 cs0, float2 cs1) {
    float x[4] = {bf_lo(u.x), bf_hi(u.x), bf_lo(u.y), bf_hi(u.y)};
    const float wgt[4] = {bf_lo(wv.x), bf_hi(wv.x), bf_lo(wv.y), bf_hi(wv.y)};
    const float ss = warp_sum(x[0] * x[0] + x[1] * x[1] + x[2] * x[2] + x[3] * x[3]);
    const float inv = 1.0f / sqrtf(ss / float(head_dim) + eps);
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = bf_lo(uint32_t(f2bf(x[e] * inv * wgt[e])));
    float y[4];
    // rotary table entries (cos, sin) of the lane's two dim pairs
    y[0] = x[0] * cs0.x - x[1] * cs0.y;
    y[1] = x[0] * cs0.y + x[1] * cs0.x;
    y[2] = x[2] * cs1.x - x[3] * cs1.y;
    y[3] = x[2] * cs1.y + x[3] * cs1.x;
    return make_uint2(pack2(y[0], y[1]), pack2(y[2], y[3]));
}

// tensor-core attention helpers (mma.sync m16n8k16 bf16 -> fp32; ldmatrix
// from swizzled KV page rows)
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// 16-byte chunk c of KV page row r (r & 7 = r7) in the swizzled page layout
__device__ __forceinline__ uint32_t kv_swz(uint32_t c, uint32_t r7) { return (c & 8u) | ((c & 7u) ^ r7); }

// TP exchange: this thread's output row rg for requests c0 .. c0 + nh - 1
// into slot `off` of every rank's buffer (batched BGEMM epilogue)
// (T = uint16_t: bf16 partials; float: fp32 partials)
template <typename T>
__device__ __noinline__ void sym_store_rows(char* const* bases, uint32_t world, int64_t off, int64_t M, int rg, int c0, int nb, int nh,
                                            const float* v) {
    for (uint32_t qr = 0; qr < world; ++qr) {
        T* dst = reinterpret_cast<T*>(bases[qr] + VDC_SYM_HEADER_BYTES) + off;
        for (int c = 0; c < nh; ++c) {
            if (c0 + c >= nb) continue;
            if constexpr (sizeof(T) == 2)
                dst[int64_t(c0 + c) * M + rg] = f2bf(v[c]);
            else
                dst[int64_t(c0 + c) * M + rg] = v[c];
        }
    }
}

// BATCHED: the kernel instance for batched programs (BGEMM µops, paged
// attention); single-request programs run the instance without those paths
// so their register allocation and scheduling are unaffected
template <bool BATCHED, bool QKNORM = false>
struct Vcc {
    const RingParams* P;
    Shared* S;
    uint32_t ring;   // shared address of slot 0
    uint32_t sm;
    uint32_t ct, lane, w;
    uint32_t kt = 0;  // ring tiles consumed so far (program order, uniform over the VCC)
    uint32_t R;
    uint32_t ep = 0;  // epoch of the running decode step (readiness targets are producers x epoch)
    bool ok = true;
    // wait-site cycle counters (thread 0, shared memory): VS_* slots of S->vstat
    enum : int { VS_FULL = 0, VS_DEP, VS_EPI, VS_XF, VS_XE, VS_MMA, VS_PRO };
    __device__ void stat_add(int k, long long c) const { S->vstat[k] += (unsigned long long)c; }
    uint32_t n_attn = 0;             // debug stamps
    float resid = 0.f;               // GEMV_ADD: this thread's residual element, loaded before the tile sweep
    int32_t rope_hd = 0;             // head dim of the cached rotary table (0 = none)
    float rope_theta = 0.f;
    // x held in registers across jobs that share it
    int32_t xk_t = -2, xk_off = 0, xk_flags = 0, xk_a = 0;
    // RMS jobs stage bf16(x * w) and scale the row sums by 1/rms in the
    // epilogue (the batched GEMMs' order), so the tile sweep starts without
    // waiting for the sum-of-squares reduction: xinv of the staged x, taken
    // from the per-warp partials (S->bc) at the first epilogue
    float rs_scale = 1.f, xinv = 1.f;
    bool xinv_pending = false;

    __device__ void sync() const { named_bar(BAR_VCC, NCT); }
    __device__ bool aborted() const { return *reinterpret_cast<volatile int32_t*>(&P->status->abort) != 0; }
    __device__ void fire(uint32_t code, uint32_t info) const {
        if (atomicCAS(&P->status->abort, 0, code == 0 ? 1 : 2) == 0) {
            P->status->fault_code = code;
            P->status->fault_info = info;
            P->status->stalled_core[0] = 2 * sm + 1;
            P->status->n_stalled = 1;
        }
    }
    __device__ char* tptr(int32_t t) const { return P->descs[t].ptr; }
    // symmetric (TP) tensors keep their readiness counter in their buffer header
    __device__ char* sym_base(int32_t t, uint32_t q) const { return P->sym ? P->sym[size_t(t) * VDC_RING_MAX_TP + q] : nullptr; }
    __device__ uint32_t* ctr(int32_t t) const {
        char* b = t >= 0 ? sym_base(t, P->tp_rank) : nullptr;
        return b ? reinterpret_cast<uint32_t*>(b) : &P->counters[t < 0 ? 0 : t];
    }
    __device__ int64_t token() const { return S->sstep[0]; }
    __device__ int32_t tdtype(int32_t t) const { return P->descs[t].dtype; }

    // all compute threads: wait for ring tile k (slot full)
    __device__ bool wait_full(uint32_t slot, uint32_t parity) {
        const long long c0 = clock64();
        if (mbar_try(&S->full[slot], parity)) {
            if (ct == 0) stat_add(VS_FULL, clock64() - c0);
            return true;
        }
        const unsigned long long t0 = now_ns();
        for (uint32_t n = 1;; ++n) {
            if (mbar_wait_hint(&S->full[slot], parity)) break;
            if ((n & 15) == 0) {
                if (aborted()) return false;
                if (P->watchdog_ns && now_ns() - t0 > P->watchdog_ns) {
                    fire(0, 0x10000u | slot);
                    return false;
                }
            }
        }
        if (ct == 0) stat_add(VS_FULL, clock64() - c0);
        return true;
    }
    __device__ void release(uint32_t slot) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&S->empty[slot]);
    }

    // thread 0 waits for every (tensor, target) then the VCC syncs; returns
    // false (everywhere) if the launch aborted
    __device__ bool wait_ready(int32_t t0, int32_t n0, int32_t t1, int32_t n1, int32_t t2, int32_t n2) {
        if (ct == 0) {
            // the (up to three) counters are polled together: one L2 round
            // trip per poll, not one per counter; one acquire fence at the end
            const long long c0 = clock64();
            const bool u0 = t0 >= 0 && n0 > 0, u1 = t1 >= 0 && n1 > 0, u2 = t2 >= 0 && n2 > 0;
            const uint32_t g0 = uint32_t(n0) * ep, g1 = uint32_t(n1) * ep, g2 = uint32_t(n2) * ep;
            const uint32_t* c0p = ctr(u0 ? t0 : -1);
            const uint32_t* c1p = ctr(u1 ? t1 : -1);
            const uint32_t* c2p = ctr(u2 ? t2 : -1);
            const bool sys = P->tp_world > 1;  // peers publish at system scope
            bool good = true;
            if (u0 || u1 || u2) {
                const unsigned long long w0 = now_ns();
                for (uint32_t n = 1;; ++n) {
                    const uint32_t v0 = u0 ? (sys ? ld_relaxed_sys(c0p) : ld_relaxed(c0p)) : 0u;
                    const uint32_t v1 = u1 ? (sys ? ld_relaxed_sys(c1p) : ld_relaxed(c1p)) : 0u;
                    const uint32_t v2 = u2 ? (sys ? ld_relaxed_sys(c2p) : ld_relaxed(c2p)) : 0u;
                    // signed distance: counters grow monotonically across launches and
                    // wrap at 2^32; a target is reached when v - g (mod 2^32) is
                    // non-negative as a signed value (gaps stay far below 2^31)
                    if ((!u0 || int32_t(v0 - g0) >= 0) && (!u1 || int32_t(v1 - g1) >= 0) && (!u2 || int32_t(v2 - g2) >= 0)) break;
                    if ((n & 255) == 0) {
                        if (aborted()) {
                            good = false;
                            break;
                        }
                        if (P->watchdog_ns && now_ns() - w0 > P->watchdog_ns) {
                            fire(0, 0x20000u | uint32_t(u0 ? t0 : u1 ? t1 : t2));
                            good = false;
                            break;
                        }
                    }
                }
                if (sys)
                    asm volatile("fence.acq_rel.sys;" ::: "memory");
                else
                    fence_acquire_gpu();
            }
            S->flag = good ? 1 : 0;
            stat_add(VS_DEP, clock64() - c0);
            if (P->trace) S->t_ready = now_ns();
        }
        sync();
        return S->flag != 0;
    }

    // after all threads stored the job's outputs
    __device__ void publish(int32_t t) {
        sync();
        if (ct == 0 && t >= 0) red_release_add(ctr(t), 1u);  // release is cumulative over the CTA barrier
    }

    // ---------------------------------------------------------------- GEMV
    template <bool BF>
    __device__ void gemv(const vdc_job& J) {
        constexpr int EPC = BF ? 8 : 4;  // elements per 16-byte chunk
        const int K = J.k, nch = K / EPC;
        const int32_t rmsf = J.flags & VDC_JOB_RMS;
        const bool reuse = xk_t == J.x_t && xk_off == J.x_off && xk_flags == rmsf && xk_a == J.a_t;
        // the norm weight is immutable: its chunks are requested before the
        // readiness wait (read once per step, it is usually evicted from L2 by
        // then, and its DRAM latency would otherwise follow the wait)
        // (single-request kernel only: the batched instance, which runs GEMV
        // µops rarely, would spill holding them across the wait)
        uint4 gr[XPT];
        const uint4* ws = rmsf ? reinterpret_cast<const uint4*>(tptr(J.a_t)) : nullptr;
        if constexpr (!BATCHED) {
            if (!reuse && rmsf) {
#pragma unroll
                for (int i = 0; i < XPT; ++i) {
                    const int c = int(ct) + i * NCT;
                    gr[i] = c < nch ? __ldg(ws + c) : make_uint4(0, 0, 0, 0);
                }
            }
        }
        if (!wait_ready(reuse ? -1 : J.x_t, J.x_need, (J.flags & VDC_JOB_RESID) ? J.a_t : -1, J.a_need, -1, 0)) {
            ok = false;
            return;
        }
        if (!reuse) {  // stage x (RMS-normalised, rounded to the model dtype) in shared memory
            // every chunk of x is requested before any is used: one L2 round
            // trip instead of one per loop iteration
            const uint4* xs = reinterpret_cast<const uint4*>(tptr(J.x_t)) +
                              (J.x_off + (J.flags & VDC_JOB_TOKEN_ROW ? token() * int64_t(K) : 0)) / EPC;
            uint4 xr[XPT];
#pragma unroll
            for (int i = 0; i < XPT; ++i) {
                const int c = int(ct) + i * NCT;
                xr[i] = c < nch ? ldcg128(xs + c) : make_uint4(0, 0, 0, 0);
                if constexpr (BATCHED) gr[i] = (rmsf && c < nch) ? __ldg(ws + c) : make_uint4(0, 0, 0, 0);
            }
            if (rmsf) {  // this warp's sum of squares; 1/rms is formed at the epilogue
                float ss = 0.f;
#pragma unroll
                for (int i = 0; i < XPT; ++i) ss += dot16<BF>(xr[i], xr[i]);
                ss = warp_sum(ss);
                if (lane == 0) S->bc[w] = ss;
                xinv_pending = true;
            }
#pragma unroll
            for (int i = 0; i < XPT; ++i) {
                const int c = int(ct) + i * NCT;
                if (c >= nch) break;
                uint4 v = xr[i];
                if (rmsf) {
                    const uint4 g = gr[i];
                    if constexpr (BF) {
                        v.x = pack2(bf_lo(v.x) * bf_lo(g.x), bf_hi(v.x) * bf_hi(g.x));
                        v.y = pack2(bf_lo(v.y) * bf_lo(g.y), bf_hi(v.y) * bf_hi(g.y));
                        v.z = pack2(bf_lo(v.z) * bf_lo(g.z), bf_hi(v.z) * bf_hi(g.z));
                        v.w = pack2(bf_lo(v.w) * bf_lo(g.w), bf_hi(v.w) * bf_hi(g.w));
                    } else {
                        v.x = __float_as_uint(__uint_as_float(v.x) * __uint_as_float(g.x));
                        v.y = __float_as_uint(__uint_as_float(v.y) * __uint_as_float(g.y));
                        v.z = __float_as_uint(__uint_as_float(v.z) * __uint_as_float(g.z));
                        v.w = __float_as_uint(__uint_as_float(v.w) * __uint_as_float(g.w));
                    }
                }
                S->x[c] = v;
            }
            xk_t = J.x_t;
            xk_off = J.x_off;
            xk_flags = rmsf;
            xk_a = J.a_t;
            sync();
            if ((P->debug & 4u) && P->trace && ct == 0) S->t_ready = now_ns();  // debug: trace "ready" = x staged
        }
        if (J.flags & VDC_JOB_RESID) {  // residual element of this thread's output row (hidden behind the sweep)
            const int i = int(ct);
            resid = 0.f;
            if (i < J.r1 - J.r0) {
                const char* ab = tptr(J.a_t);
                const int64_t ai = int64_t(J.a_off) + (J.r0 - J.out_row0) + i + (J.flags & VDC_JOB_TOKEN_AUX ? token() * int64_t(J.cache_rows) : 0);
                resid = tdtype(J.a_t) == VDC_DTYPE_BF16 ? bf_lo(ldcg_u16(reinterpret_cast<const uint16_t*>(ab) + ai))
                                                        : ldcg_f32(reinterpret_cast<const float*>(ab) + ai);
            }
        }
        if ((J.flags & (VDC_JOB_ROPE | VDC_JOB_QKV)) && (rope_hd != J.head_dim || rope_theta != J.theta)) {
            // rotary table of this launch's position: cos/sin per dim pair, angles in double precision
            const int64_t pos = S->sstep[1];
            for (int d2 = int(ct); d2 < J.head_dim / 2; d2 += NCT) {
                const double ang = double(pos) * pow(double(J.theta), -double(2 * d2) / double(J.head_dim));
                S->rope_cs[d2] = float(cos(ang));
                S->rope_sn[d2] = float(sin(ang));
            }
            rope_hd = J.head_dim;
            rope_theta = J.theta;
            sync();
        }
        if constexpr (BF) {
            switch (J.tile_rows) {  // lowering guarantees 2/4/8-row tiles with 16 * (16 / TR) | chunks per row
                case 2: tiles_mma<2>(J); break;
                case 4: tiles_mma<4>(J); break;
                default: tiles_mma<8>(J); break;
            }
        } else {
            switch (J.tile_rows) {
                case 1: tiles<false, 1>(J); break;
                case 2: tiles<false, 2>(J); break;
                case 4: tiles<false, 4>(J); break;
                default: tiles<false, 8>(J); break;
            }
        }
        sync();  // (an aborted launch runs on through the epilogue: every warp must reach the same barriers)
        if (rmsf) {
            if (xinv_pending) {  // the staging's per-warp sums of squares (S->bc, before the staging barrier)
                float tot = 0.f;
#pragma unroll
                for (int i = 0; i < CW; ++i) tot += S->bc[i];
                xinv = 1.0f / sqrtf(tot / float(K) + J.eps);
                xinv_pending = false;
            }
            rs_scale = xinv;
        }
        const long long e0 = clock64();
        gemv_epilogue(J, J.r1 - J.r0);
        if (ct == 0) stat_add(VS_EPI, clock64() - e0);
        if (J.flags & VDC_JOB_QKV) {
            const int qrows = J.block, kvr = J.split;
            sync();
            if (ct == 0) {
                if (J.r0 < qrows) red_release_add(&P->counters[J.o_t], 1u);
                if (J.r0 < qrows + kvr && J.r1 > qrows) red_release_add(&P->counters[J.b_t], 1u);
                if (J.r1 > qrows + kvr) red_release_add(&P->counters[J.o2_t], 1u);
            }
        } else if (J.flags & VDC_JOB_SYM_OUT) {
            sync();  // the partial rows were stored into every rank's slot: publish on every rank
            if (ct == 0)
                for (uint32_t q = 0; q < P->tp_world; ++q)
                    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(sym_base(J.o_t, q)) : "memory");
        } else {
            if (J.flags & VDC_JOB_ARGMAX) argmax_rows(J, J.r1 - J.r0);
            publish(J.o_t);
        }
        rs_scale = 1.f;
    }

    // TP sampling exchange (one thread): spin at system scope until the
    // symmetric header of t reaches n x epoch; false if the launch aborted
    __device__ bool wait_sym(int32_t t, uint32_t n) const {
        const uint32_t* c = reinterpret_cast<const uint32_t*>(sym_base(t, P->tp_rank));
        const uint32_t g = n * ep;
        const unsigned long long w0 = now_ns();
        for (uint32_t k = 1;; ++k) {
            if (int32_t(ld_relaxed_sys(c) - g) >= 0) break;
            if ((k & 255) == 0) {
                if (aborted()) return false;
                if (P->watchdog_ns && now_ns() - w0 > P->watchdog_ns) {
                    fire(0, 0x50000u | uint32_t(t));
                    return false;
                }
            }
        }
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        return true;
    }
    // (one thread) post n (value, index) pairs into slot tp_rank of every
    // rank's exchange buffer t (slot = n pairs), release on every header
    __device__ void post_sym_pairs(int32_t t, int n, const float* v, const int* idx) const {
        for (uint32_t q = 0; q < P->tp_world; ++q) {
            float* d = reinterpret_cast<float*>(sym_base(t, q) + VDC_SYM_HEADER_BYTES) + size_t(P->tp_rank) * 2 * n;
            for (int i = 0; i < n; ++i) {
                d[2 * i] = v[i];
                d[2 * i + 1] = __int_as_float(idx[i]);
            }
        }
        for (uint32_t q = 0; q < P->tp_world; ++q)
            asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(sym_base(t, q)) : "memory");
    }

    // greedy sampling fused into the lm_head epilogue: (max, first argmax)
    // of this job's logit rows, merged into the SM's running best; the SM's
    // last lm_head job posts it to its slot, and the last SM to arrive
    // reduces the slots (one warp, ties -> lowest vocab index like numpy
    // argmax) and writes the token
    float am_v = -INFINITY;
    int am_i = 0x7fffffff;
    __device__ static void am_merge(float& bv, int& bi, float ov, int oi) {
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    __device__ void argmax_rows(const vdc_job& J, int rows) {
        const int tpr = J.k / J.tile_cols;
        float bv = -INFINITY;
        int bi = 0x7fffffff;
        for (int i = int(ct); i < rows; i += NCT) am_merge(bv, bi, row_sum(i, tpr), J.r0 - J.out_row0 + i);
#pragma unroll
        for (int o = 16; o; o >>= 1) am_merge(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
        if (lane == 0) {
            S->bc[w] = bv;
            S->bc[CW + w] = __int_as_float(bi);
        }
        sync();
        if (ct == 0) {
            for (int q = 0; q < CW; ++q) am_merge(am_v, am_i, S->bc[q], __float_as_int(S->bc[CW + q]));
            S->flag = 0;
            if (J.block) {  // the SM's last lm_head job: post, arrive
                float* part = reinterpret_cast<float*>(tptr(J.b_t)) + 2 * J.split;
                part[0] = am_v;
                part[1] = __int_as_float(am_i);
                uint32_t old;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&P->counters[J.arrive_ctr]) : "memory");
                S->flag = (old + 1u == uint32_t(J.arrive_need) * ep) ? 1 : 0;
            }
        }
        sync();
        if (S->flag && w == 0) {
            const float* all = reinterpret_cast<const float*>(tptr(J.b_t));
            float v0 = -INFINITY;
            int i0 = 0x7fffffff;
            for (int q = int(lane); q < J.arrive_need; q += 32)
                am_merge(v0, i0, ldcg_f32(all + 2 * q), __float_as_int(ldcg_f32(all + 2 * q + 1)));
#pragma unroll
            for (int o = 16; o; o >>= 1) am_merge(v0, i0, __shfl_xor_sync(0xffffffffu, v0, o), __shfl_xor_sync(0xffffffffu, i0, o));
            if (J.flags & VDC_JOB_TP_ARGMAX) {
                // vocab-parallel: this rank's best with its global index -> every
                // rank; reduce the W posts in rank order (ties -> lowest index)
                const int gi = i0 == 0x7fffffff ? i0 : i0 + J.o2_off;
                int good = 1;
                if (lane == 0) {
                    post_sym_pairs(J.group, 1, &v0, &gi);
                    good = wait_sym(J.group, P->tp_world) ? 1 : 0;
                }
                good = __shfl_sync(0xffffffffu, good, 0);
                v0 = -INFINITY;
                i0 = 0x7fffffff;
                if (good && lane < P->tp_world) {
                    const float* x = reinterpret_cast<const float*>(sym_base(J.group, P->tp_rank) + VDC_SYM_HEADER_BYTES) + 2 * lane;
                    v0 = ldcg_f32(x);
                    i0 = __float_as_int(ldcg_f32(x + 1));
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) am_merge(v0, i0, __shfl_xor_sync(0xffffffffu, v0, o), __shfl_xor_sync(0xffffffffu, i0, o));
                if (!good) ok = false;
            }
            if (lane == 0) {
                *reinterpret_cast<int64_t*>(tptr(J.o2_t)) = int64_t(i0);
                if (J.flags & VDC_JOB_FEEDBACK) {  // next launch: this token at the next position
                    int64_t* st = const_cast<int64_t*>(P->step);
                    st[VDC_STEP_TOKEN] = int64_t(i0);
                    st[VDC_STEP_POS] += 1;
                    st[VDC_STEP_CTX] += 1;
                }
                red_release_add(ctr(J.o2_t), 1u);
            }
        }
    }

    // bf16 GEMV tile on the tensor cores (mma.sync m16n8k16, fp32 accumulate).
    // A TR-row x (cpt x 8)-column tile is viewed as 16 "virtual rows"
    // v = r * NC + c (NC = 16 / TR chunk classes): virtual row v holds the
    // 16-byte chunks c, c + NC, c + 2 NC, ... of W row r, so one ldmatrix.x4
    // reads 8 consecutive chunks per matrix (bank-conflict free). B column n
    // holds the matching x chunks of class n; the partial dot products of row
    // r are the diagonal entries D[r * NC + c][c], summed over c. Tensor-core
    // work is 8x redundant (only the diagonal is used) but the instruction
    // count per 16 KB tile drops from ~1200 FFMA/unpack to ~100, which is
    // what bounds the slot hold time of warp-per-tile consumption.
    template <int TR>
    __device__ void tiles_mma(const vdc_job& J) {
        constexpr int NC = 16 / TR;
        const int K = J.k, tc = J.tile_cols, tpr = K / tc, cpt = tc / 8;
        const int rows = J.r1 - J.r0, ntiles = (rows / TR) * tpr;
        const uint32_t row_bytes = uint32_t(cpt) * 16u;
        const uint32_t xb = smem_addr(S->x);
        const int ksteps = cpt / (2 * NC);
        // ldmatrix source of this lane: matrix mi = lane / 8 -> (virtual row block, k half)
        const int mi = int(lane) >> 3, vi = int(lane & 7u) + 8 * (mi & 1), kh = mi >> 1;
        const uint32_t a_lane = uint32_t(vi / NC) * row_bytes + uint32_t(vi % NC + NC * kh) * 16u;
        // B fragment: n = lane / 4 (class), k = (lane % 4) * 2
        const int bn = int(lane) >> 2;
        const uint32_t b_lane = uint32_t(bn % NC) * 16u + (lane & 3u) * 4u;
        // diagonal ownership: lanes with lane % 4 == c / 2 hold D[v][c] for v = lane / 4 (+8)
        const int c_lo = (int(lane) >> 2) % NC;
        const bool diag = int(lane & 3u) == (c_lo >> 1);
        const bool odd = c_lo & 1;
        const int r_lo = (int(lane) >> 2) / NC, r_hi = ((int(lane) >> 2) + 8) / NC;
        uint32_t g = kt - 1u, gs = kt % R, gph = (kt / R) & 1u;
        for (int t = 0; t < ntiles; ++t) {
            // ring tile g lives in slot g % R and belongs to compute warp (g % R) % 8
            const uint32_t wslot = gs, wphase = gph;
            ++g;
            if (++gs == R) {
                gs = 0;
                gph ^= 1u;
            }
            if ((wslot & uint32_t(CW - 1)) != w) continue;
            const int rg = t / tpr, c = t - rg * tpr;
            if (!wait_full(wslot, wphase)) {
                // aborted launch: keep the VCC's control flow uniform (every
                // warp reaches the same barriers), skip the arithmetic
                ok = false;
                release(wslot);
                continue;
            }
            const bool ttr = P->tile_trace && sm == (P->debug >> 8) && g < P->tile_trace_cap && lane == 0;
            if (ttr) P->tile_trace[3 * g + 1] = now_ns();
            const uint32_t abase = ring + wslot * SLOT + a_lane;
            const uint32_t bbase = xb + uint32_t(c * cpt) * 16u + b_lane;
            float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
            float d2[4] = {0.f, 0.f, 0.f, 0.f}, d3[4] = {0.f, 0.f, 0.f, 0.f};
            if (!(P->debug & 1u)) {
                // groups of 8 (then 4) k-steps: all fragment loads first, then the
                // MMAs (volatile asm keeps program order, so the order is
                // explicit); k-step u of a group accumulates into d[u % 4], the
                // same per-accumulator order as groups of 4
                int st = 0;
                for (; st + 8 <= ksteps; st += 8) {
                    uint32_t a[8][4], b[8][2];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t off = uint32_t((st + u) * 2 * NC) * 16u;
                        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(a[u][0]), "=r"(a[u][1]), "=r"(a[u][2]), "=r"(a[u][3])
                                     : "r"(abase + off));
                        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b[u][0]) : "r"(bbase + off));
                        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b[u][1]) : "r"(bbase + off + uint32_t(NC) * 16u));
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        float* d = (u & 3) == 0 ? d0 : (u & 3) == 1 ? d1 : (u & 3) == 2 ? d2 : d3;
                        asm volatile(
                            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                            "{%0,%1,%2,%3};"
                            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                            : "r"(a[u][0]), "r"(a[u][1]), "r"(a[u][2]), "r"(a[u][3]), "r"(b[u][0]), "r"(b[u][1]));
                    }
                }
                for (; st + 4 <= ksteps; st += 4) {
                    uint32_t a[4][4], b[4][2];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t off = uint32_t((st + u) * 2 * NC) * 16u;
                        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(a[u][0]), "=r"(a[u][1]), "=r"(a[u][2]), "=r"(a[u][3])
                                     : "r"(abase + off));
                        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b[u][0]) : "r"(bbase + off));
                        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b[u][1]) : "r"(bbase + off + uint32_t(NC) * 16u));
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        float* d = u == 0 ? d0 : u == 1 ? d1 : u == 2 ? d2 : d3;
                        asm volatile(
                            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                            "{%0,%1,%2,%3};"
                            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                            : "r"(a[u][0]), "r"(a[u][1]), "r"(a[u][2]), "r"(a[u][3]), "r"(b[u][0]), "r"(b[u][1]));
                    }
                }
                for (; st < ksteps; ++st) {
                    const uint32_t off = uint32_t(st * 2 * NC) * 16u;
                    uint32_t a0, a1, a2, a3, b0, b1;
                    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                                 : "r"(abase + off));
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b0) : "r"(bbase + off));
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b1) : "r"(bbase + off + uint32_t(NC) * 16u));
                    asm volatile(
                        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                        "{%0,%1,%2,%3};"
                        : "+f"(d0[0]), "+f"(d0[1]), "+f"(d0[2]), "+f"(d0[3])
                        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
                }
            }
            __syncwarp();
            if (ttr) P->tile_trace[3 * g + 2] = now_ns();
            if (lane == 0) mbar_arrive(&S->empty[wslot]);  // the tile goes back to the memory core
#pragma unroll
            for (int e = 0; e < 4; ++e) d0[e] = (d0[e] + d1[e]) + (d2[e] + d3[e]);
            const float vlo = diag ? (odd ? d0[1] : d0[0]) : 0.f;
            const float vhi = diag ? (odd ? d0[3] : d0[2]) : 0.f;
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                const float v = warp_sum((r_lo == r ? vlo : 0.f) + (r_hi == r ? vhi : 0.f));
                if (lane == 0) S->red[c][rg * TR + r] = v;
            }
        }
        kt += uint32_t(ntiles);
    }

    // Consume the job's W tiles warp-per-tile: ring tile g (global consumption
    // index) belongs to compute warp g % 8, so eight tiles are in the compute
    // pipeline at once and each tile costs one full-wait and one release. A
    // warp accumulates its tile's rows over its 32 lanes (x chunks from the
    // staged vector in shared memory), releases the slot, reduces across the
    // warp and adds the row sums to red[warp][row]; column-split rows (K
    // larger than a slot) are summed over warps in the epilogue.
    template <bool BF, int TR>
    __device__ void tiles(const vdc_job& J) {
        constexpr int EPC = BF ? 8 : 4;
        const int K = J.k, tc = J.tile_cols, tpr = K / tc, cpt = tc / EPC;
        const int rows = J.r1 - J.r0, ntiles = (rows / TR) * tpr;
        const uint32_t row_bytes = uint32_t(cpt) * 16u;
        const uint32_t xb = smem_addr(S->x);
        uint32_t g = kt - 1u, gs = kt % R, gph = (kt / R) & 1u;
        for (int t = 0; t < ntiles; ++t) {
            // ring tile g lives in slot g % R and belongs to compute warp (g % R) % 8
            const uint32_t wslot = gs, wphase = gph;
            ++g;
            if (++gs == R) {
                gs = 0;
                gph ^= 1u;
            }
            if ((wslot & uint32_t(CW - 1)) != w) continue;
            const int rg = t / tpr, c = t - rg * tpr;
            if (!wait_full(wslot, wphase)) {  // aborted launch: uniform control flow, no arithmetic
                ok = false;
                release(wslot);
                continue;
            }
            const uint32_t base = ring + wslot * SLOT;
            const bool ttr = P->tile_trace && sm == (P->debug >> 8) && g < P->tile_trace_cap && lane == 0;
            if (ttr) P->tile_trace[3 * g + 1] = now_ns();
            if (P->debug & 1u) {
                release(wslot);
                continue;
            }
            // two independent accumulators per row (even / odd chunk steps)
            // halve the FMA dependency chain of the 16-step sweep
            float acc[2][TR];
#pragma unroll
            for (int r = 0; r < TR; ++r) acc[0][r] = acc[1][r] = 0.f;
#pragma unroll 2
            for (int j = int(lane); j < cpt; j += 64) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int jj = j + 32 * h;
                    if (jj >= cpt) break;
                    const uint4 xv = lds128(xb + uint32_t(c * cpt + jj) * 16u);
                    float x[EPC];
                    if constexpr (BF) {
                        x[0] = bf_lo(xv.x); x[1] = bf_hi(xv.x); x[2] = bf_lo(xv.y); x[3] = bf_hi(xv.y);
                        x[4] = bf_lo(xv.z); x[5] = bf_hi(xv.z); x[6] = bf_lo(xv.w); x[7] = bf_hi(xv.w);
                    } else {
                        x[0] = __uint_as_float(xv.x); x[1] = __uint_as_float(xv.y);
                        x[2] = __uint_as_float(xv.z); x[3] = __uint_as_float(xv.w);
                    }
#pragma unroll
                    for (int r = 0; r < TR; ++r) {
                        const uint4 wv = lds128(base + uint32_t(r) * row_bytes + uint32_t(jj) * 16u);
                        float s = acc[h][r];
                        if constexpr (BF) {
                            s = fmaf(bf_lo(wv.x), x[0], s);
                            s = fmaf(bf_hi(wv.x), x[1], s);
                            s = fmaf(bf_lo(wv.y), x[2], s);
                            s = fmaf(bf_hi(wv.y), x[3], s);
                            s = fmaf(bf_lo(wv.z), x[4], s);
                            s = fmaf(bf_hi(wv.z), x[5], s);
                            s = fmaf(bf_lo(wv.w), x[6], s);
                            s = fmaf(bf_hi(wv.w), x[7], s);
                        } else {
                            s = fmaf(__uint_as_float(wv.x), x[0], s);
                            s = fmaf(__uint_as_float(wv.y), x[1], s);
                            s = fmaf(__uint_as_float(wv.z), x[2], s);
                            s = fmaf(__uint_as_float(wv.w), x[3], s);
                        }
                        acc[h][r] = s;
                    }
                }
            }
            __syncwarp();
            if (ttr) P->tile_trace[3 * g + 2] = now_ns();
            if (lane == 0) mbar_arrive(&S->empty[wslot]);  // the tile goes back to the memory core
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                const float v = warp_sum(acc[0][r] + acc[1][r]);
                if (lane == 0) S->red[c][rg * TR + r] = v;
            }
        }
        kt += uint32_t(ntiles);
    }

    // (rs_scale: the RMS jobs' 1/rms, applied to the row sums in the epilogue)
    __device__ float row_sum(int i, int tpr) const {
        float v = S->red[0][i];
        for (int c = 1; c < tpr; ++c) v += S->red[c][i];
        return v * rs_scale;
    }

    __device__ void store_out(char* base, bool bf, int64_t idx, float v) const {
        if (bf)
            reinterpret_cast<uint16_t*>(base)[idx] = f2bf(v);
        else
            reinterpret_cast<float*>(base)[idx] = v;
    }

    __device__ void gemv_epilogue(const vdc_job& J, int rows) {
        const int tpr = J.k / J.tile_cols;
        char* ob = tptr(J.o_t);
        const bool obf = tdtype(J.o_t) == VDC_DTYPE_BF16;
        const int lr0 = J.r0 - J.out_row0;  // first output row (region-local)
        const int64_t pos = S->sstep[1];
        const bool swz = J.flags & VDC_JOB_KVSWZ;  // swizzled cache page rows
        // element d of a cache row at position pos, in storage order
        auto cache_col = [&](int d) -> int { return swz ? int((kv_swz(uint32_t(d) >> 3, uint32_t(pos & 7)) << 3) | uint32_t(d & 7)) : d; };
        auto out_index = [&](int lr) -> int64_t {
            if (J.flags & VDC_JOB_KV_APPEND)
                return (int64_t(lr / J.head_dim) * J.cache_rows + pos) * J.head_dim + cache_col(lr % J.head_dim);
            return int64_t(J.o_off) + lr;
        };
        if (J.flags & VDC_JOB_QKV) {
            // fused q | k | v rows of one SM's share: rotary on q and k rows,
            // k and v rows appended to the caches at the step position
            const int qrows = J.block, kvr = J.split, hd = J.head_dim;
            char* kb = tptr(J.b_t);
            char* vb = tptr(J.o2_t);
            if (pos >= J.cache_rows) {  // past the cache capacity (e.g. a device decode loop ran too long)
                if (ct == 0) fire(7, uint32_t(pos));
                return;
            }
            for (int p = int(ct); p < rows / 2; p += NCT) {
                const int wr = J.r0 + 2 * p;  // W row (pairs never straddle a region boundary)
                float a = row_sum(2 * p, tpr), b = row_sum(2 * p + 1, tpr);
                if (wr < qrows + kvr && !(J.flags & VDC_JOB_QKNORM)) {
                    const int d = (wr < qrows ? wr : wr - qrows) % hd;
                    const float cs = S->rope_cs[d / 2], sn = S->rope_sn[d / 2];
                    const float na = a * cs - b * sn, nb = a * sn + b * cs;
                    a = na;
                    b = nb;
                }
                if (wr < qrows) {
                    store_out(ob, obf, int64_t(J.o_off) + wr, a);
                    store_out(ob, obf, int64_t(J.o_off) + wr + 1, b);
                } else {
                    const bool isk = wr < qrows + kvr;
                    const int lr = isk ? wr - qrows : wr - qrows - kvr;
                    // (a pair of dims never straddles a 16-byte chunk)
                    const int64_t at = (int64_t(lr / hd) * J.cache_rows + pos) * hd + cache_col(lr % hd);
                    store_out(isk ? kb : vb, obf, at, a);
                    store_out(isk ? kb : vb, obf, at + 1, b);
                }
            }
        } else if (J.flags & VDC_JOB_SWIGLU) {
            const int B = J.block, hb = B / 2;
            for (int j = int(ct); j < rows / 2; j += NCT) {
                const int blk = j / hb, jj = j % hb;
                const float gt = row_sum(blk * B + jj, tpr), up = row_sum(blk * B + hb + jj, tpr);
                store_out(ob, obf, int64_t(J.o_off) + lr0 / 2 + j, gt / (1.0f + expf(-gt)) * up);
            }
        } else if (J.flags & VDC_JOB_ROPE) {
            for (int p = int(ct); p < rows / 2; p += NCT) {
                const int lr = lr0 + 2 * p;
                float a = row_sum(2 * p, tpr), b = row_sum(2 * p + 1, tpr);
                const int d = lr % J.head_dim;
                const float cs = S->rope_cs[d / 2], sn = S->rope_sn[d / 2];
                const float na = a * cs - b * sn, nb = a * sn + b * cs;
                store_out(ob, obf, out_index(lr), na);
                store_out(ob, obf, out_index(lr + 1), nb);
            }
        } else {
            const bool res = J.flags & VDC_JOB_RESID;
            const bool symo = J.flags & VDC_JOB_SYM_OUT;
            for (int i = int(ct); i < rows; i += NCT) {
                float v = row_sum(i, tpr);
                if (res) v += resid;
                if (symo) {  // TP partial sum -> slot `tp_rank` of every rank's buffer (NVLink peer stores)
                    for (uint32_t q = 0; q < P->tp_world; ++q)
                        store_out(sym_base(J.o_t, q) + VDC_SYM_HEADER_BYTES, obf, int64_t(J.o_off) + lr0 + i, v);
                } else {
                    store_out(ob, obf, out_index(lr0 + i), v);
                }
            }
        }
    }

    // ------------------------------------------------------------ BGEMM
    // Batched GEMM µop (batched programs): out[b][r] = sum_k W[r][k] X[b][k]
    // for the 128 W rows [r0, r0 + 128) and the nb requests, reduction tiles
    // [kt0, kt1) (a stream-K piece of the row block).
    //  * W tiles (128 x 64 bf16, 128-byte swizzle) arrive in the ring from
    //    the memory core (TMA tensor copies, prefetched across operators).
    //  * activation chunks (npad x 64) are loaded by the MMA issuer (thread 0)
    //    after the readiness wait, into a small ring in the x buffer; the
    //    issuer keeps NX - 1 chunks in flight.
    //  * thread 0 issues 4 tcgen05.mma (M=128, N=npad, K=16) per tile into the
    //    TMEM accumulator; tcgen05.commit hands the W slot back to the memory
    //    core (its empty barrier) and the chunk buffer back to the issuer once
    //    the MMAs that read them completed.
    //  * epilogue: tcgen05.ld (warp w: TMEM lanes 32 (w % 4) .. , columns
    //    (w / 4) * npad / 2 ..); pieces of a split row block add their fp32
    //    partials in piece order (the last to arrive finishes the block);
    //    per-request rms scale, rotary / KV append / SwiGLU / residual, stores.
    uint32_t tmem = 0;
    uint32_t xq = 0, xd = 0;  // activation chunks issued / consumed (issuer thread)
    uint32_t nmma = 0;        // BGEMM µops completed (mma_bar phase)
    int32_t binv_t = -2;      // activations the cached rms scales belong to

    __device__ float* f32p(int32_t t) const { return reinterpret_cast<float*>(tptr(t)); }
    __device__ uint16_t* u16p(int32_t t) const { return reinterpret_cast<uint16_t*>(tptr(t)); }
    __device__ int64_t req_pos(int b) const { return S->bpos[b]; }

    // wait for an mbarrier phase; returns the cycles waited, or -1 if the
    // launch aborted (no member addresses escape: the Vcc stays in registers)
    __device__ long long spin(uint64_t* bar, uint32_t parity) {
        const long long c0 = clock64();
        if (mbar_try(bar, parity)) return clock64() - c0;
        const unsigned long long t0 = now_ns();
        for (uint32_t n = 1;; ++n) {
            if (mbar_wait_hint(bar, parity)) return clock64() - c0;
            if ((n & 15) == 0) {
                if (aborted()) return -1;
                if (P->watchdog_ns && now_ns() - t0 > P->watchdog_ns) {
                    fire(0, 0x40000u);
                    return -1;
                }
            }
        }
    }

    // debug trace (VDC_RING_DEBUG): per BGEMM µop of the traced SM, phase stamps
    // at tile_trace[200000 + 8 * (job % 4096) + ev]
    __device__ void bstamp(int ev) const {
        if (P->tile_trace && sm == (P->debug >> 8) && ct == 0) P->tile_trace[200000 + 16 * (nmma & 2047u) + ev] = now_ns();
    }
    // The RMS prologue's sums of squares move as one bulk copy (the TMA
    // engine), not as LSU loads: with every SM streaming weights, an L2-hit
    // ld.global round trip measured ~4.4 us, the bulk copy ~2.2 us (bulk copies
    // of the stream-K partials and residual rows measured no gain: 2954 vs
    // 2984 tokens/s, so those stay loads). Thread 0 issues (after the acquire
    // that made the producer's generic writes visible; the async proxy needs
    // its own fence) and every compute thread waits on S->lbar.
    uint32_t lph = 0;  // S->lbar phase (uniform over the VCC)
    __device__ void lbar_issue(uint32_t bytes) const {
        fence_proxy_async_global();
        mbar_expect_tx(&S->lbar, bytes);
    }
    __device__ bool lbar_wait() {
        const long long c = spin(&S->lbar, lph & 1u);
        ++lph;
        return c >= 0;
    }


    __device__ void bgemm(const vdc_job& J) {
        const long long p0 = clock64();
        bstamp(0);
        const int n = J.kt1 - J.kt0, K = J.k, nb = J.nb, npad = J.npad;
        const bool rms = J.flags & VDC_JOB_RMS;
        if (!wait_ready(J.x_t, J.x_need, rms ? J.x2_t : -1, J.x2_need, (J.flags & VDC_JOB_RESID) ? J.a_t : -1, J.a_need)) {
            ok = false;
            return;
        }
        bstamp(1);
        if (rms && binv_t != J.x2_t && J.ssq_t >= 0) {
            // 1 / rms from the producer's per-group sums of squares: 8 threads per
            // request each add K/32/8 groups (loads issued together), then the 8
            // partials in fixed order (deterministic)
            // the [K/32][npad] sums arrive in one bulk copy (after the staging area
            // of the per-thread partial sums), then 8 threads per request add
            // K/256 groups each and one thread adds the 8 partials in order
            const int G = K / 32, per = (G + 7) / 8;
            bstamp(9);
            float* scr = reinterpret_cast<float*>(S->x);
            float* sq = scr + 8 * VDC_RING_MAX_BATCH;
            const uint32_t sbytes = uint32_t(G * npad) * 4u;
            if (sbytes + 8u * VDC_RING_MAX_BATCH * 4u <= uint32_t(XBUF)) {
                if (ct == 0) {
                    lbar_issue(sbytes);
                    bulk_g2s(sq, f32p(J.ssq_t), sbytes, &S->lbar);
                }
                if (!lbar_wait()) {
                    ok = false;
                    return;
                }
            } else {
                for (int i = int(ct); i < G * npad; i += NCT) sq[i] = ldcg_f32(f32p(J.ssq_t) + i);
                sync();
            }
            for (int b0 = 0; b0 < nb; b0 += NCT / 8) {
                const int b = b0 + (int(ct) >> 3), part = int(ct) & 7;
                float ss = 0.f;
                if (b < nb)
                    for (int i = 0; i < per; ++i) {
                        const int g = part * per + i;
                        if (g < G) ss += sq[g * npad + b];
                    }
                scr[(b0 * 8) + int(ct)] = ss;
            }
            bstamp(8);
            sync();
            for (int b = int(ct); b < nb; b += NCT) {
                float tot = 0.f;
#pragma unroll
                for (int i = 0; i < 8; ++i) tot += scr[b * 8 + i];
                S->binv[b] = 1.0f / sqrtf(tot / float(K) + J.eps);
            }
            binv_t = J.x2_t;
            sync();
        } else if (rms && binv_t != J.x2_t) {  // per-request 1 / rms of the raw activations (warp per request)
            const uint16_t* xr = u16p(J.x2_t);
            for (int b = int(w); b < nb; b += CW) {
                const uint4* row = reinterpret_cast<const uint4*>(xr + int64_t(b) * K);
                float ss = 0.f;
                // 16 chunks per lane requested before any is used: one L2 round trip
                // per 16 (the loads are volatile asm, so the compiler keeps their order)
                for (int c0 = int(lane); c0 < K / 8; c0 += 32 * 16) {
                    uint4 u[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) u[i] = c0 + 32 * i < K / 8 ? ldcg128(row + c0 + 32 * i) : make_uint4(0, 0, 0, 0);
#pragma unroll
                    for (int i = 0; i < 16; ++i) ss += dot16<true>(u[i], u[i]);
                }
                ss = warp_sum(ss);
                if (lane == 0) S->binv[b] = 1.0f / sqrtf(ss / float(K) + J.eps);
            }
            binv_t = J.x2_t;
            sync();
        }
        const uint32_t xbytes = uint32_t(npad) * 128u;
        // activation-chunk buffers after the control block (1 KB aligned: the
        // 128-byte swizzle atoms repeat every 1 KB), NXW per compute warp
        const uint32_t xb0 = (smem_addr(S) + uint32_t(sizeof(Shared)) + 1023u) & ~1023u;
        const uint32_t NXW = min(2u, XRING_BYTES / xbytes / uint32_t(CW));
        if (ct == 0) stat_add(VS_PRO, clock64() - p0);
        if (ct == 0) S->flag = 1;
        sync();
        bstamp(2);
        // Every compute warp is an MMA issuer (lane 0) for the tiles of its own
        // ring slot (slot w of the 8-slot ring) into its own TMEM accumulator
        // (columns w * npad): like the single-request GEMV, each slot's
        // turnaround is independent, so one late tile does not hold the other
        // slots (head-of-line blocking of a single in-order issuer). The
        // epilogue adds the 8 accumulators in warp order (deterministic).
        if (lane == 0) {
            fence_proxy_async_global();
            fence_proxy_async_smem();
            const void* xm = static_cast<const char*>(P->tmaps) + size_t(J.x_t) * 128;
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(npad >> 3) << 17) | (uint32_t(128 >> 4) << 24);
            const uint32_t acc = tmem + w * uint32_t(npad);
            const int t0 = int((w + uint32_t(CW) - kt % uint32_t(CW)) % uint32_t(CW));  // first tile of this warp's slot
            bool good = true;
            auto xload = [&](int t) {  // activation chunk of tile t -> this warp's buffer xq % NXW
                const uint32_t i = w * NXW + xq % NXW;
                if (xq >= NXW) {
                    const long long c = spin(&S->xempty[i], ((xq / NXW) - 1u) & 1u);
                    if (c < 0) return false;
                    if (ct == 0) stat_add(VS_XE, c);
                }
                mbar_expect_tx(&S->xfull[i], xbytes);
                tma_2d(xb0 + i * xbytes, xm, (J.kt0 + t) * VDC_RING_BGEMM_KT, 0, &S->xfull[i]);
                ++xq;
                return true;
            };
            for (int t = t0, u = 0; t < n && u < int(NXW) && good; t += CW, ++u) good = xload(t);
            // debug tile trace (VDC_RING_DEBUG): loop top / activation chunk landed,
            // weight tile landed / MMAs committed
            unsigned long long* tt = (P->tile_trace && sm == (P->debug >> 8)) ? P->tile_trace : nullptr;
            for (int t = t0; t < n && good; t += CW) {
                const uint32_t g = kt + uint32_t(t), slot = g % R;
                const bool ttr = tt && g < 30000u;
                if (ttr) tt[100000 + 2 * g] = now_ns();
                const uint32_t xi = w * NXW + xd % NXW;
                const long long wc = spin(&S->xfull[xi], (xd / NXW) & 1u);
                if (ttr) tt[100000 + 2 * g + 1] = now_ns();
                if (wc < 0 || !wait_full(slot, (g / R) & 1u)) {
                    good = false;
                    break;
                }
                if (ttr) tt[3 * g + 1] = now_ns();
                if (ct == 0) stat_add(VS_XF, wc);
                tc_fence_after();
                if (!(P->debug & 1u)) {
                    const uint32_t a0 = ring + slot * SLOT, b0 = xb0 + xi * xbytes;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_bf16(acc, umma_sw128_desc(a0 + kk * 32), umma_sw128_desc(b0 + kk * 32), idesc,
                                  (t == t0 && kk == 0) ? 0u : 1u);
                }
                umma_commit(&S->empty[slot]);  // W slot -> memory core when its MMAs are done
                umma_commit(&S->xempty[xi]);
                if (ttr) tt[3 * g + 2] = now_ns();
                ++xd;
                if (t + int(NXW) * CW < n && !xload(t + int(NXW) * CW)) {
                    good = false;
                    break;
                }
            }
            umma_commit(&S->mma_bar);  // count 8: one per warp issuer (arrives at once if it issued nothing)
            if (!good) S->flag = 0;
        }
        kt += uint32_t(n);
        sync();
        bstamp(3);
        if (!S->flag) {
            ok = false;
            return;
        }
        // every warp issuer commits mma_bar (also after an abort), so this wait
        // always completes: never abandoned (no tcgen05 work may outlive the job)
        long long wm = 0;
        {
            const long long c0 = clock64();
            while (!mbar_wait_hint(&S->mma_bar, nmma & 1u)) {
            }
            wm = clock64() - c0;
        }
        if (ct == 0) stat_add(VS_MMA, wm);
        bstamp(4);
        tc_fence_after();
        const long long e0 = clock64();
        bool fin = false;
        switch (npad) {
            case 16: fin = bgemm_epilogue<8>(J); break;
            case 32: fin = bgemm_epilogue<16>(J); break;
            default: fin = bgemm_epilogue<32>(J); break;
        }
        if (ct == 0) stat_add(VS_EPI, clock64() - e0);
        bstamp(5);
        ++nmma;
        if ((J.flags & VDC_JOB_ARGMAX) && J.block) post_argmax_batched(J);
        if (!fin) return;  // a piece of a split row block that was not the last to arrive
        fence_proxy_async_global();  // consumers read these activations with TMA (async proxy)
        sync();
        if (ct == 0 && (J.flags & VDC_JOB_SYM_OUT)) {  // publish on every rank (system scope)
            for (uint32_t qr = 0; qr < P->tp_world; ++qr)
                asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(sym_base(J.o_t, qr)) : "memory");
        } else if (ct == 0) {
            red_release_add(ctr(J.o_t), 1u);
            if (J.flags & VDC_JOB_QKV) {
                red_release_add(ctr(J.b_t), 1u);
                red_release_add(ctr(J.o2_t), 1u);
            }
            if (J.o3_t >= 0) red_release_add(ctr(J.o3_t), 1u);
        }
    }

    template <int NH>
    __device__ __forceinline__ void tmem_ld(uint32_t addr, float (&v)[NH]) const {
        uint32_t r[NH];
        if constexpr (NH == 8) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "r"(addr));
        } else {
#pragma unroll
            for (int c = 0; c < NH; c += 16)
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[c]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]), "=r"(r[c + 6]),
                      "=r"(r[c + 7]), "=r"(r[c + 8]), "=r"(r[c + 9]), "=r"(r[c + 10]), "=r"(r[c + 11]), "=r"(r[c + 12]),
                      "=r"(r[c + 13]), "=r"(r[c + 14]), "=r"(r[c + 15])
                    : "r"(addr + uint32_t(c)));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int c = 0; c < NH; ++c) v[c] = __uint_as_float(r[c]);
    }

    // returns false when this piece is not the one that finishes its row block
    template <int NH>
    __device__ bool bgemm_epilogue(const vdc_job& J) {
        const int q = int(w & 3u);
        const int row = q * 32 + int(lane);  // row within the 128-row block (TMEM lane)
        const int c0 = int(w >> 2) * NH;     // first request column of this thread
        const int nb = J.nb, npad = J.npad;
        const int64_t M = J.cache_rows;      // output row stride (elements per request)
        const int rg = J.r0 + row;           // global W row
        float v[NH];
#pragma unroll
        for (int c = 0; c < NH; ++c) v[c] = 0.f;
        const int ntile = J.kt1 - J.kt0;
        // the per-warp accumulators in the order of their first tile (warp a took
        // tiles t = a - k0 mod 8), so the association of the sum does not depend
        // on where the job started in the ring; a warp without tiles wrote none
        const uint32_t k0 = (kt - uint32_t(ntile)) % uint32_t(CW);
        for (int tt = 0; tt < CW && tt < ntile; ++tt) {
            const int a = int((uint32_t(tt) + k0) % uint32_t(CW));
            float va[NH];
            tmem_ld<NH>(tmem + (uint32_t(q * 32) << 16) + uint32_t(a * npad) + uint32_t(c0), va);
#pragma unroll
            for (int c = 0; c < NH; ++c) v[c] += va[c];
        }
        tc_fence_before();  // the accumulator may be overwritten after the next barrier
        bstamp(6);
        if (J.arrive_need > 1) {
            // stream-K: this piece's partial -> global; the last piece of the
            // row block to arrive adds all partials in piece order
            float* part = f32p(J.part_t);
            float* mine = part + size_t(J.part_off) * size_t(npad) * 128;
#pragma unroll
            for (int c = 0; c < NH; ++c) mine[(c0 + c) * 128 + row] = v[c];
            sync();
            if (ct == 0) {
                uint32_t old;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&P->counters[J.arrive_ctr]) : "memory");
                S->flag = (old + 1u == uint32_t(J.arrive_need) * ep) ? 1 : 0;
            }
            sync();
            bstamp(7);
            if (!S->flag) return false;
            const float* p0 = part + size_t(J.part_off - J.split) * size_t(npad) * 128;
            float acc[NH];
#pragma unroll
            for (int c = 0; c < NH; ++c) acc[c] = 0.f;
#pragma unroll 4
            for (int s = 0; s < J.arrive_need; ++s) {
                float t[NH];
                if (s == J.split) {
#pragma unroll
                    for (int c = 0; c < NH; ++c) t[c] = v[c];
                } else {
                    const float* ps = p0 + size_t(s) * size_t(npad) * 128;
#pragma unroll
                    for (int c = 0; c < NH; ++c) t[c] = ldcg_f32(ps + (c0 + c) * 128 + row);
                }
#pragma unroll
                for (int c = 0; c < NH; ++c) acc[c] += t[c];
            }
#pragma unroll
            for (int c = 0; c < NH; ++c) v[c] = acc[c];
        }
        if (J.flags & VDC_JOB_RMS) {
#pragma unroll
            for (int c = 0; c < NH; ++c) v[c] *= S->binv[min(c0 + c, VDC_RING_MAX_BATCH - 1)];
        }
        if (J.flags & VDC_JOB_QKV) {
            const int qrows = J.block, kvr = J.kvrows, hd = J.head_dim, hkv = kvr / hd;
            const bool isq = rg < qrows, isk = !isq && rg < qrows + kvr;
            const int lr = isq ? rg : isk ? rg - qrows : rg - qrows - kvr;
            const int d = lr % hd;
            const double invf = pow(double(J.theta), -double(d & ~1) / double(hd));
            const bool even = (lane & 1u) == 0;
#pragma unroll
            for (int c = 0; c < NH; ++c) {
                const int b = c0 + c;
                const float other = __shfl_xor_sync(0xffffffffu, v[c], 1);
                if (b >= nb) continue;
                const int64_t pos = req_pos(b);
                if ((isq || isk) && !(J.flags & VDC_JOB_QKNORM)) {
                    double ang = double(pos) * invf;
                    ang -= 6.283185307179586 * rint(ang * 0.15915494309189535);
                    float sn, cs;
                    __sincosf(float(ang), &sn, &cs);  // |ang| <= pi after the reduction
                    v[c] = even ? v[c] * cs - other * sn : other * sn + v[c] * cs;
                }
                if (isq) {
                    u16p(J.o_t)[int64_t(b) * qrows + rg] = f2bf(v[c]);
                } else {
                    const int64_t page = S->bpage[b];  // (request b's page of pos, -1 if none)
                    if (page < 0) {  // no KV page allocated for this position: fail loudly, write nothing
                        fire(7, uint32_t(b));
                        continue;
                    }
                    // K and V rows are stored pre-swizzled: 16-byte chunk ch of page
                    // row r at (ch & 8) | ((ch & 7) ^ (r & 7)), so attention's
                    // ldmatrix reads of 8 consecutive rows are bank-conflict free
                    const int ch = d >> 3, r7 = int(pos & 7);
                    const int dk = (((ch & 8) | ((ch & 7) ^ r7)) << 3) | (d & 7);
                    const int64_t at = ((page * hkv + lr / hd) * 64 + pos % 64) * hd + dk;
                    u16p(isk ? J.b_t : J.o2_t)[at] = f2bf(v[c]);
                }
            }
        } else if (J.flags & VDC_JOB_SWIGLU) {
            // 128-row blocks = [64 gate rows | 64 up rows]: up rows go through shared memory
            float* scr = reinterpret_cast<float*>(S->x);
            if (row >= 64) {
#pragma unroll
                for (int c = 0; c < NH; ++c) scr[(c0 + c) * 64 + (row - 64)] = v[c];
            }
            sync();
            if (row < 64) {
                const int64_t orow = int64_t(J.r0 / 128) * 64 + row;
#pragma unroll
                for (int c = 0; c < NH; ++c) {
                    const int b = c0 + c;
                    if (b >= nb) continue;
                    const float gt = v[c], up = scr[(c0 + c) * 64 + row];
                    u16p(J.o_t)[int64_t(b) * M + orow] = f2bf(gt / (1.0f + expf(-gt)) * up);
                }
            }
        } else if (J.flags & VDC_JOB_RESID) {
            const uint16_t* res = u16p(J.a_t);
            const float wn = J.o3_t >= 0 ? bf_lo(u16p(J.w3_t)[rg]) : 0.f;
            float r[NH];
#pragma unroll
            for (int c = 0; c < NH; ++c) r[c] = c0 + c < nb ? bf_lo(ldcg_u16(res + int64_t(c0 + c) * M + rg)) : 0.f;
#pragma unroll
            for (int c = 0; c < NH; ++c) {
                const int b = c0 + c;
                const uint16_t xo = f2bf(v[c] + r[c]);
                if (J.ssq_t >= 0) {  // this warp's 32 rows: the sum of squares of request b's group
                    const float ss = warp_sum(b < nb ? bf_lo(xo) * bf_lo(xo) : 0.f);
                    if (lane == 0 && b < nb) f32p(J.ssq_t)[int64_t(rg >> 5) * J.npad + b] = ss;
                }
                if (b >= nb) continue;
                u16p(J.o_t)[int64_t(b) * M + rg] = xo;
                if (J.o3_t >= 0) u16p(J.o3_t)[int64_t(b) * M + rg] = f2bf(bf_lo(xo) * wn);
            }
        } else if (J.flags & VDC_JOB_SYM_OUT) {
            // TP partial sums (fp32) -> slot tp_rank of every rank's exchange buffer
            // (peer stores; out of line: keeps the other epilogues' registers)
            float vs[NH];
#pragma unroll
            for (int c = 0; c < NH; ++c) vs[c] = v[c];
            if (tdtype(J.o_t) == VDC_DTYPE_BF16)
                sym_store_rows<uint16_t>(P->sym + size_t(J.o_t) * VDC_RING_MAX_TP, P->tp_world, J.o_off, M, rg, c0, nb, NH, vs);
            else
                sym_store_rows<float>(P->sym + size_t(J.o_t) * VDC_RING_MAX_TP, P->tp_world, J.o_off, M, rg, c0, nb, NH, vs);
        } else {
            const bool obf = tdtype(J.o_t) == VDC_DTYPE_BF16;
#pragma unroll
            for (int c = 0; c < NH; ++c)
                if (c0 + c < nb) store_out(tptr(J.o_t), obf, int64_t(c0 + c) * M + rg, v[c]);
            if (J.flags & VDC_JOB_ARGMAX) {
                // per request: (max, first argmax) over this block's 128 rows,
                // merged into the SM's running best (S->am_*)
                float* scr = reinterpret_cast<float*>(S->x);  // [4 row quarters][npad] x (value, index)
#pragma unroll
                for (int c = 0; c < NH; ++c) {
                    const bool real_row = !(J.flags & VDC_JOB_TP_ARGMAX) || rg < J.am_valid;  // TP: padding rows never win
                    float bv = real_row ? v[c] : -INFINITY;
                    int bi = real_row ? rg + ((J.flags & VDC_JOB_TP_ARGMAX) ? J.am_base : 0) : 0x7fffffff;
#pragma unroll
                    for (int o = 16; o; o >>= 1)
                        am_merge(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
                    if (lane == 0) {
                        scr[2 * (q * npad + c0 + c)] = bv;
                        scr[2 * (q * npad + c0 + c) + 1] = __int_as_float(bi);
                    }
                }
                sync();
                if (int(ct) < npad) {
                    float bv = S->am_v[ct];
                    int bi = S->am_i[ct];
                    for (int qq = 0; qq < 4; ++qq)
                        am_merge(bv, bi, scr[2 * (qq * npad + int(ct))], __float_as_int(scr[2 * (qq * npad + int(ct)) + 1]));
                    S->am_v[ct] = bv;
                    S->am_i[ct] = bi;
                }
            }
        }
        (void)npad;
        return true;
    }

    // batched greedy sampling: the SM's last lm_head piece posts the SM's
    // per-request best (slot J.req); the last SM to arrive reduces the slots
    // per request (warp per request) and writes the tokens
    __device__ void post_argmax_batched(const vdc_job& J) {
        const int npad = J.npad, nb = J.nb;
        float* slot = reinterpret_cast<float*>(tptr(J.b_t)) + size_t(J.req) * npad * 2;
        sync();
        if (int(ct) < npad) {
            slot[2 * ct] = S->am_v[ct];
            slot[2 * ct + 1] = __int_as_float(S->am_i[ct]);
        }
        sync();
        if (ct == 0) {
            uint32_t old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&P->counters[J.am_ctr]) : "memory");
            S->flag = (old + 1u == uint32_t(J.am_need) * ep) ? 1 : 0;
        }
        sync();
        if (!S->flag) return;
        const float* all = reinterpret_cast<const float*>(tptr(J.b_t));
        const bool tpx = J.flags & VDC_JOB_TP_ARGMAX;
        if (tpx) {
            // vocab-parallel: this rank's best per request -> every rank (one post
            // of nb pairs), then each request's W posts reduced in rank order
            for (int b = int(w); b < nb; b += CW) {
                float bv = -INFINITY;
                int bi = 0x7fffffff;
                for (int s2 = int(lane); s2 < J.am_need; s2 += 32)
                    am_merge(bv, bi, ldcg_f32(all + (size_t(s2) * npad + b) * 2), __float_as_int(ldcg_f32(all + (size_t(s2) * npad + b) * 2 + 1)));
#pragma unroll
                for (int o = 16; o; o >>= 1) am_merge(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
                if (lane == 0) {
                    S->am_v[b] = bv;
                    S->am_i[b] = bi;
                }
            }
            sync();
            if (ct == 0) {
                post_sym_pairs(J.am_sym, nb, S->am_v, S->am_i);
                S->flag = wait_sym(J.am_sym, P->tp_world) ? 1 : 0;
            }
            sync();
            if (!S->flag) {
                ok = false;
                publish(J.o2_t);
                return;
            }
        }
        const float* xs = tpx ? reinterpret_cast<const float*>(sym_base(J.am_sym, P->tp_rank) + VDC_SYM_HEADER_BYTES) : nullptr;
        for (int b = int(w); b < nb; b += CW) {
            float bv = -INFINITY;
            int bi = 0x7fffffff;
            if (tpx) {
                if (int(lane) < int(P->tp_world)) {
                    bv = ldcg_f32(xs + (size_t(lane) * nb + b) * 2);
                    bi = __float_as_int(ldcg_f32(xs + (size_t(lane) * nb + b) * 2 + 1));
                }
            } else {
                for (int s2 = int(lane); s2 < J.am_need; s2 += 32)
                    am_merge(bv, bi, ldcg_f32(all + (size_t(s2) * npad + b) * 2), __float_as_int(ldcg_f32(all + (size_t(s2) * npad + b) * 2 + 1)));
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) am_merge(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
            if (lane == 0) {
                reinterpret_cast<int64_t*>(tptr(J.o2_t))[b] = int64_t(bi);
                if (J.flags & VDC_JOB_FEEDBACK) {  // next launch: request b's token at its next position
                    int64_t* st = const_cast<int64_t*>(P->step);
                    st[3 * b] = int64_t(bi);
                    st[3 * b + 1] += 1;
                    st[3 * b + 2] += 1;
                }
            }
        }
        publish(J.o2_t);
    }

    // ELEMWISE (batched): embedding rows of requests [r0, r1) -> x, and the
    // normalised-weight copy x * w3 the first layer's qkv GEMM reads
    __device__ void embed_rows(const vdc_job& J) {
        const int d = J.k, nch = d / 8;
        const uint4* tab = reinterpret_cast<const uint4*>(tptr(J.x_t));
        const uint4* wv = reinterpret_cast<const uint4*>(tptr(J.w3_t));
        uint4* xo = reinterpret_cast<uint4*>(tptr(J.o_t));
        uint4* xn = reinterpret_cast<uint4*>(tptr(J.o3_t));
        for (int i = int(ct); i < (J.r1 - J.r0) * nch; i += NCT) {
            const int b = J.r0 + i / nch, c = i % nch;
            const int64_t tok = S->btok[b];
            const uint4 u = __ldg(tab + tok * nch + c), g = __ldg(wv + c);
            xo[int64_t(b) * nch + c] = u;
            uint4 o;
            o.x = pack2(bf_lo(u.x) * bf_lo(g.x), bf_hi(u.x) * bf_hi(g.x));
            o.y = pack2(bf_lo(u.y) * bf_lo(g.y), bf_hi(u.y) * bf_hi(g.y));
            o.z = pack2(bf_lo(u.z) * bf_lo(g.z), bf_hi(u.z) * bf_hi(g.z));
            o.w = pack2(bf_lo(u.w) * bf_lo(g.w), bf_hi(u.w) * bf_hi(g.w));
            xn[int64_t(b) * nch + c] = o;
            if (J.ssq_t >= 0) {  // sum of squares of each 32-element group (4 chunks = 4 consecutive lanes)
                float ss = dot16<true>(u, u);
                const uint32_t m = __activemask();
                ss += __shfl_xor_sync(m, ss, 1);
                ss += __shfl_xor_sync(m, ss, 2);
                if ((c & 3) == 0) f32p(J.ssq_t)[int64_t(c >> 2) * J.npad + b] = ss;
            }
        }
        fence_proxy_async_global();
        sync();
        if (ct == 0) {
            red_release_add(ctr(J.o_t), 1u);
            red_release_add(ctr(J.o3_t), 1u);
        }
    }

    // ------------------------------------------------------ ATTN_DECODE
    // Split-KV q-len-1 attention of one kv head (G q heads) over pages
    // [r0, r1), fused with the split combine.
    //  * page i = ring tiles (K, V) at global indices kt + 2i, kt + 2i + 1,
    //    processed by warp pair i mod 4 (rows split in halves, each warp
    //    keeps its own online softmax). The job's tiles (<= ring depth) were
    //    issued after every earlier tile was released, so any warp may wait
    //    on their slots' next phase; each warp of the pair hands one slot back.
    //  * scores: a lane owns a row (q staged in shared memory in the cache
    //    dtype, chunks rotated per lane: conflict free); P.V: lanes own head
    //    dim slices. The appended K/V row was produced in this launch by the
    //    qkv µop, so it is patched into the slots from global.
    //  * the 8 warp states are merged per head in shared memory and written
    //    as this split's partial; the last split of the kv head to arrive
    //    (per-head arrival counter) merges all partials in split order and
    //    publishes the head's attention output (reference finalize,
    //    handlers.cpp:155-168).
    // One warp's 32 rows of a KV page on the tensor cores (mma.sync m16n8k16,
    // bf16 -> fp32), K and V rows swizzled (kv_swz): conflict-free ldmatrix.
    //  S = Q K^T: M = 16 q heads (rows >= G zero), N = 8 keys per n-tile, K = 16 dims;
    //    K rows are the B operand as stored (ldmatrix).
    //  online softmax in the log2 domain on the S fragments (lane (g, t) holds
    //    head g, keys 8 nt + 2t, +1); masked keys (past the context) get p = 0.
    //  O^T += V^T P^T: M = 16 dims, N = 8 heads, K = 16 keys; V rows through
    //    ldmatrix.trans, P^T straight from the S fragments (same lane layout),
    //    P split hi + mid + lo into three bf16 MMAs (24 significant bits, so the
    //    products are fp32 P x bf16 V up to fp32 accumulation order).
    template <int G>
    __device__ __forceinline__ void attn_page_mma(uint32_t kb, uint32_t vb, int nvalid, float sl2, uint32_t qs,
                                                  float (&mo)[8][4], float& mm, float& ml) const {
        const uint32_t i7 = lane & 7u, mi = lane >> 3;
        const int g = int(lane >> 2), t = int(lane & 3u);
        // q A fragments (rows = heads) by ldmatrix from the staged q (swizzled
        // like the KV rows); rows >= G read 16 zero bytes after the staged q
        const bool qrow = int(i7) < G;
        const uint32_t qa = qrow ? qs + i7 * 256u : qs + uint32_t(G) * 256u;
        float sc[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) sc[nt][e] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 8; ks += 2) {
            uint32_t q[4];  // a0, a2 of k-steps ks and ks + 1 (heads x dims 16 ks .. 16 ks + 31)
            ldsm_x4(qa + (qrow ? kv_swz(uint32_t(2 * ks) + mi, i7) * 16u : 0u), q);
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                uint32_t b[4];  // dims 16 ks .. 16 ks + 31 of keys 8 nt .. 8 nt + 7
                ldsm_x4(kb + (uint32_t(8 * nt) + i7) * 256u + kv_swz(uint32_t(2 * ks) + mi, i7) * 16u, b);
                mma_bf16(sc[nt], q[0], 0u, q[1], 0u, b[0], b[1]);
                mma_bf16(sc[nt], q[2], 0u, q[3], 0u, b[2], b[3]);
            }
        }
        float mx = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int key = 8 * nt + 2 * t + e;
                const float v = (g < G && key < nvalid) ? sc[nt][e] * sl2 : -INFINITY;
                sc[nt][e] = v;
                mx = fmaxf(mx, v);
            }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float mn = fmaxf(mm, mx);
        const float corr = mn == -INFINITY ? 1.f : exp2f(mm - mn);
        float ls = 0.f;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float p = sc[nt][e] == -INFINITY ? 0.f : exp2f(sc[nt][e] - mn);
                sc[nt][e] = p;
                ls += p;
            }
        ml = ml * corr + ls;
        mm = mn;
        // O^T columns of this lane are heads 2t, 2t + 1: their corrections sit on lanes 8t, 8t + 4
        const float ca = __shfl_sync(0xffffffffu, corr, 8 * t), cb = __shfl_sync(0xffffffffu, corr, 8 * t + 4);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            mo[mt][0] *= ca;
            mo[mt][1] *= cb;
            mo[mt][2] *= ca;
            mo[mt][3] *= cb;
        }
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            // P = hi + mid + lo in bf16 (24 significant bits: fp32 P)
            uint32_t ph[2], pm[2], pl[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float x0 = sc[2 * kk + u][0], x1 = sc[2 * kk + u][1];
                ph[u] = pack2(x0, x1);
                const float r0 = x0 - bf_lo(ph[u]), r1 = x1 - bf_hi(ph[u]);
                pm[u] = pack2(r0, r1);
                pl[u] = pack2(r0 - bf_lo(pm[u]), r1 - bf_hi(pm[u]));
            }
            const uint32_t row = uint32_t(16 * kk) + (mi >> 1) * 8u + i7;
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                uint32_t a[4];  // V^T: dims 16 mt .. 16 mt + 15 x keys 16 kk .. 16 kk + 15
                ldsm_x4_t(vb + row * 256u + kv_swz(uint32_t(2 * mt) + (mi & 1u), i7) * 16u, a);
                mma_bf16(mo[mt], a[0], a[1], a[2], a[3], pl[0], pl[1]);  // smallest terms first
                mma_bf16(mo[mt], a[0], a[1], a[2], a[3], pm[0], pm[1]);
                mma_bf16(mo[mt], a[0], a[1], a[2], a[3], ph[0], ph[1]);
            }
        }
    }

    // merge round of the split-KV attention: warp hh < HPR merges the 8 warp
    // states of head h0 + hh from the scratch (warp order) into the split's
    // partial (o[HD], m, l)
    template <int DPL, int HD, int HPR>
    __device__ void merge_round(float* part, const float* scr, int h0) const {
        constexpr int SST = HD + 2;
        if (int(w) < HPR) {
            const int h = h0 + int(w);
            const float* base = scr + size_t(w) * CW * SST;
            float M = -INFINITY;
            for (int q2 = 0; q2 < CW; ++q2) M = fmaxf(M, base[q2 * SST]);
            float L = 0.f, O[DPL];
#pragma unroll
            for (int d = 0; d < DPL; ++d) O[d] = 0.f;
            for (int q2 = 0; q2 < CW; ++q2) {
                const float* t = base + q2 * SST;
                if (t[0] == -INFINITY) continue;
                const float f = expf(t[0] - M);
                L = fmaf(t[1], f, L);
#pragma unroll
                for (int d = 0; d < DPL; ++d) O[d] = fmaf(t[2 + lane * DPL + d], f, O[d]);
            }
            float* out = part + h * (HD + 2);
#pragma unroll
            for (int d = 0; d < DPL; ++d) out[lane * DPL + d] = O[d];
            if (lane == 0) {
                out[HD] = M;
                out[HD + 1] = L;
            }
        }
    }

    __device__ void astamp(int ev) {
        if (P->tile_trace && sm == (P->debug >> 8) && ct == 0) P->tile_trace[60000 + 8 * (n_attn & 7) + ev] = now_ns();
    }
    // QKN: Qwen3 QK-norm instance (separate, so the other instances carry no
    // call to the double-precision norm/rotary helper)
    template <bool BF, int DPL, int G, bool QKN = false>
    __device__ void attn(const vdc_job& J) {
        constexpr int EB = BF ? 2 : 4;
        astamp(0);
        constexpr int HD = 32 * DPL;
        constexpr int NCH = HD * EB / 16;  // 16-byte chunks per K/V row
        if (!wait_ready(J.x_t, J.x_need, J.a_t, J.a_need, J.b_t, J.b_need)) {
            ok = false;
            return;
        }
        astamp(1);
        const int PR = J.tile_rows;
        const uint32_t rowb = uint32_t(HD * EB);
        // batched programs: per-request position / context, paged pools, and
        // pages mapped to warp pairs by ring slot (slot s -> pair (s % 8) / 2,
        // K on even slots: a leading pad tile aligns the job), so every slot
        // keeps a single consumer pair and jobs may span more than the ring
        const bool batched = BATCHED && (J.flags & VDC_JOB_BATCH);
        const int64_t pos = batched ? S->bpos[J.req] : S->sstep[1];
        const int64_t ctx = batched ? S->bctx[J.req] : S->sstep[2];
        if (batched && J.lead_pad) {
            const uint32_t s0 = kt % R;
            if ((s0 & uint32_t(CW - 1)) == w) {
                if (!wait_full(s0, (kt / R) & 1u)) ok = false;  // aborted: carry on (uniform control flow)
                release(s0);
            }
            kt += 1;
        }
        const int rows_w = PR / 2;  // rows per warp (<= 32: one per lane)
        // bf16 head-dim-128 caches (K and V page rows swizzled: batched pools and
        // VDC_JOB_KVSWZ single-request caches): scores and P.V on the tensor
        // cores (attn_page_mma); the fp32 geometry: CUDA-core path
        constexpr bool MMA = BF && DPL == 4;
        const bool swz = batched || (J.flags & VDC_JOB_KVSWZ);
        if (MMA && !swz) {  // ring bf16 head-dim-128 caches are always swizzled (decode_graph.cpp)
            if (ct == 0) fire(6, 0x2A00u | uint32_t(sm));
            ok = false;
        }
        // q of the group -> shared memory in the cache dtype, same 16-byte chunk
        // layout as a K row: the rotated chunk reads of the score loop hit 8
        // consecutive chunks per phase (bank-conflict free)
        xk_t = -2;  // the staged-x buffer holds q (and the merge scratch) now
        const uint32_t qs = smem_addr(S->x);
        {
            const uint4* qb = reinterpret_cast<const uint4*>(tptr(J.x_t) + size_t(J.x_off) * EB);
            uint4* qd = S->x;
            if constexpr (BF && DPL == 4 && QKN) {  // Qwen3: per-head RMSNorm of q, then the rotary (warp per head)
                // rotary table of this job's position (q and the appended k row share it)
                for (int d2 = int(ct); d2 < HD / 2; d2 += NCT) {
                    const double ang = double(pos) * pow(double(J.theta), -double(2 * d2) / double(HD));
                    S->rope_cs[d2] = float(cos(ang));
                    S->rope_sn[d2] = float(sin(ang));
                }
                rope_hd = 0;  // the GEMV's cached table is overwritten
                sync();
                const float2 cs0 = make_float2(S->rope_cs[2 * lane], S->rope_sn[2 * lane]);
                const float2 cs1 = make_float2(S->rope_cs[2 * lane + 1], S->rope_sn[2 * lane + 1]);
                const uint2 wv = *reinterpret_cast<const uint2*>(tptr(J.out_row0) + lane * 8);
                for (int h = int(w); h < G; h += CW) {
                    const uint2 u = ldcg64(reinterpret_cast<const char*>(qb) + h * HD * 2 + lane * 8);
                    const uint2 o = qk_norm_rope4(u, wv, J.head_dim, J.eps, cs0, cs1);
                    if constexpr (MMA) {  // bf16 rows [head][dim], chunks swizzled like KV rows (ldmatrix A fragments)
                        *reinterpret_cast<uint2*>(reinterpret_cast<char*>(qd) + h * HD * 2 +
                                                  kv_swz(lane >> 1, uint32_t(h) & 7u) * 16 + (lane & 1u) * 8) = o;
                    } else {
                        // lane's dims 4 lane .. 4 lane + 3 = chunk lane / 2, half lane % 2
                        qd[(h * 2 + int(lane & 1u)) * NCH + int(lane >> 1)] =
                            make_uint4(__float_as_uint(bf_lo(o.x)), __float_as_uint(bf_hi(o.x)), __float_as_uint(bf_lo(o.y)),
                                       __float_as_uint(bf_hi(o.y)));
                    }
                }
            } else if constexpr (MMA) {  // bf16 rows [head][dim], chunks swizzled like KV rows (ldmatrix A fragments)
                for (int i = int(ct); i < G * NCH; i += NCT)
                    qd[(i / NCH) * NCH + int(kv_swz(uint32_t(i % NCH), uint32_t(i / NCH) & 7u))] = ldcg128(qb + i);
            } else if constexpr (BF) {
                // bf16 caches: q staged as fp32 in split halves, [head][half][chunk]
                // x 4 floats (dims 8c..8c+3 | 8c+4..8c+7), so the score loop's
                // packed-fp32 FMAs read q without unpacking (conflict-free)
                for (int i = int(ct); i < G * NCH; i += NCT) {
                    const uint4 u = ldcg128(qb + i);
                    const int h = i / NCH, c = i % NCH;
                    qd[(h * 2) * NCH + c] = make_uint4(__float_as_uint(bf_lo(u.x)), __float_as_uint(bf_hi(u.x)),
                                                       __float_as_uint(bf_lo(u.y)), __float_as_uint(bf_hi(u.y)));
                    qd[(h * 2 + 1) * NCH + c] = make_uint4(__float_as_uint(bf_lo(u.z)), __float_as_uint(bf_hi(u.z)),
                                                           __float_as_uint(bf_lo(u.w)), __float_as_uint(bf_hi(u.w)));
                }
            } else {
                for (int i = int(ct); i < G * NCH; i += NCT) qd[i] = ldcg128(qb + i);
            }
            if constexpr (MMA) {
                if (ct == 0) qd[G * NCH] = make_uint4(0u, 0u, 0u, 0u);  // the zero rows of the q fragments
            }
        }
        sync();
        astamp(2);
        float m[G], l[G], o[G][DPL];
#pragma unroll
        for (int h = 0; h < G; ++h) {
            m[h] = -INFINITY;
            l[h] = 0.f;
#pragma unroll
            for (int d = 0; d < DPL; ++d) o[h][d] = 0.f;
        }
        // tensor-core state: q A fragments (head lane / 4), O^T accumulators
        // (dims x heads), running max (log2 domain) and per-lane partial sum
        constexpr int NMT = HD / 16;
        float mo[NMT][4], mm = -INFINITY, ml = 0.f;
        if constexpr (MMA) {
#pragma unroll
            for (int mt = 0; mt < NMT; ++mt)
#pragma unroll
                for (int e = 0; e < 4; ++e) mo[mt][e] = 0.f;
        }
        const uint32_t npages = uint32_t(J.r1 - J.r0), ntiles = 2u * npages;
        for (uint32_t i = 0; i < npages; ++i) {
            const uint32_t gk = kt + 2u * i;
            const uint32_t sk = gk % R, pk = (gk / R) & 1u, sv = (gk + 1u) % R, pv = ((gk + 1u) / R) & 1u;
            // page i -> warp pair i mod 4 (balanced over the 8 warps); the
            // job's tiles (<= ring depth) were issued after every earlier
            // tile was released, so any warp may wait on their slots
            // single-request programs: page i -> pair i % 4; batched programs on
            // an 8-slot ring: pair (sk % 8) / 2 (one consumer pair per slot)
            const uint32_t pair = batched ? ((sk & uint32_t(CW - 1)) >> 1) : i % uint32_t(CW / 2);
            if ((w >> 1) != pair) continue;
            const int half = int(w & 1u);
            const int my_row0 = half * rows_w;
            if (!wait_full(sk, pk) || !wait_full(sv, pv)) ok = false;  // aborted: garbage pages, same barriers
            const bool ttr = P->tile_trace && sm == (P->debug >> 8) && gk < P->tile_trace_cap && lane == 0;
            if (ttr) P->tile_trace[3 * (gk + half) + 1] = now_ns();
            const uint32_t kb = ring + sk * SLOT + uint32_t(my_row0) * rowb, vb = ring + sv * SLOT + uint32_t(my_row0) * rowb;
            const int64_t prow0 = int64_t(J.r0 + int(i)) * PR + my_row0;  // global row of this warp's first row
            if (batched && (J.flags & VDC_JOB_PREFILL)) {
                // prefill chunk: every row appended in this launch (request 0's
                // position .. this row's position) comes from global
                const int64_t lo = max(prow0, int64_t(S->bpos[0])), hi = min(prow0 + int64_t(rows_w), ctx);
                for (int64_t rr = lo; rr < hi; ++rr) {
                    const size_t crow =
                        size_t(ldstep(P->step + (J.ptab + int64_t(J.req) * J.maxp + rr / PR))) * size_t(J.cache_rows) + size_t(rr % PR);
                    const char* kn = tptr(J.a_t) + (size_t(J.a_off) + crow * HD) * EB;
                    const char* vn = tptr(J.b_t) + (size_t(J.b_off) + crow * HD) * EB;
                    for (int c = int(lane); c < 2 * NCH; c += 32) {
                        const bool isk = c < NCH;
                        const int cc = isk ? c : c - NCH;
                        const uint4 v = ldcg128(reinterpret_cast<const uint4*>(isk ? kn : vn) + cc);
                        const uint32_t dst = (isk ? kb : vb) + uint32_t(rr - prow0) * rowb + uint32_t(cc) * 16u;
                        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
                    }
                }
                if (lo < hi) {
                    fence_proxy_async_smem();
                    __syncwarp();
                }
            }
            const bool fresh = pos >= prow0 && pos < prow0 + rows_w && !(batched && (J.flags & VDC_JOB_PREFILL));
            if (fresh) {
                // the appended row was produced in this launch (after the page's
                // bulk copy may have been issued): patch it into the slots
                const int r = int(pos - prow0);
                // cache row of the appended position: (hkv, T, hd) cache, or
                // page pool (pages, hkv * 64, hd) through the page table
                const size_t crow = batched ? size_t(ldstep(P->step + (J.ptab + int64_t(J.req) * J.maxp + pos / PR))) * size_t(J.cache_rows) +
                                                  size_t(pos % PR)
                                            : size_t(pos);
                const char* kn = tptr(J.a_t) + (size_t(J.a_off) + crow * HD) * EB;
                const char* vn = tptr(J.b_t) + (size_t(J.b_off) + crow * HD) * EB;
                constexpr bool qkn = BF && DPL == 4 && QKN;
                if constexpr (qkn) {  // QK-norm + rotary of the appended k row, written back to the cache
                    // the lane's 4 stored dims; batched pools hold K rows swizzled
                    const int pc = int(lane >> 1);
                    const int lc = swz ? ((pc & 8) | ((pc & 7) ^ int(pos & 7))) : pc;
                    const int dbase = lc * 8 + int(lane & 1u) * 4;
                    const uint2 u = ldcg64(kn + lane * 8);
                    const uint2 wv = *reinterpret_cast<const uint2*>(tptr(J.block) + dbase * 2);
                    const uint2 o = qk_norm_rope4(u, wv, J.head_dim, J.eps, make_float2(S->rope_cs[dbase / 2], S->rope_sn[dbase / 2]),
                                                  make_float2(S->rope_cs[dbase / 2 + 1], S->rope_sn[dbase / 2 + 1]));
                    *reinterpret_cast<uint2*>(const_cast<char*>(kn) + lane * 8) = o;
                    asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(kb + uint32_t(r) * rowb + lane * 8u), "r"(o.x), "r"(o.y) : "memory");
                }
                for (int c = int(lane); c < 2 * NCH; c += 32) {
                    const bool isk = c < NCH;
                    if (isk && qkn) continue;
                    const int cc = isk ? c : c - NCH;
                    const uint4 v = ldcg128(reinterpret_cast<const uint4*>(isk ? kn : vn) + cc);
                    const uint32_t dst = (isk ? kb : vb) + uint32_t(r) * rowb + uint32_t(cc) * 16u;
                    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
                }
                fence_proxy_async_smem();  // these generic writes precede the slot's next bulk refill
                __syncwarp();
            }
            if constexpr (MMA) {
                const int nvalid = int(ctx - prow0 < 0 ? 0 : (ctx - prow0 < int64_t(rows_w) ? ctx - prow0 : int64_t(rows_w)));
                if (nvalid > 0) {
                    if (nvalid < 32) {
                        // rows past the context: zero V (P is 0 there, 0 x NaN is not), scores masked
                        for (int idx = int(lane); idx < (32 - nvalid) * NCH; idx += 32) {
                            const uint32_t dst = vb + uint32_t(nvalid + idx / NCH) * rowb + uint32_t(idx % NCH) * 16u;
                            asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(dst), "r"(0u) : "memory");
                        }
                        fence_proxy_async_smem();
                        __syncwarp();
                    }
                    attn_page_mma<G>(kb, vb, nvalid, J.scale * 1.4426950408889634f, qs, mo, mm, ml);
                }
            } else {
                // ---- scores: lane = row; chunks rotated by lane (conflict-free K reads)
                const bool valid = int(lane) < rows_w && prow0 + int(lane) < ctx;
                float s[G];
    #pragma unroll
                for (int h = 0; h < G; ++h) s[h] = 0.f;
                if (int(lane) < rows_w) {
                    const uint32_t krow = kb + lane * rowb;
                    if constexpr (BF) {  // packed fp32 FMAs (FFMA2): even / odd dims in the two halves
                        float2 acc[G];
    #pragma unroll
                        for (int h = 0; h < G; ++h) acc[h] = make_float2(0.f, 0.f);
    #pragma unroll 4
                        for (int c = 0; c < NCH; ++c) {
                            // single-request caches: chunk order rotated per lane; batched
                            // pools: K rows pre-swizzled, so every lane reads logical chunk c
                            // (q loads are broadcasts) from its row's physical chunk
                            const int cc = batched ? c : (c + int(lane)) & (NCH - 1);
                            const int kc = batched ? ((c & 8) | ((c & 7) ^ int(lane & 7u))) : cc;
                            const uint4 kv = lds128(krow + uint32_t(kc) * 16u);
                            const float2 k01 = make_float2(bf_lo(kv.x), bf_hi(kv.x)), k23 = make_float2(bf_lo(kv.y), bf_hi(kv.y));
                            const float2 k45 = make_float2(bf_lo(kv.z), bf_hi(kv.z)), k67 = make_float2(bf_lo(kv.w), bf_hi(kv.w));
    #pragma unroll
                            for (int h = 0; h < G; ++h) {
                                const uint4 qa = lds128(qs + uint32_t((h * 2) * NCH + cc) * 16u);
                                const uint4 qb2 = lds128(qs + uint32_t((h * 2 + 1) * NCH + cc) * 16u);
                                acc[h] = __ffma2_rn(k01, make_float2(__uint_as_float(qa.x), __uint_as_float(qa.y)), acc[h]);
                                acc[h] = __ffma2_rn(k23, make_float2(__uint_as_float(qa.z), __uint_as_float(qa.w)), acc[h]);
                                acc[h] = __ffma2_rn(k45, make_float2(__uint_as_float(qb2.x), __uint_as_float(qb2.y)), acc[h]);
                                acc[h] = __ffma2_rn(k67, make_float2(__uint_as_float(qb2.z), __uint_as_float(qb2.w)), acc[h]);
                            }
                        }
    #pragma unroll
                        for (int h = 0; h < G; ++h) s[h] = acc[h].x + acc[h].y;
                    } else {
    #pragma unroll 4
                        for (int c = 0; c < NCH; ++c) {
                            const int cc = (c + int(lane)) & (NCH - 1);
                            const uint4 kv = lds128(krow + uint32_t(cc) * 16u);
    #pragma unroll
                            for (int h = 0; h < G; ++h) {
                                const uint4 qv = lds128(qs + uint32_t(h * NCH + cc) * 16u);
                                s[h] += dot16<BF>(qv, kv);
                            }
                        }
                    }
                }
                // ---- online softmax per head over the warp's rows
                float p[G];
    #pragma unroll
                for (int h = 0; h < G; ++h) {
                    const float sc = valid ? s[h] * J.scale : -INFINITY;
                    const float mx = warp_max(sc);
                    const float mn = fmaxf(m[h], mx);
                    const float corr = (mn == -INFINITY) ? 1.f : (m[h] == -INFINITY ? 0.f : expf(m[h] - mn));
                    p[h] = valid ? expf(sc - mn) : 0.f;
                    l[h] = l[h] * corr + warp_sum(p[h]);
                    m[h] = mn;
    #pragma unroll
                    for (int d = 0; d < DPL; ++d) o[h][d] *= corr;
                }
                // ---- o += p V (lanes own DPL dims)
                const int nrow = int(ctx - prow0 < int64_t(rows_w) ? ctx - prow0 : int64_t(rows_w));
    #pragma unroll 4
                for (int r = 0; r < nrow; ++r) {
                    float vv[DPL];
                    load_row<BF, DPL>(vb + uint32_t(r) * rowb + lane * uint32_t(DPL * EB), vv);
    #pragma unroll
                    for (int h = 0; h < G; ++h) {
                        const float ph = __shfl_sync(0xffffffffu, p[h], r);
                        if constexpr (DPL % 2 == 0) {  // packed fp32 FMAs over dim pairs
    #pragma unroll
                            for (int d = 0; d < DPL; d += 2) {
                                const float2 a = __ffma2_rn(make_float2(vv[d], vv[d + 1]), make_float2(ph, ph),
                                                            make_float2(o[h][d], o[h][d + 1]));
                                o[h][d] = a.x;
                                o[h][d + 1] = a.y;
                            }
                        } else {
    #pragma unroll
                            for (int d = 0; d < DPL; ++d) o[h][d] = fmaf(ph, vv[d], o[h][d]);
                        }
                    }
                }
            }
            // both warps of the pair are done with K and V: each returns its slot
            if (ttr) P->tile_trace[3 * (gk + half) + 2] = now_ns();
            named_bar(2 + int(pair), 64);  // the pair is done with K and V
            release(half ? sv : sk);
        }
        kt += ntiles;
        sync();
        astamp(3);
        // ---- merge the 8 warp states per head (warp order), write this split's partial;
        // scratch = the staged-x buffer, up to 4 heads per round (2 barriers per round)
        float* part = reinterpret_cast<float*>(tptr(J.o_t)) + J.o_off;
        float* scr = reinterpret_cast<float*>(S->x) + G * HD;  // after the staged q
        constexpr int HPR = G < 4 ? G : 4;
        constexpr int SST = HD + 2;
        if constexpr (MMA) {
            // lane (g, t): m, l of head g; O^T of heads 2t, 2t + 1 at dims 16 mt + g (+ 8)
            ml += __shfl_xor_sync(0xffffffffu, ml, 1);
            ml += __shfl_xor_sync(0xffffffffu, ml, 2);
            const int g = int(lane >> 2), t = int(lane & 3u);
#pragma unroll
            for (int h0 = 0; h0 < G; h0 += HPR) {
                if (t == 0 && g >= h0 && g < h0 + HPR) {
                    float* st = scr + (size_t(g - h0) * CW + w) * SST;
                    st[0] = mm == -INFINITY ? -INFINITY : mm * 0.69314718055994531f;  // natural-log domain
                    st[1] = ml;
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int h = 2 * t + e;
                    if (h >= h0 && h < h0 + HPR && h < G) {
                        float* st = scr + (size_t(h - h0) * CW + w) * SST + 2;
#pragma unroll
                        for (int mt = 0; mt < NMT; ++mt) {
                            st[16 * mt + g] = mo[mt][e];
                            st[16 * mt + 8 + g] = mo[mt][2 + e];
                        }
                    }
                }
                sync();
                merge_round<DPL, HD, HPR>(part, scr, h0);
                sync();
            }
        } else {
#pragma unroll
        for (int h0 = 0; h0 < G; h0 += HPR) {
#pragma unroll
            for (int hh = 0; hh < HPR; ++hh) {
                float* st = scr + (size_t(hh) * CW + w) * SST;
                if (lane == 0) {
                    st[0] = m[h0 + hh];
                    st[1] = l[h0 + hh];
                }
#pragma unroll
                for (int d = 0; d < DPL; ++d) st[2 + lane * DPL + d] = o[h0 + hh][d];
            }
            sync();
            merge_round<DPL, HD, HPR>(part, scr, h0);
            sync();
        }
        }
        astamp(4);
        // ---- arrival: the last split of this kv head combines (the
        // reference-form ATTN_COMBINE, fused: saves one dependency hop)
        if (ct == 0) {
            uint32_t old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&P->counters[J.arrive_ctr]) : "memory");
            S->flag = (old + 1u == uint32_t(J.arrive_need) * ep) ? 1 : 0;
        }
        sync();
        astamp(5);
        if (S->flag) {
            if (int(w) < G) combine_head<DPL, HD>(J, int(w));
            publish(J.o2_t);
        }
        astamp(6);
        ++n_attn;
    }

    // ATTN_COMBINE as a separate µop (waits for all splits of a kv head on its
    // arrival counter); ring programs fuse it into ATTN_DECODE by default
    __device__ void combine(const vdc_job& J) {
        if (!wait_ready(J.arrive_ctr, J.arrive_need, -1, 0, -1, 0)) {
            ok = false;
            return;
        }
        if (int(w) < J.group) {
            if (J.head_dim == 128)
                combine_head<4, 128>(J, int(w));
            else
                combine_head<2, 64>(J, int(w));
        }
        publish(J.o2_t);
    }

    template <bool BF, int DPL>
    __device__ __forceinline__ void load_row(uint32_t a, float (&v)[DPL]) const {
        if constexpr (BF) {
            if constexpr (DPL == 4) {
                const uint2 u = lds64(a);
                v[0] = bf_lo(u.x); v[1] = bf_hi(u.x); v[2] = bf_lo(u.y); v[3] = bf_hi(u.y);
            } else if constexpr (DPL == 8) {
                const uint4 u = lds128(a);
                v[0] = bf_lo(u.x); v[1] = bf_hi(u.x); v[2] = bf_lo(u.y); v[3] = bf_hi(u.y);
                v[4] = bf_lo(u.z); v[5] = bf_hi(u.z); v[6] = bf_lo(u.w); v[7] = bf_hi(u.w);
            } else {
#pragma unroll
                for (int d = 0; d < DPL; ++d) {
                    unsigned short x;
                    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(x) : "r"(a + uint32_t(d) * 2u));
                    v[d] = __uint_as_float(uint32_t(x) << 16);
                }
            }
        } else {
            if constexpr (DPL == 2) {
                const uint2 u = lds64(a);
                v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y);
            } else if constexpr (DPL == 4) {
                const uint4 u = lds128(a);
                v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y); v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
            } else {
#pragma unroll
                for (int d = 0; d < DPL; ++d) {
                    float x;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a + uint32_t(d) * 4u));
                    v[d] = x;
                }
            }
        }
    }

    // butterfly reduce-scatter: 32 values per lane -> lane l holds the warp
    // sum of value l
    __device__ __forceinline__ float reduce_scatter32(float (&v)[32]) const {
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const bool up = lane & uint32_t(step);
#pragma unroll
            for (int i = 0; i < step; ++i) {
                const float send = up ? v[i] : v[i + step], keep = up ? v[i + step] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, step);
            }
        }
        return v[0];
    }

    // merge all split partials of q head h of this kv head (warp-wide): the
    // splits' (m, l) are loaded in parallel across lanes, then o in split order
    template <int DPL, int HD>
    __device__ void combine_head(const vdc_job& J, int h) {
        const int S2 = J.arrive_need, G = J.group;
        // split 0 of this kv head's partials
        const float* part0 = reinterpret_cast<const float*>(tptr(J.o_t)) + (J.o_off - J.split * G * (HD + 2));
        float M = -INFINITY, L = 0.f, O[DPL];
#pragma unroll
        for (int d = 0; d < DPL; ++d) O[d] = 0.f;
        constexpr int SB = 16;  // splits per block: every load of a block is issued before any is used
        for (int s0 = 0; s0 < S2; s0 += SB) {
            const int n = min(SB, S2 - s0);
            float ms = -INFINITY, ls = 0.f;
            if (int(lane) < n) {
                const float* pr = part0 + size_t((s0 + int(lane)) * G + h) * (HD + 2);
                ms = ldcg_f32(pr + HD);
                ls = ldcg_f32(pr + HD + 1);
            }
            float4 ov[SB];
#pragma unroll
            for (int k2 = 0; k2 < SB; ++k2) {
                const int kk = min(k2, n - 1);
                const float* pr = part0 + size_t((s0 + kk) * G + h) * (HD + 2) + lane * DPL;
                if constexpr (DPL == 4) {
                    ov[k2] = make_float4(ldcg_f32(pr), ldcg_f32(pr + 1), ldcg_f32(pr + 2), ldcg_f32(pr + 3));
                } else {
                    ov[k2] = make_float4(ldcg_f32(pr), DPL > 1 ? ldcg_f32(pr + 1) : 0.f, 0.f, 0.f);
                }
            }
            const bool ok_s = ms != -INFINITY && ls > 0.f;
            const float bm = warp_max(ok_s ? ms : -INFINITY);
            const float mn = fmaxf(M, bm);
            if (mn == -INFINITY) continue;
            const float a = M == -INFINITY ? 0.f : expf(M - mn);
            const float ws = ok_s ? expf(ms - mn) : 0.f;
            L = L * a + warp_sum(ls * ws);
#pragma unroll
            for (int d = 0; d < DPL; ++d) O[d] *= a;
#pragma unroll
            for (int k2 = 0; k2 < SB; ++k2) {
                const float wk = __shfl_sync(0xffffffffu, ws, k2);
                if (k2 < n) {
                    const float v[4] = {ov[k2].x, ov[k2].y, ov[k2].z, ov[k2].w};
#pragma unroll
                    for (int d = 0; d < DPL; ++d) O[d] = fmaf(v[d], wk, O[d]);
                }
            }
            M = mn;
        }
        char* ob = tptr(J.o2_t);
        const bool obf = tdtype(J.o2_t) == VDC_DTYPE_BF16;
#pragma unroll
        for (int d = 0; d < DPL; ++d)
            store_out(ob, obf, int64_t(J.o2_off) + h * HD + lane * DPL + d, L > 0.f ? O[d] / L : 0.f);
    }

    // ------------------------------------------- ALLREDUCE_ADD (tensor parallel)
    // rows [r0, r1): x_next = residual + sum over the W rank slots of the
    // symmetric partial buffer, in rank order (same result on every rank)
    __device__ void allreduce(const vdc_job& J) {
        if constexpr (BATCHED) {
            if (J.flags & VDC_JOB_BATCH) {
                allreduce_batched(J);
                return;
            }
        }
        if (!wait_ready(J.x_t, J.x_need, J.a_t, J.a_need, -1, 0)) {
            ok = false;
            return;
        }
        const char* part = tptr(J.x_t);
        const bool pbf = tdtype(J.x_t) == VDC_DTYPE_BF16;  // bf16 exchange partials
        const char* ab = tptr(J.a_t);
        const bool abf = tdtype(J.a_t) == VDC_DTYPE_BF16;
        const int64_t aoff = J.a_off + (J.flags & VDC_JOB_TOKEN_AUX ? token() * int64_t(J.cache_rows) : 0);
        char* ob = tptr(J.o_t);
        const bool obf = tdtype(J.o_t) == VDC_DTYPE_BF16;
        for (int r = J.r0 + int(ct); r < J.r1; r += NCT) {
            float acc[VDC_RING_MAX_TP];
#pragma unroll
            for (int q = 0; q < VDC_RING_MAX_TP; ++q)
                acc[q] = q >= J.group ? 0.f
                         : pbf ? bf_lo(ldcg_u16(reinterpret_cast<const uint16_t*>(part) + int64_t(q) * J.k + r))
                               : ldcg_f32(reinterpret_cast<const float*>(part) + int64_t(q) * J.k + r);
            float v = 0.f;
#pragma unroll
            for (int q = 0; q < VDC_RING_MAX_TP; ++q)
                if (q < J.group) v += acc[q];
            v += abf ? bf_lo(ldcg_u16(reinterpret_cast<const uint16_t*>(ab) + aoff + r))
                     : ldcg_f32(reinterpret_cast<const float*>(ab) + aoff + r);
            store_out(ob, obf, r, v);
        }
        publish(J.o_t);
    }

    // batched (npad, d) hidden states: x = residual + sum of the rank slots
    // (rank order), and the next RMSNorm's operand bf16(x * w)
    __device__ void allreduce_batched(const vdc_job& J) {
        if (!wait_ready(J.x_t, J.x_need, J.a_t, J.a_need, -1, 0)) {
            ok = false;
            return;
        }
        const char* part = tptr(J.x_t);
        const bool pbf = tdtype(J.x_t) == VDC_DTYPE_BF16;  // bf16 exchange partials
        const uint16_t* res = u16p(J.a_t);
        const uint16_t* wn = u16p(J.w3_t);
        const int64_t M = J.k, slot = int64_t(J.npad) * M;
        const int rows = J.r1 - J.r0;
        for (int i = int(ct); i < J.nb * rows; i += NCT) {
            const int b = i / rows, r = J.r0 + i % rows;
            const int64_t e = int64_t(b) * M + r;
            float v = 0.f;
            for (int qr = 0; qr < J.group; ++qr)
                v += pbf ? bf_lo(ldcg_u16(reinterpret_cast<const uint16_t*>(part) + qr * slot + e))
                         : ldcg_f32(reinterpret_cast<const float*>(part) + qr * slot + e);
            const uint16_t xo = f2bf(v + bf_lo(ldcg_u16(res + e)));
            u16p(J.o_t)[e] = xo;
            u16p(J.o3_t)[e] = f2bf(bf_lo(xo) * bf_lo(wn[r]));
        }
        fence_proxy_async_global();  // the next GEMM reads x * w with TMA
        sync();
        if (ct == 0) {
            red_release_add(ctr(J.o_t), 1u);
            red_release_add(ctr(J.o3_t), 1u);
        }
    }

    // ------------------------------------------- ELEMWISE copy (embedding row)
    __device__ void copy_row(const vdc_job& J) {
        const int32_t eb = P->descs[J.x_t].elem;
        int64_t off = J.x_off;
        if (J.flags & VDC_JOB_TOKEN_ROW) off += token() * J.k;
        const uint4* src = reinterpret_cast<const uint4*>(tptr(J.x_t) + off * eb);
        uint4* dst = reinterpret_cast<uint4*>(tptr(J.o_t) + int64_t(J.o_off) * eb);
        for (int c = int(ct); c < J.k * eb / 16; c += NCT) dst[c] = __ldg(src + c);
        publish(J.o_t);
    }
};

template <bool BATCHED, bool QKNORM>
__device__ __forceinline__ void vcc_role(const RingParams& P, Shared& S, char* ring) {
    Vcc<BATCHED, QKNORM> v;
    v.P = &P;
    v.S = &S;
    v.ring = smem_addr(ring);
    v.sm = blockIdx.x;
    v.ct = threadIdx.x;
    v.lane = threadIdx.x & 31;
    v.w = threadIdx.x >> 5;
    v.R = P.ring_slots;
    v.tmem = S.tmem_base;
    const uint32_t core = 2 * blockIdx.x + 1;
    const uint32_t w0 = P.core_off[core], n = P.core_off[core + 1] - w0;
    const long long t0 = clock64();
    uint32_t jobs = 0;
    // resident decode: n_epochs decode steps in this launch. Step e > 0 waits
    // (thread 0) until step e - 1 fed its token back (every SM has finished
    // step e - 1 by then: its lm_head jobs are each SM's last µops), then the
    // per-step caches are refreshed (rotary table, staged x, rms scales,
    // request positions / append pages)
    for (uint32_t e = 0; e < P.n_epochs; ++e) {
    v.ep = P.epoch + e;
    if (e > 0) {
        if (v.ct == 0) {
            const uint32_t* fb = &P.counters[P.fb_ctr];
            const uint32_t want = v.ep - 1u;
            const unsigned long long w0t = now_ns();
            for (uint32_t k = 1; int32_t(ld_relaxed(fb) - want) < 0; ++k) {
                if ((k & 255) == 0) {
                    if (v.aborted()) break;
                    if (P.watchdog_ns && now_ns() - w0t > P.watchdog_ns) {
                        v.fire(0, 0x60000u | e);
                        break;
                    }
                }
                __nanosleep(64);
            }
            fence_acquire_gpu();
        }
        // the sampler's running bests start over (single-request: per thread;
        // batched: the SM's per-request slots)
        v.am_v = -INFINITY;
        v.am_i = 0x7fffffff;
        if (BATCHED && v.ct < VDC_RING_MAX_BATCH) {
            S.am_v[v.ct] = -INFINITY;
            S.am_i[v.ct] = 0x7fffffff;
        }
        v.sync();
        v.xk_t = -2;
        v.rope_hd = 0;
        v.binv_t = -2;
    }
    // the step's scalars (constant within a step) -> shared memory, read once
    // here instead of an L2 round trip in every µop that needs them
    if constexpr (BATCHED) {  // per request: token, position, context, append page
        const int b = int(v.ct);
        if (b < VDC_RING_MAX_BATCH) {
            const int64_t pos = 3 * b + 1 < P.n_step ? ldstep(P.step + (3 * b + 1)) : 0;
            const int64_t lp = pos / 64, at = int64_t(P.ptab) + int64_t(b) * P.maxp + lp;
            S.bpos[b] = int32_t(pos);
            S.btok[b] = 3 * b < P.n_step ? int32_t(ldstep(P.step + 3 * b)) : 0;
            S.bctx[b] = 3 * b + 2 < P.n_step ? int32_t(ldstep(P.step + (3 * b + 2))) : 0;
            S.bpage[b] = (P.maxp > 0 && pos >= 0 && lp < P.maxp && at < P.n_step) ? int32_t(ldstep(P.step + (at))) : -1;
        }
    }
    if (v.ct < 3) S.sstep[v.ct] = int32_t(v.ct) < P.n_step ? ldstep(P.step + v.ct) : 0;
    v.sync();
    // the stream runs to its end even after an abort (every wait then returns
    // at once), so all compute warps reach the same barriers; only a
    // dispatch fault (uniform over the VCC) stops it early
    bool halt = false;
    for (uint32_t pc = 0; pc < n && !halt; ++pc) {
        const uint4 raw = __ldg(&P.words[w0 + pc]);
        const uint32_t op = raw.x & 0xff;
        if (op == OP_HALT) break;
        // batched programs read whole 256-byte operand blocks, single-request
        // programs the packed first halves (the only fields their µops use)
        const char* jb = BATCHED ? reinterpret_cast<const char*>(P.jobs) : P.jobs_core;
        const size_t js = BATCHED ? sizeof(vdc_job) : 128;
        if (pc + 1 < n) {  // the next µop's operand block -> L1 while this one runs
            const uint4 nx = __ldg(&P.words[w0 + pc + 1]);
            if ((nx.x & 0xff) != OP_HALT && v.ct * 128u < js)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(jb + size_t(nx.z) * js + 128 * v.ct));
        }
        // single-request µops: the 128-byte core of the block by value (all
        // fields requested in one round trip, kept in registers; measured
        // ~2% faster per token than field loads through a reference)
        vdc_job Jv;
        if constexpr (!BATCHED) {
            const uint4* src = reinterpret_cast<const uint4*>(jb + size_t(raw.z) * js);
#pragma unroll
            for (int i = 0; i < 8; ++i) reinterpret_cast<uint4*>(&Jv)[i] = __ldg(src + i);
        }
        const vdc_job& J = BATCHED ? *reinterpret_cast<const vdc_job*>(jb + size_t(raw.z) * js) : Jv;
        const bool bf = J.x_t >= 0 && v.tdtype(J.x_t) == VDC_DTYPE_BF16;
        const unsigned long long t_enter = P.trace ? now_ns() : 0;
        if (v.ct == 0) S.t_ready = 0;
        switch (op) {
            case OP_GEMV:
            case OP_RMS_GEMV:
            case OP_GEMV_ADD:
                if (bf) v.template gemv<true>(J); else v.template gemv<false>(J);
                break;
            case OP_ATTN_DECODE: {
                const bool kbf = v.tdtype(J.a_t) == VDC_DTYPE_BF16;
                const int dpl = J.head_dim / 32, G = J.group;
#define VDC_ATTN_CASE(B, D, GG) \
    if (kbf == B && dpl == D && G == GG) { v.template attn<B, D, GG>(J); break; }
#define VDC_ATTN_QKN_CASE(GG) \
    if (kbf && dpl == 4 && G == GG && (J.flags & VDC_JOB_QKNORM)) { v.template attn<true, 4, GG, true>(J); break; }
                if constexpr (QKNORM) {  // Qwen3 programs run their own kernel instance
                    VDC_ATTN_QKN_CASE(4)
                    VDC_ATTN_QKN_CASE(8)
                }
                if (J.flags & VDC_JOB_QKNORM) {  // QK-norm geometry without an instance: fail loudly
                    if (v.ct == 0) v.fire(6, (core << 16) | pc);
                    halt = true;
                    break;
                }
#undef VDC_ATTN_QKN_CASE
                VDC_ATTN_CASE(true, 4, 4)
                VDC_ATTN_CASE(true, 4, 8)
                VDC_ATTN_CASE(false, 2, 1)
#undef VDC_ATTN_CASE
                if (v.ct == 0) v.fire(6, (core << 16) | pc);  // unsupported head geometry
                halt = true;
                break;
            }
            case OP_ATTN_COMBINE: v.combine(J); break;
            case OP_ALLREDUCE_ADD: v.allreduce(J); break;
            case OP_BGEMM:
                if constexpr (BATCHED) {
                    v.bgemm(J);
                    break;
                }
                if (v.ct == 0) v.fire(4, (core << 16) | pc);
                halt = true;
                break;
            case OP_ELEMWISE:
                if constexpr (BATCHED) {
                    if (J.flags & VDC_JOB_BATCH) {
                        v.embed_rows(J);
                        break;
                    }
                }
                v.copy_row(J);
                break;
            default:
                if (v.ct == 0) v.fire(4, (core << 16) | pc);
                halt = true;
                break;
        }
        if (P.trace && v.ct == 0 && jobs < P.trace_cap) {
            unsigned long long* rec = P.trace + (size_t(core) * P.trace_cap + jobs) * 4;
            rec[0] = (static_cast<unsigned long long>(core) << 32) | pc;
            rec[1] = t_enter;
            rec[2] = S.t_ready ? S.t_ready : t_enter;
            rec[3] = now_ns();
        }
        ++jobs;
    }
    if constexpr (BATCHED) {  // resident steps of odd tile count end with the memory core's pad tile
        if (P.n_epochs > 1) {
            if (P.vtiles[blockIdx.x] & 1u) {
                const uint32_t s0 = v.kt % v.R;
                if ((s0 & uint32_t(CW - 1)) == v.w) {
                    if (!v.wait_full(s0, (v.kt / v.R) & 1u)) v.ok = false;
                    v.release(s0);
                }
                v.kt += 1;
            }
        }
    }
    }
    if (v.ct == 0) {
        SmStats& st = P.stats[blockIdx.x];
        st.wait[S_VCC_FULL] = S.vstat[v.VS_FULL];
        st.wait[S_VCC_DEP] = S.vstat[v.VS_DEP];
        st.wait[S_VCC_EPI] = S.vstat[v.VS_EPI];
        st.wait[S_VCC_TOTAL] = clock64() - t0;
        st.wait[S_NJOBS] = jobs;
        st.tiles_consumed = v.kt;  // ring tiles taken from (and handed back to) the memory core
        if constexpr (BATCHED) {
            st.wait[S_X_FULL] = S.vstat[v.VS_XF];
            st.wait[S_X_EMPTY] = S.vstat[v.VS_XE];
            st.wait[S_MMA_DONE] = S.vstat[v.VS_MMA];
            st.wait[S_BG_PRO] = S.vstat[v.VS_PRO];
        }
    }
}

// One LOAD word resolved to its global runs: `copies` runs of `run` bytes,
// `pitch` apart (whole-row tiles are a single run).
struct Tile {
    const char* src = nullptr;
    uint32_t copies = 0, run = 0, pitch = 0;
    bool bad = false, halt = false;
    bool empty = false;  // a KV page past the context (or unallocated): the slot completes without data
    __device__ uint32_t bytes() const { return copies * run; }
};

template <bool BATCHED>
__device__ __forceinline__ Tile resolve_load(const RingParams& P, uint4 raw) {
    Tile t;
    const uint32_t op = raw.x & 0xff;
    if (op == OP_HALT) {
        t.halt = true;
        return t;
    }
    if (op != OP_LOAD) {
        t.bad = true;
        return t;
    }
    const uint32_t b1 = (raw.x >> 8) & 0xff;
    const uint32_t kind = (b1 >> 4) & 3, rank = (b1 >> 6) + 1;
    const uint32_t ti = raw.z & 0xffff;
    const uint64_t pl = uint64_t(raw.z >> 16) | (uint64_t(raw.w) << 16);
    const DevDesc& d = P.descs[ti];
    if (kind != 2 || int32_t(rank) != d.grid_rank) {
        t.bad = true;
        return t;
    }
    const int64_t c0 = int64_t(pl & 0xfff), c1 = int64_t((pl >> 12) & 0xfff), c2 = int64_t((pl >> 24) & 0xfff);
    const uint32_t mode = (raw.y >> 24) & 0xfu;  // reg1 (ring_abi.h VDC_LOAD_*)
    if (mode == VDC_LOAD_PAGED) {
        // (request, logical page, kv head) -> physical page through the step
        // block's page table; pages past the request's context are not loaded
        if (!BATCHED || rank != 3 || c1 >= P.maxp) {
            t.bad = true;
            return t;
        }
        // (plain loads: the memory core resolves every KV tile, an L2 round trip
        // each would stall its issue loop; a later resident step only reads
        // them after the acquire at its token gate)
        const int64_t ctx = P.step[3 * c0 + 2];
        const int64_t page = P.step[P.ptab + c0 * P.maxp + c1];
        if (c1 * d.tile_rows >= ctx || page < 0) {
            t.empty = true;
            return t;
        }
        t.src = d.ptr + (page * d.lead_stride[0] + c2 * d.tile_rows * d.cols) * d.elem;
        t.copies = 1;
        t.run = uint32_t(d.tile_rows * d.cols * d.elem);
        t.bad = page >= d.grid[0] || c2 >= d.grid[1] || t.run > SLOT;
        return t;
    }
    if (mode == VDC_LOAD_CTX && c1 * d.tile_rows >= (P.n_step > VDC_STEP_CTX ? P.step[VDC_STEP_CTX] : 0)) {
        t.empty = true;  // single-request cache page past the step's context
        return t;
    }
    if (BATCHED && mode == VDC_LOAD_PACKED) {  // reg1 = 1: packed, pre-swizzled 16 KB weight tile (one bulk copy)
        t.src = d.ptr + (c0 * d.grid[1] + c1) * (d.tile_rows * d.tile_cols * d.elem);
        t.copies = 1;
        t.run = uint32_t(d.tile_rows * d.tile_cols * d.elem);
        t.pitch = 0;
        t.bad = t.run != SLOT || rank != 2 || c0 >= d.grid[0] || c1 >= d.grid[1];
        return t;
    }
    const int64_t rt = rank == 3 ? c1 : c0, ctile = rank == 3 ? c2 : c1, plane = rank == 3 ? c0 : 0;
    const int64_t off = plane * d.lead_stride[0] + rt * d.tile_rows * d.cols + ctile * d.tile_cols;
    const int64_t rows_at = min(d.tile_rows, d.rows - rt * d.tile_rows);
    t.src = d.ptr + off * d.elem;
    t.copies = d.tile_cols == d.cols ? 1u : uint32_t(rows_at);
    t.run = uint32_t((d.tile_cols == d.cols ? rows_at * d.cols : d.tile_cols) * d.elem);
    t.pitch = uint32_t(d.cols * d.elem);
    t.bad = t.bytes() == 0 || t.bytes() > SLOT || (reinterpret_cast<uintptr_t>(t.src) & 15) || (t.run & 15) ||
            (t.copies > 1 && (t.pitch & 15));
    return t;
}

// one folded run entry (ring_abi.h vdc_run) as the memory core caches it:
// the two raw 16-byte halves (fields decoded per tile: the memory warpgroup
// runs on few registers) and 1 / n_in
struct Run {
    uint4 b, m;
    float rcp;
};
__device__ __forceinline__ uint32_t run_count(const Run& r) { return r.m.x & 0xffffffu; }
__device__ __forceinline__ Run load_run(const RingParams& P, uint32_t i) {
    const uint4* rp = reinterpret_cast<const uint4*>(P.runs + i);
    Run r;
    r.b = __ldg(rp);
    r.m = __ldg(rp + 1);
    r.rcp = 1.f / float(r.m.y & 0xfffu);
    return r;
}
// tile k of a run as a LOAD word (the host reference is host/ring_fold.cpp
// expand_run): the division by n_in is a multiply by its reciprocal with a
// one-step correction
__device__ __forceinline__ uint4 expand_run(const Run& r, uint32_t k) {
    const uint32_t n_alt = r.m.x >> 24, n_in = r.m.y & 0xfffu;
    const uint32_t a = n_alt == 2u ? (k & 1u) : 0u, j = n_alt == 2u ? (k >> 1) : k;
    uint32_t o = __float2uint_rz(float(j) * r.rcp);
    if (o * n_in > j) --o;
    if ((o + 1u) * n_in <= j) ++o;
    const int32_t i = int32_t(j - o * n_in), oo = int32_t(o);
    auto s8 = [](uint32_t v, int q) { return int32_t(int8_t(uint8_t((v >> (8 * q)) & 0xffu))); };
    const uint64_t pl = uint64_t(r.b.z >> 16) | (uint64_t(r.b.w) << 16);
    const int32_t c0 = int32_t(pl & 0xfff) + i * s8(r.m.z, 0) + oo * s8(r.m.z, 3);
    const int32_t c1 = int32_t((pl >> 12) & 0xfff) + i * s8(r.m.z, 1) + oo * s8(r.m.w, 0);
    const int32_t c2 = int32_t((pl >> 24) & 0xfff) + i * s8(r.m.z, 2) + oo * s8(r.m.w, 1);
    const uint64_t np = uint64_t(c0 & 0xfff) | (uint64_t(c1 & 0xfff) << 12) | (uint64_t(c2 & 0xfff) << 24) | (pl & ~0xfffffffffull);
    const uint32_t ti = a ? (r.m.y >> 12) : (r.b.z & 0xffffu);
    return make_uint4(r.b.x, r.b.y, ti | (uint32_t(np & 0xffffu) << 16), uint32_t(np >> 16));
}

__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

// The memory core: eight issuing lanes, one per compute warp. Ring tile g
// is consumed by compute warp g % 8 and lives in slot (g % 8) + 8 * ((g / 8)
// % S) (S = ring_slots / 8), so lane w walks tiles w, w + 8, w + 16, ... of
// the stream and refills only warp w's slots: each (issuing lane, compute
// warp) pair is an independent pipeline and a slow tile never blocks the
// refill of another warp's slot. Lanes poll their own slot's `empty`
// barrier (non-blocking test_wait) in one converged loop and issue the bulk
// copy of their next tile as soon as it is free.
// The stream is folded (ring_abi.h vdc_run): each lane keeps a cursor (folded
// word, offset in it) that it advances by R tiles per issue.
// RESIDENT: launches of several decode steps (vdc_set_steps) walk the stream
// once per step with token-gated KV pages; single-step launches run the
// instance without that bookkeeping on the issue path
template <bool BATCHED, bool RESIDENT>
__device__ __forceinline__ void vmc_loop(const RingParams& P, Shared& S, char* ring) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t core = 2 * blockIdx.x;
    const uint32_t R = P.ring_slots;
    // the folded stream of this SM and its length in tiles
    const uint32_t v0 = P.voff[blockIdx.x], fn = P.voff[blockIdx.x + 1] - v0;  // run entries
    const uint32_t ntiles = P.vtiles[blockIdx.x];
    // resident decode: the stream is walked once per step; tile g is word
    // g % ntiles of step g / ntiles. Weight tiles stream across the step
    // boundary; a KV page of step e > 0 is resolved (context, page table) and
    // loaded only after step e - 1 fed its token back: by then every append of
    // step e - 1 is in memory and the step block holds step e's positions.
    // batched programs place every attention page's K tile on an even ring
    // index (lead pads); a step of odd length would flip that parity for the
    // next step, so resident steps are padded to even length with one
    // data-less tile (the compute core consumes it at the step's end)
    const uint32_t ept = RESIDENT ? ntiles + (BATCHED ? (ntiles & 1u) : 0u) : ntiles;
    const uint32_t total = RESIDENT ? ept * P.n_epochs : ntiles;
    // (word index, step) of the lane's tile g, advanced incrementally (no
    // per-tile division on the issue path)
    uint32_t wi = lane, ei = 0;
    while (ept && wi >= ept) {
        wi -= ept;
        ++ei;
    }
    uint32_t gate_ep = 0;  // resident: the latest step whose token gate this lane saw open
    auto kv_gated = [&](uint4 r) {
        if constexpr (!RESIDENT) return false;
        const uint32_t mode = (r.y >> 24) & 0xfu;
        // once the lane saw the step's gate open, its later KV tiles of the step
        // are resolved ahead like any other tile
        return ei > gate_ep && wi < ntiles && (mode == VDC_LOAD_CTX || mode == VDC_LOAD_PAGED);
    };
    // cursor: run entry fw (cached in run), tile fk of it; the next entry is
    // prefetched into L1 whenever the cursor enters one
    uint32_t fw = 0, fk = 0;
    Run run{};
    auto enter = [&](uint32_t i) {
        fw = i;
        if (i < fn) {
            run = load_run(P, v0 + i);
            if (i + 1 < fn) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.runs + v0 + i + 1));
        } else {
            run.m.x = 0xffffffu;  // past the end: a run no cursor leaves
        }
    };
    auto advance = [&](uint32_t d) {
        fk += d;
        while (fw < fn && fk >= run_count(run)) {
            fk -= run_count(run);
            enter(fw + 1);
        }
    };
    auto seek = [&](uint32_t t) {
        fk = 0;
        enter(0);
        advance(t);
    };
    seek(wi);
    auto word = [&]() {  // the LOAD word of the lane's tile (the step pad: a data-less tile)
        if (wi >= ntiles) return make_uint4(0, 0, 0, 0);
        return expand_run(run, fk);
    };
    auto resolve = [&](uint4 r) {
        if (RESIDENT && wi >= ntiles) {
            Tile t;
            t.empty = true;
            return t;
        }
        return resolve_load<BATCHED>(P, r);
    };
    const bool issuer = lane < R;
    uint32_t g = lane, m = 0;  // lane s issues tiles s, s + R, s + 2R, ... into slot s
    unsigned long long st_empty = 0, bytes = 0, uops = 0;
    const long long t_start = clock64();
    uint4 raw = issuer && g < total ? word() : make_uint4(0, 0, 0, 0);
    // the lane's next tile is resolved as soon as its word arrives (descriptor,
    // page table and context loads overlap the slot polling), not when the
    // slot frees up
    bool deferred = issuer && g < total && kv_gated(raw);
    Tile cur = issuer && g < total && !deferred ? resolve(raw) : Tile{};
    long long idle_since = 0;
    unsigned long long t_idle = 0;
    bool real_last = false;  // this lane's last issue was a bulk copy (bytes may still be landing)
    for (;;) {
        const bool pending = issuer && g < total;
        if (!__any_sync(0xffffffffu, pending)) break;
        bool ready = false;
        uint32_t slot = 0;
        if (pending) {
            slot = lane;
            ready = m == 0 || mbar_test(&S.empty[slot], (m - 1u) & 1u);
            if (RESIDENT && ready && deferred) {  // KV page of a later step: wait for the previous step's token
                // (polled until it opens, once per step and lane: the lane's later
                // KV tiles of the step follow the acquire in program order and are
                // resolved ahead like any other tile, see kv_gated; a counter load
                // per tile stalled the whole issue warp)
                if (int32_t(ld_relaxed(&P.counters[P.fb_ctr]) - (P.epoch + ei - 1u)) >= 0) {
                    fence_acquire_gpu();
                    fence_proxy_async_global();  // the appends were generic stores; the copy is async-proxy
                    gate_ep = ei;
                    cur = resolve(raw);
                    deferred = false;
                } else {
                    ready = false;
                }
            }
        }
        if (ready) {
            const Tile t = cur;
            if (t.bad || t.halt) {
                if (atomicCAS(&P.status->abort, 0, 2) == 0) {
                    P.status->fault_code = 5;
                    P.status->fault_info = g;
                    P.status->stalled_core[0] = core;
                }
            } else if (t.empty) {
                mbar_arrive(&S.full[slot]);  // no data: the consumer masks the page
                ++uops;
                real_last = false;
            } else {
                real_last = true;
                if (P.tile_trace && blockIdx.x == (P.debug >> 8) && g < P.tile_trace_cap) P.tile_trace[3 * g] = now_ns();
                mbar_expect_tx(&S.full[slot], t.bytes());
                char* dst = ring + size_t(slot) * SLOT;
                for (uint32_t q = 0; q < t.copies; ++q)
                    bulk_g2s(dst + q * t.run, t.src + size_t(q) * t.pitch, t.run, &S.full[slot]);
                bytes += t.bytes();
                ++uops;
            }
            g += R;
            ++m;
            wi += R;
            bool wrapped = false;
            if constexpr (RESIDENT) {
                while (ept && wi >= ept) {
                    wi -= ept;
                    ++ei;
                    wrapped = true;
                }
            }
            if (wrapped)
                seek(wi);
            else
                advance(R);
            raw = g < total ? word() : make_uint4(0, 0, 0, 0);
            deferred = g < total && kv_gated(raw);
            if (g < total && !deferred) cur = resolve(raw);
        }
        if (!__any_sync(0xffffffffu, ready)) {
            const long long now = clock64();
            if (!idle_since) {
                idle_since = now;
                t_idle = now_ns();
            }
            __nanosleep(32);
            if (*reinterpret_cast<volatile int32_t*>(&P.status->abort)) break;
            if (P.watchdog_ns && now_ns() - t_idle > P.watchdog_ns) {
                if (lane == 0 && atomicCAS(&P.status->abort, 0, 1) == 0) {
                    P.status->stalled_core[0] = core;
                    P.status->n_stalled = 1;
                    P.status->fault_info = 0x30000u | (g & 0xffffu);
                }
                break;
            }
        } else if (idle_since) {
            st_empty += clock64() - idle_since;
            idle_since = 0;
        }
    }
    if (idle_since) st_empty += clock64() - idle_since;
    if (*reinterpret_cast<volatile int32_t*>(&P.status->abort) && issuer && m > 0 && real_last) {
        // aborted launch: the consumers may not wait for this lane's last
        // copy; let its bytes land before the CTA can exit (bounded)
        const unsigned long long t0 = now_ns();
        while (!mbar_test(&S.full[lane], (m - 1u) & 1u) && now_ns() - t0 < 100000000ull) __nanosleep(64);
    }
    for (int o = 16; o; o >>= 1) {
        bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
        uops += __shfl_xor_sync(0xffffffffu, uops, o);
    }
    if (lane == 0) {
        SmStats& st = P.stats[blockIdx.x];
        st.wait[S_VMC_EMPTY] = st_empty;
        st.wait[S_VMC_TOTAL] = clock64() - t_start;
        st.bytes_loaded = bytes;
        st.uops = uops;
        st.bytes_stored = 0;
        st.tiles_issued = uops;
    }
}

template <bool BATCHED>
__device__ void vmc_role(const RingParams& P, Shared& S, char* ring) {
    if (P.n_epochs > 1)
        vmc_loop<BATCHED, true>(P, S, ring);
    else
        vmc_loop<BATCHED, false>(P, S, ring);
}

// register split per SM sub-partition (16384 registers = 512 per lane slot,
// one warp of each warpgroup): 2 x 224 (compute) + 56 (memory warpgroup);
// (the full 512 is not available: an inc to 2 x 224 + 64 never returns)
constexpr uint32_t kVccRegs = 224, kVmcRegs = 56;
static_assert(2 * kVccRegs + kVmcRegs < 512 && kRingThreads == 3 * 128 && NCT == 256);

template <bool BATCHED, bool QKNORM>
__global__ void __launch_bounds__(kRingThreads, 1) ring_kernel(const __grid_constant__ RingParams P) {
    extern __shared__ __align__(1024) char smem[];
    char* ring = smem;
    Shared& S = *reinterpret_cast<Shared*>(smem + size_t(P.ring_slots) * SLOT);
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < P.ring_slots; ++i) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], 1);
        }
        if (BATCHED) {
            for (int i = 0; i < NXMAX; ++i) {
                mbar_init(&S.xfull[i], 1);
                mbar_init(&S.xempty[i], 1);
            }
            mbar_init(&S.mma_bar, CW);
            mbar_init(&S.lbar, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 8) S.vstat[threadIdx.x] = 0;
    if (threadIdx.x == 0) S.t_ready = 0;
    if (BATCHED && threadIdx.x < VDC_RING_MAX_BATCH) {
        S.am_v[threadIdx.x] = -INFINITY;
        S.am_i[threadIdx.x] = 0x7fffffff;
    }
    if (BATCHED && threadIdx.x < 32) {  // TMEM accumulator of the batched GEMM µops (one CTA per SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&S.tmem_base)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (BATCHED) tc_fence_before();
    __syncthreads();
    if (BATCHED) tc_fence_after();
    if (threadIdx.x < NCT) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kVccRegs));
        vcc_role<BATCHED, QKNORM>(P, S, ring);
        if (BATCHED) {
            tc_fence_before();
            named_bar(BAR_VCC, NCT);
            tc_fence_after();
            if (threadIdx.x < 32)
                asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(S.tmem_base), "r"(TMEM_COLS));
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kVmcRegs));
        if (threadIdx.x < NCT + 32) vmc_role<BATCHED>(P, S, ring);  // warps 9..11 only donate registers
    }
}

}  // namespace ring

size_t ring_smem_bytes(uint32_t ring_slots, bool batched) { return ring::smem_bytes(ring_slots, batched); }
// four instances: single-request / batched x without / with Qwen3 QK-norm,
// so each program type keeps its own register allocation
const void* ring_kernel_entry(bool batched, bool qknorm) {
    if (batched)
        return qknorm ? reinterpret_cast<const void*>(&ring::ring_kernel<true, true>)
                      : reinterpret_cast<const void*>(&ring::ring_kernel<true, false>);
    return qknorm ? reinterpret_cast<const void*>(&ring::ring_kernel<false, true>)
                  : reinterpret_cast<const void*>(&ring::ring_kernel<false, false>);
}

}  // namespace vdc_dev
