/* Ring-mode µop programs: the operand block of a compute µop and the
 * constants shared by the host lowering (ring_lower.cpp), the sm_100a ring
 * engine (device/ring_engine.cu) and the tests.
 *
 * A ring-mode program is an ordinary LoweredProgram (per-core streams of
 * 16-byte isa words, CoreId order sm<i>.vmc, sm<i>.vcc0) with the decoupled
 * execution model of the paper (§3-4) specialised for decode:
 *
 *   sm<i>.vmc  : LOAD [send] size=1 words only. Each LOAD moves one tile
 *                (contiguous, <= VDC_RING_SLOT_BYTES) into the next slot of
 *                the SM's shared-memory ring with one cp.async.bulk; the
 *                slot's `full` mbarrier is the m2c message. The memory core
 *                never waits on data dependencies (weights and KV pages of
 *                earlier steps are immutable during a launch), so it
 *                prefetches across operator boundaries, bounded only by the
 *                ring's `empty` mbarriers (slot release = the c2m FREE).
 *   sm<i>.vcc0 : compute µops (GEMV / RMS_GEMV / GEMV_ADD / ATTN_DECODE /
 *                ATTN_COMBINE / ELEMWISE) with size = ring tiles consumed and
 *                imm = index of a vdc_job operand block. Activation operands
 *                (the LOAD_WAIT of the reference-form decode program) are
 *                read by the compute core itself after its readiness counter
 *                reaches the target; results are stored by the compute core
 *                and published with a release increment of the output
 *                tensor's counter (the STORE_DEP of the reference form).
 *
 * Readiness counters are per storage tensor and monotonic across launches:
 * launch e (1-based) waits for counter >= need * e.
 */
#ifndef UOPSIM_RING_ABI_H
#define UOPSIM_RING_ABI_H

#include <stdint.h>

#define VDC_RING_SLOT_BYTES 16384
#define VDC_RING_MAX_SLOTS 12  /* 12 x 16 KB ring + 28 KB staged x + scratch <= 227 KB */
#define VDC_RING_COMPUTE_WARPS 8
#define VDC_RING_MAX_JOB_ROWS 256  /* output rows per GEMV job (smem partials) */
#define VDC_RING_MAX_COL_TILES 4   /* column tiles per W row group (one partial plane each) */
#define VDC_RING_MAX_TILE_ROWS 8   /* W rows per ring tile */
#define VDC_RING_MAX_K 14336       /* GEMV reduction length (bf16) staged in shared memory */

/* ATTN_DECODE in ring programs also performs the split-KV combine (the
 * reference-form ATTN_COMBINE): every split job writes its partial
 * (o, m, l per q head), increments the kv head's arrival counter, and the
 * last arriving job merges the partials and publishes the output. */

/* vdc_job.flags */
#define VDC_JOB_RMS 0x01        /* x <- bf16/f32(x * rsqrt(mean(x^2)+eps) * a) */
#define VDC_JOB_ROPE 0x02       /* interleaved-pair rotary on the output rows */
#define VDC_JOB_SWIGLU 0x04     /* W rows in blocks [gate x B/2 | up x B/2] */
#define VDC_JOB_RESID 0x08      /* out = a + W x */
#define VDC_JOB_KV_APPEND 0x10  /* output row r -> cache[(r/hd)*T + pos][r%hd] */
#define VDC_JOB_TOKEN_ROW 0x20  /* x offset += step[TOKEN] * k (embedding row) */
#define VDC_JOB_TOKEN_AUX 0x40  /* aux offset += step[TOKEN] * cache_rows (residual = embedding row) */
#define VDC_JOB_SYM_OUT 0x100   /* output rows go to every rank's slot `tp_rank` of a symmetric tensor */
#define VDC_JOB_SYM_IN 0x200    /* x is a symmetric tensor: readiness on its header counter (sys scope) */
#define VDC_RING_MAX_TP 8       /* tensor-parallel ranks */
#define VDC_SYM_HEADER_BYTES 128 /* symmetric buffer = header (u32 readiness counter) + data */
#define VDC_JOB_QKV 0x80        /* fused q|k|v rows: q -> o_t, k -> cache b_t, v -> cache o2_t;
                                   block = q rows, split = k (= v) rows; rotary on q and k */
#define VDC_JOB_ARGMAX 0x800     /* lm_head GEMV: greedy sampling fused into the logits epilogue: each
                                   job posts (max, argmax) of its rows to b_t[split]; the last of
                                   arrive_need jobs writes the token (int64) to o2_t */
#define VDC_JOB_QKNORM 0x1000    /* Qwen3 QK-norm. qkv µops store q and k un-rotated; ATTN_DECODE
                                   normalises q (and the appended k row, written back to the
                                   cache) per head with weights out_row0 (q) / block (k) and
                                   eps, then applies the rotary (theta) */
#define VDC_JOB_FEEDBACK 0x2000  /* with ARGMAX: the sampled token is fed back on the device: the step
                                   block's token becomes it and pos / ctx advance by one, so the
                                   next launch decodes the next position without the host */
#define VDC_JOB_PREFILL 0x4000  /* batched ATTN of a prefill chunk: the batch's rows are consecutive
                                   positions of one sequence sharing its pages; every row appended
                                   in this launch (from request 0's position on) is patched in */
#define VDC_JOB_KVSWZ 0x8000   /* single-request KV caches with swizzled page rows (VDC_DESC_KPAGE_SWZ):
                                   the qkv epilogue appends k / v rows swizzled and ATTN_DECODE reads
                                   them on the tensor cores (batched pools are always swizzled) */
#define VDC_JOB_TP_ARGMAX 0x10000 /* with ARGMAX under tensor parallelism (vocab-parallel lm_head): the
                                   rank's best (logit, global vocab index) per request is posted to
                                   slot tp_rank of every rank's symmetric exchange buffer and each
                                   rank reduces the W posts in rank order (ties -> lowest index), so
                                   all ranks sample the same token. Single-request jobs: group =
                                   exchange tensor, o2_off = the rank's first vocab row; batched:
                                   am_sym, am_base, am_valid (rows >= am_valid are vocab padding) */
#define VDC_JOB_BATCH 0x400     /* batched program (nb requests): per-request token / pos / ctx in
                                   the step block (3 int64 each), paged KV pools, page table at
                                   step[ptab + b * maxp + logical page] */

/* Batched programs (BGEMM and friends, layout.batch > 1):
 *  - activations are (npad, K) bf16 row-major, request b = row b; rows
 *    >= nb stay zero. npad in {16, 32, 64} is the tcgen05 MMA N.
 *  - weight tiles are 128 rows x 64 columns, stored packed and
 *    pre-swizzled (VDC_DESC_PACKED_SW128) and moved by one bulk copy each;
 *    activation chunks (npad x 64) are loaded by the compute core's MMA
 *    issuer with TMA tensor copies (128-byte swizzle, vdc_desc.tma = npad)
 *    after the readiness wait.
 *  - KV caches are page pools (pages, hkv * 64, hd): tile (page, head). */
#define VDC_RING_BGEMM_ROWS 128  /* output rows per BGEMM job (MMA M) */
/* vdc_desc.tma value of a weight stored as packed tiles: tile (rb, kt) of
 * 128 rows x 64 columns is 16 KB contiguous at ((rb * K/64) + kt) * 16 KB,
 * pre-swizzled (16-byte chunk c of row r at chunk c ^ (r % 8)), i.e. the
 * K-major 128-byte-swizzle operand layout of tcgen05.mma: one contiguous
 * bulk copy per ring tile (row-major 128 x 64 boxes would be 128 separate
 * 128-byte DRAM bursts per tile, ~half the HBM rate). */
#define VDC_DESC_PACKED_SW128 0x80000000u
/* vdc_desc.tma value of a batched K or V page pool (pages, hkv * 64, hd), and
 * of a single-request bf16 head-dim-128 ring cache (hkv, max_ctx, hd):
 * each page row's 16-byte chunks are stored swizzled, logical chunk c of page
 * row r at chunk (c & 8) | ((c & 7) ^ (r & 7)) (written that way by the qkv
 * epilogue; attention's ldmatrix reads of 8 consecutive rows, K for Q.K^T and
 * V transposed for P.V, are bank-conflict free). Hosts that import or export
 * row-major KV caches apply / undo this permutation (engine.py swizzle_k /
 * unswizzle_k). */
#define VDC_DESC_KPAGE_SWZ 0x40000000u
/* LOAD word reg1 (ring programs): how the memory core resolves a tile.
 *  1 VDC_LOAD_PACKED: packed 16 KB weight tile (VDC_DESC_PACKED_SW128).
 *  2 VDC_LOAD_PAGED: KV page of a page pool, coords (request b, logical page
 *    i, kv head h): physical page = step[ptab + b * maxp + i] (the program's
 *    page table); pages with i * 64 >= ctx_b, or unallocated entries (< 0),
 *    are not loaded (the slot completes empty; attention masks them).
 *  3 VDC_LOAD_CTX: KV page of a single-request cache, coords (h, i): not
 *    loaded when i * 64 >= the step's ctx. */
#define VDC_LOAD_PACKED 1
#define VDC_LOAD_PAGED 2
#define VDC_LOAD_CTX 3
#define VDC_RING_BGEMM_KT 64     /* reduction columns per weight tile (128-byte swizzle atom) */
#define VDC_RING_MAX_BATCH 64

typedef struct vdc_job {
    int32_t op;               /* isa opcode of the compute µop                */
    int32_t flags;            /* VDC_JOB_*                                    */
    int32_t r0, r1;           /* GEMV: W rows; ATTN: pages; COMBINE: r1 = splits */
    int32_t k;                /* GEMV reduction length; ATTN/COMBINE: head dim; copy: elements */
    int32_t tile_rows;        /* ring tile rows (GEMV W rows / KV page rows)  */
    int32_t tile_cols;        /* ring tile columns                            */
    int32_t x_t, x_off, x_need; /* input vector: tensor, element offset, readiness target */
    int32_t a_t, a_off, a_need; /* aux: rms weight / residual / K cache       */
    int32_t b_t, b_off, b_need; /* aux 2: V cache                              */
    int32_t o_t, o_off;       /* output tensor + element offset               */
    int32_t out_row0;         /* W row of output row 0 (region start)         */
    int32_t head_dim;         /* rope / attention head dim                    */
    int32_t group;            /* attention: q heads per kv head               */
    int32_t block;            /* swiglu block                                 */
    int32_t cache_rows;       /* KV cache rows per kv head (T)                */
    float eps, theta, scale;
    int32_t lead_pad;         /* ATTN: leading padding tiles (keeps K pages on even ring indices) */
    int32_t arrive_ctr;       /* ATTN: per-kv-head arrival counter (index into the counter array) */
    int32_t arrive_need;      /* ATTN: split jobs per kv head; the last to arrive combines */
    int32_t o2_t, o2_off;     /* ATTN: combined output (attention vector of the head's q heads) */
    int32_t split;            /* ATTN: split index of this job within its kv head;
                                 BGEMM: piece index within its row block */
    /* ---- batched programs (VDC_JOB_BATCH) ---- */
    int32_t kt0, kt1;         /* BGEMM: reduction tiles [kt0, kt1) of this piece (stream-K share) */
    int32_t nb, npad;         /* requests in the batch; MMA N (activation rows incl. padding) */
    int32_t x2_t, x2_need;    /* BGEMM + RMS: raw activations the per-request rms scale is taken from */
    int32_t o3_t, w3_t;       /* BGEMM + RESID: second output o3 = bf16(out * w3) (next RMSNorm's operand) */
    int32_t part_t, part_off; /* BGEMM stream-K: fp32 partial buffer, this piece's slot (npad x 128 floats) */
    int32_t req;              /* ATTN / ELEMWISE: request index (first request of an embed job) */
    int32_t ptab, maxp;       /* page table: step-block offset and pages per request row */
    int32_t kvrows;           /* BGEMM + QKV: k (= v) rows */
    int32_t am_ctr, am_need;  /* BGEMM + ARGMAX: sampling arrival counter, SMs posting (slot = req) */
    int32_t am_sym, am_base;  /* BGEMM + TP_ARGMAX: exchange tensor, the rank's first vocab row */
    int32_t am_valid;         /* BGEMM + TP_ARGMAX: this rank's real vocab rows (the rest is padding) */
    int32_t ssq_t;            /* batched activations: sums of squares per 32-row group and request
                                 (f32 [d/32][npad]), written by x's producer (embedding, residual
                                 epilogue) and read by the RMS GEMM for its 1/rms (-1: none, the
                                 consumer sums x itself) */
    int32_t rsv[12];          /* pads the block to 256 bytes: the single-request fields stay in
                                 the first 128-byte line, the batched ones in the second */
} vdc_job;  /* 256 bytes */

/* Folded memory-core streams (the loop folding of PAPER.md:773 / fold.cpp on
 * the ring hot path). A ring program's memory-core stream is one LOAD word per
 * ring tile. At vdc_load_jobs the engine folds each SM's stream into a
 * sequence of vdc_run entries, every maximal regular stretch of tiles one
 * entry (a lone tile is a run of 1); the device expands them tile by tile.
 * Tile k of a run (k < count):
 *   a = k % n_alt, j = k / n_alt, i = j % n_in, o = j / n_in;
 *   tensor = a ? t_alt : the base word's tensor;
 *   coordinate c = base c + i * d_in[c] + o * d_out[c]   (c = 0, 1, 2);
 *   every other field is the base word's.
 * So a GEMV job (row blocks x column tiles, row-major) is one run, and an
 * attention job (K page, V page, K page, ...) is one run with n_alt = 2.
 * 32 bytes, self-contained: one load per run on the device. */
typedef struct vdc_run {
    uint32_t base[4];         /* the LOAD word of tile 0 */
    uint32_t count_alt;       /* tiles in the run (bits 0..23) | n_alt (1 or 2) << 24 */
    uint32_t nin_talt;        /* groups per inner line n_in (bits 0..11) | t_alt << 12 (tensor of odd tiles) */
    int8_t d_in[3], d_out[3]; /* coordinate steps per inner group / per outer line */
    uint16_t rsv;
} vdc_run;  /* 32 bytes */

#endif
