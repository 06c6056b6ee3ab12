/* Shared constants of the decode µop extension: step-block slots, handler
 * parameter layouts and imm encodings. Included by the host lowering (C++),
 * the sm_100a engine (CUDA) and the CPU oracle (test infrastructure), so all
 * three agree on the meaning of every extension word.
 *
 * Step block: int64 scalars bound per launch (vdc_set_step); SET_ACC_MEM
 * reads them: acc[reg0] = step[imm & 0xff] * max(1, imm >> 8).
 */
#ifndef UOPSIM_DECODE_ABI_H
#define UOPSIM_DECODE_ABI_H

#define VDC_STEP_TOKEN 0 /* token id fed to the embedding row gather      */
#define VDC_STEP_POS 1   /* position of the token being decoded          */
#define VDC_STEP_CTX 2   /* valid KV length after the append (= pos + 1) */
#define VDC_STEP_MAX 8

/* GEMV / RMS_GEMV / GEMV_ADD: imm = (param_base << 8) | variant.
 * acc[reg0] = position (rope).                                           */
#define VDC_GEMV_ROPE 0x1   /* interleaved-pair rotary on rows < rope_rows */
#define VDC_GEMV_SWIGLU 0x2 /* W rows in blocks [gate x B/2 | up x B/2]    */
#define VDC_GEMV_P_EPS 0
#define VDC_GEMV_P_THETA 1
#define VDC_GEMV_P_HEAD_DIM 2
#define VDC_GEMV_P_ROPE_ROWS 3
#define VDC_GEMV_P_SWIGLU_BLOCK 4
#define VDC_GEMV_NPARAMS 5

/* ATTN_DECODE: imm = param_base << 8; acc[reg0] = ctx (valid KV rows).
 * prologue: q group (G*D); groups: (K page, V page) tiles of `page_rows`
 * rows of the (Hkv, T, D) caches; result: G x (D + 2) fp32 partial
 * [o_unnormalised(D), running max m, running sum l] per q head.            */
#define VDC_ATTN_P_SCALE 0
#define VDC_ATTN_P_HEAD_DIM 1
#define VDC_ATTN_P_GROUP 2
#define VDC_ATTN_P_PAGE_ROWS 3
#define VDC_ATTN_NPARAMS 4

/* ATTN_COMBINE: imm = param_base << 8; groups: S partial tiles.           */
#define VDC_COMB_P_HEAD_DIM 0
#define VDC_COMB_P_GROUP 1
#define VDC_COMB_NPARAMS 2

#endif
