#pragma once
// Decode-layer graph builder (ext): a Llama/Qwen-style decoder expressed as
// an OperatorGraph of decode kinds, ready for generator::generate().
//
// Per layer l (B = 1, all vectors (M,1)):
//   L.qkv  rms_gemv  [L.wqkv, x.all, L.attn_norm] -> [L.q, L.kc.seg, L.vc.seg]
//          (RMSNorm fused, interleaved-pair RoPE on q/k rows, k/v rows appended
//           to the caches at the step position: the KV append)
//   L.attn attn_decode [L.q.grp, L.kc.page, L.vc.page] -> [L.part]  (split-KV, GQA)
//   L.comb attn_combine [L.part] -> [L.attn]
//   L.o    gemv_add  [L.wo, L.attn.all, x.blk] -> [L.x1]      (residual fused)
//   L.gu   rms_gemv  [L.wgu, L.x1.all, L.mlp_norm] -> [L.a]   (SwiGLU fused)
//   L.down gemv_add  [L.wd, L.a.all, L.x1.blk] -> [L.x2]
// plus `embed` (embed_row, token from the step block) and `head`
// (rms_gemv: final norm + lm_head -> fp32 logits).
// Weight layout conventions (part of the model definition, mirrored by the
// oracle): wqkv rows = [q heads | k heads | v heads]; wgu rows come in blocks
// of `gu_block` = [gate x gu_block/2 | up x gu_block/2].

#include <cstdint>
#include <string>
#include <vector>

#include "uopsim/workload.hpp"

namespace uopsim::decode {

struct ModelConfig {
    std::string name = "tiny";
    int layers = 2;
    int hidden = 256;
    int heads = 4;
    int kv_heads = 4;
    int head_dim = 64;
    int ffn = 512;
    int vocab = 512;
    float eps = 1e-5f;
    float theta = 10000.0f;
    workload::ElemType dtype = workload::ElemType::f32;
    bool scaled_init = false;  // (u-1)/2/sqrt(fan_in) weights instead of raw unit_float
    bool qk_norm = false;      // Qwen3: per-head RMSNorm of q and k (weights L.q_norm / L.k_norm) before the rotary
};

struct LayoutConfig {
    int ctx_pages = 1;       // KV pages covered by the program (ctx <= ctx_pages * page_rows)
    int max_ctx = 64;        // cache capacity T (>= ctx_pages * page_rows)
    int page_rows = 64;
    int pages_per_job = 1;   // split-KV granularity
    int job_rows = 16;       // output rows per GEMV job (divides head_dim)
    int head_job_rows = 64;  // output rows per lm_head job
    int gu_block = 16;       // swiglu interleave block (== job_rows for the gu node)
    int wtile_bytes = 32768; // target weight tile bytes (32 KB: full 4096-wide rows)
    bool ring = false;       // ring-mode tiling: contiguous weight tiles of <= one ring slot
    // tensor parallelism (ext): 0 = single-device graph; >= 1 = the graph of
    // rank `tp_rank` of `tp_world` (Megatron split: column-parallel qkv and
    // gate/up, row-parallel o and down followed by ALLREDUCE_ADD of the
    // hidden vector, vocab-parallel lm_head, replicated embedding and norms)
    int tp_world = 0;
    int tp_rank = 0;
    // element type of the TP exchange partials (the W slots each rank stores
    // its partial sums into), layout.tp_partials "f32" (default) or "bf16":
    // bf16 halves the NVLink bytes of the in-kernel allreduce at the cost of
    // one more bf16 rounding of each partial before the residual add
    bool tp_bf16_partials = false;
    // batched decode (ext): batch >= 1 builds the graph of
    // `batch` concurrent requests: activations (npad, width) with the
    // request index as the row, 128 x 64 weight tiles for the tcgen05 GEMM
    // µops (BGEMM), KV caches as page pools (pool_pages, kv_heads * 64, hd)
    // addressed through a page table; request b covers req_pages[b] logical
    // pages (its context capacity in this program). KV tiles are addressed
    // (request, logical page, head) and resolved through the step block's
    // page table at run time, so pages can be allocated, freed and grown
    // between launches (vdc_kv_* block allocator) without a rebuild; pages
    // past a request's context are not loaded. pool_pages = 0: the pool holds
    // sum(req_pages) pages allocated contiguously (the lowered program's
    // default page table); > 0: a shared pool of that many pages, every
    // page-table entry unallocated (-1) until the host allocates it.
    int pool_pages = 0;
    bool argmax = false;  // greedy sampling fused into lm_head (single-request, no TP): next_token (int64)
    bool feedback = false;  // with argmax: token fed back + position advanced in the step block on the device
    int batch = 0;
    std::vector<int> req_pages;
    // prefill chunk (ext, §8f rank 3): the `batch` rows are consecutive
    // positions of ONE sequence (causal: row b attends to ctx_b = pos_b + 1)
    // sharing one page allocation (req_pages all equal); one launch appends
    // all their K/V rows and returns every row's logits
    bool prefill = false;
    int attn_job_cost = -1;  // batched attention load balance: fixed cost per split-KV job in ring tiles (-1: default)
};

ModelConfig llama3_8b();
ModelConfig qwen3_8b();
ModelConfig llama3_70b();
ModelConfig tiny_llama();

workload::OperatorGraph build_decode_graph(const ModelConfig& m, const LayoutConfig& l);
workload::OperatorGraph build_decode_graph_batched(const ModelConfig& m, const LayoutConfig& l);
int batch_npad(int batch);  // MMA N of a batch: 16, 32 or 64

// weight tile shape (rows, cols) used for a (M,K) matrix under `l`
std::pair<int64_t, int64_t> weight_tile(int64_t rows, int64_t cols, workload::ElemType e, const LayoutConfig& l);

}  // namespace uopsim::decode
