// Decode-layer graph builder (ext). See include/uopsim/decode.hpp for the
// operator sequence and weight-layout conventions.
#include <cmath>

#include "uopsim/decode.hpp"
#include "uopsim/util.hpp"
#include "uopsim/ring_abi.h"

namespace uopsim::decode {

using workload::ElemType;
using workload::InitKind;
using workload::OperatorGraph;
using workload::OperatorNode;
using workload::OpKind;
using workload::TensorRef;

ModelConfig llama3_8b() {
    ModelConfig m;
    m.name = "llama3-8b";
    m.layers = 32;
    m.hidden = 4096;
    m.heads = 32;
    m.kv_heads = 8;
    m.head_dim = 128;
    m.ffn = 14336;
    m.vocab = 128256;
    m.eps = 1e-5f;
    m.theta = 500000.0f;
    m.dtype = ElemType::bf16;
    m.scaled_init = true;
    return m;
}
ModelConfig qwen3_8b() {
    ModelConfig m = llama3_8b();
    m.name = "qwen3-8b";
    m.layers = 36;
    m.ffn = 12288;
    m.vocab = 151936;
    m.eps = 1e-6f;
    m.theta = 1000000.0f;
    m.qk_norm = true;
    return m;
}
ModelConfig llama3_70b() {
    ModelConfig m = llama3_8b();
    m.name = "llama3-70b";
    m.layers = 80;
    m.hidden = 8192;
    m.heads = 64;
    m.kv_heads = 8;
    m.ffn = 28672;
    return m;
}
ModelConfig tiny_llama() {
    ModelConfig m;  // C1: 2 layers, hidden 256, 4 heads x 64, fp32
    m.scaled_init = true;
    return m;
}

std::pair<int64_t, int64_t> weight_tile(int64_t rows, int64_t cols, ElemType e, const LayoutConfig& l) {
    (void)rows;
    const int64_t eb = workload::elem_bytes(e);
    if (l.ring) {
        // ring mode: tiles of <= one ring slot moved by bulk copies. Rows of
        // <= 8 KB: whole rows (power-of-two count <= VDC_RING_MAX_TILE_ROWS,
        // one contiguous copy). Longer rows: 2-row tiles of equal column
        // chunks (one copy per row), chunk a multiple of 128 elements so the
        // tensor-core GEMV's 16-chunk k-steps divide it; 2-row units keep the
        // per-SM split of an operator fine grained (+-1 unit of 2 rows).
        const int64_t row_bytes = cols * eb;
        if (row_bytes <= VDC_RING_SLOT_BYTES / 2) {
            int64_t tr = 1;
            while (tr * 2 <= VDC_RING_MAX_TILE_ROWS && tr * 2 * row_bytes <= VDC_RING_SLOT_BYTES) tr *= 2;
            return {tr, cols};
        }
        for (int64_t parts = (2 * row_bytes + VDC_RING_SLOT_BYTES - 1) / VDC_RING_SLOT_BYTES; parts <= cols; ++parts)
            if (cols % parts == 0 && (cols / parts) % 128 == 0) return {2, cols / parts};
        for (int64_t parts = (row_bytes + VDC_RING_SLOT_BYTES - 1) / VDC_RING_SLOT_BYTES; parts <= cols; ++parts)
            if (cols % parts == 0 && ((cols / parts) * eb) % 16 == 0) return {1, cols / parts};
        throw workload::WorkloadError("no ring tiling for a row of " + std::to_string(cols) + " elements");
    }
    const int64_t tc = std::min<int64_t>(cols, std::max<int64_t>(1, l.wtile_bytes / (eb * 4)));
    int64_t tr = std::max<int64_t>(1, l.wtile_bytes / (tc * eb));
    return {tr, tc};
}

namespace {

struct Builder {
    OperatorGraph g;
    const ModelConfig& m;
    const LayoutConfig& l;

    TensorRef& add(const std::string& name, std::vector<int64_t> shape, int64_t tr, int64_t tc, InitKind init,
                   ElemType e, float scale = 1.0f) {
        TensorRef t;
        t.name = name;
        t.shape = std::move(shape);
        t.tile_rows = tr;
        t.tile_cols = tc;
        t.init = init;
        t.elem = e;
        t.init_scale = scale;
        g.tensors.push_back(t);
        return g.tensors.back();
    }
    // vector (rows, 1) produced in tiles of `tile` rows
    std::string vec(const std::string& name, int64_t rows, int64_t tile, ElemType e) {
        add(name, {rows, 1}, tile, 1, InitKind::zeros, e);
        return name;
    }
    // a view of `base` with a different row tiling (same row-major storage)
    std::string view(const std::string& base, const std::string& suffix, int64_t tile_rows, int64_t tile_cols = 0) {
        const TensorRef& b = g.tensor(base);
        if (tile_rows == b.tile_rows && (tile_cols == 0 || tile_cols == b.tile_cols)) return base;
        const std::string name = base + suffix;
        if (g.find_tensor(name)) return name;
        TensorRef v = b;
        v.name = name;
        v.tile_rows = tile_rows;
        if (tile_cols) v.tile_cols = tile_cols;
        v.init = InitKind::zeros;
        v.state = false;
        v.view_of = base;
        g.tensors.push_back(v);
        return name;
    }
    // weight matrix (rows x cols) with the layout's tile shape; job_rows must
    // be a multiple of the tile rows so tiles never straddle two jobs
    std::string weight(const std::string& name, int64_t rows, int64_t cols, int64_t job_rows, float fan_in) {
        auto [tr, tc] = weight_tile(rows, cols, m.dtype, l);
        if (l.ring)
            job_rows = tr;  // ring jobs are tile aligned only (the lowering splits rows per SM)
        else
            while (job_rows % tr) --tr;
        const InitKind init = m.scaled_init ? InitKind::centered : InitKind::random;
        const float scale = m.scaled_init ? float(1.0 / std::sqrt(double(fan_in))) : 1.0f;
        // the word format encodes tile coordinates in 12 bits: tall matrices
        // become (planes, rows/plane, K) — same row-major storage — with the
        // fewest planes that keep every coordinate < 4096 and jobs inside a plane
        int64_t planes = 1;
        while (rows / planes / tr > 4095 || rows % planes || (rows / planes) % job_rows) {
            if (++planes > rows) throw workload::WorkloadError(name + ": no plane split fits the 12-bit tile coordinates");
        }
        if (planes == 1)
            add(name, {rows, cols}, tr, tc, init, m.dtype, scale);
        else
            add(name, {planes, rows / planes, cols}, tr, tc, init, m.dtype, scale);
        return name;
    }
    std::string norm(const std::string& name, int64_t rows) {
        add(name, {rows, 1}, rows, 1, InitKind::ones, m.dtype);
        return name;
    }
    void node(const std::string& id, OpKind k, std::vector<std::string> in, std::vector<std::string> out,
              std::map<std::string, std::string> attrs = {}) {
        g.nodes.push_back(OperatorNode{id, k, std::move(in), std::move(out), std::move(attrs)});
    }
};

std::string num(double v) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.9g", v);
    return buf;
}

}  // namespace

OperatorGraph build_decode_graph(const ModelConfig& m, const LayoutConfig& l) {
    if (l.batch >= 1) return build_decode_graph_batched(m, l);
    if (m.head_dim % l.job_rows || l.job_rows % 2) throw workload::WorkloadError("job_rows must divide head_dim and be even");
    if (m.heads % m.kv_heads) throw workload::WorkloadError("heads must be a multiple of kv_heads");
    if (l.max_ctx < l.ctx_pages * l.page_rows) throw workload::WorkloadError("max_ctx below ctx_pages*page_rows");
    const bool tp = l.tp_world >= 1;
    const int64_t W = tp ? l.tp_world : 1;
    if (tp && (l.tp_rank < 0 || l.tp_rank >= W || m.kv_heads % W || m.ffn % (W * (l.gu_block / 2)) || m.vocab % W))
        throw workload::WorkloadError("tensor parallelism needs kv_heads, ffn (in gu blocks) and vocab divisible by tp_world");
    Builder b{{}, m, l};
    const ElemType e = m.dtype;
    const int64_t d = m.hidden, hd = m.head_dim, hq = m.heads / W, hkv = m.kv_heads / W, grp = hq / hkv;
    const int64_t qrows = hq * hd, kvrows = hkv * hd, R = l.job_rows, ffn = m.ffn / W, vocab = m.vocab / W;
    const int64_t splits = (l.ctx_pages + l.pages_per_job - 1) / l.pages_per_job;
    const std::string eps = num(m.eps), theta = num(m.theta);
    const std::map<std::string, std::string> tp_attrs = {{"tp_world", std::to_string(W)}, {"tp_rank", std::to_string(l.tp_rank)}};
    auto with = [](std::map<std::string, std::string> a, const std::map<std::string, std::string>& extra) {
        a.insert(extra.begin(), extra.end());
        return a;
    };
    // TP exchange buffer: one (D,1) slot of partials per rank (bf16 or fp32), peer mapped
    auto sym = [&](const std::string& name) {
        TensorRef& t = b.add(name, {W * d, 1}, d, 1, InitKind::zeros, l.tp_bf16_partials ? ElemType::bf16 : ElemType::f32);
        t.symmetric = true;
        return name;
    };

    b.add("embed.table", {m.vocab, d}, 1, d, m.scaled_init ? InitKind::centered : InitKind::random, e);
    b.vec("embed.x", d, d, e);
    b.node("embed", OpKind::EMBED_ROW, {"embed.table"}, {"embed.x"});
    std::string x = "embed.x";

    for (int li = 0; li < m.layers; ++li) {
        const std::string L = "L" + std::to_string(li) + ".";
        // attention block
        b.norm(L + "attn_norm", d);
        b.weight(L + "wqkv", qrows + 2 * kvrows, d, R, float(d));
        b.vec(L + "q", qrows, R, e);
        for (const char* c : {"kc", "vc"}) {
            TensorRef& t = b.add(L + c, {hkv, l.max_ctx, hd}, l.page_rows, hd,
                                 m.scaled_init ? InitKind::centered : InitKind::random, e);
            t.state = true;
            // ring programs: bf16 head-dim-128 caches keep their page rows swizzled
            // for the tensor-core attention (ring_abi.h VDC_DESC_KPAGE_SWZ)
            if (l.ring && e == ElemType::bf16 && hd == 128 && l.page_rows == 64 && l.max_ctx % 64 == 0)
                t.tma = VDC_DESC_KPAGE_SWZ;
            b.view(L + c, ".seg", 1, R);
        }
        std::map<std::string, std::string> qkv_attrs = {{"eps", eps}, {"theta", theta}, {"rope", "1"}, {"job_rows", std::to_string(R)}};
        if (m.qk_norm) {
            b.norm(L + "q_norm", hd);
            b.norm(L + "k_norm", hd);
            qkv_attrs["qk_norm"] = "1";
        }
        b.node(L + "qkv", OpKind::RMS_GEMV, {L + "wqkv", b.view(x, ".all", d), L + "attn_norm"},
               {L + "q", L + "kc.seg", L + "vc.seg"}, qkv_attrs);
        b.add(L + "part", {hkv * splits * grp, hd + 2}, grp, hd + 2, InitKind::zeros, ElemType::f32);
        std::map<std::string, std::string> attn_attrs = {{"ctx_pages", std::to_string(l.ctx_pages)},
                                                         {"pages_per_job", std::to_string(l.pages_per_job)}};
        if (m.qk_norm) {
            attn_attrs["q_norm"] = L + "q_norm";
            attn_attrs["k_norm"] = L + "k_norm";
            attn_attrs["eps"] = eps;
            attn_attrs["theta"] = theta;
        }
        b.node(L + "attn", OpKind::ATTN_DECODE, {b.view(L + "q", ".grp", grp * hd), L + "kc", L + "vc"}, {L + "part"}, attn_attrs);
        b.vec(L + "attn", qrows, grp * hd, e);
        // the combine reads all partials of one kv head as a single tile
        b.node(L + "comb", OpKind::ATTN_COMBINE, {b.view(L + "part", ".head", splits * grp)}, {L + "attn"});
        b.weight(L + "wo", d, qrows, R, float(qrows * W));
        b.vec(L + "x1", d, R, e);
        if (tp) {  // row-parallel o-proj: partial sums -> all ranks' slots -> allreduce + residual
            b.node(L + "o", OpKind::GEMV, {L + "wo", b.view(L + "attn", ".all", qrows)}, {sym(L + "o.part")},
                   with({{"job_rows", std::to_string(R)}}, tp_attrs));
            b.node(L + "o.ar", OpKind::ALLREDUCE_ADD, {L + "o.part", x}, {L + "x1"}, tp_attrs);
        } else {
            b.node(L + "o", OpKind::GEMV_ADD, {L + "wo", b.view(L + "attn", ".all", qrows), b.view(x, ".blk", R)}, {L + "x1"},
                   {{"job_rows", std::to_string(R)}});
        }
        // MLP block
        b.norm(L + "mlp_norm", d);
        b.weight(L + "wgu", 2 * ffn, d, l.gu_block, float(d));
        b.vec(L + "a", ffn, l.gu_block / 2, e);
        b.node(L + "gu", OpKind::RMS_GEMV, {L + "wgu", b.view(L + "x1", ".all", d), L + "mlp_norm"}, {L + "a"},
               {{"eps", eps}, {"swiglu", std::to_string(l.gu_block)}, {"job_rows", std::to_string(l.gu_block)}});
        b.weight(L + "wd", d, ffn, R, float(ffn * W));
        b.vec(L + "x2", d, R, e);
        if (tp) {
            b.node(L + "down", OpKind::GEMV, {L + "wd", b.view(L + "a", ".all", ffn)}, {sym(L + "d.part")},
                   with({{"job_rows", std::to_string(R)}}, tp_attrs));
            b.node(L + "down.ar", OpKind::ALLREDUCE_ADD, {L + "d.part", L + "x1"}, {L + "x2"}, tp_attrs);
        } else {
            b.node(L + "down", OpKind::GEMV_ADD, {L + "wd", b.view(L + "a", ".all", ffn), L + "x1"}, {L + "x2"},
                   {{"job_rows", std::to_string(R)}});
        }
        x = L + "x2";
    }
    b.norm("final_norm", d);
    b.weight("lm_head", vocab, d, l.head_job_rows, float(d));  // vocab-parallel: this rank's logit rows
    b.add("logits", {vocab, 1}, l.head_job_rows, 1, InitKind::zeros, ElemType::f32);
    std::map<std::string, std::string> head_attrs = {{"eps", eps}, {"job_rows", std::to_string(l.head_job_rows)}};
    if (l.argmax) {
        // per-job (max, argmax) slots and the sampled token
        b.add("head.amax", {4096, 2}, 4096, 2, InitKind::zeros, ElemType::f32);
        b.add("next_token", {1, 1}, 1, 1, InitKind::zeros, ElemType::i64);
        head_attrs["argmax"] = "1";
        if (l.feedback) head_attrs["feedback"] = "1";
        if (tp) {  // vocab-parallel logits: the ranks exchange their (max, global index) pairs
            TensorRef& t = b.add("head.amx", {W * 2, 1}, 2, 1, InitKind::zeros, ElemType::f32);
            t.symmetric = true;
            head_attrs["tp_argmax"] = "head.amx";
            head_attrs["vocab_base"] = std::to_string(l.tp_rank * vocab);
            head_attrs["vocab_valid"] = std::to_string(vocab);
        }
    }
    b.node("head", OpKind::RMS_GEMV, {"lm_head", b.view(x, ".all", d), "final_norm"}, {"logits"}, head_attrs);
    b.g.validate();
    return std::move(b.g);
}

int batch_npad(int batch) {
    if (batch < 1 || batch > VDC_RING_MAX_BATCH) throw workload::WorkloadError("batch must be 1..64");
    return batch <= 16 ? 16 : batch <= 32 ? 32 : 64;
}

// Batched decode graph (see LayoutConfig::batch). Node kinds label the
// operators for the ring lowering's batched planner (attr "batch"); the
// tensor shapes are batched, so the single-request shape rules of
// check_node_shapes do not apply and are not run.
//   embed   [embed.table, L0.attn_norm]            -> [embed.x, embed.xn]
//   L.qkv   [L.wqkv, xn, x]                        -> [L.q, L.kc, L.vc]
//   L.attn  [L.q, L.kc, L.vc]                      -> [L.part]
//   L.comb  [L.part]                               -> [L.attn]
//   L.o     [L.wo, L.attn, x, L.mlp_norm]          -> [L.x1, L.x1n]
//   L.gu    [L.wgu, L.x1n, L.x1]                   -> [L.a]
//   L.down  [L.wd, L.a, L.x1, next norm]           -> [L.x2, L.x2n]
//   head    [lm_head, xn, x]                       -> [logits]
// xn = bf16(x * w_norm) of the next RMSNorm (its per-request 1/rms is
// applied in the consuming GEMM's epilogue); gate/up rows come in blocks of
// 128 = [64 gate | 64 up] (gu_block 128: one MMA row block).
static std::map<std::string, std::string> with_attrs(std::map<std::string, std::string> a, const std::map<std::string, std::string>& extra) {
    a.insert(extra.begin(), extra.end());
    return a;
}

OperatorGraph build_decode_graph_batched(const ModelConfig& m, const LayoutConfig& l) {
    const int B = l.batch, N = batch_npad(B);
    if (m.dtype != ElemType::bf16 || m.head_dim != 128 || l.page_rows != 64)
        throw workload::WorkloadError("batched decode is built for bf16 models with head_dim 128 and 64-row pages");
    if (int(l.req_pages.size()) != B) throw workload::WorkloadError("layout.req_pages needs one entry per request");
    if (l.gu_block != 128) throw workload::WorkloadError("batched decode uses gu_block 128");
    // tensor parallelism (rank tp_rank of tp_world): column-parallel qkv and
    // gate/up, row-parallel o / down into symmetric fp32 partial buffers,
    // in-kernel ALLREDUCE_ADD (+ residual, + the next norm's operand),
    // vocab-parallel lm_head
    const bool tp = l.tp_world >= 1;
    const int64_t W = tp ? l.tp_world : 1;
    if (tp && (l.tp_rank < 0 || l.tp_rank >= W || m.kv_heads % W || m.ffn % (W * 64)))
        throw workload::WorkloadError("tensor parallelism needs kv_heads and ffn / 64 divisible by tp_world");
    const int64_t d = m.hidden, hd = m.head_dim, hq = m.heads / W, hkv = m.kv_heads / W, grp = hq / hkv;
    // vocab shard per rank: ceil(vocab / W) rounded up to whole 128-row MMA
    // blocks; rank r holds vocabulary rows [r * shard, (r + 1) * shard), rows
    // past the vocabulary are zero padding (their logits are not tokens:
    // sampling and callers use the first `vocab` columns of the gathered logits)
    const int64_t vocab = ((m.vocab + W - 1) / W + 127) / 128 * 128;
    const int64_t qrows = hq * hd, kvrows = hkv * hd, ffn = m.ffn / W;
    if (d % 128 || qrows % 128 || kvrows % 128 || ffn % 64 || hq % hkv)
        throw workload::WorkloadError("batched decode needs 128-row aligned projections");
    const std::map<std::string, std::string> tp_attrs = {{"tp_world", std::to_string(W)}, {"tp_rank", std::to_string(l.tp_rank)}};

    int64_t pool = 0, jobs = 0;
    for (int p : l.req_pages) {
        if (p < 1) throw workload::WorkloadError("every request covers at least one page");
        pool += p;
        jobs += (p + l.pages_per_job - 1) / l.pages_per_job;
    }
    if (l.prefill) {  // one sequence: every row shares request 0's pages
        for (int p : l.req_pages)
            if (p != l.req_pages[0]) throw workload::WorkloadError("a prefill chunk's rows share one page allocation");
        if (m.qk_norm) throw workload::WorkloadError("prefill chunks of QK-norm models are not supported");
        pool = l.req_pages[0];
    }
    // KV tiles are addressed (request, logical page, head) through the page
    // table, so the pool size is not bounded by the 12-bit tile coordinates
    if (l.batch > 4095) throw workload::WorkloadError("at most 4095 requests per batched program (12-bit tile coordinates)");
    for (int p : l.req_pages)
        if (p > 4095) throw workload::WorkloadError("at most 4095 pages per request (12-bit tile coordinates)");
    if (l.pool_pages > 0) {
        if (l.prefill) throw workload::WorkloadError("prefill chunks use the contiguous default pool");
        pool = l.pool_pages;
    }
    Builder b{{}, m, l};
    auto sym = [&](const std::string& name) {  // exchange buffer: one (npad, d) slot of partials per rank
        TensorRef& t = b.add(name, {W * N * d, 1}, N * d, 1, InitKind::zeros, l.tp_bf16_partials ? ElemType::bf16 : ElemType::f32);
        t.symmetric = true;
        return name;
    };
    const ElemType e = m.dtype;
    const InitKind winit = m.scaled_init ? InitKind::centered : InitKind::random;
    const std::string eps = num(m.eps), theta = num(m.theta), bs = std::to_string(B);
    std::string rp;
    for (int p : l.req_pages) rp += (rp.empty() ? "" : ",") + std::to_string(p);
    auto act = [&](const std::string& name, int64_t width, bool tma) {
        TensorRef& t = b.add(name, {N, width}, N, 64, InitKind::zeros, e);
        t.tma = tma ? uint32_t(N) : 0u;
        return name;
    };
    auto wgt = [&](const std::string& name, int64_t rows, int64_t cols, double fan_in) {
        TensorRef& t = b.add(name, {rows, cols}, VDC_RING_BGEMM_ROWS, VDC_RING_BGEMM_KT, winit, e,
                             m.scaled_init ? float(1.0 / std::sqrt(fan_in)) : 1.0f);
        t.tma = VDC_DESC_PACKED_SW128;
        return name;
    };
    auto sk = [&](const std::string& name, int64_t row_blocks) {  // stream-K partials (shared by all layers)
        b.add(name, {(row_blocks + 256) * N * 128, 1}, N * 128, 1, InitKind::zeros, ElemType::f32);
        return name;
    };
    b.add("ring.pad", {1, 8}, 1, 8, InitKind::zeros, e);  // 16-byte tile that realigns attention jobs in the ring
    b.add("embed.table", {m.vocab, d}, 1, d, winit, e);
    sk("qkv.sk", (qrows + 2 * kvrows) / 128);
    sk("o.sk", d / 128);
    sk("gu.sk", 2 * ffn / 128);
    sk("down.sk", d / 128);
    sk("head.sk", vocab / 128);
    // sums of squares of a residual-stream activation per 32-row group and
    // request, written by its producer so RMS consumers need not re-read it
    auto ssq = [&](const std::string& xname) {
        if (!tp) b.add(xname + ".ssq", {d / 32, N}, 1, N, InitKind::zeros, ElemType::f32);
    };
    std::string x = act("embed.x", d, false), xn = act("embed.xn", d, true);
    ssq(x);
    b.norm("L0.attn_norm", d);
    b.node("embed", OpKind::EMBED_ROW, {"embed.table", "L0.attn_norm"}, {x, xn}, {{"batch", bs}});
    for (int li = 0; li < m.layers; ++li) {
        const std::string L = "L" + std::to_string(li) + ".";
        wgt(L + "wqkv", qrows + 2 * kvrows, d, double(d));
        b.add(L + "q", {B, qrows}, 1, qrows, InitKind::zeros, e);
        for (const char* c : {"kc", "vc"}) {
            TensorRef& t = b.add(L + c, {pool, hkv * l.page_rows, hd}, l.page_rows, hd, winit, e);
            t.state = true;
            t.tma = VDC_DESC_KPAGE_SWZ;  // K and V page rows swizzled (tensor-core attention)
        }
        std::map<std::string, std::string> qkv_attrs = {{"eps", eps}, {"theta", theta}, {"rope", "1"}, {"batch", bs}};
        std::map<std::string, std::string> attn_attrs = {{"pages_per_job", std::to_string(l.pages_per_job)}, {"batch", bs},
                                                         {"req_pages", rp}};
        if (l.prefill) attn_attrs["prefill"] = "1";
        if (l.pool_pages > 0) attn_attrs["pool_pages"] = std::to_string(l.pool_pages);
        if (l.attn_job_cost >= 0) attn_attrs["job_cost"] = std::to_string(l.attn_job_cost);
        if (m.qk_norm) {
            b.norm(L + "q_norm", hd);
            b.norm(L + "k_norm", hd);
            qkv_attrs["qk_norm"] = "1";
            attn_attrs["q_norm"] = L + "q_norm";
            attn_attrs["k_norm"] = L + "k_norm";
            attn_attrs["eps"] = eps;
            attn_attrs["theta"] = theta;
        }
        b.node(L + "qkv", OpKind::RMS_GEMV, {L + "wqkv", xn, x}, {L + "q", L + "kc", L + "vc"}, qkv_attrs);
        b.add(L + "part", {jobs * hkv * grp, hd + 2}, grp, hd + 2, InitKind::zeros, ElemType::f32);
        b.node(L + "attn", OpKind::ATTN_DECODE, {L + "q", L + "kc", L + "vc"}, {L + "part"}, attn_attrs);
        act(L + "attn", qrows, true);
        b.node(L + "comb", OpKind::ATTN_COMBINE, {L + "part"}, {L + "attn"}, {{"batch", bs}});
        wgt(L + "wo", d, qrows, double(qrows * W));
        b.norm(L + "mlp_norm", d);
        act(L + "x1", d, false);
        act(L + "x1n", d, true);
        ssq(L + "x1");
        if (tp) {
            b.node(L + "o", OpKind::GEMV, {L + "wo", L + "attn"}, {sym(L + "o.part")}, with_attrs({{"batch", bs}}, tp_attrs));
            b.node(L + "o.ar", OpKind::ALLREDUCE_ADD, {L + "o.part", x, L + "mlp_norm"}, {L + "x1", L + "x1n"},
                   with_attrs({{"batch", bs}}, tp_attrs));
        } else {
            b.node(L + "o", OpKind::GEMV_ADD, {L + "wo", L + "attn", x, L + "mlp_norm"}, {L + "x1", L + "x1n"}, {{"batch", bs}});
        }
        wgt(L + "wgu", 2 * ffn, d, double(d));
        act(L + "a", ffn, true);
        b.node(L + "gu", OpKind::RMS_GEMV, {L + "wgu", L + "x1n", L + "x1"}, {L + "a"},
               {{"eps", eps}, {"swiglu", "128"}, {"batch", bs}});
        wgt(L + "wd", d, ffn, double(ffn * W));
        const std::string next_norm = li + 1 < m.layers ? "L" + std::to_string(li + 1) + ".attn_norm" : "final_norm";
        b.norm(next_norm, d);
        x = act(L + "x2", d, false);
        xn = act(L + "x2n", d, true);
        ssq(x);
        if (tp) {
            b.node(L + "down", OpKind::GEMV, {L + "wd", L + "a"}, {sym(L + "d.part")}, with_attrs({{"batch", bs}}, tp_attrs));
            b.node(L + "down.ar", OpKind::ALLREDUCE_ADD, {L + "d.part", L + "x1", next_norm}, {x, xn}, with_attrs({{"batch", bs}}, tp_attrs));
        } else {
            b.node(L + "down", OpKind::GEMV_ADD, {L + "wd", L + "a", L + "x1", next_norm}, {x, xn}, {{"batch", bs}});
        }
    }
    wgt("lm_head", vocab, d, double(d));  // vocab-parallel: this rank's logit columns
    b.add("logits", {B, vocab}, 1, vocab, InitKind::zeros, ElemType::f32);
    std::map<std::string, std::string> head_attrs = {{"eps", eps}, {"batch", bs}};
    if (!tp && vocab != m.vocab) throw workload::WorkloadError("batched decode needs the vocabulary in whole 128-row blocks");
    if (l.argmax) {  // greedy sampling fused into the lm_head GEMM: per-SM slots, tokens per request
        b.add("head.amax", {256 * N, 2}, N, 2, InitKind::zeros, ElemType::f32);
        b.add("next_token", {B, 1}, 1, 1, InitKind::zeros, ElemType::i64);
        head_attrs["argmax"] = "1";
        if (l.feedback) head_attrs["feedback"] = "1";
        if (tp) {  // vocab-parallel logits: the ranks exchange their (max, global index) pairs per request
            TensorRef& t = b.add("head.amx", {W * N * 2, 1}, N * 2, 1, InitKind::zeros, ElemType::f32);
            t.symmetric = true;
            head_attrs["tp_argmax"] = "head.amx";
            head_attrs["vocab_base"] = std::to_string(l.tp_rank * vocab);
            head_attrs["vocab_valid"] = std::to_string(std::max<int64_t>(0, std::min<int64_t>(vocab, m.vocab - l.tp_rank * vocab)));
        }
    }
    b.node("head", OpKind::RMS_GEMV, {"lm_head", xn, x}, {"logits"}, head_attrs);
    return std::move(b.g);
}

}  // namespace uopsim::decode
