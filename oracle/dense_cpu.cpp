// TEST / BASELINE INFRASTRUCTURE ONLY (never linked into the product).
//
// The optional dense fp32 CPU decode of BASELINE.md §3.2: one Llama-3-8B
// decode step (batch 1) evaluated directly on the host with every core
// (std::thread; the image's gcc ships no OpenMP runtime), for context beside the GPU numbers — not the reference path (that
// is oracle_interp + the reference HandlerState, single-threaded by design)
// and not an optimisation target.
//
// Model math as in tests/decode_ref.py (fp32 throughout): RMSNorm, fused
// q|k|v projection, interleaved-pair RoPE, GQA attention over a ctx-row
// cache + the appended row, o-proj + residual, RMSNorm, gate/up + SwiGLU,
// down + residual; final RMSNorm + lm_head + argmax.
//
// Memory: one layer's weights (~0.87 GB fp32) are allocated and reused for
// every layer (a bandwidth-bound step touches each layer's weights once
// either way) plus the lm_head (2.1 GB). Weights are splitmix64 uniform
// values scaled by 1/sqrt(fan_in).
//
// usage: dense_cpu <layers> <ctx> <steps> [threads]   prints one JSON line
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

namespace {

constexpr int D = 4096, HQ = 32, HKV = 8, HD = 128, FFN = 14336, VOCAB = 128256;
constexpr float EPS = 1e-5f, THETA = 500000.f;

int g_threads = 1;

// f(lo, hi) over [0, n) split into g_threads contiguous ranges
template <class F>
void parallel_for(size_t n, F f) {
    std::vector<std::thread> ts;
    for (int t = 1; t < g_threads; ++t) ts.emplace_back([&, t] { f(n * t / g_threads, n * (t + 1) / g_threads); });
    f(0, n / g_threads);
    for (auto& th : ts) th.join();
}

uint64_t splitmix(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void fill(std::vector<float>& v, uint64_t seed, float scale) {
    parallel_for(v.size(), [&](size_t lo, size_t hi) {
        uint64_t s = seed ^ (0x1234567ull * (lo + 1));
        for (size_t i = lo; i < hi; ++i) v[i] = (float(splitmix(s) >> 40) * (1.f / 16777216.f) * 2.f - 1.f) * scale;
    });
}

// y = W x, W (M x K) row-major, rows split over the threads
void matvec(const float* W, const float* x, float* y, int M, int K) {
    parallel_for(size_t(M), [&](size_t lo, size_t hi) {
        for (size_t r = lo; r < hi; ++r) {
            const float* w = W + r * K;
            float s[8] = {};
            for (int k = 0; k < K; k += 8)
                for (int j = 0; j < 8; ++j) s[j] += w[k + j] * x[k + j];
            y[r] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
        }
    });
}

void rmsnorm(const float* x, const float* w, float* y, int n) {
    double ss = 0;
    for (int i = 0; i < n; ++i) ss += double(x[i]) * x[i];
    const float inv = 1.f / std::sqrt(float(ss / n) + EPS);
    for (int i = 0; i < n; ++i) y[i] = x[i] * inv * w[i];
}

void rope(float* v, int n, int pos) {
    for (int i = 0; i < n; i += 2) {
        const double ang = double(pos) * std::pow(double(THETA), -double(i % HD) / HD);
        const float c = float(std::cos(ang)), s = float(std::sin(ang)), a = v[i], b = v[i + 1];
        v[i] = a * c - b * s;
        v[i + 1] = a * s + b * c;
    }
}

}  // namespace

int main(int argc, char** argv) {
    const int layers = argc > 1 ? std::atoi(argv[1]) : 32, ctx = argc > 2 ? std::atoi(argv[2]) : 4096;
    const int steps = argc > 3 ? std::atoi(argv[3]) : 2;
    g_threads = argc > 4 ? std::atoi(argv[4]) : int(std::max(1u, std::thread::hardware_concurrency()));
    const int qr = HQ * HD, kvr = HKV * HD, G = HQ / HKV;
    std::vector<float> wqkv(size_t(qr + 2 * kvr) * D), wo(size_t(D) * qr), wgu(size_t(2 * FFN) * D), wd(size_t(D) * FFN);
    std::vector<float> lm(size_t(VOCAB) * D), emb(D), nrm(D, 1.f);  // emb: the token's embedding row
    std::vector<float> kc(size_t(HKV) * (ctx + steps) * HD), vc(kc.size());
    fill(wqkv, 1, 1.f / std::sqrt(float(D)));
    fill(wo, 2, 1.f / std::sqrt(float(qr)));
    fill(wgu, 3, 1.f / std::sqrt(float(D)));
    fill(wd, 4, 1.f / std::sqrt(float(FFN)));
    fill(lm, 5, 1.f / std::sqrt(float(D)));
    fill(emb, 6, 1.f);
    fill(kc, 7, 1.f);
    fill(vc, 8, 1.f);
    std::vector<float> x(D), xn(D), qkv(qr + 2 * kvr), att(qr), t(D), gu(2 * FFN), a(FFN), logits(VOCAB);
    double best = 1e30;
    int token = 0;
    for (int st = 0; st < steps; ++st) {
        const int pos = ctx - 1 + st;
        const auto t0 = std::chrono::steady_clock::now();
        x = emb;
        for (int l = 0; l < layers; ++l) {
            rmsnorm(x.data(), nrm.data(), xn.data(), D);
            matvec(wqkv.data(), xn.data(), qkv.data(), qr + 2 * kvr, D);
            rope(qkv.data(), qr + kvr, pos);
            const int T = ctx + steps;
            for (int h = 0; h < HKV; ++h)
                for (int e = 0; e < HD; ++e) {
                    kc[(size_t(h) * T + pos) * HD + e] = qkv[qr + h * HD + e];
                    vc[(size_t(h) * T + pos) * HD + e] = qkv[qr + kvr + h * HD + e];
                }
            parallel_for(HQ, [&](size_t hlo, size_t hhi) {
            for (size_t hq = hlo; hq < hhi; ++hq) {
                const int h = hq / G;
                const float* q = qkv.data() + hq * HD;
                std::vector<float> p(pos + 1);
                float m = -1e30f;
                for (int r = 0; r <= pos; ++r) {
                    const float* k = kc.data() + (size_t(h) * T + r) * HD;
                    float s = 0.f;
                    for (int e = 0; e < HD; ++e) s += q[e] * k[e];
                    p[r] = s / std::sqrt(float(HD));
                    m = std::max(m, p[r]);
                }
                float l = 0.f;
                float o[HD] = {};
                for (int r = 0; r <= pos; ++r) {
                    const float w = std::exp(p[r] - m);
                    l += w;
                    const float* v = vc.data() + (size_t(h) * T + r) * HD;
                    for (int e = 0; e < HD; ++e) o[e] += w * v[e];
                }
                for (int e = 0; e < HD; ++e) att[hq * HD + e] = o[e] / l;
            }
            });
            matvec(wo.data(), att.data(), t.data(), D, qr);
            for (int i = 0; i < D; ++i) x[i] += t[i];
            rmsnorm(x.data(), nrm.data(), xn.data(), D);
            matvec(wgu.data(), xn.data(), gu.data(), 2 * FFN, D);
            for (int i = 0; i < FFN; ++i) a[i] = gu[i] / (1.f + std::exp(-gu[i])) * gu[FFN + i];
            matvec(wd.data(), a.data(), t.data(), D, FFN);
            for (int i = 0; i < D; ++i) x[i] += t[i];
        }
        rmsnorm(x.data(), nrm.data(), xn.data(), D);
        matvec(lm.data(), xn.data(), logits.data(), VOCAB, D);
        int arg = 0;
        for (int i = 1; i < VOCAB; ++i)
            if (logits[i] > logits[arg]) arg = i;
        token = arg;
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        best = std::min(best, s);
    }
    std::printf("{\"layers\": %d, \"ctx\": %d, \"threads\": %d, \"seconds_per_token\": %.6f, \"tokens_per_s\": %.4f, \"token\": %d}\n",
                layers, ctx, g_threads, best, 1.0 / best, token);
    return 0;
}
