// Probe: tcgen05.mma (kind::f16, cta_group::1, M=128) fed by TMA 2-D tensor
// tiles with 128-byte swizzle, accumulator in TMEM, read back with
// tcgen05.ld.32x32b. Validates the descriptor encodings the batched ring
// GEMM uses:  D[m][n] = sum_k W[m][k] * X[n][k]  (W: M x K, X: N x K, bf16).
//   nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a probe_umma.cu -lcuda -o probe_umma
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);        // start address
    d |= uint64_t(1) << 16;                       // LBO (unused for swizzled K-major)
    d |= uint64_t(1024 >> 4) << 32;               // SBO: 8 rows x 128 B
    d |= uint64_t(1) << 46;                       // version (sm_100)
    d |= uint64_t(2) << 61;                       // SWIZZLE_128B
    return d;
}

template <int N>
__global__ void __launch_bounds__(128) probe(const CUtensorMap* tw, const CUtensorMap* tx, int K, float* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* a_s = sm;                 // 128 x 64 bf16 = 16 KB
    uint8_t* b_s = sm + 16384;         // N x 64 bf16
    __shared__ uint64_t full_bar, mma_bar;
    __shared__ uint32_t tmem_base;
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full_bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mma_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tmem_base)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = tmem_base;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    if (threadIdx.x == 0) {
        for (int kt = 0; kt < K / 64; ++kt) {
            uint32_t ph = kt & 1;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full_bar)), "r"(16384 + N * 128) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sa(a_s)), "l"(tw), "r"(kt * 64), "r"(0), "r"(sa(&full_bar)) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sa(b_s)), "l"(tx), "r"(kt * 64), "r"(0), "r"(sa(&full_bar)) : "memory");
            asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa(&full_bar)), "r"(ph) : "memory");
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int kk = 0; kk < 4; ++kk) {
                uint64_t ad = sw128_desc(sa(a_s) + kk * 32), bd = sw128_desc(sa(b_s) + kk * 32);
                uint32_t acc = (kt | kk) ? 1u : 0u;
                asm volatile("{\n.reg .pred p;\nsetp.ne.u32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                             ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&mma_bar)) : "memory");
            asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}" ::"r"(sa(&mma_bar)), "r"(ph) : "memory");
        }
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[N];
    uint32_t taddr = tmem + (uint32_t(warp * 32) << 16);
    if constexpr (N == 16)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(taddr));
    else {
#pragma unroll
        for (int c = 0; c < N; c += 8)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[c]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]), "=r"(r[c + 6]), "=r"(r[c + 7])
                         : "r"(taddr + c));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int row = warp * 32 + lane;
    for (int n = 0; n < N; ++n) out[row * N + n] = __uint_as_float(r[n]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void make_map(EncodeFn enc, CUtensorMap* m, void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); exit(1); }
}

template <int N>
static int run(EncodeFn enc, int K) {
    const int M = 128;
    std::vector<__nv_bfloat16> w(size_t(M) * K), x(size_t(N) * K);
    std::vector<float> wf(w.size()), xf(x.size());
    srand(7);
    for (size_t i = 0; i < w.size(); ++i) { w[i] = __float2bfloat16(float(rand() % 2001 - 1000) / 1000.f); wf[i] = __bfloat162float(w[i]); }
    for (size_t i = 0; i < x.size(); ++i) { x[i] = __float2bfloat16(float(rand() % 2001 - 1000) / 1000.f); xf[i] = __bfloat162float(x[i]); }
    void *dw, *dx; float* dout; CUtensorMap* dmaps;
    CK(cudaMalloc(&dw, w.size() * 2)); CK(cudaMalloc(&dx, x.size() * 2)); CK(cudaMalloc(&dout, M * N * 4)); CK(cudaMalloc(&dmaps, 256));
    CK(cudaMemcpy(dw, w.data(), w.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, x.data(), x.size() * 2, cudaMemcpyHostToDevice));
    alignas(64) CUtensorMap maps[2];
    make_map(enc, &maps[0], dw, K, M, 128);
    make_map(enc, &maps[1], dx, K, N, N);
    CK(cudaMemcpy(dmaps, maps, sizeof(maps), cudaMemcpyHostToDevice));
    int smem = 16384 + N * 128 + 1024;
    CK(cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    probe<N><<<1, 128, smem>>>(dmaps, dmaps + 1, K, dout);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    std::vector<float> out(M * N);
    CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += double(wf[size_t(m) * K + k]) * xf[size_t(n) * K + k];
            maxerr = fmax(maxerr, fabs(s - out[m * N + n])); maxref = fmax(maxref, fabs(s));
        }
    printf("N=%d K=%d max|err|=%.3e max|ref|=%.3e %s\n", N, K, maxerr, maxref, maxerr <= 1e-3 * maxref ? "OK" : "FAIL");
    cudaFree(dw); cudaFree(dx); cudaFree(dout); cudaFree(dmaps);
    return maxerr <= 1e-3 * maxref ? 0 : 1;
}

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    int bad = 0;
    bad += run<16>(enc, 64);
    bad += run<16>(enc, 1024);
    bad += run<32>(enc, 4096);
    bad += run<48>(enc, 512);
    bad += run<64>(enc, 512);
    printf(bad ? "PROBE FAIL\n" : "PROBE OK\n");
    return bad;
}
