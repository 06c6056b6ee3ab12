// Calibration probe: achievable HBM read bandwidth on B200 for
//  (a) plain vectorised LDG streaming, (b) a persistent single-issuer
//  cp.async.bulk ring (the memory-virtual-core pattern) at several tile sizes.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void ldg_stream(const int4* __restrict__ p, size_t n, float* out) {
  float s = 0.f;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  #pragma unroll 4
  for (; i < n; i += stride) {
    int4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    s += __int_as_float(v.x) + __int_as_float(v.w);
  }
  if (s == 1234.5f) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// warp 0 lane 0 = issuer; warps 1..NC = consumers (round-robin slots)
template <int NC>
__global__ void __launch_bounds__(32 * (NC + 1), 1) ring_stream(const uint8_t* __restrict__ base, size_t tiles, uint32_t tile_bytes, int nslots, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 32;
  uint8_t* slots = smem + 1024;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t my0 = blockIdx.x, step = gridDim.x;
  if (warp == 0) {
    if (lane == 0) {
      size_t k = 0;
      for (size_t t = my0; t < tiles; t += step, ++k) {
        int s = k % nslots; uint32_t ph = (k / nslots) & 1;
        if (k >= (size_t)nslots) mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], tile_bytes);
        bulk_g2s(slots + (size_t)s * tile_bytes, base + t * (size_t)tile_bytes, tile_bytes, &full[s]);
      }
    }
  } else {
    int c = warp - 1;
    float acc = 0.f;
    size_t k = 0;
    for (size_t t = my0; t < tiles; t += step, ++k) {
      if ((int)(k % NC) != c) continue;
      int s = k % nslots; uint32_t ph = (k / nslots) & 1;
      mbar_wait(&full[s], ph);
      const int4* d = (const int4*)(slots + (size_t)s * tile_bytes);
      for (uint32_t i = lane; i < tile_bytes / 16; i += 32) { int4 v = d[i]; acc += __int_as_float(v.x); }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 1234.5f) out[0] = acc;
  }
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  printf("device %s sms=%d smem/block optin=%zu l2=%d\n", prop.name, sms, prop.sharedMemPerBlockOptin, prop.l2CacheSize);
  size_t bytes = 4ull << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  float* out; CK(cudaMalloc(&out, 4));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks : {sms, sms * 2, sms * 4}) for (int th : {256, 512, 1024}) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); ldg_stream<<<blocks, th>>>((const int4*)buf, bytes / 16, out); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("LDG  blocks=%d th=%d : %.1f GB/s\n", blocks, th, bytes / best / 1e6);
  }
  auto run_ring = [&](auto kern, int nc, uint32_t tb, int nslots) {
    size_t smem = 1024 + (size_t)tb * nslots;
    if (smem > prop.sharedMemPerBlockOptin) return;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    size_t tiles = bytes / tb;
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); kern<<<sms, 32 * (nc + 1), smem>>>(buf, tiles, tb, nslots, out); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("RING nc=%d tile=%6u slots=%2d inflight=%4zu KB : %.1f GB/s\n", nc, tb, nslots, (size_t)tb * nslots / 1024, bytes / best / 1e6);
  };
  for (uint32_t tb : {8192u, 16384u, 32768u})
    for (int inflight_kb : {64, 128, 160, 192, 208}) {
      int ns = inflight_kb * 1024 / tb; if (ns < 2 || ns > 32) continue;
      if (ns % 2 == 0) run_ring(ring_stream<2>, 2, tb, ns);
      if (ns % 4 == 0) run_ring(ring_stream<4>, 4, tb, ns);
    }
  return 0;
}
