// Microbenchmark: per-SM TMA ingest (global -> shared) from L2-resident vs HBM-resident data,
// 148 CTAs, 16 KB boxes ({64 bf16, 128 rows}, SW128) into a ring of S slots, one producer
// thread that re-issues a slot as soon as its previous load landed (no consumer work).
//   usage: tma_ingest <slots> <src MB> [iters]
// src MB <= 64: L2-resident (after the first pass); src MB >= 1024: streams from HBM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(32, 1) ingest_kernel(const __grid_constant__ CUtensorMap map, int slots, int rows_total,
                                                       int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < slots; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const int boxes = rows_total / 128;
  int b = blockIdx.x;
  uint32_t phase[16] = {};
  for (int it = 0; it < iters; ++it) {
    const int s = it % slots;
    if (it >= slots) {  // wait for the slot's previous load
      const uint32_t a = smem_u32(&bar[s]);
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                     : "=r"(ok) : "r"(a), "r"(phase[s]));
      phase[s] ^= 1u;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(16384));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(base + s * 16384)), "l"(&map), "r"(smem_u32(&bar[s])), "r"(0), "r"((b % boxes) * 128));
    b += gridDim.x;
  }
  for (int s = 0; s < slots; ++s) {
    const uint32_t a = smem_u32(&bar[s]);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                   : "=r"(ok) : "r"(a), "r"(phase[s]));
  }
  sink[blockIdx.x] = *reinterpret_cast<volatile unsigned long long*>(base);
}

int main(int argc, char** argv) {
  const int slots = argc > 1 ? atoi(argv[1]) : 6;
  const long long mb = argc > 2 ? atoll(argv[2]) : 32;
  const int iters = argc > 3 ? atoi(argv[3]) : 2000;
  const long long rows = mb * 1024 * 1024 / 128;  // rows of 128 B (64 bf16)
  void* src;
  cudaMalloc(&src, rows * 128);
  cudaMemset(src, 0, rows * 128);
  unsigned long long* sink;
  cudaMalloc(&sink, 148 * 8);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m;
  cuuint64_t gd[2] = {64, (cuuint64_t)rows}, gs[1] = {128};
  cuuint32_t bd[2] = {64, 128}, es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = slots * 16384 + 1024;
  cudaFuncSetAttribute(ingest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  ingest_kernel<<<148, 32, smem>>>(m, slots, (int)rows, iters, sink);
  cudaEventRecord(a);
  ingest_kernel<<<148, 32, smem>>>(m, slots, (int)rows, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 148.0 * iters * 16384;
  printf("slots %2d src %5lld MB: %.1f GB/s total, %.1f GB/s per SM (%s)\n", slots, mb, bytes / (ms * 1e-3) / 1e9,
         bytes / 148 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
