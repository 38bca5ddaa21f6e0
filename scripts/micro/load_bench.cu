// Microbenchmark: HBM read bandwidth of TMA tile loads (the logits GEMM's W stream):
// each CTA streams its own class rows of a [C x 2048] bf16 matrix in K-major boxes
// {64, BN}; stages x box bytes in flight per SM; no MMA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2011_09208_b200/csrc/ptx_sm100.cuh"
using namespace whale;

constexpr int D = 2048;

__global__ void __launch_bounds__(128, 1) tma_load_kernel(const __grid_constant__ CUtensorMap map, int C, int BN,
                                                          int stages, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int stage_bytes = BN * 128;
  const int tiles = (C + BN - 1) / BN;
  const int kbs = D / 64;
  int issued = 0, done = 0;
  uint32_t phase[16] = {0};
  // flat sequence of (tile, kb) loads; keep `stages` in flight
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    for (int kb = 0; kb < kbs; ++kb) {
      const int s = issued % stages;
      if (issued >= stages) {  // wait for the load that used this slot
        mbar_wait(&full[s], phase[s]);
        phase[s] ^= 1;
        ++done;
      }
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      tma_load_2d(base + s * stage_bytes, &map, &full[s], kb * 64, t * BN);
      ++issued;
    }
  }
  while (done < issued) {
    const int s = done % stages;
    mbar_wait(&full[s], phase[s]);
    phase[s] ^= 1;
    ++done;
  }
  if (issued < 0) *sink = 1;
}

int main() {
  const int C = 100000;
  void* buf;
  cudaMalloc(&buf, (size_t)C * D * 2);
  cudaMemset(buf, 0, (size_t)C * D * 2);
  int* sink;
  cudaMalloc(&sink, 4);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(tma_load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int BN : {128, 192, 256}) {
    CUtensorMap m;
    cuuint64_t gd[2] = {D, (cuuint64_t)C}, gs[1] = {D * 2};
    cuuint32_t bd[2] = {64, (cuuint32_t)BN}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int stages : {2, 4, 6, 8, 12, 16}) {
      if (stages * BN * 128 + 1024 > 220 * 1024) continue;
      for (int grid : {74, 148}) {
        int smem = stages * BN * 128 + 1024;
        for (int it = 0; it < 2; ++it) tma_load_kernel<<<grid, 128, smem>>>(m, C, BN, stages, sink);
        cudaEventRecord(a);
        for (int it = 0; it < 5; ++it) tma_load_kernel<<<grid, 128, smem>>>(m, C, BN, stages, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("BN %d stages %2d (%3d KB in flight) grid %3d: %.0f GB/s  %s\n", BN, stages, stages * BN * 128 / 1024,
               grid, 5.0 * C * D * 2 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
