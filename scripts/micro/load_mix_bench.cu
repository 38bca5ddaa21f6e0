// Microbenchmark: the logits GEMM's operand stream without the MMA -- per stage one W box
// {64, BN} (HBM, this CTA's class rows) plus optionally one X box {64, XR} (a small matrix all
// CTAs read: L2 hits), `stages` in flight per CTA, one tile of D = 2048 per CTA (the N = 4
// shard shape: 131 CTAs x 192 classes).  Prints the W bandwidth.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2011_09208_b200/csrc/ptx_sm100.cuh"
using namespace whale;

constexpr int D = 2048;

__global__ void __launch_bounds__(128, 1) mix_kernel(const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap mx,
                                                     int C, int BN, int XR, int stages, int tiles_per_cta, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int wbytes = BN * 128, xbytes = XR * 128, stage_bytes = wbytes + xbytes;
  const int tiles = (C + BN - 1) / BN;
  const int kbs = D / 64;
  int issued = 0, done = 0;
  uint32_t phase[16] = {0};
  for (int i = 0; i < tiles_per_cta; ++i) {
    const int t = blockIdx.x + i * gridDim.x;
    if (t >= tiles) break;
    for (int kb = 0; kb < kbs; ++kb) {
      const int s = issued % stages;
      if (issued >= stages) {
        mbar_wait(&full[s], phase[s]);
        phase[s] ^= 1;
        ++done;
      }
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      tma_load_2d(base + s * stage_bytes, &mw, &full[s], kb * 64, t * BN);
      if (XR) tma_load_2d(base + s * stage_bytes + wbytes, &mx, &full[s], kb * 64, 0);
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
  const int C = 25000;
  void *w, *x;
  cudaMalloc(&w, (size_t)C * D * 2);
  cudaMemset(w, 0, (size_t)C * D * 2);
  cudaMalloc(&x, (size_t)256 * D * 2);
  cudaMemset(x, 0, (size_t)256 * D * 2);
  int* sink;
  cudaMalloc(&sink, 4);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int BN = 192;
  CUtensorMap mw, mx;
  cuuint64_t gd[2] = {D, (cuuint64_t)C}, gs[1] = {D * 2};
  cuuint32_t bd[2] = {64, (cuuint32_t)BN}, es[2] = {1, 1};
  enc(&mw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  for (int XR : {0, 64, 128}) {
    cuuint64_t gx[2] = {D, 256};
    cuuint32_t bx[2] = {64, (cuuint32_t)(XR ? XR : 64)};
    enc(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, gx, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int stages : {4, 5, 6, 8}) {
      const int sb = BN * 128 + XR * 128;
      if (stages * sb + 1024 > 220 * 1024) continue;
      for (int grid : {131, 148}) {
        const int tiles = (C + BN - 1) / BN, tpc = (tiles + grid - 1) / grid;
        int smem = stages * sb + 1024;
        for (int it = 0; it < 2; ++it) mix_kernel<<<grid, 128, smem>>>(mw, mx, C, BN, XR, stages, tpc, sink);
        cudaEventRecord(a);
        for (int it = 0; it < 10; ++it) mix_kernel<<<grid, 128, smem>>>(mw, mx, C, BN, XR, stages, tpc, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("X rows %3d stages %d (W %3d KB + X %3d KB in flight) grid %3d: %6.1f us/launch, W %.0f GB/s  %s\n", XR,
               stages, stages * BN * 128 / 1024, stages * XR * 128 / 1024, grid, ms * 100, 10.0 * C * D * 2 / (ms / 1e3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
