// Microbenchmark for the F1 load pattern: 2-CTA clusters, CTA q streams D half q of its
// cluster's 128-class tiles ({64, 128} boxes, `stages` in flight), tiles cl, cl + ncl, ...
// Compares against the plain pattern (no cluster, whole D per CTA).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2011_09208_b200/csrc/ptx_sm100.cuh"
using namespace whale;

constexpr int D = 2048;

__global__ void __launch_bounds__(128, 1) f1_load_kernel(const __grid_constant__ CUtensorMap map, int C, int stages,
                                                         int mode, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  __shared__ uint64_t full[16], empty[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (mode & 2) {  // producer (thread 0) / consumer (thread 32) handoff through empty barriers
    const int stage_bytes = 128 * 128;
    const int tiles = (C + 127) / 128;
    int q = 0, cl = blockIdx.x, ncl = gridDim.x, kb0 = 0, kb1 = D / 64;
    if (mode & 1) {
      q = cluster_ctarank();
      cl = cluster_id_x();
      ncl = ncluster_x();
      kb0 = q * (D / 128);
      kb1 = kb0 + D / 128;
    }
    int n = 0;
    for (int t = cl; t < tiles; t += ncl) n += kb1 - kb0;
    if (threadIdx.x == 0) {
      int s = 0; uint32_t ph = 0, i = 0;
      for (int t = cl; t < tiles; t += ncl)
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_arrive_expect_tx(&full[s], stage_bytes);
          tma_load_2d(base + s * stage_bytes, &map, &full[s], kb * 64, t * 128);
          if (++s == stages) { s = 0; ph ^= 1u; }
        }
    } else if (threadIdx.x == 32) {
      int s = 0; uint32_t ph = 0;
      for (int i = 0; i < n; ++i) {
        mbar_wait(&full[s], ph);
        mbar_arrive(&empty[s]);
        if (++s == stages) { s = 0; ph ^= 1u; }
      }
    }
    return;
  }
  if (threadIdx.x != 0) return;
  const int stage_bytes = 128 * 128;
  const int tiles = (C + 127) / 128;
  int q = 0, cl = blockIdx.x, ncl = gridDim.x, kb0 = 0, kb1 = D / 64;
  if (mode & 1) {  // clusters of 2: D halves
    q = cluster_ctarank();
    cl = cluster_id_x();
    ncl = ncluster_x();
    kb0 = q * (D / 128);
    kb1 = kb0 + D / 128;
  }
  int issued = 0, done = 0;
  uint32_t phase[16] = {0};
  for (int t = cl; t < tiles; t += ncl) {
    for (int kb = kb0; kb < kb1; ++kb) {
      const int s = issued % stages;
      if (issued >= stages) {
        mbar_wait(&full[s], phase[s]);
        phase[s] ^= 1;
        ++done;
      }
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      tma_load_2d(base + s * stage_bytes, &map, &full[s], kb * 64, t * 128);
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
  void* fn; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(f1_load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (auto prom : {CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B}) {
    CUtensorMap m;
    cuuint64_t gd[2] = {D, (cuuint64_t)C}, gs[1] = {D * 2};
    cuuint32_t bd[2] = {64, 128}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode : {0, 1, 3}) {
      for (int stages : {4, 8, 12}) {
        int smem = stages * 128 * 128 + 1024;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (mode & 1) ? 2 : 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        for (int it = 0; it < 2; ++it) cudaLaunchKernelEx(&cfg, f1_load_kernel, m, C, stages, mode, sink);
        cudaEventRecord(a);
        for (int it = 0; it < 5; ++it) cudaLaunchKernelEx(&cfg, f1_load_kernel, m, C, stages, mode, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("prom %s mode %d stages %2d: %.0f GB/s  %s\n", prom == CU_TENSOR_MAP_L2_PROMOTION_L2_256B ? "256" : "128",
               mode, stages, 5.0 * C * D * 2 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
