// Microbenchmark: HBM write bandwidth of TMA bulk-tensor stores (various boxes) vs
// coalesced st.global, 148 persistent CTAs writing a 1 GiB fp32 [rows x 2048] buffer in
// 128-row x 256-col tiles (the dW epilogue's pattern).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2011_09208_b200/csrc/ptx_sm100.cuh"
using namespace whale;

constexpr int N = 2048, ROWS = 131072;  // 1 GiB
constexpr int TILE_R = 128, TILE_C = 256;

__global__ void __launch_bounds__(128, 1) tma_store_kernel(const __grid_constant__ CUtensorMap map, int box_rows, int nbuf, int order) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const int tiles = (ROWS / TILE_R) * (N / TILE_C);
  // fill staging buffers once
  for (int i = threadIdx.x; i < nbuf * 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 1.0f;
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x != 0) return;
  int buf = 0;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    int mr, nc;
    if (order == 0) { mr = (t % (ROWS / TILE_R)) * TILE_R; nc = (t / (ROWS / TILE_R)) * TILE_C; }
    else if (order == 1) { nc = (t % (N / TILE_C)) * TILE_C; mr = (t / (N / TILE_C)) * TILE_R; }
    else {  // order 2: CTA-contiguous -- this CTA's tiles walk whole 8 KB rows
      const int rb = t / (N / TILE_C);
      nc = (t % (N / TILE_C)) * TILE_C; mr = rb * TILE_R;
      // remap so that consecutive tiles of ONE cta cover the same row block
      const int per = tiles / gridDim.x;
      (void)per;
    }
    for (int c0 = 0; c0 < TILE_C; c0 += 32) {
      for (int r0 = 0; r0 < TILE_R; r0 += box_rows) {
        bulk_wait_read<7>();
        tma_store_2d(&map, base + buf * 16384, nc + c0, mr + r0);
        bulk_commit();
        buf = (buf + 1) % nbuf;
      }
    }
  }
  bulk_wait<0>();
}

__global__ void __launch_bounds__(256) stg_kernel(float* out) {
  // coalesced: a warp writes 4 rows x 128 B per instruction
  const int tiles = (ROWS / TILE_R) * (N / TILE_C);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int mr = (t % (ROWS / TILE_R)) * TILE_R, nc = (t / (ROWS / TILE_R)) * TILE_C;
    for (int c0 = 0; c0 < TILE_C; c0 += 32)
      for (int r = warp * 4 + (lane >> 3); r < TILE_R; r += 32) {
        float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
        __stcs(reinterpret_cast<float4*>(out + (size_t)(mr + r) * N + nc + c0 + (lane & 7) * 4), v);
      }
  }
}

__global__ void __launch_bounds__(128, 1) tma_store_contig(const __grid_constant__ CUtensorMap map, int nbuf) {
  // map: [ROWS*N/32 rows x 32 cols] fp32 = fully contiguous rows of 128 B
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < nbuf * 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 1.0f;
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long rows = (long long)ROWS * N / 32;
  int buf = 0;
  for (long long r0 = (long long)blockIdx.x * 128; r0 < rows; r0 += (long long)gridDim.x * 128) {
    bulk_wait_read<7>();
    tma_store_2d(&map, base + buf * 16384, 0, (int)r0);
    bulk_commit();
    buf = (buf + 1) % nbuf;
  }
  bulk_wait<0>();
}

int main() {
  float* out;
  cudaMalloc(&out, (size_t)ROWS * N * 4);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int order : {1})
  for (int box_rows : {32, 128}) {
    for (int sw : {1}) {
      CUtensorMap m;
      cuuint64_t gd[2] = {N, ROWS}, gs[1] = {N * 4};
      cuuint32_t bd[2] = {32, (cuuint32_t)box_rows}, es[2] = {1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      int smem = 8 * 16384 + 1024;
      cudaFuncSetAttribute(tma_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int it = 0; it < 3; ++it) tma_store_kernel<<<148, 128, smem>>>(m, box_rows, 8, order);
      cudaEventRecord(a);
      for (int it = 0; it < 5; ++it) tma_store_kernel<<<148, 128, smem>>>(m, box_rows, 8, order);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("order %d tma box {32,%d} sw%d: %.1f GB/s  (%s)\n", order, box_rows, sw, 5.0 * ROWS * N * 4 / (ms / 1e3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  {
    CUtensorMap m;
    cuuint64_t gd[2] = {32, (cuuint64_t)ROWS * N / 32}, gs[1] = {128};
    cuuint32_t bd[2] = {32, 128}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int smem = 8 * 16384 + 1024;
    cudaFuncSetAttribute(tma_store_contig, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int it = 0; it < 3; ++it) tma_store_contig<<<148, 128, smem>>>(m, 8);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) tma_store_contig<<<148, 128, smem>>>(m, 8);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("tma contiguous 16KB boxes: %.1f GB/s (%s)\n", 5.0 * ROWS * N * 4 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  for (int grid : {148}) {
    for (int it = 0; it < 3; ++it) stg_kernel<<<grid, 256>>>(out);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) stg_kernel<<<grid, 256>>>(out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("st.global.cs grid %d: %.1f GB/s\n", grid, 5.0 * ROWS * N * 4 / (ms / 1e3) / 1e9);
  }
  return 0;
}
