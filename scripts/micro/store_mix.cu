// Microbenchmark: fp32 HBM write bandwidth for the dW output pattern (1 GiB [rows x 2048]),
// comparing plain vector stores (16 B / 32 B, many CTAs vs a persistent grid) with the TMA
// tile stores the dW epilogue uses, and a mix of both paths inside one persistent CTA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2011_09208_b200/csrc/ptx_sm100.cuh"
using namespace whale;

constexpr int N = 2048, ROWS = 131072;  // 1 GiB fp32
constexpr int TILE_R = 128, TILE_C = 256;

__global__ void fill16(float4* o, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    o[i] = make_float4(1.f, 1.f, 1.f, 1.f);
}
__global__ void fill32(float* o, long long n8) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const float a = 1.f;
    asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(o + i * 8), "f"(a) : "memory");
  }
}
// persistent tile writer: 148 CTAs x (4 TMA-warps-worth via one thread + 8 st.global warps);
// frac_tma of every tile's 32-column chunks go through TMA (16 KB boxes), the rest via STG.256
// in row-contiguous 1 KB pieces (a warp writes 32 lanes x 32 B = one row's 256 columns).
__global__ void __launch_bounds__(384, 1) mix_kernel(const __grid_constant__ CUtensorMap map, float* out, int tma_chunks) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 8 * 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 1.0f;
  fence_proxy_async_smem();
  __syncthreads();
  const int tiles = (ROWS / TILE_R) * (N / TILE_C);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int buf = 0;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int nc = (t % (N / TILE_C)) * TILE_C, mr = (t / (N / TILE_C)) * TILE_R;
    if (threadIdx.x == 0) {
      for (int c = 0; c < tma_chunks; ++c) {
        bulk_wait_read<7>();
        tma_store_2d(&map, base + buf * 16384, nc + c * 32, mr);
        bulk_commit();
        buf = (buf + 1) % 8;
      }
    } else if (warp >= 4) {
      // STG part: columns [tma_chunks*32, 256) of the tile's 128 rows; each lane 8 floats
      const int c_lo = tma_chunks * 32, ncols = TILE_C - c_lo;
      if (ncols > 0) {
        const int lanes_per_row = ncols / 8;  // 32 B per lane
        const int rows_per_pass = 32 / lanes_per_row > 0 ? 32 / lanes_per_row : 1;
        for (int r = (warp - 4) * rows_per_pass + lane / lanes_per_row; r < TILE_R; r += 8 * rows_per_pass) {
          const int col = c_lo + (lane % lanes_per_row) * 8;
          if (lane / lanes_per_row < rows_per_pass) {
            const float a = 1.f;
            asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(out + (size_t)(mr + r) * N + nc + col),
                         "f"(a) : "memory");
          }
        }
      }
    }
  }
  if (threadIdx.x == 0) bulk_wait<0>();
}

// the dW epilogue's natural layout: thread = one tile row (TMEM lane), 32 consecutive columns
// per TMEM load -> 4 x STG.256 (full 32-byte sectors) per thread, rows 8 KB apart within a warp
__global__ void __launch_bounds__(256, 1) rowthread_kernel(float* out) {
  const int tiles = (ROWS / TILE_R) * (N / TILE_C);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int nc = (t % (N / TILE_C)) * TILE_C, mr = (t / (N / TILE_C)) * TILE_R;
    if (warp >= 4) {
      const int r = (warp - 4) * 32 + lane;
      for (int c0 = 0; c0 < TILE_C; c0 += 32)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float a = 1.f;
          asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(out + (size_t)(mr + r) * N + nc + c0 + 8 * k),
                       "f"(a) : "memory");
        }
    }
  }
}

int main() {
  float* out;
  cudaMalloc(&out, (size_t)ROWS * N * 4);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double bytes = (double)ROWS * N * 4;
  auto timeit = [&](const char* name, auto&& launch) {
    for (int it = 0; it < 3; ++it) launch();
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-44s %.0f GB/s  (%s)\n", name, 5.0 * bytes / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  const long long n4 = (long long)ROWS * N / 4, n8 = n4 / 2;
  for (int g : {148, 148 * 4, 148 * 16}) {
    char nm[64];
    snprintf(nm, 64, "fill16 grid %d x 256", g); timeit(nm, [&] { fill16<<<g, 256>>>((float4*)out, n4); });
    snprintf(nm, 64, "fill32 (STG.256) grid %d x 256", g); timeit(nm, [&] { fill32<<<g, 256>>>(out, n8); });
  }
  CUtensorMap m;
  cuuint64_t gd[2] = {N, ROWS}, gs[1] = {N * 4};
  cuuint32_t bd[2] = {32, 128}, es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 8 * 16384 + 1024;
  cudaFuncSetAttribute(mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int tc : {8, 6, 4, 2, 0}) {
    char nm[64];
    snprintf(nm, 64, "persistent mix: %d/8 chunks TMA, rest STG.256", tc);
    timeit(nm, [&] { mix_kernel<<<148, 384, smem>>>(m, out, tc); });
  }
  timeit("persistent row-thread STG.256 (4 warps)", [&] { rowthread_kernel<<<148, 256>>>(out); });
  return 0;
}
