// Microbenchmark: HBM write bandwidth of the dW epilogue's store pattern, 148 persistent CTAs
// writing a 1 GiB fp32 [rows x 2048] buffer in 128-row x 256-col tiles, N-fastest tile order
// (the backward's dW schedule):
//   mode 0: 2-D TMA tensor stores, box {32 cols, 128 rows} (the current epilogue)
//   mode 1: 1-D bulk copies (cp.async.bulk.global.shared::cta), one 1 KB row segment per
//           thread per tile (128 threads, each its own row)
//   mode 2: 1-D bulk copies of 512 B (half rows, 2 per thread per tile)
//   mode 3: st.global.v4 from registers, a warp writes 512 contiguous bytes per instruction
//   mode 4: 1-D bulk copies, 1 KB rows, issued by one elected lane per warp (32 per lane)
//   mode 5: as mode 1 with ONE copy in flight per thread (128 KB per SM: a single staging
//           buffer of one 128 x 256 fp32 tile)
// usage: bulk1d_store <mode> [reps]
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

constexpr int N = 2048, ROWS = 131072;  // 1 GiB
constexpr int TILE_R = 128, TILE_C = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(K) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__global__ void __launch_bounds__(128, 1) store_kernel(float* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int tiles = (ROWS / TILE_R) * (N / TILE_C);
  const int t0 = threadIdx.x;
  // staging: 4 buffers of one tile's rows (128 rows x 1 KB = 128 KB each would not fit: use
  // 2 buffers of 64 KB = 64 rows x 1 KB per half tile)
  float* stage = reinterpret_cast<float*>(sm);
  for (int i = t0; i < 2 * 64 * 256; i += blockDim.x) stage[i] = 1.0f;
  fence_async_smem();
  __syncthreads();
  const int lane = t0 & 31, warp = t0 >> 5;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int nc = (t % (N / TILE_C)) * TILE_C, mr = (t / (N / TILE_C)) * TILE_R;  // N fastest
    if (mode == 1) {
      bulk_wait_read<1>();
      const int r = t0;
      bulk_s2g(out + (size_t)(mr + r) * N + nc, stage + ((r & 63) + 64 * (r >> 6)) * 256 % (2 * 64 * 256), 1024);
      bulk_commit();
    } else if (mode == 2) {
      bulk_wait_read<3>();
      const int r = t0;
      for (int h = 0; h < 2; ++h) {
        bulk_s2g(out + (size_t)(mr + r) * N + nc + h * 128, stage + ((r & 63) * 256 + h * 128), 512);
        bulk_commit();
      }
    } else if (mode == 3) {
      const float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
      for (int r = warp; r < TILE_R; r += 4)
#pragma unroll
        for (int c = 0; c < TILE_C; c += 128)
          *reinterpret_cast<float4*>(out + (size_t)(mr + r) * N + nc + c + lane * 4) = v;
    } else if (mode == 5) {
      bulk_wait_read<0>();
      const int r = t0;
      bulk_s2g(out + (size_t)(mr + r) * N + nc, stage + (r & 63) * 256, 1024);
      bulk_commit();
    } else if (mode == 4) {
      if (lane == 0) {
        bulk_wait_read<0>();
        for (int k = 0; k < 32; ++k) bulk_s2g(out + (size_t)(mr + warp * 32 + k) * N + nc, stage + (k & 63) * 256, 1024);
        bulk_commit();
      }
    }
  }
  bulk_wait_all();
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 1;
  const int reps = argc > 2 ? atoi(argv[2]) : 5;
  float* out;
  cudaMalloc(&out, (size_t)ROWS * N * 4);
  const int smem = 2 * 64 * 1024;
  cudaFuncSetAttribute(store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    store_kernel<<<148, 128, smem>>>(out, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i > 0 && ms < best) best = ms;
  }
  const cudaError_t e = cudaGetLastError();
  printf("mode %d: %.3f ms  %.2f TB/s  (%s)\n", mode, best, (double)ROWS * N * 4 / (best * 1e-3) / 1e12,
         cudaGetErrorString(e));
  return 0;
}
