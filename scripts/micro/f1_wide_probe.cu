// Probe for a single-W-pass forward at B_tot = 64 (the N = 2 shard shape): the data movement and
// MMAs of an F1-like kernel with KC-CTA clusters splitting D, without the softmax / Z exchange.
//
// Per CTA (D part q of its cluster's 128-class tiles t = cluster, cluster + nclusters, ...):
//   G1: Z^T [128 classes x NB rows] += W_t chunk (K-major [128 x 64 D]) * X chunk^T ([NB x 64 D]),
//       D_q / 64 chunks per tile through ring 1 (W 16 KB + X NB*128 B per slot) from HBM;
//   G2: U^T block [128 D rows x NB] += W_t^T (the same W, MN-major, re-read from L2) * P^T
//       (a zero operand in smem), D_q / 128 blocks per tile through ring 2 (32 KB slots),
//       started when the tile's G1 is done (the real kernel waits for the softmax on top).
// KC = 2, NB = 32 is today's F1 pattern at N = 1 (calibration); KC = 4, NB = 64 the proposed
// B_tot = 64 kernel.  Prints us per launch and the W stream rate.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2011_09208_b200/csrc/ptx_sm100.cuh"
using namespace whale;

constexpr int D = 2048;

__global__ void __launch_bounds__(128, 1) probe_kernel(const __grid_constant__ CUtensorMap mw,
                                                       const __grid_constant__ CUtensorMap mx, int C, int KC, int NB,
                                                       int S1, int S2, int* sink) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t full1[8], empty1[8], full2[8], empty2[8], g1done[2], g2done[2];
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t q = cluster_ctarank();
  const int cl = static_cast<int>(cluster_id_x()), ncl = static_cast<int>(ncluster_x());
  const int Dq = D / KC, KQ = Dq / 64, NBLK = Dq / 128;
  const int slot1 = 16384 + NB * 128, slot2 = 32768;
  uint8_t* ring1 = sm;
  uint8_t* ring2 = ring1 + S1 * slot1;
  uint8_t* pbuf = ring2 + S2 * slot2;  // P^T operand: 2 atoms x NB rows x 128 B (zeros)
  const int tiles = (C + 127) / 128;
  const int my_tiles = cl < tiles ? (tiles - 1 - cl) / ncl + 1 : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S1; ++i) { mbar_init(&full1[i], 1); mbar_init(&empty1[i], 1); }
    for (int i = 0; i < S2; ++i) { mbar_init(&full2[i], 1); mbar_init(&empty2[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&g1done[i], 1); mbar_init(&g2done[i], 1); }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 2 * NB * 128 / 16; i += blockDim.x) reinterpret_cast<uint4*>(pbuf)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (warp == 2) tmem_alloc(&tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const int d0 = static_cast<int>(q) * Dq;
  if (warp == 0 && lane == 0) {  // G1 producer
    const uint64_t keep = l2_policy_evict_last();
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < my_tiles; ++it) {
      const int row0 = (cl + it * ncl) * 128;
      for (int k = 0; k < KQ; ++k) {
        mbar_wait(&empty1[st], ph ^ 1u);
        uint8_t* s = ring1 + st * slot1;
        mbar_arrive_expect_tx(&full1[st], slot1);
        tma_load_2d_hint(s, &mw, &full1[st], d0 + k * 64, row0, keep);
        tma_load_2d(s + 16384, &mx, &full1[st], d0 + k * 64, 0);
        if (++st == S1) { st = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 3 && lane == 0) {  // G2 producer (L2 re-reads of the same W)
    const uint64_t drop = l2_policy_evict_first();
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < my_tiles; ++it) {
      const int row0 = (cl + it * ncl) * 128;
      for (int m = 0; m < NBLK; ++m) {
        mbar_wait(&empty2[st], ph ^ 1u);
        uint8_t* s = ring2 + st * slot2;
        mbar_arrive_expect_tx(&full2[st], slot2);
        tma_load_2d_hint(s, &mw, &full2[st], d0 + (2 * m) * 64, row0, drop);
        tma_load_2d_hint(s + 16384, &mw, &full2[st], d0 + (2 * m + 1) * 64, row0, drop);
        if (++st == S2) { st = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1 && lane == 0) {  // G1 MMA
    const uint32_t idesc1 = umma_idesc(128, NB, false, false, 1u);
    int st = 0; uint32_t ph = 0;
    const uint32_t r1 = smem_u32(ring1);
    for (int it = 0; it < my_tiles; ++it) {
      // G1 runs at most two tiles ahead of G2 (the real kernel's Z buffers); also keeps the
      // g1done / g2done parities unambiguous
      if (it >= 2) mbar_wait(&g2done[(it - 2) & 1], ((it - 2) >> 1) & 1);
      for (int k = 0; k < KQ; ++k) {
        mbar_wait(&full1[st], ph);
        tc_fence_after();
        const uint32_t aS = r1 + st * slot1, bS = aS + 16384;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem, umma_sdesc(aS + kk * 32, 16, 1024), umma_sdesc(bS + kk * 32, 16, 1024), idesc1,
                    (k > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&empty1[st]);
        if (++st == S1) { st = 0; ph ^= 1u; }
      }
      umma_commit(&g1done[it & 1]);
    }
  } else if (warp == 2 && lane == 0) {  // G2 MMA (after the tile's G1)
    const uint32_t idesc2 = umma_idesc(128, NB, true, false, 1u);
    int st = 0; uint32_t ph = 0;
    const uint32_t r2 = smem_u32(ring2), ps = smem_u32(pbuf);
    for (int it = 0; it < my_tiles; ++it) {
      mbar_wait(&g1done[it & 1], (it >> 1) & 1);
      tc_fence_after();
      for (int i = 0; i < NBLK; ++i) {
        mbar_wait(&full2[st], ph);
        tc_fence_after();
        const uint32_t aS = r2 + st * slot2;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tmem + 64 + i * NB, umma_sdesc(aS + kk * 2048, 16384, 1024),
                    umma_sdesc(ps + (kk >> 2) * (NB * 128) + (kk & 3) * 32, 16, 1024), idesc2, (it > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&empty2[st]);
        if (++st == S2) { st = 0; ph ^= 1u; }
      }
      umma_commit(&g2done[it & 1]);
    }
    if (my_tiles > 0) mbar_wait(&g2done[(my_tiles - 1) & 1], ((my_tiles - 1) >> 1) & 1);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) { tc_fence_after(); tmem_dealloc(tmem, 512); }
  if (my_tiles < 0) *sink = 1;
}

int main() {
  void* fn; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  int* sink; cudaMalloc(&sink, 4);
  struct Cfg { int C, KC, NB, S1, S2; };
  const Cfg cfgs[] = {{100000, 2, 32, 4, 3}, {50000, 2, 32, 4, 3}, {50000, 4, 64, 4, 3}, {50000, 4, 64, 4, 2},
                      {50000, 4, 64, 3, 2}, {50000, 4, 64, 5, 2}};
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (const Cfg& c : cfgs) {
    void *w, *x;
    cudaMalloc(&w, (size_t)c.C * D * 2);
    cudaMemset(w, 0, (size_t)c.C * D * 2);
    cudaMalloc(&x, (size_t)c.NB * D * 2);
    cudaMemset(x, 0, (size_t)c.NB * D * 2);
    CUtensorMap mw, mx;
    cuuint64_t gd[2] = {D, (cuuint64_t)c.C}, gs[1] = {D * 2}, gx[2] = {D, (cuuint64_t)c.NB};
    cuuint32_t bw[2] = {64, 128}, bx[2] = {64, (cuuint32_t)c.NB}, es[2] = {1, 1};
    enc(&mw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, gd, gs, bw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, gx, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 1024 + c.S1 * (16384 + c.NB * 128) + c.S2 * 32768 + 2 * c.NB * 128;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.KC; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.gridDim = dim3(c.KC);
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, probe_kernel, &cfg);
    cfg.gridDim = dim3(c.KC * ncl);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) cudaLaunchKernelEx(&cfg, probe_kernel, mw, mx, c.C, c.KC, c.NB, c.S1, c.S2, sink);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) cudaLaunchKernelEx(&cfg, probe_kernel, mw, mx, c.C, c.KC, c.NB, c.S1, c.S2, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("C %6d KC %d NB %2d S1 %d S2 %d: %3d clusters, smem %6d B: %6.1f us/launch, W %.0f GB/s  %s\n", c.C, c.KC, c.NB,
           c.S1, c.S2, ncl, smem, ms * 100, 10.0 * c.C * D * 2 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(w); cudaFree(x);
  }
  return 0;
}
