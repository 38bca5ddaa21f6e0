// Fused backward GEMM for sm_100a: dX = G W_r (split-K, fused deterministic fixup /
// NVLink push) and dW_r = G^T X in ONE persistent launch.
//
// Why: at the paper's 100K-class point the backward is HBM-bound and its two GEMMs are
// opposite in kind -- dX streams W_r (read-bound, few long split-K units), dW streams dW_r
// out (write-bound, thousands of one-k-block tiles).  Run back to back, each leaves DRAM
// half idle in its tail (dX: split-K fixup barrier; dW: write-only stream).  Here every CTA
// first takes one dX unit (static: CTA c <- unit c, so the S splits of a tile are
// co-resident for the fixup barrier), then pulls dW tiles from a dynamic scheduler
// (atomic counter), so reads and writes overlap and the dX tail hides under dW stores.
//
//   warp 0      scheduler + TMA producer   (tile ids flow to the other roles via a 4-slot
//                                           smem ring guarded by sfull/sempty mbarriers)
//   warp 1      MMA issuer                  TMEM: 2 accumulators x 256 columns
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: fp32 tile -> swizzled smem -> one 128-row TMA store per 32
//               columns; dX units then run the split-K fixup (gemm_sm100.cuh)
#pragma once
#include "gemm_sm100.cuh"

namespace whale {

struct BwdArgs {
  GemmArgs dx;          // units [0, ux): M = B_tot, N = D, K = C_r (A = G K-major, B = W_r MN-major)
  GemmArgs dw;          // units [ux, ux + tw): M = C_r, N = D, K = B_tot (both MN-major)
  int ux, tw;
  int stages, stage_bytes, epi_bufs;  // epi_bufs: CTA-wide 16 KB store stages
  unsigned* sched_cnt;  // monotonic dynamic-scheduler counter: (e - 1) * (ux + tw) at launch
};

constexpr int kSchedSlots = 4;

template <int ES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    splitfc_bwd_kernel(const __grid_constant__ CUtensorMap tmGx, const __grid_constant__ CUtensorMap tmW,
                       const __grid_constant__ CUtensorMap tmPart, const __grid_constant__ CUtensorMap tmGw,
                       const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDW,
                       const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_fix_go;
  __shared__ int sched_tile[kSchedSlots];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi_smem = smem + a.stages * a.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + a.epi_bufs * 4 * kEpiBufBytes);
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + kSchedSlots;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sempty + kSchedSlots);

  constexpr int kBK = kRowBytes / ES;
  constexpr int kAtom = kRowBytes / ES;
  constexpr int kKStepMN = (32 / ES) * kRowBytes;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int total = a.ux + a.tw;

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    for (int i = 0; i < kSchedSlots; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 1 + 4);  // MMA thread + 4 epilogue warps
    }
    fence_mbar_init();
  }
  if (threadIdx.x == 32) {
    tma_prefetch_desc(&tmGx);
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmPart);
    tma_prefetch_desc(&tmGw);
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmDW);
  }
  if (warp == 2) tmem_alloc(tmem_holder, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();
  pdl_trigger();
  TraceScope _trace(8);
  const uint32_t e = ld_acquire_gpu(a.dx.dev_epoch) + 1u;  // this step's epoch

  if (warp == 0) {
    // ===================== scheduler + TMA producer =====================
    if (lane == 0) {
      const GemmArgs& X = a.dx;
      const GemmArgs& W = a.dw;
      const int dw_bk = W.bk;
      const int dw_box = dw_bk * kRowBytes;
      const int dw_a_bytes = (kBM / kAtom) * dw_box;
      const uint32_t tx_dx = static_cast<uint32_t>(kStageABytes + (X.BN / kAtom) * kBK * kRowBytes);
      const uint32_t tx_dw = static_cast<uint32_t>(dw_a_bytes + (W.BN / kAtom) * dw_box);
      int stage = 0;
      uint32_t phase = 0;
      int unit = blockIdx.x;
      for (int it = 0;; ++it) {
        const int slot = it % kSchedSlots;
        mbar_wait(&sempty[slot], ((it / kSchedSlots) & 1) ^ 1u);
        if (it > 0)
          unit = static_cast<int>(atomicAdd(a.sched_cnt, 1u) - (e - 1u) * static_cast<uint32_t>(total)) + gridDim.x;
        if (unit >= total) unit = -1;
        sched_tile[slot] = unit;
        mbar_arrive(&sfull[slot]);
        if (unit < 0) break;
        int mb, nb, sp, kb0, kb1;
        if (unit < a.ux) {
          decode_tile(X, unit, mb, nb, sp, kb0, kb1);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* sA = smem + stage * a.stage_bytes;
            uint8_t* sB = sA + kStageABytes;
            mbar_arrive_expect_tx(&full[stage], tx_dx);
            tma_load_2d(sA, &tmGx, &full[stage], kb * kBK, mb * kBM);
            for (int j = 0; j < X.BN / kAtom; ++j)
              tma_load_2d(sB + j * kBK * kRowBytes, &tmW, &full[stage], nb * X.BN + j * kAtom, kb * kBK);
            if (++stage == a.stages) {
              stage = 0;
              phase ^= 1u;
            }
          }
        } else {
          decode_tile(W, unit - a.ux, mb, nb, sp, kb0, kb1);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* sA = smem + stage * a.stage_bytes;
            uint8_t* sB = sA + dw_a_bytes;
            mbar_arrive_expect_tx(&full[stage], tx_dw);
#pragma unroll
            for (int j = 0; j < kBM / kAtom; ++j)
              tma_load_2d(sA + j * dw_box, &tmGw, &full[stage], mb * kBM + j * kAtom, kb * dw_bk);
            for (int j = 0; j < W.BN / kAtom; ++j)
              tma_load_2d(sB + j * dw_box, &tmX, &full[stage], nb * W.BN + j * kAtom, kb * dw_bk);
            if (++stage == a.stages) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc_dx = umma_idesc(kBM, a.dx.BN, false, true, ES == 2 ? 1u : 2u);
      const uint32_t idesc_dw = umma_idesc(kBM, a.dw.BN, true, true, ES == 2 ? 1u : 2u);
      const uint32_t dw_box = a.dw.bk * kRowBytes;
      const uint32_t dw_a_bytes = (kBM / kAtom) * dw_box;
      const int dw_kmma = a.dw.bk / (32 / ES);
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        const int slot = it % kSchedSlots;
        mbar_wait(&sfull[slot], (it / kSchedSlots) & 1);
        const int unit = sched_tile[slot];
        mbar_arrive(&sempty[slot]);
        if (unit < 0) break;
        const bool is_dx = unit < a.ux;
        int mb, nb, sp, kb0, kb1;
        if (is_dx) decode_tile(a.dx, unit, mb, nb, sp, kb0, kb1);
        else decode_tile(a.dw, unit - a.ux, mb, nb, sp, kb0, kb1);
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kMaxBN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t aS = smem_u32(smem + stage * a.stage_bytes);
          if (is_dx) {
            const uint32_t bS = aS + kStageABytes;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = umma_sdesc(aS + k * 32, 16, 1024);
              const uint64_t bd = umma_sdesc(bS + k * kKStepMN, kBK * kRowBytes, 1024);
              umma_bf16(d_tmem, ad, bd, idesc_dx, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          } else {
            const uint32_t bS = aS + dw_a_bytes;
            for (int k = 0; k < dw_kmma; ++k) {
              const uint64_t ad = umma_sdesc(aS + k * kKStepMN, dw_box, 1024);
              const uint64_t bd = umma_sdesc(bS + k * kKStepMN, dw_box, 1024);
              umma_bf16(d_tmem, ad, bd, idesc_dw, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[stage]);
          if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;
    const int nbuf = a.epi_bufs;
    int buf = 0;
    for (int it = 0;; ++it) {
      const int slot = it % kSchedSlots;
      mbar_wait(&sfull[slot], (it / kSchedSlots) & 1);
      const int unit = sched_tile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[slot]);
      if (unit < 0) break;
      const bool is_dx = unit < a.ux;
      const GemmArgs& g = is_dx ? a.dx : a.dw;
      int mb, nb, sp, kb0, kb1;
      decode_tile(g, is_dx ? unit : unit - a.ux, mb, nb, sp, kb0, kb1);
      const CUtensorMap* om = is_dx ? &tmPart : &tmDW;
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * kMaxBN + (static_cast<uint32_t>(q * 32) << 16);
      for (int c0 = 0; c0 < g.BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tbase + c0, v);
        tmem_ld_wait();
        if (c0 + 32 >= g.BN) {
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
        if (threadIdx.x == 128) bulk_wait_read_n(nbuf);
        named_bar_sync(1, 128);
        uint8_t* b = epi_smem + buf * 4 * kEpiBufBytes + (q * 32 + lane) * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          *reinterpret_cast<uint4*>(b + ((ch ^ (lane & 7)) << 4)) =
              make_uint4(v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (threadIdx.x == 128) {
          tma_store_3d(om, epi_smem + buf * 4 * kEpiBufBytes, nb * g.BN + c0, mb * kBM, sp);
          bulk_commit();
        }
        if (++buf == nbuf) buf = 0;
      }
      if (is_dx) {
        // ---- split-K fixup (see gemm_sm100.cuh): publish, wait for all splits, reduce 1/S
        if (threadIdx.x == 128) bulk_wait<0>();
        fence_proxy_async_global();
        __threadfence();
        named_bar_sync(1, 128);
        uint32_t* cnt = a.dx.tile_cnt + mb * a.dx.n_blocks + nb;
        if (threadIdx.x == 128) {
          atomicAdd(cnt, 1u);
          const uint32_t target = e * static_cast<uint32_t>(a.dx.splits);
          if (static_cast<int32_t>(ld_acquire_gpu(cnt) - target) < 0) {
            SpinGuard sg;
            while (static_cast<int32_t>(ld_acquire_gpu(cnt) - target) < 0) sg.check(a.dx.err, 16);
          }
        }
        named_bar_sync(1, 128);
        __threadfence();
        fixup_share<ES>(a.dx, mb, nb, sp, threadIdx.x - 128);
      }
    }
    if (threadIdx.x == 128) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
  end_of_step_ticket(a.dx, e, s_fix_go);  // RS flags (N > 1) + epoch++ (last CTA)
}

}  // namespace whale
