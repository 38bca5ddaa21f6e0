// Persistent, warp-specialised tcgen05 GEMM for sm_100a with the split-FC epilogues.
//
//   D[M x N] = A[M x K] * B[N x K]^T    (bf16 operands, fp32 accumulator in TMEM)
//
// A and B are each either K-major (K contiguous) or MN-major (M/N contiguous); both are
// fed by TMA into 128B-swizzled shared memory and consumed by tcgen05.mma issued from one
// thread.  One CTA per SM, grid = min(#tiles, #SMs), static round-robin tile order with
// M fastest (CTAs running concurrently share the same B tile -> it is read from HBM once).
//
//   warp 0      TMA producer (one lane)       smem ring: full/empty mbarriers
//   warp 1      MMA issuer (one lane)         TMEM ring: 2 accumulators x 256 columns
//   warp 2      TMEM allocator
//   warps 4..7  epilogue (TMEM lane quadrant = warp % 4, one thread per output row)
//
// Epilogues:
//   EPI_FWD_STATS  split-FC forward (north star (b)): the logits tile
//                  Z = X W_r^T never leaves the SM as fp32.  Per row and class tile the
//                  epilogue writes m_tile = max_j z, s_tile = sum_j exp(z - m_tile),
//                  P~ = exp(z - m_tile) (bf16, TMA store) and captures the label logit
//                  z_y when the label falls in this tile.
//   EPI_STORE_F32  fp32 tile store through a swizzled smem stage + TMA (3-D map:
//                  {N, M, split}); used for dW (A7) and the split-K dX partials (A8).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "ptx_sm100.cuh"

namespace whale {

enum EpiKind : int { EPI_FWD_STATS = 0, EPI_STORE_F32 = 1 };

constexpr int kBM = 128;               // MMA M (rows of A per tile)
constexpr int kRowBytes = 128;         // one SWIZZLE_128B row: K elements per stage = 128 / ES
constexpr int kMaxBN = 256;            // accumulator columns per TMEM buffer
constexpr int kGemmThreads = 256;      // 8 warps
constexpr int kStageABytes = kBM * kRowBytes;   // 16 KB
constexpr int kEpiBufBytes = 4096;     // per epilogue warp per buffer: 32 rows x 128 B
constexpr int kEpiBytes = 4 * 2 * kEpiBufBytes;
constexpr int kTmemCols = 512;

struct GemmArgs {
  int M, N;                 // valid output rows / cols
  int BN;                   // N tile (multiple of 128/ES when B is MN-major or EPI_FWD_STATS)
  int m_blocks, n_blocks, splits;
  int num_kb, kb_per_split; // k-blocks of 128/ES elements
  int num_tiles;
  int stages;
  int stage_bytes;
  // EPI_FWD_STATS
  const int32_t* labels;    // [M] global class ids
  long long class_offset;   // first class of this shard
  float* m_tile;            // [M x n_blocks]
  float* s_tile;            // [M x n_blocks]
  float* zy;                // [M] label logit (written by the owner tile only)
  // producer-side wait for peer data (NVLink all-gather) before the first A load
  const uint32_t* wait_flags;  // [wait_count] local flag words, NULL = no wait
  int wait_count;
  uint32_t wait_epoch;
  int* err;
};

__host__ __device__ inline int gemm_smem_bytes(int stages, int stage_bytes) {
  return 1024 /*align slack*/ + stages * stage_bytes + kEpiBytes + 256 /*barriers*/;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void decode_tile(const GemmArgs& a, int tile, int& mb, int& nb, int& sp, int& kb0,
                                            int& kb1) {
  mb = tile % a.m_blocks;
  const int r = tile / a.m_blocks;
  nb = r % a.n_blocks;
  sp = r / a.n_blocks;
  kb0 = sp * a.kb_per_split;
  kb1 = min(kb0 + a.kb_per_split, a.num_kb);
}

// ES = operand element size: 2 -> bf16 (kind::f16), 4 -> fp32 storage run as kind::tf32.
template <int EPI, bool A_MN, bool B_MN, int ES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    splitfc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmOut, const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi_smem = smem + a.stages * a.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + kEpiBytes);
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  constexpr int kBK = kRowBytes / ES;        // K elements per stage
  constexpr int kAtom = kRowBytes / ES;      // MN elements per swizzle atom (MN-major)
  constexpr int kBoxBytes = kBK * kRowBytes; // one MN-major box {kAtom, kBK}
  constexpr int kKStepMN = (32 / ES) * kRowBytes;  // MN-major: UMMA_K rows per MMA
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    fence_mbar_init();
  }
  if (threadIdx.x == 32) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmOut);
  }
  if (warp == 2) tmem_alloc(tmem_holder, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      if (a.wait_flags != nullptr) {
        // peers' rows of A were pushed over NVLink by generic-proxy stores; acquire their
        // flags, then order the async-proxy (TMA) reads after them.
        for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, a.wait_epoch, a.err, 8);
        fence_proxy_async_global();
      }
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t tx = static_cast<uint32_t>(kStageABytes + a.BN * kRowBytes);
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
        int mb, nb, sp, kb0, kb1;
        decode_tile(a, tile, mb, nb, sp, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* sA = smem + stage * a.stage_bytes;
          uint8_t* sB = sA + kStageABytes;
          mbar_arrive_expect_tx(&full[stage], tx);
          if (!A_MN) {
            tma_load_2d(sA, &tmA, &full[stage], kb * kBK, mb * kBM);
          } else {
#pragma unroll
            for (int j = 0; j < kBM / kAtom; ++j)
              tma_load_2d(sA + j * kBoxBytes, &tmA, &full[stage], mb * kBM + j * kAtom, kb * kBK);
          }
          if (!B_MN) {
            tma_load_2d(sB, &tmB, &full[stage], kb * kBK, nb * a.BN);
          } else {
            for (int j = 0; j < a.BN / kAtom; ++j)
              tma_load_2d(sB + j * kBoxBytes, &tmB, &full[stage], nb * a.BN + j * kAtom, kb * kBK);
          }
          if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(kBM, a.BN, A_MN, B_MN, ES == 2 ? 1u : 2u);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++it) {
        int mb, nb, sp, kb0, kb1;
        decode_tile(a, tile, mb, nb, sp, kb0, kb1);
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kMaxBN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t aS = smem_u32(smem + stage * a.stage_bytes);
          const uint32_t bS = aS + kStageABytes;
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 MMAs x 32 bytes of K per 128-byte row
            const uint64_t ad = A_MN ? umma_sdesc(aS + k * kKStepMN, kBoxBytes, 1024)
                                     : umma_sdesc(aS + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_sdesc(bS + k * kKStepMN, kBoxBytes, 1024)
                                     : umma_sdesc(bS + k * 32, 16, 1024);
            if constexpr (ES == 2)
              umma_bf16(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            else
              umma_tf32(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);  // frees this smem stage once the MMAs have read it
          if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    uint8_t* ebuf = epi_smem + q * 2 * kEpiBufBytes;
    int buf = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++it) {
      int mb, nb, sp, kb0, kb1;
      decode_tile(a, tile, mb, nb, sp, kb0, kb1);
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * kMaxBN + (static_cast<uint32_t>(q * 32) << 16);
      const int row0 = mb * kBM + q * 32;  // first output row of this warp
      const int row = row0 + lane;
      if (row0 < a.M) {  // warp-uniform: skip warps whose rows are all padding
        if constexpr (EPI == EPI_STORE_F32) {
          for (int c0 = 0; c0 < a.BN; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + c0, v);
            tmem_ld_wait();
            if (lane == 0) bulk_wait_read<1>();  // the store that last used this buffer has read it
            __syncwarp();
            uint8_t* b = ebuf + buf * kEpiBufBytes + lane * 128;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch)
              *reinterpret_cast<uint4*>(b + ((ch ^ (lane & 7)) << 4)) =
                  make_uint4(v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&tmOut, ebuf + buf * kEpiBufBytes, nb * a.BN + c0, row0, sp);
              bulk_commit();
            }
            buf ^= 1;
          }
        } else {
          const bool rv = row < a.M;
          const int ncol = min(a.BN, a.N - nb * a.BN);  // valid classes in this tile
          constexpr float kLog2e = 1.4426950408889634f;
          // pass 1: row max over the tile's valid classes
          float mx = -INFINITY;
          for (int c0 = 0; c0 < a.BN; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c0 + c < ncol) mx = fmaxf(mx, __uint_as_float(v[c]));
          }
          long long yl = -1;
          if (rv) yl = static_cast<long long>(a.labels[row]) - a.class_offset - static_cast<long long>(nb) * a.BN;
          const float mxl = mx * kLog2e;
          float s = 0.f, zy = 0.f;
          // pass 2: P~ = exp(z - m_tile) -> tile store (bf16, or fp32 for ES=4); s_tile; z_y
          constexpr int kChunk = kRowBytes / ES;  // P~ columns per 128-byte smem row
          for (int c0 = 0; c0 < a.BN; c0 += kChunk) {
            uint32_t v[64];
            tmem_ld32(tbase + c0, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
            if constexpr (kChunk == 64) tmem_ld32(tbase + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
            tmem_ld_wait();
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < kChunk; c += 2) {
              const float z0 = __uint_as_float(v[c]);
              const float z1 = __uint_as_float(v[c + 1]);
              const float p0 = (c0 + c < ncol) ? ex2_approx(fmaf(z0, kLog2e, -mxl)) : 0.f;
              const float p1 = (c0 + c + 1 < ncol) ? ex2_approx(fmaf(z1, kLog2e, -mxl)) : 0.f;
              s += p0 + p1;
              if (c0 + c == yl) zy = z0;
              if (c0 + c + 1 == yl) zy = z1;
              if constexpr (ES == 2) {
                pk[c >> 1] = pack_bf16x2(p0, p1);
              } else {
                pk[c] = __float_as_uint(p0);
                pk[c + 1] = __float_as_uint(p1);
              }
            }
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            uint8_t* b = ebuf + buf * kEpiBufBytes + lane * 128;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch)
              *reinterpret_cast<uint4*>(b + ((ch ^ (lane & 7)) << 4)) =
                  make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmOut, ebuf + buf * kEpiBufBytes, nb * a.BN + c0, row0);
              bulk_commit();
            }
            buf ^= 1;
          }
          if (rv) {
            a.m_tile[static_cast<size_t>(row) * a.n_blocks + nb] = mx;
            a.s_tile[static_cast<size_t>(row) * a.n_blocks + nb] = s;
            if (yl >= 0 && yl < ncol) a.zy[row] = zy;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

}  // namespace whale
