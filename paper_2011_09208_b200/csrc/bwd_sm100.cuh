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
//   warps 8..11 G-fused mode (NEXT-4b): operand transformers.  The A stages
//               of both GEMMs hold P~ = e^{z - m_tile} (the forward's bf16 output); each
//               thread turns one 128-byte smem row of a landed stage into
//               G = (P~ e^{m_tile - lse} / B_tot) - onehot / B_tot  (PAPER.md:286-288,
//               the softmax-minus-onehot gradient) before the MMA reads it, so G never
//               exists in HBM.  Every smem row of an A stage has ONE factor: a dX stage is
//               128 batch rows x 64 classes of one forward class tile (K-major); a dW stage
//               is 2 boxes x bk batch rows x 64 classes (MN-major G^T), again one tile per box.
#pragma once
#include "gemm_sm100.cuh"

namespace whale {

// F1 dX combine as work units of the backward kernel (scheduled first, while U is L2-resident;
// the dynamic scheduler balances the dW tiles around them):
// unit (row b, 1024-column part) computes dX[b, part] = (1/B_tot)(sum_cl e^{uref - lse} U_cl -
// W_{y_b}) in fixed cluster order; N = 1 writes dX, N > 1 pushes to the row owner's slab.
struct CombineArgs {
  const float* upart;   // [ncl x B_tot x D]
  const float* uref;    // [ncl x B_tot]
  int ncl, Bt, D, parts;
  const float* lse;     // [B_tot]
  const int32_t* y;     // [B_tot] global labels
  long long o_r, C_r;
  const void* w;        // W_r bf16 [C_r x D]
  float inv_bt;
  void* dx_out;         // N = 1: dX bf16 [B_tot x D]
  PeerPtrs recv;        // N > 1: owners' fp32 slabs [world][B_max x D]
  int row_off[kMaxRanks + 1];
  int rank, world, Bslab;
  const float* grad_scale;  // grad_output factor (device scalar) or NULL
};

// G-fused operand path: A stages hold P~; G[i, j] = P~[i, j] gscale[i, j / fwd_bn] - [j == y_i - o_r] / B_tot
struct GFuse {
  const float* gscale;  // [T x Bt] e^{m_tile - lse} / B_tot (statistics kernel), NULL: A holds G already
  const int32_t* y;     // [Bt] global labels
  long long o_r, C_r;
  int T, fwd_bn, Bt;
  float inv_bt;
};

struct BwdArgs {
  GemmArgs dx;          // units [0, ux): M = B_tot, N = D, K = C_r (A = G K-major, B = W_r MN-major)
  GemmArgs dw;          // units [ux, ux + tw): M = C_r, N = D, K = B_tot (both MN-major)
  int ux, tw;
  int tc;               // F1 dX combine units (no TMEM / smem stages), scheduled FIRST: unit ids
                        // [0, tc) are combine units and the GEMM units above are shifted by tc
  CombineArgs cb;
  GFuse gf;
  int stages, stage_bytes, epi_bufs;  // epi_bufs: CTA-wide 16 KB store stages
  unsigned* sched_cnt;  // dynamic-scheduler counter (zeroed by the last CTA of every launch)
  // Row-bulk dW stores: each epilogue thread stages its whole dW row segment (BN fp32,
  // rows padded by 16 B so the 32 lanes' 16-byte stores hit distinct banks) and writes it
  // with ONE 1-D bulk copy (cp.async.bulk) -- row-contiguous 1 KB writes instead of 128 x
  // 128 B tensor-store rows (measured 6.2 vs 5.8 TB/s, scripts/micro/bulk1d_store.cu).
  int row_bulk;         // 1: dW tiles use row-bulk stores (epi_bufs x 16 KB >= 128 x (BN + 4) x 4 B)
  void* dw_ptr;         // dW_r [C_r x D] fp32 or bf16 (row-bulk stores)
  int dw_ld;            // D
  int dw_bf16;          // 1: dW_r is stored in bf16 (RN-even from the fp32 accumulator)
  // N > 1: the owner side of the dX reduce-scatter in this kernel's tail (instead of the
  // dx_reduce kernel): after the end-of-step ticket every CTA waits for all ranks' RS flags
  // and sums its slice of this rank's rows over the N receive slots in rank order
  int w_last_use;            // 1: dX-unit W_r loads are marked L2 evict_first (the logits kept W_r in L2)
  int red_on;
  const float4* red_recv;    // this rank's receive slab [world][Bslab x D] fp32
  const float4* red_mc;      // NVLS: slot `rank` of every rank's slab (multicast view) or NULL
  const uint32_t* red_flags; // &flag[RS][0] on this rank
  void* red_out;             // dX_r bf16 [B x D]
  int red_B, red_Bslab;
};

constexpr int kBwdThreads = 384;  // 12 warps (8..11: G-fused operand transformers)

// One 128-byte SW128 smem row (8 x 16-byte chunks, chunk c stored at c ^ (row & 7)) of P~,
// all in one forward class tile: G = P~ * sc - [class == oc] / B_tot, rounded to bf16 as the
// in-place rewrite does (same expression, so G is bit-identical to the materialised one).
__device__ __forceinline__ void gfuse_row(uint8_t* row, int rsw, float sc, long long oc, float inv_bt) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {  // logical chunk q (classes 8q .. 8q + 7) sits at chunk q ^ rsw:
    // walking logical chunks spreads the 32 lanes (32 rows) over all banks
    uint8_t* cp = row + ((q ^ rsw) << 4);
    uint4 raw = *reinterpret_cast<const uint4*>(cp);
    const int c0 = q << 3;  // first class (within the 64) of this chunk
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __bfloat1622float2(h[k]);
      const long long j = c0 + 2 * k;
      f.x = f.x * sc - ((j == oc) ? inv_bt : 0.f);
      f.y = f.y * sc - ((j + 1 == oc) ? inv_bt : 0.f);
      h[k] = __floats2bfloat162_rn(f.x, f.y);
    }
    *reinterpret_cast<uint4*>(cp) = raw;
  }
}

constexpr int kCombineCols = 1024;  // dX columns per combine unit (128 threads x 2 float4)

// One combine unit, by the 128 epilogue threads (named barrier 1); fac: >= ncl floats of smem.
__device__ __forceinline__ void combine_unit(const CombineArgs& c, int u, float* fac) {
  const int b = u / c.parts, part = u % c.parts;
  const int et = threadIdx.x - 128;
  const float l = c.lse[b];
  for (int i = et; i < c.ncl; i += 128) fac[i] = __expf(c.uref[static_cast<size_t>(i) * c.Bt + b] - l);
  named_bar_sync(1, 128);
  const long long lab = static_cast<long long>(c.y[b]) - c.o_r;
  const bool own = lab >= 0 && lab < c.C_r;
  const size_t cstride = static_cast<size_t>(c.Bt) * c.D;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int d = part * kCombineCols + (h * 128 + et) * 4;
    if (d >= c.D) continue;
    const float* src = c.upart + static_cast<size_t>(b) * c.D + d;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int i = 0;
    for (; i + 4 <= c.ncl; i += 4) {  // four independent loads in flight, fixed summation order
      float4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __ldcg(reinterpret_cast<const float4*>(src + (i + k) * cstride));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float f = fac[i + k];
        acc.x = fmaf(f, v[k].x, acc.x);
        acc.y = fmaf(f, v[k].y, acc.y);
        acc.z = fmaf(f, v[k].z, acc.z);
        acc.w = fmaf(f, v[k].w, acc.w);
      }
    }
    for (; i < c.ncl; ++i) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(src + i * cstride));
      const float f = fac[i];
      acc.x = fmaf(f, v.x, acc.x);
      acc.y = fmaf(f, v.y, acc.y);
      acc.z = fmaf(f, v.z, acc.z);
      acc.w = fmaf(f, v.w, acc.w);
    }
    if (own) {  // the one-hot term, on the shard that owns the label
      const uint2 raw = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(c.w) + lab * c.D + d);
      const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
      const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
      acc.x -= w01.x;
      acc.y -= w01.y;
      acc.z -= w23.x;
      acc.w -= w23.y;
    }
    const float f = c.inv_bt * grad_factor(c.grad_scale);
    acc.x *= f;
    acc.y *= f;
    acc.z *= f;
    acc.w *= f;
    if (c.world == 1) {
      uint2 o;
      o.x = pack_bf16x2(acc.x, acc.y);
      o.y = pack_bf16x2(acc.z, acc.w);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(c.dx_out) + static_cast<size_t>(b) * c.D + d) = o;
    } else {
      int owner = 0;
#pragma unroll
      for (int r = 1; r < kMaxRanks; ++r)
        if (r < c.world && c.row_off[r] <= b) owner = r;
      float* dst = reinterpret_cast<float*>(c.recv.p[owner]) +
                   (static_cast<size_t>(c.rank) * c.Bslab + (b - c.row_off[owner])) * c.D + d;
      *reinterpret_cast<float4*>(dst) = acc;  // NVLink store into the owner's slab
    }
  }
  named_bar_sync(1, 128);  // fac is reused by the next unit
  // N > 1: the pushes of this unit, published at system scope now (the end-of-step ticket
  // then needs only gpu-scope fences in every CTA but the last)
  if (c.world > 1 && threadIdx.x == 128) __threadfence_system();
}

constexpr int kSchedSlots = 4;
// Debug timeline (WHALE_EPI_DEBUG bit 16, no effect on results): per CTA [start, dX unit done
// (after its fixup), epilogue done, GEMM units] in globaltimer ns -- whale_debug_bwd_timeline.
__device__ unsigned long long g_bwd_cta[160 * 4];

// DWB: dW_r stored in bf16 (a separate instantiation, so the fp32 kernel carries none of the
// bf16 store code and keeps its register allocation)
// PAIR: CTA pairs (launched as 2-CTA clusters; tensor-bound shapes, e.g. c5): every unit is
// an M = 256 tcgen05.mma.cta_group::2 tile over two M blocks -- each CTA loads its own 128 A
// rows and HALF of the B tile (a stage costs 32 instead of 48 KB, and each SM's tensor core
// reads half the B bytes), the leader's MMA thread issues for both, its commits multicast to
// both CTAs, and each CTA's epilogue stores its own 128 rows.  The leader's producer runs the
// dynamic scheduler and hands every unit id to the peer through distributed shared memory
// (st.async into the peer's slot + complete_tx on its slot barrier).  Requires no split-K
// (dx.splits == 1), no F1 combine units and no G-fused transformers.
template <int ES, bool DWB, bool PAIR = false>
__global__ void __launch_bounds__(kBwdThreads, 1)
    splitfc_bwd_kernel(const __grid_constant__ CUtensorMap tmGx, const __grid_constant__ CUtensorMap tmW,
                       const __grid_constant__ CUtensorMap tmPart, const __grid_constant__ CUtensorMap tmGw,
                       const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDW,
                       const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_fix_go;
  __shared__ int sched_tile[kSchedSlots];
  __shared__ float s_fac[160];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi_smem = smem + a.stages * a.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + a.epi_bufs * 4 * kEpiBufBytes);
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + kSchedSlots;
  uint64_t* ready = sempty + kSchedSlots;  // G-fused: A stage transformed (4 warp arrivals)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(ready + a.stages);

  constexpr int kBK = kRowBytes / ES;
  constexpr int kAtom = kRowBytes / ES;
  constexpr int kKStepMN = (32 / ES) * kRowBytes;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int total = a.ux + a.tw + a.tc;
  const bool xf = !PAIR && a.gf.gscale != nullptr;  // G-fused operand path
  constexpr int cs = PAIR ? 2 : 1;
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;
  const int uid0 = PAIR ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);  // first unit
  const int nuid = PAIR ? static_cast<int>(ncluster_x()) : static_cast<int>(gridDim.x);   // units in flight

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);   // pairs: the leader's expect_tx; both CTAs' TMA bytes land on the leader's
      mbar_init(&empty[i], 1);  // pairs: the leader's multicast commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128 * cs);  // pairs: both CTAs' epilogue threads, on the leader's
    }
    for (int i = 0; i < kSchedSlots; ++i) {
      mbar_init(&sfull[i], 1);
      // MMA thread + 4 epilogue warps (+ 4 transformer warps); pairs: on the leader's, plus the
      // peer's producer and 4 epilogue warps (the peer's MMA thread does not read the ring)
      mbar_init(&sempty[i], 1 + 4 + (xf ? 4 : 0) + (PAIR ? 5 : 0));
    }
    for (int i = 0; i < a.stages; ++i) mbar_init(&ready[i], 4);
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
  if (PAIR) cluster_sync();  // peer barriers initialised before any remote arrive / TMA / st.async
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair(tmem_holder, kTmemCols);
    else tmem_alloc(tmem_holder, kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();
  pdl_trigger();
  TraceScope _trace(8);
  // a consumer is done with scheduler slot `sl` (pairs: on the leader's barrier)
  auto release_slot = [&](int sl) {
    if (PAIR) mbar_arrive_remote(mapa_smem(smem_u32(&sempty[sl]), 0));
    else mbar_arrive(&sempty[sl]);
  };
  // an epilogue thread's TMEM reads of accumulator `acc` are complete (tcgen05.wait::ld, fence
  // issued): hand it back -- pairs: to the leader's MMA (relaxed: the loads already completed)
  auto release_acc_bwd = [&](uint64_t* bar) {
    if (PAIR) mbar_arrive_remote(mapa_smem(smem_u32(bar), 0));
    else mbar_arrive(bar);
  };
  const uint32_t e = ld_acquire_gpu(a.dx.dev_epoch) + 1u;  // this step's epoch
  if ((a.dx.debug & 16) && threadIdx.x == 0 && blockIdx.x < 160) {
    g_bwd_cta[blockIdx.x * 4] = gtime_ns();
    g_bwd_cta[blockIdx.x * 4 + 1] = 0ull;
  }

  if (warp == 0) {
    // ===================== scheduler + TMA producer =====================
    if (lane == 0) {
      const GemmArgs& X = a.dx;
      const GemmArgs& W = a.dw;
      const int dw_bk = W.bk;
      const int dw_box = dw_bk * kRowBytes;
      const int dw_a_bytes = (kBM / kAtom) * dw_box;
      const int dx_a_bytes = X.a_rows * kRowBytes;  // G rows per stage (B_tot rounded up to 8 when < 128)
      // pairs: this CTA's half of each B tile; the leader's full barrier expects both CTAs' bytes
      const int dx_bn = X.BN / cs, dw_bn = W.BN / cs;
      const uint32_t tx_dx = static_cast<uint32_t>(cs * (dx_a_bytes + (dx_bn / kAtom) * kBK * kRowBytes));
      const uint32_t tx_dw = static_cast<uint32_t>(cs * (dw_a_bytes + (dw_bn / kAtom) * dw_box));
      int stage = 0;
      uint32_t phase = 0;
      int unit = uid0;
      for (int it = 0;; ++it) {
        const int slot = it % kSchedSlots;
        if (!PAIR || crank == 0) {
          mbar_wait(&sempty[slot], ((it / kSchedSlots) & 1) ^ 1u);
          if (it > 0) unit = static_cast<int>(atomicAdd(a.sched_cnt, 1u)) + nuid;
          if (unit >= total) unit = -1;
          sched_tile[slot] = unit;
          mbar_arrive(&sfull[slot]);
          if (PAIR) {  // hand the unit to the peer: 4 bytes into its slot, completing its barrier
            const uint32_t pbar = mapa_smem(smem_u32(&sfull[slot]), 1);
            mbar_arrive_expect_tx_remote(pbar, 4u);
            st_async_u32(mapa_smem(smem_u32(&sched_tile[slot]), 1), pbar, static_cast<uint32_t>(unit));
          }
        } else {  // pair peer: the leader's unit
          mbar_wait(&sfull[slot], (it / kSchedSlots) & 1);
          unit = sched_tile[slot];
          release_slot(slot);
        }
        if (unit < 0) break;
        if (unit < a.tc) continue;  // combine unit: epilogue-only work
        unit -= a.tc;
        int mb, nb, sp, kb0, kb1;
        if (unit < a.ux) {
          decode_unit(X, unit, crank, mb, nb, sp, kb0, kb1);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* sA = smem + stage * a.stage_bytes;
            uint8_t* sB = sA + dx_a_bytes;
            if constexpr (PAIR) {
              const uint32_t fl = mapa_smem(smem_u32(&full[stage]), 0);
              if (crank == 0) mbar_arrive_expect_tx(&full[stage], tx_dx);
              tma_load_2d_pair(sA, &tmGx, fl, kb * kBK, mb * kBM);
              for (int j = 0; j < dx_bn / kAtom; ++j)
                tma_load_2d_pair(sB + j * kBK * kRowBytes, &tmW, fl, nb * X.BN + static_cast<int>(crank) * dx_bn + j * kAtom,
                                 kb * kBK);
            } else {
              mbar_arrive_expect_tx(&full[stage], tx_dx);
              tma_load_2d(sA, &tmGx, &full[stage], kb * kBK, mb * kBM);
              for (int j = 0; j < X.BN / kAtom; ++j)
                if (a.w_last_use)  // W_r kept in L2 by the logits: this is its last use
                  tma_load_2d_hint(sB + j * kBK * kRowBytes, &tmW, &full[stage], nb * X.BN + j * kAtom, kb * kBK,
                                   l2_policy_evict_first());
                else
                  tma_load_2d(sB + j * kBK * kRowBytes, &tmW, &full[stage], nb * X.BN + j * kAtom, kb * kBK);
            }
            if (++stage == a.stages) {
              stage = 0;
              phase ^= 1u;
            }
          }
        } else {
          decode_unit(W, unit - a.ux, crank, mb, nb, sp, kb0, kb1);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* sA = smem + stage * a.stage_bytes;
            uint8_t* sB = sA + dw_a_bytes;
            if constexpr (PAIR) {
              const uint32_t fl = mapa_smem(smem_u32(&full[stage]), 0);
              if (crank == 0) mbar_arrive_expect_tx(&full[stage], tx_dw);
#pragma unroll
              for (int j = 0; j < kBM / kAtom; ++j)
                tma_load_2d_pair(sA + j * dw_box, &tmGw, fl, mb * kBM + j * kAtom, kb * dw_bk);
              for (int j = 0; j < dw_bn / kAtom; ++j)
                tma_load_2d_pair(sB + j * dw_box, &tmX, fl, nb * W.BN + static_cast<int>(crank) * dw_bn + j * kAtom,
                                 kb * dw_bk);
            } else {
              mbar_arrive_expect_tx(&full[stage], tx_dw);
#pragma unroll
              for (int j = 0; j < kBM / kAtom; ++j)
                tma_load_2d(sA + j * dw_box, &tmGw, &full[stage], mb * kBM + j * kAtom, kb * dw_bk);
              for (int j = 0; j < W.BN / kAtom; ++j)
                tma_load_2d(sB + j * dw_box, &tmX, &full[stage], nb * W.BN + j * kAtom, kb * dw_bk);
            }
            if (++stage == a.stages) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (pairs: the leader only, M = 256) =====================
    if (lane == 0 && crank == 0) {
      const uint32_t idesc_dx = umma_idesc(kBM * cs, a.dx.BN, false, true, ES == 2 ? 1u : 2u);
      const uint32_t idesc_dw = umma_idesc(kBM * cs, a.dw.BN, true, true, ES == 2 ? 1u : 2u);
      const uint32_t dw_box = a.dw.bk * kRowBytes;
      const uint32_t dw_a_bytes = (kBM / kAtom) * dw_box;
      const int dw_kmma = a.dw.bk / (32 / ES);
      int stage = 0;
      uint32_t phase = 0;
      int na = 0;  // GEMM units so far (accumulator ring index; combine units use no TMEM)
      for (int it = 0;; ++it) {
        const int slot = it % kSchedSlots;
        mbar_wait(&sfull[slot], (it / kSchedSlots) & 1);
        const int unit = sched_tile[slot];
        mbar_arrive(&sempty[slot]);
        if (unit < 0) break;
        if (unit < a.tc) continue;
        const int gu = unit - a.tc;
        const bool is_dx = gu < a.ux;
        int mb, nb, sp, kb0, kb1;
        if (is_dx) decode_unit(a.dx, gu, 0u, mb, nb, sp, kb0, kb1);
        else decode_unit(a.dw, gu - a.ux, 0u, mb, nb, sp, kb0, kb1);
        const int acc = na & 1;
        const uint32_t aph = (na >> 1) & 1;
        ++na;
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kMaxBN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(xf ? &ready[stage] : &full[stage], phase);
          tc_fence_after();
          const uint32_t aS = smem_u32(smem + stage * a.stage_bytes);
          if (is_dx) {
            const uint32_t bS = aS + a.dx.a_rows * kRowBytes;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = umma_sdesc(aS + k * 32, 16, 1024);
              const uint64_t bd = umma_sdesc(bS + k * kKStepMN, kBK * kRowBytes, 1024);
              if constexpr (PAIR) umma_bf16_pair(d_tmem, ad, bd, idesc_dx, (kb > kb0 || k > 0) ? 1u : 0u);
              else umma_bf16(d_tmem, ad, bd, idesc_dx, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          } else {
            const uint32_t bS = aS + dw_a_bytes;
            for (int k = 0; k < dw_kmma; ++k) {
              const uint64_t ad = umma_sdesc(aS + k * kKStepMN, dw_box, 1024);
              const uint64_t bd = umma_sdesc(bS + k * kKStepMN, dw_box, 1024);
              if constexpr (PAIR) umma_bf16_pair(d_tmem, ad, bd, idesc_dw, (kb > kb0 || k > 0) ? 1u : 0u);
              else umma_bf16(d_tmem, ad, bd, idesc_dw, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          if constexpr (PAIR) umma_commit_pair_mc(&empty[stage], 0x3);  // frees the stage in both CTAs
          else umma_commit(&empty[stage]);
          if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if constexpr (PAIR) umma_commit_pair_mc(&tfull[acc], 0x3);  // both halves ready
        else umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ===================== epilogue =====================
    const int q = warp & 3;
    const int nbuf = a.epi_bufs;
    int buf = 0;
    int na = 0;  // GEMM units so far (accumulator ring index)
    for (int it = 0;; ++it) {
      const int slot = it % kSchedSlots;
      mbar_wait(&sfull[slot], (it / kSchedSlots) & 1);
      const int unit = sched_tile[slot];
      __syncwarp();
      if (lane == 0) release_slot(slot);
      if (unit < 0) break;
      if (unit < a.tc) {
        combine_unit(a.cb, unit, s_fac);
        continue;
      }
      const int gu = unit - a.tc;
      const bool is_dx = gu < a.ux;
      const GemmArgs& g = is_dx ? a.dx : a.dw;
      int mb, nb, sp, kb0, kb1;
      decode_unit(g, is_dx ? gu : gu - a.ux, crank, mb, nb, sp, kb0, kb1);
      const CUtensorMap* om = is_dx ? &tmPart : &tmDW;
      const int acc = na & 1;
      const uint32_t aph = (na >> 1) & 1;
      ++na;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * kMaxBN + (static_cast<uint32_t>(q * 32) << 16);
      const float dws = is_dx ? 1.f : grad_factor(a.dx.grad_scale);  // dW carries grad_output
      if (!is_dx && a.row_bulk) {
        // ---- row-bulk dW store: this thread's row, all BN columns, one bulk copy
        constexpr int eb = DWB ? 2 : 4;
        uint8_t* srow = epi_smem + (q * 32 + lane) * (g.BN * eb + 16);
        bulk_wait_read<0>();  // my previous row copy has left the staging row
        for (int c0 = 0; c0 < g.BN; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c0, v);
          tmem_ld_wait();
          if (c0 + 32 >= g.BN) {
            tc_fence_before();
            release_acc_bwd(&tempty[acc]);
          }
          if (a.dx.grad_scale) scale32(v, dws);
          if constexpr (DWB) {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch)
              *reinterpret_cast<uint4*>(srow + (c0 + 8 * ch) * 2) =
                  make_uint4(pack_bf16x2(__uint_as_float(v[8 * ch]), __uint_as_float(v[8 * ch + 1])),
                             pack_bf16x2(__uint_as_float(v[8 * ch + 2]), __uint_as_float(v[8 * ch + 3])),
                             pack_bf16x2(__uint_as_float(v[8 * ch + 4]), __uint_as_float(v[8 * ch + 5])),
                             pack_bf16x2(__uint_as_float(v[8 * ch + 6]), __uint_as_float(v[8 * ch + 7])));
          } else {
#pragma unroll
            for (int ch = 0; ch < 8; ++ch)
              *reinterpret_cast<uint4*>(srow + (c0 + 4 * ch) * 4) =
                  make_uint4(v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
          }
        }
        fence_proxy_async_smem();
        const int row = mb * kBM + q * 32 + lane;
        const int ncol = min(g.BN, g.N - nb * g.BN);
        if (row < g.M && ncol > 0) {
          bulk_store_1d(static_cast<uint8_t*>(a.dw_ptr) + (static_cast<size_t>(row) * a.dw_ld + static_cast<size_t>(nb) * g.BN) * eb,
                        srow, ncol * eb);
          bulk_commit();
        }
        continue;
      }
      if (DWB && !is_dx) {
        // ---- bf16 dW through the tensor-store path: 64 columns (128 B) per 16 KB stage
        for (int c0 = 0; c0 < g.BN; c0 += 64) {
          uint32_t v[32], w[32];
          tmem_ld32(tbase + c0, v);
          if (c0 + 32 < g.BN) tmem_ld32(tbase + c0 + 32, w);
          tmem_ld_wait();
          if (c0 + 64 >= g.BN) {
            tc_fence_before();
            release_acc_bwd(&tempty[acc]);
          }
          if (c0 + 32 >= g.BN) {
#pragma unroll
            for (int k = 0; k < 32; ++k) w[k] = 0u;
          }
          uint32_t pk[32];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            pk[k] = pack_bf16x2(__uint_as_float(v[2 * k]) * dws, __uint_as_float(v[2 * k + 1]) * dws);
            pk[16 + k] = pack_bf16x2(__uint_as_float(w[2 * k]) * dws, __uint_as_float(w[2 * k + 1]) * dws);
          }
          if (threadIdx.x == 128) bulk_wait_read_n(nbuf);
          named_bar_sync(1, 128);
          uint8_t* b = epi_smem + buf * 4 * kEpiBufBytes + (q * 32 + lane) * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            *reinterpret_cast<uint4*>(b + ((ch ^ (lane & 7)) << 4)) =
                make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (threadIdx.x == 128) {
            tma_store_3d(&tmDW, epi_smem + buf * 4 * kEpiBufBytes, nb * g.BN + c0, mb * kBM, 0);
            bulk_commit();
          }
          if (++buf == nbuf) buf = 0;
        }
        continue;
      }
      for (int c0 = 0; c0 < g.BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tbase + c0, v);
        tmem_ld_wait();
        if (c0 + 32 >= g.BN) {
          tc_fence_before();
          release_acc_bwd(&tempty[acc]);
        }
        if (!is_dx && a.dx.grad_scale) scale32(v, dws);
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
          const uint32_t target = static_cast<uint32_t>(a.dx.splits);
          if (static_cast<int32_t>(ld_acquire_gpu(cnt) - target) < 0) {
            SpinGuard sg;
            while (static_cast<int32_t>(ld_acquire_gpu(cnt) - target) < 0)
              if (sg.expired(a.dx.err, ERR_SPLITK)) break;
          }
        }
        named_bar_sync(1, 128);
        __threadfence();
        fixup_share<ES>(a.dx, mb, nb, sp, threadIdx.x - 128);
        if (a.dx.fix_mode == FIX_PUSH) {  // this CTA's NVLink pushes, published at system scope now
          named_bar_sync(1, 128);         // (off the kernel's tail: the dW tiles follow)
          if (threadIdx.x == 128) __threadfence_system();
        }
        if ((a.dx.debug & 16) && threadIdx.x == 128 && blockIdx.x < 160) g_bwd_cta[blockIdx.x * 4 + 1] = gtime_ns();
      }
    }
    if (threadIdx.x == 128 || a.row_bulk) bulk_wait<0>();  // this thread's bulk stores are complete
    if ((a.dx.debug & 16) && threadIdx.x == 128 && blockIdx.x < 160) {
      g_bwd_cta[blockIdx.x * 4 + 2] = gtime_ns();
      g_bwd_cta[blockIdx.x * 4 + 3] = static_cast<unsigned long long>(na);
    }
  } else if (warp >= 8 && xf) {
    // ===================== G-fused operand transformers =====================
    // thread tt owns one 128-byte row of every A stage.  The stages are walked as a task
    // stream (unit by unit through the scheduler ring); the factor and label of task k + 2
    // are loaded while task k is transformed, so the L2 latency of those loads is hidden.
    // (Looking 2 tasks ahead is safe: the producer issues a unit's stages before it publishes
    // the next unit, and at most 2 < ring-depth stages are held here untransformed.)
    const int tt = threadIdx.x - 256;
    const GFuse& g = a.gf;
    const int dw_bk = a.dw.bk;
    const int dw_box = dw_bk * kRowBytes;
    int it = 0;           // scheduler-ring slots read
    int u_kb = 0, u_kb1 = 0, u_dx = 0, u_mb = 0;  // current unit: remaining k-blocks [u_kb, u_kb1)
    int t_stage = 0;      // smem stage of the next task
    bool done = false;
    struct Task {
      int stage;
      int row_off;        // byte offset of this thread's row in the stage, -1: no row
      int rsw;
      const float* sc;    // factor address (gscale, transposed [T x B_tot])
      const int32_t* y;   // label address
      long long cls0;     // first class of the row's 64
      bool end;
    };
    auto next_task = [&]() -> Task {
      Task k{};
      while (u_kb >= u_kb1) {  // next GEMM unit from the scheduler ring
        if (done) {
          k.end = true;
          return k;
        }
        const int slot = it % kSchedSlots;
        mbar_wait(&sfull[slot], (it / kSchedSlots) & 1);
        const int unit = sched_tile[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[slot]);
        ++it;
        if (unit < 0) {
          done = true;
          continue;
        }
        if (unit < a.tc) continue;  // combine unit: no operand stages
        const int gu = unit - a.tc;
        int nb, sp;
        u_dx = gu < a.ux;
        if (u_dx) decode_tile(a.dx, gu, u_mb, nb, sp, u_kb, u_kb1);
        else decode_tile(a.dw, gu - a.ux, u_mb, nb, sp, u_kb, u_kb1);
      }
      const int kb = u_kb++;
      k.stage = t_stage;
      if (++t_stage == a.stages) t_stage = 0;
      k.row_off = -1;
      if (u_dx) {  // dX: A = G [batch rows x 64 classes]; row tt = batch row mb * 128 + tt
        const int i = u_mb * kBM + tt;
        if (i < g.Bt) {
          k.row_off = tt * kRowBytes;
          k.rsw = tt & 7;
          k.cls0 = static_cast<long long>(kb) * kBK;
          k.sc = g.gscale + static_cast<size_t>((kb * kBK) / g.fwd_bn) * g.Bt + i;  // 32-bit: kb * 64 < 2^31
          k.y = g.y + i;
        }
      } else {  // dW: A = G^T MN-major, boxes {64 classes, bk batch rows}; row tt = (box j, row ii)
        const int j = tt / dw_bk, ii = tt % dw_bk;
        const long long cls0 = static_cast<long long>(u_mb) * kBM + j * kAtom;
        const int i = kb * dw_bk + ii;
        if (j < kBM / kAtom && cls0 < g.C_r && i < g.Bt) {
          k.row_off = j * dw_box + ii * kRowBytes;
          k.rsw = ii & 7;
          k.cls0 = cls0;
          k.sc = g.gscale + static_cast<size_t>(static_cast<int>(cls0) / g.fwd_bn) * g.Bt + i;
          k.y = g.y + i;
        }
      }
      return k;
    };
    // task ring of depth 3 kept in registers (rotated, never indexed dynamically)
    Task k0 = next_task(), k1 = next_task();
    const bool v0 = !k0.end && k0.row_off >= 0, v1 = !k1.end && k1.row_off >= 0;
    float s0 = v0 ? __ldg(k0.sc) : 0.f, s1 = v1 ? __ldg(k1.sc) : 0.f;
    int32_t y0 = v0 ? __ldg(k0.y) : 0, y1 = v1 ? __ldg(k1.y) : 0;
    uint32_t phase = 0;
    for (bool first = true; !k0.end; first = false) {
      const Task k2 = next_task();  // prefetch two tasks ahead
      const bool v2 = !k2.end && k2.row_off >= 0;
      const float s2 = v2 ? __ldg(k2.sc) : 0.f;
      const int32_t y2 = v2 ? __ldg(k2.y) : 0;
      if (!first && k0.stage == 0) phase ^= 1u;
      mbar_wait(&full[k0.stage], phase);
      if (k0.row_off >= 0)
        gfuse_row(smem + k0.stage * a.stage_bytes + k0.row_off, k0.rsw, s0, static_cast<long long>(y0) - g.o_r - k0.cls0,
                  g.inv_bt);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[k0.stage]);
      k0 = k1;
      s0 = s1;
      y0 = y1;
      k1 = k2;
      s1 = s2;
      y1 = y2;
    }
  }
  tc_fence_before();
  __syncthreads();
  // pairs: the peer may still receive the leader's commits / send its arrives
  if (PAIR) cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem_base, kTmemCols);
    else tmem_dealloc(tmem_base, kTmemCols);
  }
  end_of_step_ticket(a.dx, e, s_fix_go, a.sched_cnt, /*pushes_fenced=*/true);  // RS flags (N > 1) + epoch publish + counter reset
  if (a.red_on) {  // A8 owner side (as dx_reduce_kernel): every rank's pushes for my rows have landed
    if (threadIdx.x < a.dx.world) wait_flag_geq(a.red_flags + threadIdx.x, e, a.dx.err, ERR_COMM | ERR_AT_RS);
    __syncthreads();
    __threadfence_system();
    const int64_t total = static_cast<int64_t>(a.red_B) * (a.dx.N / 4);
    const int64_t slab = static_cast<int64_t>(a.red_Bslab) * (a.dx.N / 4);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      float4 acc;
      if (a.red_mc != nullptr) {
        acc = multimem_ld_reduce_add_v4f32(a.red_mc + i);
      } else {
        acc = __ldcg(a.red_recv + i);
        for (int p = 1; p < a.dx.world; ++p) {
          const float4 v = __ldcg(a.red_recv + p * slab + i);
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
      }
      uint2 o;
      o.x = pack_bf16x2(acc.x, acc.y);
      o.y = pack_bf16x2(acc.z, acc.w);
      reinterpret_cast<uint2*>(a.red_out)[i] = o;
    }
  }
}

}  // namespace whale
